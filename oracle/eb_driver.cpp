// eb_driver.cpp — runs the UNMODIFIED reference's run_eb_gfn (train.cpp:875-1018) through
// its Config front door: eb_driver <out_dir> key=value ... ; prints the EbGfnResult.
// TEST INFRASTRUCTURE ONLY (tests/test_device_eb.py). A separate process because the
// reference's std::ofstream output crashes inside a Python process that has numpy's
// bundled runtime libraries loaded.
#include <cstdio>
#include <cstring>
#include <string>

#include "gfn/config.hpp"
#include "gfn/errors.hpp"
#include "gfn/train.hpp"

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: eb_driver <out_dir> key=value ...\n");
    return 2;
  }
  try {
    gfn::Config cfg;
    for (int i = 2; i < argc; ++i) {
      const char* eq = std::strchr(argv[i], '=');
      if (!eq) return 2;
      cfg.set(std::string(argv[i], eq - argv[i]), std::string(eq + 1));
    }
    const gfn::EbGfnResult r = gfn::run_eb_gfn(cfg, argv[1]);
    std::printf("%.17g %.17g %.17g %.17g\n", r.init_neg_log_rmse, r.best_neg_log_rmse, r.final_neg_log_rmse,
                r.final_loss);
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
