// Reference-side drop-in check (TEST INFRASTRUCTURE): a gfnkit driver that trains through
// include/gfnx_device.hpp. Built by oracle/Makefile (target _ref/binding_driver) against the
// reference's headers and objects plus libgfnx.so, run by tests/test_integration_binding.py.
//
//   binding_driver errors   bad descriptors surface as the reference's exception types
//   binding_driver train    mlp_init (nn.cpp:41-58) params -> device, 3 iterations, params back
//   binding_driver eb       run_eb_gfn's loop on the device through DeviceTrainer::eb_*, the
//                           data from the reference's gibbs_data_sampler, the learned coupling
//                           back into the reference's IsingCoupling
#include <cmath>
#include <cstdio>
#include <cstring>

#include "gfn/rng.hpp"
#include "gfnx_device.hpp"

int main(int argc, char** argv) {
  const char* mode = argc > 1 ? argv[1] : "errors";
  gfnx_env_desc env{};
  gfnx_train_desc train{};
  gfnx_default_env_desc(GFNX_ENV_HYPERGRID, &env);
  gfnx_default_train_desc(GFNX_ENV_HYPERGRID, &train);
  env.hg_dim = 4;
  env.hg_side = 20;
  if (!std::strcmp(mode, "eb")) {  // acceptance.cpp:365-385's EB setting, 200 iterations
    gfnx_env_desc ie{};
    gfnx_train_desc it{};
    gfnx_default_env_desc(GFNX_ENV_ISING, &ie);
    gfnx_default_train_desc(GFNX_ENV_ISING, &it);
    ie.is_side = 3;
    it.batch_size = 16;
    it.num_hidden = 2;
    it.hidden[0] = it.hidden[1] = 128;
    it.iterations = 200;
    it.seed = 5;
    it.precision = GFNX_PREC_FP64_CHECK;
    gfnx_eb_desc d{};
    gfnx_eb_default_desc(&d);
    d.data_batch = 64;
    d.coupling_lr = d.coupling_lr_end = 0.02;
    const auto data = gfn::gibbs_data_sampler(gfn::toroidal_coupling(3, 0.2),
                                              gfn::fold_in(gfn::make_key(5), 0x919B), 2000);
    gfn::DeviceTrainer dev(ie, it);
    dev.eb_init(d, data);
    const std::vector<double> m = dev.eb_run(0, 200);
    gfn::IsingCoupling jm = gfn::zero_coupling(3);
    dev.eb_coupling(jm);
    const double nlr = gfn::neg_log_rmse(gfn::toroidal_coupling(3, 0.2), jm);
    std::printf("eb init_nlr %.6f final_nlr %.6f device_nlr %.6f\n",
                gfn::neg_log_rmse(gfn::toroidal_coupling(3, 0.2), gfn::zero_coupling(3)), nlr, m[4 * 199 + 2]);
    return std::fabs(nlr - m[4 * 199 + 2]) < 1e-12 ? 0 : 1;
  }
  if (!std::strcmp(mode, "errors")) {
    gfnx_env_desc bad = env;
    bad.hg_r0 = 0.0;  // hypergrid.cpp validate: r0 must be positive
    try {
      gfn::DeviceTrainer t(bad, train);
      std::printf("no exception\n");
      return 1;
    } catch (const gfn::config_error& e) {
      std::printf("config_error: %s\n", e.what());
    }
    gfnx_train_desc badt = train;
    badt.batch_size = 0;
    try {
      gfn::DeviceTrainer t(env, badt);
      return 1;
    } catch (const gfn::config_error& e) {
      std::printf("config_error: %s\n", e.what());
    }
    return 0;
  }
  // train: the reference's own initialisation handed to the device (policy key fold_in(root, 0),
  // train.cpp:204), three iterations, parameters read back into the reference's MlpParams
  gfn::MlpParams p = gfn::mlp_init(80, {256, 256}, 5, 5, gfn::fold_in(gfn::make_key(train.seed), 0),
                                   train.logz_init);
  gfn::DeviceTrainer dev(env, train);
  dev.set_params(p);
  gfn::MlpParams back = p;
  dev.get_params(back);
  double maxdiff = 0.0;
  for (size_t i = 0; i < p.tensors().size(); ++i)
    for (size_t j = 0; j < p.tensors()[i]->data.size(); ++j)
      maxdiff = std::fmax(maxdiff, std::fabs(p.tensors()[i]->data[j] - back.tensors()[i]->data[j]));
  double loss = 0.0;
  for (int it = 0; it < 3; ++it) loss = dev.iteration(it);
  dev.get_params(back);
  std::printf("roundtrip_maxdiff %.3e loss %.6f log_z %.6f\n", maxdiff, loss, back.log_z.data[0]);
  return std::isfinite(loss) && maxdiff < 1e-6 ? 0 : 1;
}
