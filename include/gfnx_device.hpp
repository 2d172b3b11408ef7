// gfnx_device.hpp — the C++ binding a reference (gfnkit) maintainer adds over the C ABI of
// include/gfnx.h: the device trainer as a drop-in for train_scenario's per-iteration state,
// speaking the reference's own types (gfn::MlpParams, nn.hpp:17-31) and rethrowing its own
// exception classes (gfn::config_error / contract_violation / numeric_error, errors.hpp:6-16).
//
// Compiled and linked against /root/reference/proj/include and libgfnx.so by
// tests/test_integration_binding.py; INTEGRATION.md shows where it slots into train.cpp.
#pragma once

#include <algorithm>
#include <stdexcept>
#include <string>
#include <vector>

#include "gfn/errors.hpp"
#include "gfn/nn.hpp"
#include "gfnx.h"

namespace gfn {

inline void gfnx_throw(gfnx_status s, const gfnx_ctx* c) {
  if (s == GFNX_OK) return;
  const std::string m = gfnx_last_error(c);
  switch (s) {
    case GFNX_ERR_CONFIG: throw config_error(m);
    case GFNX_ERR_CONTRACT: throw contract_violation(m);
    case GFNX_ERR_NUMERIC: throw numeric_error(m);
    default: throw std::runtime_error("gfnx: " + m);
  }
}

// Device replacement of train_scenario's state (train.cpp:194-221): policy, both Adam
// states and the resident trajectory batch of this rank.
class DeviceTrainer {
 public:
  DeviceTrainer(const gfnx_env_desc& env, const gfnx_train_desc& train, int device = 0, int rank = 0,
                int world = 1, const void* nccl_id = nullptr) {
    gfnx_throw(gfnx_create(&env, &train, device, rank, world, nccl_id, &ctx_), nullptr);
  }
  DeviceTrainer(const DeviceTrainer&) = delete;
  DeviceTrainer& operator=(const DeviceTrainer&) = delete;
  ~DeviceTrainer() { gfnx_destroy(ctx_); }

  // forward_rollout(env, params, policy, B, fold_in(root, 1000 + it), eps)   env_core.hpp:232
  void forward_rollout(int64_t it, double eps) { gfnx_throw(gfnx_rollout(ctx_, it, eps), ctx_); }
  // train_step(sc, policy, opt_main, opt_z, batch, lr)                       train.cpp:164
  double train_step(double lr) {
    double loss = 0.0;
    gfnx_throw(gfnx_train_step(ctx_, lr, &loss), ctx_);
    return loss;
  }
  // one train_scenario iteration, schedules resolved from the train desc     train.cpp:224-229
  double iteration(int64_t it) {
    double loss = 0.0;
    gfnx_throw(gfnx_iteration(ctx_, it, &loss), ctx_);
    return loss;
  }
  // MlpParams import / export in MlpParams::tensors() order (nn.cpp:8-19) plus log_z
  void set_params(const MlpParams& p) {
    std::vector<double> flat;
    for (const Tensor* t : p.tensors()) flat.insert(flat.end(), t->data.begin(), t->data.end());
    gfnx_throw(gfnx_set_params(ctx_, flat.data(), (int64_t)flat.size(), p.log_z.data.at(0)), ctx_);
  }
  void get_params(MlpParams& p) {
    int64_t n = 0;
    gfnx_throw(gfnx_num_params(ctx_, &n), ctx_);
    std::vector<double> flat((size_t)n);
    double z = 0.0;
    gfnx_throw(gfnx_get_params(ctx_, flat.data(), n, &z), ctx_);
    size_t off = 0;
    for (Tensor* t : p.tensors()) {
      if (off + t->data.size() > flat.size()) throw contract_violation("get_params: layout mismatch");
      std::copy(flat.begin() + (std::ptrdiff_t)off, flat.begin() + (std::ptrdiff_t)(off + t->data.size()),
                t->data.begin());
      off += t->data.size();
    }
    if (off != flat.size()) throw contract_violation("get_params: layout mismatch");
    p.log_z.data.at(0) = z;
  }
  // save_checkpoint / load_checkpoint (checkpoint.cpp:11-107), GFNCKPT1 byte-compatible
  void save_checkpoint(const std::string& path, int64_t step) {
    gfnx_throw(gfnx_save_checkpoint(ctx_, path.c_str(), step), ctx_);
  }
  int64_t load_checkpoint(const std::string& path) {
    int64_t step = 0;
    gfnx_throw(gfnx_load_checkpoint(ctx_, path.c_str(), &step), ctx_);
    return step;
  }
  gfnx_ctx* handle() { return ctx_; }

 private:
  gfnx_ctx* ctx_ = nullptr;
};

}  // namespace gfn
