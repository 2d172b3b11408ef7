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

#include "gfn/envs/ising.hpp"
#include "gfn/errors.hpp"
#include "gfn/nn.hpp"
#include "gfn/rng.hpp"
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
  // backward_rollout(env, p, nullptr, false, terminals, key)   env_core.hpp:314-370 (uniform
  // P_B) of local_batch packed terminal states -> the resident batch (train_step acts on it)
  void backward_rollout(const std::vector<uint32_t>& packed, const RngKey& key) {
    int32_t bl = 0, b0 = 0, T = 0, sw = 0;
    gfnx_throw(gfnx_batch_dims(ctx_, &bl, &b0, &T, &sw), ctx_);
    if (packed.size() != (size_t)bl * (size_t)sw) throw contract_violation("backward_rollout: batch size mismatch");
    gfnx_throw(gfnx_backward_rollout(ctx_, packed.data(), bl, key.hi, key.lo), ctx_);
  }
  // mc_terminal_logprob (exact.hpp:229-241) of n packed terminals, one RngKey each
  std::vector<double> mc_terminal_logprob(const std::vector<uint32_t>& packed, const std::vector<RngKey>& keys,
                                          int num_samples) {
    std::vector<uint64_t> kw;
    for (const RngKey& k : keys) {
      kw.push_back(k.hi);
      kw.push_back(k.lo);
    }
    std::vector<double> out(keys.size());
    gfnx_throw(gfnx_mc_terminal_logprob(ctx_, packed.data(), (int64_t)keys.size(), num_samples, kw.data(),
                                        out.data()),
               ctx_);
    return out;
  }
  // the bitseq `pearson` metric closure of build_bitseq (train.cpp:440-454)
  double pearson(int64_t step, int mc_samples, uint64_t test_seed) {
    double r = 0.0;
    gfnx_throw(gfnx_pearson(ctx_, step, mc_samples, test_seed, &r), ctx_);
    return r;
  }

  // ---- EB-GFN (run_eb_gfn, train.cpp:875-1018) on an Ising device trainer ----
  // data: the samples run_eb_gfn would load or Gibbs-sample (empty: the device ctx samples
  // them itself with gibbs_data_sampler's algorithm and key)
  void eb_init(const gfnx_eb_desc& d, const std::vector<std::vector<int8_t>>& data = {}) {
    std::vector<int8_t> flat;
    for (const auto& x : data) flat.insert(flat.end(), x.begin(), x.end());
    gfnx_throw(gfnx_eb_init(ctx_, &d, data.empty() ? nullptr : flat.data(), (int64_t)data.size()), ctx_);
  }
  // iterations it0 .. it0 + n - 1; rows {loss, logZ, neg_log_rmse, accepted proposals}
  std::vector<double> eb_run(int64_t it0, int64_t n) {
    std::vector<double> m((size_t)(4 * n));
    gfnx_throw(gfnx_eb_run(ctx_, it0, n, m.data()), ctx_);
    return m;
  }
  // the learned coupling into the reference's IsingCoupling (ising.hpp:16-25)
  void eb_coupling(IsingCoupling& j_model) {
    gfnx_throw(gfnx_eb_coupling(ctx_, j_model.j.data(), nullptr, (int64_t)j_model.j.size(), nullptr), ctx_);
  }

  gfnx_ctx* handle() { return ctx_; }

 private:
  gfnx_ctx* ctx_ = nullptr;
};

}  // namespace gfn
