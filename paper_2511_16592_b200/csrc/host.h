// host.h — host-side setup of the engine (plain C++, no CUDA): environment tables,
// parameter initialisation and the reference drivers' defaults.
#pragma once

#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/gfnx.h"

namespace gfnx {

struct MlpLayout;

struct HostEnv {
  gfnx_env_shape shape{};
  // hypergrid
  uint32_t hg_f1[8] = {0}, hg_f2[8] = {0};
  double hg_logr[4] = {0, 0, 0, 0};
  // bitseq
  int bs_slots = 0, bs_vocab = 0, n_modes = 0, mode_words = 0;
  std::vector<uint64_t> modes;  // [n_modes][mode_words]
  std::vector<double> bs_logr;  // [n_bits + 1]
  // ising
  int is_D = 0;
  std::vector<int16_t> is_nbr;  // [D][4]
  std::vector<double> is_J;     // [D][4]
  // dag
  std::vector<double> dag_cache;  // [d][2^d]
  std::vector<uint32_t> dag_true_adj;
  // -log(k) for k = 0..max parents (entry 0 = 0)
  std::vector<double> neglog;
};

// Returns "" on success or a config_error message.
std::string build_host_env(const gfnx_env_desc& e, HostEnv* out);
std::string validate_train(const gfnx_train_desc& t, const gfnx_env_shape& s);
void make_layout(const gfnx_train_desc& t, const gfnx_env_shape& s, MlpLayout* L);
// mlp_init (nn.cpp:41-58) with key fold_in(make_key(seed), 0) (train.cpp:204)
void init_params(const gfnx_train_desc& t, const MlpLayout& L, int A, int Ab,
                 std::vector<double>* params);
double schedule_value(const gfnx_schedule& s, int64_t step);  // optim.cpp:45-66
// EB-GFN setup (train.cpp:890-920): the true toroidal coupling as a dense [D][D] matrix and the
// Gibbs data sampler over it (samples [n][D], spins +-1)
std::vector<double> ising_dense_coupling(int side, double sigma);
struct Key;
std::vector<int8_t> ising_gibbs_data(const std::vector<double>& J, int D, Key key, int64_t n_samples,
                                     int64_t burn_in, int64_t thinning, int chains, double hottest_beta);
void resolve_schedule(gfnx_schedule* s, int64_t iterations);  // train.cpp:98-101
void default_env(int kind, gfnx_env_desc* e);
void default_train(int kind, gfnx_train_desc* t);

}  // namespace gfnx
