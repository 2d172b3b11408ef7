// walk.cu — backward walks and teacher-forced batches on the device:
//
//   k_bwd_walk    backward_rollout under the uniform backward policy (env_core.hpp:314-370):
//                 one thread per walk, integer state in registers, the reference's draws
//                 (step key fold_in(key, t), categorical(fold_in(step_key, b)) over the legal
//                 backward actions with weight 1.0 each, rng.cpp:87-100), forward actions
//                 written in forward order (rollout_from_actions input) with #parents per step
//   k_replay      rollout_from_actions (env_core.hpp:166-229) for the hypergrid / DAG fast
//                 path: the batch record (state words, actions, #parents, MDB deltas, lengths,
//                 log-rewards, terminals) from given actions; the training forward is then
//                 recomputed over the rows (k_linear_rows + k_fast_fwd)
//   k_mc_*        score_trajectories (objectives.cpp:294-316) + logsumexp of
//                 mc_terminal_logprob (exact.hpp:229-241): per-walk log P_F - log P_B summed in
//                 forward order, then per terminal logsumexp over its K walks (sample order)
//
// The lockstep (bitseq, Ising) and fp64 check paths take teacher-forced actions inside their
// own rollout kernels (k_ls_sample / k_ls_persist / k_check_rollout: `forced`).
#include <cub/cub.cuh>
#include <math.h>

#include <algorithm>
#include <vector>

#include "engine.h"
#include "walk.cuh"

namespace gfnx {

namespace {

// walk j of this launch is global walk g = min(j0 + j, N - 1) (chunk tails repeat the last
// walk): terminal i = g / K; with per-terminal keys (mc_terminal_logprob: K copies of each
// terminal) the draw index is the copy g % K, else (backward_rollout of a batch, K = 1) it
// is draw_base + g under the single key
template <class Env>
__global__ void k_bwd_walk(EnvParams P, const uint32_t* __restrict__ terms, int n_walks, int64_t j0, int64_t N,
                           int K, const uint64_t* __restrict__ keys, Key key, int64_t draw_base, int T,
                           int16_t* __restrict__ act, uint16_t* __restrict__ np, int32_t* __restrict__ len,
                           uint32_t* __restrict__ stst, int32_t* err) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_walks) return;
  const int64_t g = j0 + j < N ? j0 + j : N - 1;
  const int64_t i = g / K;
  const Key base = keys ? Key{keys[2 * (size_t)i], keys[2 * (size_t)i + 1]} : key;
  const uint64_t draw = keys ? (uint64_t)(g % K) : (uint64_t)(draw_base + g);
  typename Env::State s;
  unpack_terminal<Env>(P, terms + (size_t)i * P.SW, s);
  int16_t* a_out = act + (size_t)j * T;
  uint16_t* n_out = np + (size_t)j * T;
  if (!terminal_ok<Env>(P, s)) {
    atomicExch(err, GFNX_ERR_CONTRACT);  // backward_rollout: non-terminal input
    len[j] = 0;
    for (int t = 0; t < T; ++t) {
      a_out[t] = -1;
      n_out[t] = 0;
    }
    return;
  }
  const int L = walk_length<Env>(P, s);
  len[j] = L;
  for (int t = L; t < T; ++t) {
    a_out[t] = -1;
    n_out[t] = 0;
  }
  for (int t = 0; t < L; ++t) {
    const int nl = bwd_count<Env>(P, s);
    if (nl <= 0) {  // cannot happen on a valid terminal (the walk length is exact)
      atomicExch(err, GFNX_ERR_CONTRACT);
      return;
    }
    // categorical over unit weights: the first q with u < q + 1, fallback the last legal one
    const double u = uniform_scalar(fold_in(fold_in(base, (uint64_t)t), draw)) * (double)nl;
    int q = (int)u;
    if (q >= nl) q = nl - 1;
    const int ab = bwd_pick<Env>(P, s, q);
    const int f = L - 1 - t;  // forward step index of this transition
    n_out[f] = (uint16_t)nl;  // #parents of s_{f+1}: log_pb_uniform = -log(nl)
    a_out[f] = (int16_t)bwd_apply<Env>(P, s, ab);
    if (stst) Env::pack(P, s, stst + ((size_t)j * T + f) * P.SW);  // s_f, the state the step leaves
  }
}

template <class Env>
__global__ void k_replay(EnvParams P, const int16_t* __restrict__ forced, int Bl, int T, DeviceBatch batch,
                         uint32_t* __restrict__ stst) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= Bl) return;
  typename Env::State s;
  Env::reset(P, s);
  batch.lengths[b] = 0;
  batch.log_rewards[b] = 0.0;
  for (int t = 0; t < T; ++t) {
    const size_t bt = (size_t)b * T + t;
    const int a = forced[bt];
    if (a < 0 || a >= P.A || !Env::legal(P, s, a)) {
      atomicExch(batch.counters + 3, GFNX_ERR_CONTRACT);  // illegal / missing action
      return;
    }
    Env::pack(P, s, stst + bt * P.SW);
    const double prev_r = P.mdb ? Env::log_reward(P, s) : 0.0;
    const bool term = Env::step(P, s, a);
    batch.actions[bt] = (int16_t)a;
    batch.nparents[bt] = (uint16_t)Env::num_parents(P, s);
    batch.delta[bt] = (P.mdb && !term) ? Env::log_reward(P, s) - prev_r : 0.0;
    if (term) {
      batch.lengths[b] = t + 1;
      batch.log_rewards[b] = Env::log_reward(P, s);
      Env::pack(P, s, batch.term_state + (size_t)b * P.SW);
      for (int q = t + 1; q < T; ++q) batch.actions[(size_t)b * T + q] = -1;
      return;
    }
  }
  atomicExch(batch.counters + 3, GFNX_ERR_CONTRACT);  // never reached a terminal state
}

// per walk j of a chunk: log P_F(tau) - log P_B(tau | x), both summed in forward order
// (score_trajectories objectives.cpp:294-316 over the row log-probabilities [n][T]); log P_B
// is the uniform -log(#parents) or, with the learned backward policy, row_logpb
__global__ void k_mc_terms(const double* __restrict__ row_logpf, const double* __restrict__ row_logpb,
                           const uint16_t* __restrict__ np, const int32_t* __restrict__ len,
                           const double* __restrict__ neglog, int n, int T, double* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double lpf = 0.0, lpb = 0.0;
  for (int t = 0; t < len[j]; ++t) {
    lpf += row_logpf[(size_t)j * T + t];
    lpb += row_logpb ? row_logpb[(size_t)j * T + t] : neglog[np[(size_t)j * T + t]];
  }
  out[j] = lpf - lpb;
}

// the same from a fast-path eval record: row slot of (j, t) = row0[j] + t, log pi(a|s) at
// rowbuf[slot * rs + A]
__global__ void k_mc_terms_rows(const float* __restrict__ rowbuf, int rs, int A, const int32_t* __restrict__ row0,
                                const uint16_t* __restrict__ np, const int32_t* __restrict__ len,
                                const double* __restrict__ neglog, int n, int T, double* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double lpf = 0.0, lpb = 0.0;
  for (int t = 0; t < len[j]; ++t) {
    lpf += (double)rowbuf[(size_t)(row0[j] + t) * rs + A];
    lpb += neglog[np[(size_t)j * T + t]];
  }
  out[j] = lpf - lpb;
}

// logsumexp over the K walks of each terminal (sample order) - log K  (exact.hpp:236-240)
__global__ void k_mc_lse(const double* __restrict__ terms, int n, int K, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* x = terms + (size_t)i * K;
  double m = -INFINITY;
  for (int k = 0; k < K; ++k) m = x[k] > m ? x[k] : m;
  if (!isfinite(m)) {  // logsumexp (tensor.cpp:112-120) returns the non-finite max
    out[i] = m - log((double)K);
    return;
  }
  double se = 0.0;
  for (int k = 0; k < K; ++k) se += exp(x[k] - m);
  out[i] = m + log(se) - log((double)K);
}

// slot map of a compact row layout: rows of walk j at row0[j] .. row0[j] + len[j]
__global__ void k_walk_rows(const int32_t* __restrict__ len, const int32_t* __restrict__ row0, int n, int T,
                            int32_t* __restrict__ rows, int32_t* __restrict__ tiles, int kTileRows) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int R = row0[n];
  const int nt = (R + kTileRows - 1) / kTileRows;
  if (j < n)
    for (int t = 0; t < len[j]; ++t) rows[row0[j] + t] = j * T + t;
  if (j < kTileRows && R + j < nt * kTileRows) rows[R + j] = -1;
  if (j == 0) *tiles = nt;
}

template <class F>
void env_dispatch(const Ctx& c, F&& fn) {
  switch (c.env.kind) {
    case GFNX_ENV_HYPERGRID: fn(HypergridEnv{}); break;
    case GFNX_ENV_BITSEQ: fn(BitseqEnv{}); break;
    case GFNX_ENV_ISING: fn(IsingEnv{}); break;
    case GFNX_ENV_DAG: fn(DagEnv{}); break;
  }
}

// generate_test_set (sequences.cpp:100-119): for every mode m and flips f < n, the mode
// string with f distinct positions flipped, chosen by a partial Fisher-Yates shuffle whose
// draw counter runs across items (item (m, f) starts at draw m n(n-1)/2 + f(f-1)/2); written
// as packed terminal states (k-bit tokens MSB first, all slots filled) + the item keys
// fold_in(mkey, i) of the pearson metric (train.cpp:446-448)
__global__ void k_bs_testset(EnvParams P, Key key, Key mkey, uint32_t* __restrict__ terms, uint64_t* __restrict__ keys) {
  const int n = P.bs_nbits;
  const int item = blockIdx.x * blockDim.x + threadIdx.x;
  if (item >= P.n_modes * n) return;
  const int m = item / n, f = item % n;
  uint64_t bits[kMaxModeWords];
  for (int w = 0; w < kMaxModeWords; ++w) bits[w] = w < P.bs_words ? P.modes[(size_t)m * P.bs_words + w] : 0ull;
  uint16_t pos[kMaxModeWords * 64];
  for (int i = 0; i < n; ++i) pos[i] = (uint16_t)i;
  uint64_t draw = (uint64_t)m * ((uint64_t)n * (n - 1) / 2) + (uint64_t)f * (f - 1) / 2;
  for (int i = 0; i < f; ++i) {
    const int r = n - i;  // random_range (rng.cpp:82-85)
    const int j = i + (int)(uniform_scalar(fold_in(key, draw++)) * r) % r;
    const uint16_t x = pos[i];
    pos[i] = pos[j];
    pos[j] = x;
    const int b = pos[i];
    bits[b >> 6] ^= 1ull << (63 - (b & 63));
  }
  uint32_t* w = terms + (size_t)item * P.SW;
  for (int q = 0; q < P.SW; ++q) w[q] = 0u;
  const int tw = (P.bs_slots + 3) / 4;
  for (int s = 0; s < P.bs_slots; ++s) {
    uint32_t tok = 0;
    for (int b = 0; b < P.bs_k; ++b) {
      const int i = s * P.bs_k + b;
      tok = (tok << 1) | (uint32_t)((bits[i >> 6] >> (63 - (i & 63))) & 1ull);
    }
    w[s >> 2] |= tok << (8 * (s & 3));
    w[tw + (s >> 5)] |= 1u << (s & 31);
  }
  const Key k = fold_in(mkey, (uint64_t)item);
  keys[2 * (size_t)item] = k.hi;
  keys[2 * (size_t)item + 1] = k.lo;
}

__global__ void k_bs_log_reward(EnvParams P, const uint32_t* __restrict__ terms, int n, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  BitseqEnv::State s;
  BitseqEnv::unpack(P, terms + (size_t)i * P.SW, s);
  out[i] = BitseqEnv::log_reward(P, s);
}

// pearson (metrics.cpp:96-116), sequential in the reference's order
__global__ void k_pearson(const double* __restrict__ xs, const double* __restrict__ ys, int n, double* out,
                          int32_t* err) {
  const double nn = (double)n;
  double mx = 0.0, my = 0.0;
  for (int i = 0; i < n; ++i) {
    mx += xs[i];
    my += ys[i];
  }
  mx /= nn;
  my /= nn;
  double sxy = 0.0, sxx = 0.0, syy = 0.0;
  for (int i = 0; i < n; ++i) {
    const double dx = xs[i] - mx, dy = ys[i] - my;
    sxy += dx * dy;
    sxx += dx * dx;
    syy += dy * dy;
  }
  if (!(sxx > 0.0) || !(syy > 0.0)) {
    atomicExch(err, GFNX_ERR_NUMERIC);  // pearson: zero variance
    *out = 0.0;
    return;
  }
  *out = sxy / sqrt(sxx * syy);
}

}  // namespace

// the bitseq `pearson` metric (train.cpp:440-454): Pearson correlation of the device MC
// terminal log-probabilities (mc samples per string) and the log-rewards over the builder's
// test set (generate_test_set with key fold_in(make_key(test_seed), 0x7E57)); result in d_out
void bitseq_pearson(Ctx& c, int64_t step, int mc, uint64_t test_seed, double* d_out) {
  if (c.env.kind != GFNX_ENV_BITSEQ) raise_error(GFNX_ERR_CONFIG, "pearson: bitseq only");
  const int n = c.P.n_modes * c.P.bs_nbits;
  if (n < 2) raise_error(GFNX_ERR_CONTRACT, "pearson: need two equal-length series");
  uint32_t* d_t = nullptr;
  uint64_t* d_k = nullptr;
  double *d_lp = nullptr, *d_lr = nullptr;
  cuda_check(cudaMallocAsync(&d_t, sizeof(uint32_t) * (size_t)n * c.P.SW, c.stream), "pearson");
  cuda_check(cudaMallocAsync(&d_k, sizeof(uint64_t) * 2 * (size_t)n, c.stream), "pearson");
  cuda_check(cudaMallocAsync(&d_lp, sizeof(double) * (size_t)n, c.stream), "pearson");
  cuda_check(cudaMallocAsync(&d_lr, sizeof(double) * (size_t)n, c.stream), "pearson");
  const Key tkey = fold_in(make_key(test_seed), 0x7E57);
  const Key mkey = fold_in(fold_in(make_key(c.train.seed), 0x3E7A), (uint64_t)step);
  k_bs_testset<<<(n + 127) / 128, 128, 0, c.stream>>>(c.P, tkey, mkey, d_t, d_k);
  k_bs_log_reward<<<(n + 127) / 128, 128, 0, c.stream>>>(c.P, d_t, n, d_lr);
  c.launches += 2;
  mc_terminal_logprob_chunked(c, d_t, n, mc, d_k, d_lp);
  k_pearson<<<1, 1, 0, c.stream>>>(d_lp, d_lr, n, d_out, c.batch.counters + 3);
  c.launches++;
  for (void* p : {(void*)d_t, (void*)d_k, (void*)d_lp, (void*)d_lr}) cudaFreeAsync(p, c.stream);
}

void launch_bwd_walk(Ctx& c, const uint32_t* d_terms, int n_walks, int64_t j0, int64_t N, int K,
                     const uint64_t* d_keys, Key key, int64_t draw_base, int16_t* d_act, uint16_t* d_np,
                     int32_t* d_len, uint32_t* d_stst) {
  if (n_walks <= 0) return;
  if (c.train.learned_backward) {  // walks sampled from the policy's backward head (check mode)
    check_bwd_walk(c, d_terms, n_walks, j0, N, K, d_keys, key, draw_base, d_act, d_np, d_len);
    return;
  }
  env_dispatch(c, [&](auto e) {
    using Env = decltype(e);
    k_bwd_walk<Env><<<(n_walks + 127) / 128, 128, 0, c.stream>>>(c.P, d_terms, n_walks, j0, N, K, d_keys, key,
                                                                  draw_base, c.P.T, d_act, d_np, d_len, d_stst,
                                                                  c.batch.counters + 3);
  });
  c.launches++;
}

void launch_replay(Ctx& c, const int16_t* d_forced, uint32_t* d_stst) {
  env_dispatch(c, [&](auto e) {
    using Env = decltype(e);
    k_replay<Env><<<(c.Bl + 127) / 128, 128, 0, c.stream>>>(c.P, d_forced, c.Bl, c.P.T, c.batch, d_stst);
  });
  c.launches++;
}

void exclusive_scan_i32(Ctx& c, const int32_t* d_in, int32_t* d_out, int n) {
  // d_out[0..n]: exclusive prefix, d_out[n] = total (inclusive sums written one slot on)
  size_t tmp = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tmp, d_in, d_out + 1, n, c.stream);
  void* d_tmp = nullptr;
  cuda_check(cudaMallocAsync(&d_tmp, tmp, c.stream), "scan");
  cub::DeviceScan::InclusiveSum(d_tmp, tmp, d_in, d_out + 1, n, c.stream);
  cudaMemsetAsync(d_out, 0, sizeof(int32_t), c.stream);
  cuda_check(cudaFreeAsync(d_tmp, c.stream), "scan");
}

void launch_walk_rows(Ctx& c, const int32_t* d_len, const int32_t* d_row0, int n, int32_t* d_rows,
                      int32_t* d_tiles, int tile_rows) {
  k_walk_rows<<<(std::max(n, tile_rows) + 127) / 128, 128, 0, c.stream>>>(d_len, d_row0, n, c.P.T, d_rows, d_tiles,
                                                                           tile_rows);
  c.launches++;
}

void launch_mc_terms_rows(Ctx& c, const float* rowbuf, int rs, const int32_t* d_row0, const uint16_t* d_np,
                          const int32_t* d_len, int n, double* d_terms) {
  k_mc_terms_rows<<<(n + 127) / 128, 128, 0, c.stream>>>(rowbuf, rs, c.P.A, d_row0, d_np, d_len, c.d_neglog, n,
                                                          c.P.T, d_terms);
  c.launches++;
}

void launch_mc_lse(Ctx& c, const double* d_terms, int n, int K, double* d_out) {
  k_mc_lse<<<(n + 127) / 128, 128, 0, c.stream>>>(d_terms, n, K, d_out);
  c.launches++;
}

// teacher-forced batch of this rank's Bl trajectories from device actions [Bl * T]
void forced_rollout(Ctx& c, const int16_t* d_forced) {
  if (c.check_mode()) check_rollout(c, Key{0, 0}, 0.0, d_forced);
  else fast_forced_rollout(c, d_forced);
}

// backward_rollout (env_core.hpp:314-370) of Bl packed terminals (device) into the resident
// batch: walk draws b = b0 + j of `key`, then rollout_from_actions
void backward_rollout(Ctx& c, const uint32_t* d_terms, Key key) {
  const int Bl = c.Bl, T = c.P.T;
  int16_t* d_act = nullptr;
  uint16_t* d_np = nullptr;
  int32_t* d_len = nullptr;
  cuda_check(cudaMallocAsync(&d_act, sizeof(int16_t) * (size_t)Bl * T, c.stream), "walk");
  cuda_check(cudaMallocAsync(&d_np, sizeof(uint16_t) * (size_t)Bl * T, c.stream), "walk");
  cuda_check(cudaMallocAsync(&d_len, sizeof(int32_t) * (size_t)Bl, c.stream), "walk");
  launch_bwd_walk(c, d_terms, Bl, 0, Bl, 1, nullptr, key, c.b0, d_act, d_np, d_len, nullptr);
  forced_rollout(c, d_act);
  cudaFreeAsync(d_act, c.stream);
  cudaFreeAsync(d_np, c.stream);
  cudaFreeAsync(d_len, c.stream);
}

// mc_terminal_logprob through teacher-forced batches of Bl walks (lockstep and check paths):
// each chunk of walks becomes the resident batch, whose per-row log pi is then summed
void mc_terminal_logprob_chunked(Ctx& c, const uint32_t* d_terms, int64_t n, int K, const uint64_t* d_keys,
                                 double* d_out) {
  const int Bl = c.Bl, T = c.P.T;
  const int64_t N = n * K;
  int16_t* d_act = nullptr;
  uint16_t* d_np = nullptr;
  int32_t* d_len = nullptr;
  double *d_row = nullptr, *d_terms_all = nullptr;
  cuda_check(cudaMallocAsync(&d_act, sizeof(int16_t) * (size_t)Bl * T, c.stream), "mc");
  cuda_check(cudaMallocAsync(&d_np, sizeof(uint16_t) * (size_t)Bl * T, c.stream), "mc");
  cuda_check(cudaMallocAsync(&d_len, sizeof(int32_t) * (size_t)Bl, c.stream), "mc");
  cuda_check(cudaMallocAsync(&d_row, sizeof(double) * (size_t)Bl * T, c.stream), "mc");
  double* d_rowb = nullptr;  // learned backward policy: per-row log P_B of the bwd head
  if (c.train.learned_backward)
    cuda_check(cudaMallocAsync(&d_rowb, sizeof(double) * (size_t)Bl * T, c.stream), "mc");
  cuda_check(cudaMallocAsync(&d_terms_all, sizeof(double) * (size_t)((N + Bl - 1) / Bl) * Bl, c.stream), "mc");
  for (int64_t j0 = 0; j0 < N; j0 += Bl) {
    launch_bwd_walk(c, d_terms, Bl, j0, N, K, d_keys, Key{0, 0}, 0, d_act, d_np, d_len, nullptr);
    forced_rollout(c, d_act);
    launch_row_scan(c);
    c.rows_stale = false;
    if (c.check_mode()) {
      check_forward(c);
      check_row_logpf(c, d_row);
      if (d_rowb) check_row_logpb(c, d_rowb);
    } else {
      fast_row_logpf(c, d_row);
    }
    k_mc_terms<<<(Bl + 127) / 128, 128, 0, c.stream>>>(d_row, d_rowb, d_np, d_len, c.d_neglog, Bl, T,
                                                       d_terms_all + j0);
    c.launches++;
  }
  launch_mc_lse(c, d_terms_all, (int)n, K, d_out);
  for (void* p : {(void*)d_act, (void*)d_np, (void*)d_len, (void*)d_row, (void*)d_terms_all})
    cudaFreeAsync(p, c.stream);
  if (d_rowb) cudaFreeAsync(d_rowb, c.stream);
  c.has_batch = false;  // the resident batch now holds the last chunk of walks
  c.has_grads = false;
}

}  // namespace gfnx
