// eb.cu — EB-GFN on the device (run_eb_gfn, proj/src/train.cpp:875-1018): an energy-based
// Ising model J fitted by contrastive divergence while a GFlowNet sampler is trained with TB
// on the energy of the current J. One iteration = the kernels below + the ctx's own rollout
// (sampled + teacher-forced rows) and train step (api.cu gfnx_eb_run):
//
//   k_eb_select   sampler batch mixture (train.cpp:946-957): trajectory b is on-policy when
//                 uniform(fold_in(fold_in(it_key, 1), b)) < alpha, else it replays data row
//                 random_range(fold_in(fold_in(it_key, 2), b), N); on-policy rows first
//                 (forward_rollout of n_fwd), then the data-backed ones (backward_rollout,
//                 key fold_in(it_key, 4)) — TrajectoryBatch::concat order
//   k_eb_compose  forced-action rows of the mixed batch (-1 rows are sampled)
//   k_eb_pick     the CD data batch xs (train.cpp:976-980)
//   k_eb_bnf      back_and_forth_batch (ising.cpp:252-360): k uniform backward steps, the
//                 forward replay of tau scored by the policy, k fresh policy steps (tau'),
//                 the uniform backward score of tau'; fp64 SIMT in the reference's order
//                 (check mode); k_eb_bnf_fast: the same on the bf16 sampler's fp32 weights
//                 with block-parallel layers, softmax and draw (bf16 mode)
//   k_eb_mh       MH acceptance with the current J (mh_accept ising.cpp:369-373, dense
//                 ising_energy :40-51)
//   k_eb_cd       cd_gradient (ising.cpp:222-250: per element in data order, then the
//                 symmetrisation), J -= lr_J * grad, neg_log_rmse (:375-386), the metrics row
//
// Compiled with --fmad=false: the fp64 arithmetic of the proposal / acceptance / CD step is
// the reference's, so in fp64 check mode the whole loop is bit-exact with run_eb_gfn.
#include <math.h>

#include <algorithm>
#include <vector>

#include "check_common.cuh"
#include "engine.h"
#include "host.h"

namespace gfnx {

struct EbState {
  gfnx_eb_desc d{};
  int D = 0, N = 0, k = 0, db = 0, SW = 0;
  uint32_t* data = nullptr;  // [N][SW] packed terminal states
  double *Jm = nullptr, *Jt = nullptr, *grad = nullptr;
  int32_t* nfwd = nullptr;
  uint32_t* terms = nullptr;  // [B][SW] data-backed terminals, data slot order
  int16_t* wact = nullptr;    // [B][T] backward-walk forward actions
  uint16_t* wnp = nullptr;
  int32_t* wlen = nullptr;
  int16_t* forced = nullptr;  // [B][T]
  uint32_t *xs = nullptr, *props = nullptr, *acc = nullptr;  // [db][SW]
  double* logratio = nullptr;  // [db]
  int32_t* take = nullptr;     // [db]
  double *obs = nullptr, *logit = nullptr;  // [db][O], [db][A] scratch of the proposal kernel
  double* metrics = nullptr;   // [cap][4]
  int64_t cap = 0;
  double init_nlr = 0.0;
  std::vector<int8_t> host_data;
};

namespace {

EbState& EB(Ctx& c) {
  if (!c.eb) raise_error(GFNX_ERR_CONTRACT, "eb-gfn: call gfnx_eb_init first");
  return *static_cast<EbState*>(c.eb);
}

__device__ __forceinline__ int spin_of(const uint32_t* w, int half, int i) {
  if (!((w[i >> 5] >> (i & 31)) & 1u)) return 0;
  return ((w[half + (i >> 5)] >> (i & 31)) & 1u) ? 1 : -1;
}

__device__ double dense_energy(const uint32_t* w, int half, const double* J, int D) {  // ising.cpp:40-51
  double quad = 0.0;
  for (int a = 0; a < D; ++a) {
    double row = 0.0;
    for (int b = 0; b < D; ++b) row += J[(size_t)a * D + b] * (double)spin_of(w, half, b);
    quad += (double)spin_of(w, half, a) * row;
  }
  return -quad;
}

__global__ void __launch_bounds__(1024) k_eb_select(Key it_key, double alpha, int B, int N, const uint32_t* data,
                                                    int SW, int32_t* nfwd, uint32_t* terms) {
  __shared__ int wsum[32];
  __shared__ int carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < B; b0 += 1024) {
    const int b = b0 + tid;
    int row = -1;
    if (b < B && !(uniform_scalar(fold_in(fold_in(it_key, 1), (uint64_t)b)) < alpha)) {
      const double u = uniform_scalar(fold_in(fold_in(it_key, 2), (uint64_t)b));  // random_range rng.cpp:82-85
      row = (int)(u * N) % N;
    }
    const int v = row >= 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int w = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      wsum[lane] = w;
    }
    __syncthreads();
    const int i = carry + (warp ? wsum[warp - 1] : 0) + x - v;  // data slot of this row
    if (v)
      for (int q = 0; q < SW; ++q) terms[(size_t)i * SW + q] = data[(size_t)row * SW + q];
    __syncthreads();
    if (tid == 0) carry += wsum[31];
    __syncthreads();
  }
  const int n_data = carry;
  for (int i = n_data + tid; i < B; i += 1024)  // unused walk slots: any valid terminal
    for (int q = 0; q < SW; ++q) terms[(size_t)i * SW + q] = data[q];
  if (tid == 0) *nfwd = B - n_data;
}

__global__ void k_eb_compose(const int32_t* __restrict__ nfwd, const int16_t* __restrict__ wact, int B, int T,
                             int16_t* __restrict__ forced) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B * T) return;
  const int p = i / T, t = i % T, nf = *nfwd;
  forced[i] = p < nf ? (int16_t)-1 : wact[(size_t)(p - nf) * T + t];
}

__global__ void k_eb_pick(Key it_key, int db, int N, const uint32_t* __restrict__ data, int SW, uint32_t* xs) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= db) return;
  const double u = uniform_scalar(fold_in(fold_in(it_key, 5), (uint64_t)b));
  const int row = (int)(u * N) % N;
  for (int q = 0; q < SW; ++q) xs[(size_t)b * SW + q] = data[(size_t)row * SW + q];
}

// policy logits of state s into w[A] (mlp_forward, nn.cpp:60-89; every thread of the block)
// (Dl = the bwd-head layout with nout = Ab for the learned backward policy)
__device__ void policy_logits(const EnvParams& P, const DevLayout& Dl, const double* params, const IsingEnv::State& s,
                              double* obs, double (*hbuf)[512], double* w, int nout) {
  for (int i = threadIdx.x; i < P.O; i += blockDim.x) obs[i] = 0.0;
  __syncthreads();
  if (threadIdx.x == 0) IsingEnv::features(P, s, [&](int f, double v) { obs[f] = v; });
  __syncthreads();
  const double* h = obs;
  int in = P.O;
  for (int l = 0; l < Dl.n_trunk; ++l) {
    double* z = hbuf[l & 1];
    dense_block(h, in, params + Dl.off_w[l], params + Dl.off_b[l], Dl.dims[l + 1], z, true);
    __syncthreads();
    h = z;
    in = Dl.dims[l + 1];
  }
  dense_block(h, in, params + Dl.off_fw, params + Dl.off_fb, nout, w, false);
  __syncthreads();
}

// eps_uniform(logits, action_mask, A, 0.0) (objectives.cpp:242-264) in place; false on a
// non-finite maximum / no legal action (numeric_error / contract_violation)
__device__ bool eps0_probs(const EnvParams& P, const IsingEnv::State& s, double* w, bool bwd = false) {
  const int n = bwd ? P.Ab : P.A;
  auto ok = [&](int i) { return bwd ? (bool)((s.asg[i >> 5] >> (i & 31)) & 1u) : IsingEnv::legal(P, s, i); };
  int legal = 0;
  double hi = -INFINITY;
  for (int i = 0; i < n; ++i)
    if (ok(i)) {
      ++legal;
      if (w[i] > hi) hi = w[i];
    }
  if (legal == 0 || !isfinite(hi)) return false;
  double z = 0.0;
  for (int i = 0; i < n; ++i) {
    if (ok(i)) {
      const double p = exp(w[i] - hi);
      w[i] = p;
      z += p;
    } else {
      w[i] = 0.0;
    }
  }
  const double u = 0.0 / legal;
  for (int i = 0; i < n; ++i)
    if (ok(i)) w[i] = (1.0 - 0.0) * w[i] / z + u;
  return true;
}

__device__ int nth_assigned(const IsingEnv::State& s, int D, int q) {
  for (int w = 0; w < (D + 31) / 32; ++w) {
    const int n = __popc(s.asg[w]);
    if (q < n) {
      uint32_t x = s.asg[w];
      for (int i = 0; i < q; ++i) x &= x - 1;
      return 32 * w + __ffs(x) - 1;
    }
    q -= n;
  }
  return -1;
}

__device__ void unassign(IsingEnv::State& s, int site) {  // backward_step_instance
  const uint32_t bit = 1u << (site & 31);
  s.asg[site >> 5] &= ~bit;
  s.up[site >> 5] &= ~bit;
  s.count -= 1;
  s.step -= 1;
  s.term = false;
}

__global__ void k_eb_bnf(EnvParams P, DevLayout Dl, const double* __restrict__ params, Key key, int k,
                         const uint32_t* __restrict__ xs, uint32_t* __restrict__ props, double* __restrict__ logratio,
                         double* obs_scratch, double* logit_scratch, int32_t* err, int learned, DevLayout Db) {
  const int b = blockIdx.x;
  const int D = P.is_D, half = P.SW / 2;
  __shared__ IsingEnv::State s, partial;
  __shared__ double hbuf[2][512];
  __shared__ int16_t removed[kMaxIsingD], added[kMaxIsingD];
  __shared__ int bad;
  double* obs = obs_scratch + (size_t)b * P.O;
  double* w = logit_scratch + (size_t)b * (P.A > P.Ab ? P.A : P.Ab);
  const uint32_t* x = xs + (size_t)b * P.SW;
  double lr = 0.0;  // thread 0
  if (threadIdx.x == 0) {
    bad = 0;
    IsingEnv::unpack(P, x, s);
    s.term = true;
    s.step = s.count;
    // phase 1: k backward steps under the uniform backward policy, - log P_B(tau | x)
    for (int step = 0; step < k && !learned; ++step) {
      const int nl = s.count;
      const Key sk = fold_in(fold_in(key, 100), (uint64_t)step);
      int q = (int)(uniform_scalar(fold_in(sk, (uint64_t)b)) * (double)nl);
      if (q >= nl) q = nl - 1;
      const int site = nth_assigned(s, D, q);
      lr -= log(1.0 / (double)nl);  // probs[site] / total with unit weights
      unassign(s, site);
      removed[step] = (int16_t)site;
    }
  }
  __syncthreads();
  for (int step = 0; step < k && learned; ++step) {  // phase 1 under the learned backward head
    policy_logits(P, Db, params, s, obs, hbuf, w, P.Ab);
    if (threadIdx.x == 0) {
      if (!eps0_probs(P, s, w, true)) bad = GFNX_ERR_NUMERIC;
      double total = 0.0;  // categorical (rng.cpp:87-100)
      for (int i = 0; i < P.Ab; ++i) total += w[i];
      const Key sk = fold_in(fold_in(key, 100), (uint64_t)step);
      const double uu = uniform_scalar(fold_in(sk, (uint64_t)b)) * total;
      int site = -1;
      double acc = 0.0;
      for (int i = 0; i < P.Ab; ++i) {
        acc += w[i];
        if (uu < acc) {
          site = i;
          break;
        }
      }
      if (site < 0)
        for (int i = P.Ab - 1; i >= 0; --i)
          if (w[i] > 0.0) {
            site = i;
            break;
          }
      if (site < 0) {
        bad = GFNX_ERR_CONTRACT;
        site = nth_assigned(s, D, 0);
      }
      lr -= log(w[site] / total);
      unassign(s, site);
      removed[step] = (int16_t)site;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) partial = s;
  __syncthreads();
  // phase 2: forward replay of tau from the partial state, + log P_F(tau)
  for (int step = 0; step < k; ++step) {
    policy_logits(P, Dl, params, s, obs, hbuf, w, P.A);
    if (threadIdx.x == 0) {
      if (!eps0_probs(P, s, w)) bad = GFNX_ERR_NUMERIC;
      const int site = removed[k - 1 - step];
      const int action = 2 * site + (spin_of(x, half, site) > 0 ? 1 : 0);
      lr += log(w[action]);
      IsingEnv::step(P, s, action);
    }
    __syncthreads();
  }
  // phase 3: k fresh policy steps from the partial state (tau'), - log P_F(tau')
  if (threadIdx.x == 0) s = partial;
  __syncthreads();
  for (int step = 0; step < k; ++step) {
    policy_logits(P, Dl, params, s, obs, hbuf, w, P.A);
    if (threadIdx.x == 0) {
      if (!eps0_probs(P, s, w)) bad = GFNX_ERR_NUMERIC;
      double total = 0.0;  // categorical (rng.cpp:87-100)
      for (int i = 0; i < P.A; ++i) total += w[i];
      const Key sk = fold_in(fold_in(key, 300), (uint64_t)step);
      const double uu = uniform_scalar(fold_in(sk, (uint64_t)b)) * total;
      int a = -1;
      double acc = 0.0;
      for (int i = 0; i < P.A; ++i) {
        acc += w[i];
        if (uu < acc) {
          a = i;
          break;
        }
      }
      if (a < 0)
        for (int i = P.A - 1; i >= 0; --i)
          if (w[i] > 0.0) {
            a = i;
            break;
          }
      if (a < 0) {
        bad = GFNX_ERR_CONTRACT;
        a = 0;
      }
      lr -= log(w[a]);
      IsingEnv::step(P, s, a);
      added[step] = (int16_t)(a / 2);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    IsingEnv::pack(P, s, props + (size_t)b * P.SW);
    // phase 4: the uniform backward score of tau' from x', + log P_B(tau' | x')
    for (int step = 0; step < k && !learned; ++step) {
      lr += -log((double)s.count);
      unassign(s, added[k - 1 - step]);
    }
  }
  __syncthreads();
  for (int step = 0; step < k && learned; ++step) {  // phase 4 under the learned backward head
    policy_logits(P, Db, params, s, obs, hbuf, w, P.Ab);
    if (threadIdx.x == 0) {
      if (!eps0_probs(P, s, w, true)) bad = GFNX_ERR_NUMERIC;
      const int site = added[k - 1 - step];
      lr += log(w[site]);
      unassign(s, site);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    logratio[b] = lr;
    if (bad) atomicExch(err, bad);
  }
}

// ---- bf16 mode: the proposal's policy evaluations in fp32 on the block (the sampler is the
// bf16 policy, so the fp64 reference order buys nothing here): layer 1 as the sum of the D
// active one-hot rows (ising.cpp:122-129 features), dense layers with four independent
// accumulators per output, softmax statistics and the inverse-CDF draw by block reductions /
// a block scan in fp64 instead of thread 0's serial loops.
constexpr int kBnfThreads = 256;

__device__ float block_reduce_f(float v, float* red, bool is_max) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float y = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmaxf(v, y) : v + y;
  }
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float t = red[0];
  for (int q = 1; q < kBnfThreads / 32; ++q) t = is_max ? fmaxf(t, red[q]) : t + red[q];
  return t;
}

// logits of state s (fp32) into lg[nout]; h[2][512] fp32 scratch
__device__ void policy_logits_f32(const EnvParams& P, const DevLayout& Dl, const float* __restrict__ params,
                                  const IsingEnv::State& s, float (*h)[512], float* lg, int nout) {
  const int H1 = Dl.dims[1];
  for (int j = threadIdx.x; j < H1; j += blockDim.x) {  // layer 1: b1 + sum of the active rows
    float acc[4] = {params[Dl.off_b[0] + j], 0.f, 0.f, 0.f};
    for (int i = 0; i < P.is_D; ++i) {
      const int v = IsingEnv::spin(s, i);
      const int f = 3 * i + (v == 0 ? 2 : (v > 0 ? 1 : 0));
      acc[i & 3] += params[Dl.off_w[0] + (size_t)f * H1 + j];
    }
    h[0][j] = fmaxf((acc[0] + acc[1]) + (acc[2] + acc[3]), 0.f);
  }
  __syncthreads();
  int in = H1, cur = 0;
  auto dense = [&](int64_t off_w, int64_t off_b, int out, const float* x, float* y, bool relu) {
    for (int j = threadIdx.x; j < out; j += blockDim.x) {
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      const float* W = params + off_w + j;
      int p = 0;
      for (; p + 3 < in; p += 4) {
        acc[0] += x[p] * W[(size_t)p * out];
        acc[1] += x[p + 1] * W[(size_t)(p + 1) * out];
        acc[2] += x[p + 2] * W[(size_t)(p + 2) * out];
        acc[3] += x[p + 3] * W[(size_t)(p + 3) * out];
      }
      for (; p < in; ++p) acc[0] += x[p] * W[(size_t)p * out];
      const float z = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + params[off_b + j];
      y[j] = relu ? fmaxf(z, 0.f) : z;
    }
  };
  for (int l = 1; l < Dl.n_trunk; ++l) {
    dense(Dl.off_w[l], Dl.off_b[l], Dl.dims[l + 1], h[cur], h[cur ^ 1], true);
    __syncthreads();
    cur ^= 1;
    in = Dl.dims[l + 1];
  }
  dense(Dl.off_fw, Dl.off_fb, nout, h[cur], lg, false);
  __syncthreads();
}

// log pi(a | s) of every action (masked log-softmax, eps = 0) -> logp[A]; returns nothing
__device__ void masked_logp_f32(const EnvParams& P, const IsingEnv::State& s, const float* lg, float* logp,
                                float* red) {
  float hi = -INFINITY;
  for (int c = threadIdx.x; c < P.A; c += blockDim.x)
    if (IsingEnv::legal(P, s, c)) hi = fmaxf(hi, lg[c]);
  hi = block_reduce_f(hi, red, true);
  float z = 0.f;
  for (int c = threadIdx.x; c < P.A; c += blockDim.x)
    if (IsingEnv::legal(P, s, c)) z += __expf(lg[c] - hi);
  z = block_reduce_f(z, red, false);
  const float lse = hi + __logf(z);
  for (int c = threadIdx.x; c < P.A; c += blockDim.x) logp[c] = IsingEnv::legal(P, s, c) ? lg[c] - lse : -INFINITY;
  __syncthreads();
}

__global__ void __launch_bounds__(kBnfThreads) k_eb_bnf_fast(EnvParams P, DevLayout Dl, const float* __restrict__ params,
                                                            Key key, int k, const uint32_t* __restrict__ xs,
                                                            uint32_t* __restrict__ props,
                                                            double* __restrict__ logratio, int32_t* err) {
  const int b = blockIdx.x;
  const int D = P.is_D, half = P.SW / 2;
  __shared__ IsingEnv::State s, partial;
  __shared__ float h[2][512];
  __shared__ float lg[512], logp[512];
  __shared__ float red[kBnfThreads / 32];
  __shared__ double scan[kBnfThreads];
  __shared__ int16_t removed[kMaxIsingD], added[kMaxIsingD];
  __shared__ int s_pick;
  const uint32_t* x = xs + (size_t)b * P.SW;
  double lr = 0.0;  // thread 0
  if (threadIdx.x == 0) {  // phase 1: k uniform backward steps, - log P_B(tau | x)
    IsingEnv::unpack(P, x, s);
    s.term = true;
    s.step = s.count;
    for (int step = 0; step < k; ++step) {
      const int nl = s.count;
      const Key sk = fold_in(fold_in(key, 100), (uint64_t)step);
      int q = (int)(uniform_scalar(fold_in(sk, (uint64_t)b)) * (double)nl);
      if (q >= nl) q = nl - 1;
      const int site = nth_assigned(s, D, q);
      lr -= log(1.0 / (double)nl);
      unassign(s, site);
      removed[step] = (int16_t)site;
    }
    partial = s;
  }
  __syncthreads();
  for (int step = 0; step < k; ++step) {  // phase 2: forward replay of tau, + log P_F(tau)
    policy_logits_f32(P, Dl, params, s, h, lg, P.A);
    masked_logp_f32(P, s, lg, logp, red);
    if (threadIdx.x == 0) {
      const int site = removed[k - 1 - step];
      const int action = 2 * site + (spin_of(x, half, site) > 0 ? 1 : 0);
      lr += (double)logp[action];
      IsingEnv::step(P, s, action);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) s = partial;
  __syncthreads();
  for (int step = 0; step < k; ++step) {  // phase 3: k fresh policy steps (tau'), - log P_F(tau')
    policy_logits_f32(P, Dl, params, s, h, lg, P.A);
    masked_logp_f32(P, s, lg, logp, red);
    // categorical (rng.cpp:87-100) over p_c = exp(logp_c): fp64 block scan in column order
    const Key sk = fold_in(fold_in(key, 300), (uint64_t)step);
    const double u01 = uniform_scalar(fold_in(sk, (uint64_t)b));
    double carry = 0.0;
    if (threadIdx.x == 0) s_pick = -1;
    for (int c0 = 0; c0 < P.A; c0 += kBnfThreads) {
      const int c = c0 + threadIdx.x;
      const double wv = c < P.A && logp[c] > -INFINITY ? (double)__expf(logp[c]) : 0.0;
      scan[threadIdx.x] = wv;
      __syncthreads();
      for (int o = 1; o < kBnfThreads; o <<= 1) {  // inclusive Hillis-Steele scan
        const double y = threadIdx.x >= o ? scan[threadIdx.x - o] : 0.0;
        __syncthreads();
        scan[threadIdx.x] += y;
        __syncthreads();
      }
      scan[threadIdx.x] += carry;
      __syncthreads();
      carry = scan[kBnfThreads - 1];
      __syncthreads();
      // the pick needs the total: keep this chunk's running sums (h is free scratch here;
      // its 4 KB hold A <= 512 doubles)
      if (c < P.A) reinterpret_cast<double*>(h)[c] = scan[threadIdx.x];
      __syncthreads();
    }
    const double total = carry;
    const double target = u01 * total;
    for (int c = threadIdx.x; c < P.A; c += blockDim.x) {
      const double incl = reinterpret_cast<const double*>(h)[c];
      const double excl = c > 0 ? reinterpret_cast<const double*>(h)[c - 1] : 0.0;
      if (incl > excl && target < incl && target >= excl) atomicMax(&s_pick, c);  // the unique crossing column
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int a = s_pick;
      if (a < 0)  // rounding fallback: the last legal column
        for (int c = P.A - 1; c >= 0; --c)
          if (logp[c] > -INFINITY) {
            a = c;
            break;
          }
      if (a < 0) {
        atomicExch(err, GFNX_ERR_CONTRACT);
        a = 0;
      }
      lr -= (double)logp[a];
      IsingEnv::step(P, s, a);
      added[step] = (int16_t)(a / 2);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    IsingEnv::pack(P, s, props + (size_t)b * P.SW);
    for (int step = 0; step < k; ++step) {  // phase 4: the uniform backward score of tau' from x'
      lr += -log((double)s.count);
      unassign(s, added[k - 1 - step]);
    }
    logratio[b] = lr;
  }
}

// one block per sample: thread a computes row a of both energies (sequential over b, the
// reference's order), thread 0 then folds quad += s_a * row_a in a order -> bit-exact
__global__ void __launch_bounds__(128) k_eb_mh(Key it_key, int db, const EnvParams P, const double* __restrict__ Jm,
                                               const uint32_t* __restrict__ xs, const uint32_t* __restrict__ props,
                                               const double* __restrict__ logratio, uint32_t* __restrict__ acc,
                                               int32_t* __restrict__ take) {
  const int b = blockIdx.x;
  if (b >= db) return;
  const int D = P.is_D, half = P.SW / 2;
  const uint32_t* x = xs + (size_t)b * P.SW;
  const uint32_t* y = props + (size_t)b * P.SW;
  __shared__ double rx[kMaxIsingD], ry[kMaxIsingD];
  __shared__ int8_t sx[kMaxIsingD], sy[kMaxIsingD];
  for (int i = threadIdx.x; i < D; i += blockDim.x) {
    sx[i] = (int8_t)spin_of(x, half, i);
    sy[i] = (int8_t)spin_of(y, half, i);
  }
  __syncthreads();
  for (int a = threadIdx.x; a < D; a += blockDim.x) {  // ising_energy's row sums (ising.cpp:44-48)
    const double* J = Jm + (size_t)a * D;
    double r1 = 0.0, r2 = 0.0;
    for (int c = 0; c < D; ++c) {
      r1 += J[c] * (double)sx[c];
      r2 += J[c] * (double)sy[c];
    }
    rx[a] = r1;
    ry[a] = r2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double qx = 0.0, qy = 0.0;
    for (int a = 0; a < D; ++a) {
      qx += (double)sx[a] * rx[a];
      qy += (double)sy[a] * ry[a];
    }
    const double ex = -qx, ep = -qy;
    const double log_a = -ep + ex + logratio[b];  // mh_accept ising.cpp:369-373
    bool t = log_a >= 0.0;
    if (!t) t = log(uniform_scalar(fold_in(fold_in(it_key, 7), (uint64_t)b))) < log_a;
    take[b] = t ? 1 : 0;
    for (int q = 0; q < P.SW; ++q) acc[(size_t)b * P.SW + q] = t ? y[q] : x[q];
  }
}

// cd_gradient's per-element sums (ising.cpp:230-240: grad[a][b] += scale * (-x_a x_b + y_a y_b)
// over the data in order): the batch's spins are staged in shared memory, thread per element
constexpr int kCdThreads = 256, kCdGrid = 148, kCdMaxSmem = 96 * 1024;
__global__ void __launch_bounds__(kCdThreads) k_eb_cd_grad(int db, int chunk, const EnvParams P,
                                                           const uint32_t* __restrict__ xs,
                                                           const uint32_t* __restrict__ ys, double* __restrict__ g) {
  extern __shared__ int8_t sp[];  // [chunk][D] data spins, then [chunk][D] accepted spins
  const int D = P.is_D, half = P.SW / 2, n = D * D;
  const double scale = 1.0 / (double)db;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};  // elements e0 + k * stride of this thread (n <= 4 * stride)
  const int e0 = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  for (int i0 = 0; i0 < db; i0 += chunk) {  // samples in order, chunk by chunk
    const int m = min(chunk, db - i0);
    __syncthreads();
    for (int q = threadIdx.x; q < m * D; q += blockDim.x) {
      const int i = q / D, c = q % D;
      sp[q] = (int8_t)spin_of(xs + (size_t)(i0 + i) * P.SW, half, c);
      sp[m * D + q] = (int8_t)spin_of(ys + (size_t)(i0 + i) * P.SW, half, c);
    }
    __syncthreads();
    const int8_t* X = sp;
    const int8_t* Y = sp + m * D;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = e0 + k * stride;
      if (e >= n) break;
      const int a = e / D, c = e % D;
      if (a == c) continue;
      double v = acc[k];
      for (int i = 0; i < m; ++i)
        v += scale * (-(double)X[i * D + a] * (double)X[i * D + c] + (double)Y[i * D + a] * (double)Y[i * D + c]);
      acc[k] = v;
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (e0 + k * stride < n) g[e0 + k * stride] = acc[k];
}

// symmetrisation, J -= lr_J * grad, neg_log_rmse (ising.cpp:241-250, 375-386), the metrics row
__global__ void __launch_bounds__(1024) k_eb_cd_update(int db, const EnvParams P, const int32_t* __restrict__ take,
                                                       double* Jm, const double* __restrict__ Jt, double* g,
                                                       double j_lr, const double* __restrict__ scalars,
                                                       double* metrics_row) {
  const int D = P.is_D, n = D * D;
  for (int e = threadIdx.x; e < n; e += blockDim.x) {  // symmetrize
    const int a = e / D, c = e % D;
    if (c < a) {
      const double m = 0.5 * (g[(size_t)a * D + c] + g[(size_t)c * D + a]);
      g[(size_t)a * D + c] = m;
      g[(size_t)c * D + a] = m;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n; e += blockDim.x) Jm[e] -= j_lr * g[e];
  __syncthreads();
  if (threadIdx.x == 0) {
    double acc = 0.0;  // neg_log_rmse (ising.cpp:375-386)
    for (int e = 0; e < n; ++e) {
      const double diff = Jt[e] - Jm[e];
      acc += diff * diff;
    }
    const double rmse = sqrt(acc / ((double)D * D));
    int nacc = 0;
    for (int i = 0; i < db; ++i) nacc += take[i];
    metrics_row[0] = scalars[4];  // the train_step loss of this iteration
    metrics_row[1] = scalars[0];  // log Z after the update
    metrics_row[2] = rmse == 0.0 ? INFINITY : -log(rmse);
    metrics_row[3] = (double)nacc;
  }
}


double host_nlr(const std::vector<double>& jt, const std::vector<double>& jm, int D) {
  double acc = 0.0;
  for (size_t i = 0; i < jt.size(); ++i) {
    const double diff = jt[i] - jm[i];
    acc += diff * diff;
  }
  const double rmse = sqrt(acc / ((double)D * D));
  return rmse == 0.0 ? INFINITY : -log(rmse);
}

}  // namespace

void eb_default_desc(gfnx_eb_desc* d) {  // run_eb_gfn's cfg defaults (train.cpp:899-913)
  *d = gfnx_eb_desc{};
  d->data_samples = 2000;
  d->k = 0;
  d->gibbs_burn_in = 2000;
  d->gibbs_thinning = 10;
  d->gibbs_chains = 1;
  d->data_batch = 0;
  d->gibbs_hottest_beta = 0.2;
  d->alpha = 0.5;
  d->coupling_lr = 0.05;
  d->coupling_lr_end = 0.05;
}

void eb_free(Ctx& c) {
  if (!c.eb) return;
  EbState& e = *static_cast<EbState*>(c.eb);
  void* ptrs[] = {e.data, e.Jm, e.Jt, e.grad, e.nfwd, e.terms, e.wact, e.wnp, e.wlen, e.forced, e.xs, e.props,
                  e.acc, e.logratio, e.take, e.obs, e.logit, e.metrics};
  for (void* p : ptrs) cudaFree(p);
  delete &e;
  c.eb = nullptr;
}

void eb_init(Ctx& c, const gfnx_eb_desc& d, const int8_t* data, int64_t n) {
  if (c.env.kind != GFNX_ENV_ISING) raise_error(GFNX_ERR_CONFIG, "eb-gfn: Ising env only");
  if (c.train.objective != GFNX_OBJ_TB) raise_error(GFNX_ERR_CONFIG, "eb-gfn: the sampler objective must be tb");
  if (c.world != 1) raise_error(GFNX_ERR_CONFIG, "eb-gfn: single-rank loop");
  const int D = c.P.is_D;
  if (d.k > D) raise_error(GFNX_ERR_CONFIG, "back_and_forth: k must lie in [0, D]");
  if (!(d.alpha >= 0.0 && d.alpha <= 1.0)) raise_error(GFNX_ERR_CONFIG, "eb-gfn: alpha must lie in [0, 1]");
  eb_free(c);
  auto* e = new EbState();
  c.eb = e;
  e->d = d;
  e->D = D;
  e->SW = c.P.SW;
  e->k = d.k <= 0 ? D : d.k;
  e->db = d.data_batch > 0 ? d.data_batch : c.B;
  // data: caller-supplied or the reference's Gibbs sampler on the true coupling
  const std::vector<double> jt = ising_dense_coupling(c.env.is_side, c.env.is_sigma);
  if (data) {
    if (n < 1) raise_error(GFNX_ERR_CONFIG, "eb-gfn: empty data set");
    e->host_data.assign(data, data + (size_t)n * D);
    for (int8_t v : e->host_data)
      if (v != 1 && v != -1) raise_error(GFNX_ERR_CONTRACT, "ising: incomplete terminal spins");
  } else {
    if (d.gibbs_chains < 1) raise_error(GFNX_ERR_CONFIG, "gibbs: need at least one chain");
    if (d.data_samples < 1 || d.gibbs_thinning < 1) raise_error(GFNX_ERR_CONFIG, "gibbs: bad sample counts");
    e->host_data = ising_gibbs_data(jt, D, fold_in(make_key(c.train.seed), 0x919B), d.data_samples,
                                    d.gibbs_burn_in, d.gibbs_thinning, d.gibbs_chains, d.gibbs_hottest_beta);
  }
  e->N = (int)(e->host_data.size() / D);
  std::vector<uint32_t> packed((size_t)e->N * e->SW, 0u);
  const int half = e->SW / 2;
  for (int r = 0; r < e->N; ++r)
    for (int i = 0; i < D; ++i) {
      packed[(size_t)r * e->SW + (i >> 5)] |= 1u << (i & 31);
      if (e->host_data[(size_t)r * D + i] > 0) packed[(size_t)r * e->SW + half + (i >> 5)] |= 1u << (i & 31);
    }
  const int B = c.Bl, T = c.P.T, db = e->db;
  auto alloc = [&](auto** p, size_t bytes) { cuda_check(cudaMalloc((void**)p, bytes), "eb-gfn alloc"); };
  alloc(&e->data, sizeof(uint32_t) * packed.size());
  alloc(&e->Jm, sizeof(double) * D * D);
  alloc(&e->Jt, sizeof(double) * D * D);
  alloc(&e->grad, sizeof(double) * D * D);
  alloc(&e->nfwd, sizeof(int32_t));
  alloc(&e->terms, sizeof(uint32_t) * (size_t)B * e->SW);
  alloc(&e->wact, sizeof(int16_t) * (size_t)B * T);
  alloc(&e->wnp, sizeof(uint16_t) * (size_t)B * T);
  alloc(&e->wlen, sizeof(int32_t) * (size_t)B);
  alloc(&e->forced, sizeof(int16_t) * (size_t)B * T);
  alloc(&e->xs, sizeof(uint32_t) * (size_t)db * e->SW);
  alloc(&e->props, sizeof(uint32_t) * (size_t)db * e->SW);
  alloc(&e->acc, sizeof(uint32_t) * (size_t)db * e->SW);
  alloc(&e->logratio, sizeof(double) * db);
  alloc(&e->take, sizeof(int32_t) * db);
  alloc(&e->obs, sizeof(double) * (size_t)db * c.P.O);
  alloc(&e->logit, sizeof(double) * (size_t)db * std::max(c.P.A, c.P.Ab));
  cuda_check(cudaMemcpy(e->data, packed.data(), sizeof(uint32_t) * packed.size(), cudaMemcpyHostToDevice), "eb data");
  cuda_check(cudaMemcpy(e->Jt, jt.data(), sizeof(double) * D * D, cudaMemcpyHostToDevice), "eb J*");
  cuda_check(cudaMemset(e->Jm, 0, sizeof(double) * D * D), "eb J");  // zero_coupling
  e->init_nlr = host_nlr(jt, std::vector<double>((size_t)D * D, 0.0), D);
  c.P.is_Jd = e->Jm;  // the sampler's reward is the model energy from now on
}

void eb_ensure_metrics(Ctx& c, int64_t n) {
  EbState& e = EB(c);
  if (n <= e.cap) return;
  cudaFree(e.metrics);
  cuda_check(cudaMalloc(&e.metrics, sizeof(double) * 4 * n), "eb metrics");
  e.cap = n;
}

// the mixture rows of iteration it: returns the device forced-action matrix of the batch
const int16_t* eb_pre(Ctx& c, Key it_key) {
  EbState& e = EB(c);
  const int B = c.Bl, T = c.P.T;
  k_eb_select<<<1, 1024, 0, c.stream>>>(it_key, e.d.alpha, B, e.N, e.data, e.SW, e.nfwd, e.terms);
  // backward_rollout(terms, fold_in(it_key, 4)): draw i for data slot i (walks past n_data unused)
  launch_bwd_walk(c, e.terms, B, 0, B, 1, nullptr, fold_in(it_key, 4), 0, e.wact, e.wnp, e.wlen, nullptr);
  k_eb_compose<<<(B * T + 255) / 256, 256, 0, c.stream>>>(e.nfwd, e.wact, B, T, e.forced);
  c.launches += 2;
  return e.forced;
}

// the energy-model half of iteration it (train.cpp:974-995), metrics into row i
void eb_post(Ctx& c, Key it_key, double j_lr, int64_t i) {
  EbState& e = EB(c);
  const DevLayout Dl = make_dev_layout(c);
  DevLayout Db = Dl;  // the learned backward head (LossConfig::learned_backward)
  Db.off_fw = c.L.off_bw;
  Db.off_fb = c.L.off_bb;
  Db.A = c.P.Ab;
  k_eb_pick<<<(e.db + 127) / 128, 128, 0, c.stream>>>(it_key, e.db, e.N, e.data, e.SW, e.xs);
  if (c.check_mode()) {  // fp64, the reference's operation order (bit-exact with run_eb_gfn)
    k_eb_bnf<<<e.db, 256, 0, c.stream>>>(c.P, Dl, c.p64, fold_in(it_key, 6), e.k, e.xs, e.props, e.logratio, e.obs,
                                         e.logit, c.batch.counters + 3, c.train.learned_backward, Db);
  } else {  // the bf16 sampler's fp32 master weights, block-parallel evaluation
    k_eb_bnf_fast<<<e.db, kBnfThreads, 0, c.stream>>>(c.P, Dl, c.p32, fold_in(it_key, 6), e.k, e.xs, e.props,
                                                      e.logratio, c.batch.counters + 3);
  }
  k_eb_mh<<<e.db, 128, 0, c.stream>>>(it_key, e.db, c.P, e.Jm, e.xs, e.props, e.logratio, e.acc, e.take);
  const int chunk = std::min(e.db, kCdMaxSmem / (2 * e.D));
  static bool cd_attr = false;
  if (!cd_attr) {
    cudaFuncSetAttribute(k_eb_cd_grad, cudaFuncAttributeMaxDynamicSharedMemorySize, kCdMaxSmem);
    cd_attr = true;
  }
  k_eb_cd_grad<<<kCdGrid, kCdThreads, 2 * chunk * e.D, c.stream>>>(e.db, chunk, c.P, e.xs, e.acc, e.grad);
  k_eb_cd_update<<<1, 1024, 0, c.stream>>>(e.db, c.P, e.take, e.Jm, e.Jt, e.grad, j_lr, c.d_scalars,
                                           e.metrics + 4 * i);
  c.launches += 5;
}

const double* eb_metrics(Ctx& c) { return EB(c).metrics; }

// coupling_sched (train.cpp:913-914): linear coupling_lr -> coupling_lr_end over the run
double eb_coupling_lr(Ctx& c, int64_t it) {
  EbState& e = EB(c);
  gfnx_schedule s{};
  s.kind = 1;
  s.start_value = e.d.coupling_lr;
  s.end_value = e.d.coupling_lr_end;
  s.warmup = 0;
  s.horizon = std::max<int64_t>(1, c.train.iterations);
  return schedule_value(s, it);
}

void eb_coupling(Ctx& c, double* jm, double* jt, double* init_nlr) {
  EbState& e = EB(c);
  const size_t n = (size_t)e.D * e.D;
  cuda_check(cudaStreamSynchronize(c.stream), "eb sync");
  if (jm) cuda_check(cudaMemcpy(jm, e.Jm, sizeof(double) * n, cudaMemcpyDeviceToHost), "eb J");
  if (jt) cuda_check(cudaMemcpy(jt, e.Jt, sizeof(double) * n, cudaMemcpyDeviceToHost), "eb J*");
  if (init_nlr) *init_nlr = e.init_nlr;
}

int64_t eb_dataset(Ctx& c, int8_t* out, int64_t n) {
  EbState& e = EB(c);
  if (out) {
    if (n != (int64_t)e.host_data.size()) raise_error(GFNX_ERR_CONFIG, "eb dataset: size must be n_samples * D");
    std::copy(e.host_data.begin(), e.host_data.end(), out);
  }
  return e.N;
}

}  // namespace gfnx
