// bitseq.cu — bf16 tcgen05 fast path for the non-autoregressive bit-sequence environment
// (SequenceEnv NAR scheme + ModeSet reward, proj/src/envs/sequences.cpp; BASELINE config
// #3: n = 120, k = 8 -> 15 slots x 256 words, A = 3840, obs 3856, T = 15, MLP 2 x 256, TB).
//
// Every trajectory takes exactly T = #slots steps, so the batch advances in lockstep and
// the rows of the training pass are laid out step-major: row r = t * Bl + b. The rollout's
// forward IS the training forward (same parameters inside an iteration): the h1 / h2
// activation images, ReLU masks and the per-row log-softmax statistics it produces are
// consumed by the backward directly, with no second forward pass.
//
// Per rollout step t (4 launches):
//   k_bs_layer1   warp per trajectory: incremental layer-1 pre-activation (fp32, resident
//                 in HBM/L2) from the 3 features the last action changed; coalesced W1 row
//                 reads; ReLU -> h1 tile image + mask
//   k_gemm<Hid>   h1 W2^T (+b2, ReLU) -> h2 tile image + mask        (tcgen05)
//   k_gemm<Log>   h2 Wf^T (+bf) -> bf16 logits [Bl x A]              (tcgen05, 15 n-tiles)
//   k_bs_sample   warp per trajectory: two-level inverse-CDF epsilon-uniform categorical
//                 over the legal slots (eps_uniform objectives.cpp:242-264 + categorical
//                 rng.cpp:87-100 with the reference's single uniform), env step, record
// Training (TB, tb_loss objectives.cpp:120-142):
//   k_bs_loss     per trajectory residual -> per-row coefficient
//   k_gemm<Dlog>  recompute logits, dlogits = g (onehot - softmax) on legal words -> image
//   k_gemm<Dz2>   dlogits Wf (K = A) masked by h2 > 0 -> dz2 image
//   k_gemm<Dz1>   dz2 W2 masked by h1 > 0 -> dz1 image
//   k_bs_wgrad    dW2 = h1^T dz2, dWf = h2^T dlogits (per 256-word chunk), dW1 = obs^T dz1
//                 (per 128-feature block): tcgen05 with MN-major operands read from the
//                 images, rows split across CTAs; then fixed-order reductions and Adam.
#include <math.h>

#include <vector>

#include "engine.h"
#include "gemm.cuh"

namespace gfnx {

namespace {

constexpr int kH = 256;  // hidden width supported by this path

struct BsState {
  int num_sms = 0;
  int H = kH, A = 0, O = 0, V = 0, S = 0, T = 0, NT = 0, KBA = 0, OB = 0;
  int Bl = 0, R = 0, tilesB = 0, tilesR = 0;
  __nv_bfloat16* w1 = nullptr;    // [O][H] row-major
  __nv_bfloat16* w2f = nullptr;   // [H out][H in] image
  __nv_bfloat16* w2d = nullptr;   // [H in][H out] image
  __nv_bfloat16* wff = nullptr;   // head fwd image: NT n-tiles x 4 K-blocks x (256 x 128 B)
  __nv_bfloat16* wfd = nullptr;   // head dgrad image: 1 n-tile (H rows) x A/64 K-blocks
  float* h1init = nullptr;        // [H]
  float* preact = nullptr;        // [Bl][H]
  uint32_t* cur = nullptr;        // [Bl][SW] current packed state
  uint32_t* stst = nullptr;       // [Bl*T][SW] state before each step
  int32_t* last_act = nullptr;    // [Bl]
  __nv_bfloat16 *h1 = nullptr, *h2 = nullptr, *dz1 = nullptr, *dz2 = nullptr;  // [R] images
  __nv_bfloat16* logits = nullptr;  // [Bl][A] row-major, per-step scratch
  __nv_bfloat16* dlog = nullptr;    // [R] x A images (A/64 K-blocks per tile)
  uint8_t *mask1 = nullptr, *mask2 = nullptr;  // [R][H/8]
  float* rowbuf = nullptr;        // [R][2]: logp(a), lse
  float* coef = nullptr;          // [R]
  float* bpart = nullptr;         // [tilesR][2H + A] bias column sums per tile
  float* wpart = nullptr;         // wgrad partial slabs
  int nranges = 0, ntasks = 0;
  double* lpart = nullptr;
  int loss_blocks = 0;
};

BsState& BS(Ctx& c) { return *static_cast<BsState*>(c.fast); }

// ---------------------------------------------------------------------------
// rollout kernels

struct L1Args {
  EnvParams P;
  const __nv_bfloat16* w1;
  const float* h1init;
  float* preact;
  const int32_t* last_act;
  uint8_t* h1;
  uint8_t* mask1;
  int Bl, t;
};

// warp per trajectory; lane l owns hidden columns [8l, 8l + 8)
__global__ void __launch_bounds__(256) k_bs_layer1(L1Args a) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * 8 + warp;
  if (b >= a.Bl) return;
  const EnvParams& P = a.P;
  float v[8];
  float* pre = a.preact + (size_t)b * kH + 8 * lane;
  if (a.t == 0) {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = a.h1init[8 * lane + j];
  } else {
    const float4 p0 = *reinterpret_cast<const float4*>(pre), p1 = *reinterpret_cast<const float4*>(pre + 4);
    v[0] = p0.x; v[1] = p0.y; v[2] = p0.z; v[3] = p0.w;
    v[4] = p1.x; v[5] = p1.y; v[6] = p1.z; v[7] = p1.w;
    const int act = a.last_act[b];
    const int W = P.bs_vocab + 1, pos = act / P.bs_vocab, tok = act % P.bs_vocab;
    const int f0 = pos * W + P.bs_vocab, f1 = pos * W + tok, f2 = P.bs_slots * W;
    const float dv2 = 1.0f / (float)P.bs_slots;
    const uint4 w0 = __ldg(reinterpret_cast<const uint4*>(a.w1 + (size_t)f0 * kH) + lane);
    const uint4 w1v = __ldg(reinterpret_cast<const uint4*>(a.w1 + (size_t)f1 * kH) + lane);
    const uint4 w2 = __ldg(reinterpret_cast<const uint4*>(a.w1 + (size_t)f2 * kH) + lane);
    const uint32_t x0[4] = {w0.x, w0.y, w0.z, w0.w}, x1[4] = {w1v.x, w1v.y, w1v.z, w1v.w},
                   x2[4] = {w2.x, w2.y, w2.z, w2.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      v[2 * e] += -bf16_lo(x0[e]) + bf16_lo(x1[e]) + dv2 * bf16_lo(x2[e]);
      v[2 * e + 1] += -bf16_hi(x0[e]) + bf16_hi(x1[e]) + dv2 * bf16_hi(x2[e]);
    }
  }
  *reinterpret_cast<float4*>(pre) = make_float4(v[0], v[1], v[2], v[3]);
  *reinterpret_cast<float4*>(pre + 4) = make_float4(v[4], v[5], v[6], v[7]);
  uint32_t pk[4];
  uint32_t mb = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    pk[e] = pack_bf16x2(fmaxf(v[2 * e], 0.f), fmaxf(v[2 * e + 1], 0.f));
    mb |= (bf16_lo(pk[e]) > 0.f ? 1u : 0u) << (2 * e);
    mb |= (bf16_hi(pk[e]) > 0.f ? 1u : 0u) << (2 * e + 1);
  }
  const size_t r = (size_t)a.t * a.Bl + b;
  uint8_t* tile = a.h1 + (r / kTile) * (kTile * kH * 2);
  *reinterpret_cast<uint4*>(tile + sw128_offset((uint32_t)(r % kTile), 8 * lane, kTile)) =
      make_uint4(pk[0], pk[1], pk[2], pk[3]);
  a.mask1[r * (kH / 8) + lane] = (uint8_t)mb;
}

struct HidEpi {  // +b2, ReLU -> h2 tile image + mask
  struct Args {
    const float* b2;
    uint8_t* h2;
    uint8_t* mask2;
  };
  static __device__ void finish(const Args&, int, int, const float*) {}
  static __device__ void apply(const Args& e, int m, int, int row, int col0, float (&v)[32], float*) {
    uint32_t pk[16], mb = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      pk[i] = pack_bf16x2(fmaxf(v[2 * i] + __ldg(e.b2 + col0 + 2 * i), 0.f),
                          fmaxf(v[2 * i + 1] + __ldg(e.b2 + col0 + 2 * i + 1), 0.f));
      mb |= (bf16_lo(pk[i]) > 0.f ? 1u : 0u) << (2 * i);
      mb |= (bf16_hi(pk[i]) > 0.f ? 1u : 0u) << (2 * i + 1);
    }
    st_row32(e.h2 + (size_t)m * (kTile * kH * 2), row, col0, pk);
    const size_t r = (size_t)m * kTile + row;
    *reinterpret_cast<uint32_t*>(e.mask2 + r * (kH / 8) + col0 / 8) = mb;
  }
};

struct LogEpi {  // +bf -> bf16 logits row-major [Bl][A] (rows of the current step)
  struct Args {
    const float* bf;
    __nv_bfloat16* logits;
    int A, row_base;  // global row of tile 0 of this launch
  };
  static __device__ void finish(const Args&, int, int, const float*) {}
  static __device__ void apply(const Args& e, int m, int n, int row, int col0, float (&v)[32], float*) {
    const int b = m * kTile + row - e.row_base;
    const int c = n * 256 + col0;
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 16; ++i)
      pk[i] = pack_bf16x2(v[2 * i] + __ldg(e.bf + c + 2 * i), v[2 * i + 1] + __ldg(e.bf + c + 2 * i + 1));
    uint4* dst = reinterpret_cast<uint4*>(e.logits + (size_t)b * e.A + c);
#pragma unroll
    for (int q = 0; q < 4; ++q) dst[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
  }
};

struct SampleArgs {
  EnvParams P;
  Key key;
  double eps;
  int b0, Bl, t, T;
  const __nv_bfloat16* logits;
  uint32_t* cur;
  uint32_t* stst;
  int32_t* last_act;
  float* rowbuf;
  DeviceBatch batch;
};

// warp per trajectory: eps-uniform masked categorical with ONE uniform per draw, as the
// reference: slot chosen by cumulative slot mass, then the word inside the slot.
__global__ void __launch_bounds__(256) k_bs_sample(SampleArgs a) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * 8 + warp;
  if (b >= a.Bl) return;
  const EnvParams& P = a.P;
  const int V = P.bs_vocab, S = P.bs_slots, A = P.A;
  BitseqEnv::State s;
  BitseqEnv::unpack(P, a.cur + (size_t)b * P.SW, s);
  const __nv_bfloat16* lg = a.logits + (size_t)b * A;
  const int per = A / 32;  // logits per lane, lane-contiguous chunks of 8 words
  // pass 1: max over legal logits
  float hi = -INFINITY;
  for (int i0 = lane * 8; i0 < A; i0 += 256) {
    const int slot = i0 / V;
    if ((s.filled >> slot) & 1) continue;
    const uint4 q = *reinterpret_cast<const uint4*>(lg + i0);
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) hi = fmaxf(hi, fmaxf(bf16_lo(w[e]), bf16_hi(w[e])));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  (void)per;
  // pass 2: per-slot sums of exp(x - hi) (fp64 accumulation, fixed lane order)
  double slot_sum[kMaxSlots > 64 ? 64 : kMaxSlots];
  int legal_slots = 0;
  double z = 0.0;
  for (int p = 0; p < S; ++p) {
    double part = 0.0;
    if (!((s.filled >> p) & 1)) {
      for (int i0 = p * V + lane * 8; i0 < (p + 1) * V; i0 += 256) {
        const uint4 q = *reinterpret_cast<const uint4*>(lg + i0);
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int e = 0; e < 4; ++e)
          part += (double)__expf(bf16_lo(w[e]) - hi) + (double)__expf(bf16_hi(w[e]) - hi);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      ++legal_slots;
    }
    slot_sum[p < 64 ? p : 63] = part;
    z += part;
  }
  const int legal = legal_slots * V;
  const double eps = a.eps;
  const double u_eps = eps / legal;
  double total = 0.0;
  for (int p = 0; p < S; ++p)
    if (!((s.filled >> p) & 1)) total += (1.0 - eps) * slot_sum[p] / z + u_eps * V;
  const double u01 = uniform_scalar(fold_in(fold_in(a.key, (uint64_t)a.t), (uint64_t)(a.b0 + b)));
  double x = u01 * total;
  int slot = -1;
  for (int p = 0; p < S; ++p) {
    if ((s.filled >> p) & 1) continue;
    const double m = (1.0 - eps) * slot_sum[p] / z + u_eps * V;
    slot = p;
    if (x < m) break;
    x -= m;
  }
  // within the slot: lane-contiguous 8-word groups, warp prefix over group masses
  int act = -1;
  if (slot >= 0) {
    for (int i0 = slot * V; i0 < (slot + 1) * V && act < 0; i0 += 256) {
      const int base = i0 + lane * 8;
      double w8[8];
      double gsum = 0.0;
      if (base < (slot + 1) * V) {
        const uint4 q = *reinterpret_cast<const uint4*>(lg + base);
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          w8[2 * e] = (1.0 - eps) * (double)__expf(bf16_lo(w[e]) - hi) / z + u_eps;
          w8[2 * e + 1] = (1.0 - eps) * (double)__expf(bf16_hi(w[e]) - hi) / z + u_eps;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) gsum += w8[e];
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) w8[e] = 0.0;
      }
      double incl = gsum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const double excl = incl - gsum;
      const unsigned hit = __ballot_sync(0xffffffffu, gsum > 0.0 && x < incl);
      if (hit) {
        const int src = __ffs(hit) - 1;
        int pick = 7;
        double acc = excl;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          acc += w8[e];
          if (x < acc) {
            pick = e;
            break;
          }
        }
        pick = __shfl_sync(0xffffffffu, pick, src);
        act = i0 + src * 8 + pick;
      } else {
        x -= __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    if (act < 0) act = (slot + 1) * V - 1;  // categorical fallback: last positive weight
  }
  if (lane == 0) {
    const int T = a.T;
    const size_t bt = (size_t)b * T + a.t;
    const size_t r = (size_t)a.t * a.Bl + b;
    if (act < 0) {
      atomicExch(a.batch.counters + 3, GFNX_ERR_CONTRACT);
      return;
    }
    const float xa = __bfloat162float(lg[act]);
    const float lse = hi + __logf((float)z);
    a.rowbuf[2 * r] = xa - lse;
    a.rowbuf[2 * r + 1] = lse;
    for (int w = 0; w < P.SW; ++w) a.stst[bt * P.SW + w] = a.cur[(size_t)b * P.SW + w];
    const bool term = BitseqEnv::step(P, s, act);
    BitseqEnv::pack(P, s, a.cur + (size_t)b * P.SW);
    a.batch.actions[bt] = (int16_t)act;
    a.batch.nparents[bt] = (uint16_t)BitseqEnv::num_parents(P, s);
    a.last_act[b] = act;
    if (term) {
      a.batch.lengths[b] = a.t + 1;
      a.batch.log_rewards[b] = BitseqEnv::log_reward(P, s);
      BitseqEnv::pack(P, s, a.batch.term_state + (size_t)b * P.SW);
    }
    if (!isfinite(lse)) atomicExch(a.batch.counters + 3, GFNX_ERR_NUMERIC);
  }
}

__global__ void k_bs_h1init(EnvParams P, const __nv_bfloat16* w1, const float* b1, float* h1init) {
  const int j = threadIdx.x;
  if (j >= kH) return;
  float v = b1[j];
  const int W = P.bs_vocab + 1;
  for (int p = 0; p < P.bs_slots; ++p) v += __bfloat162float(w1[(size_t)(p * W + P.bs_vocab) * kH + j]);
  h1init[j] = v;  // count feature is 0 at s0
}

__global__ void k_bs_reset(EnvParams P, int Bl, uint32_t* cur) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < Bl * P.SW) cur[i] = 0;
}

// ---------------------------------------------------------------------------
// training kernels

struct BsLossArgs {
  DeviceBatch batch;
  int Bl, T;
  double B_global;
  const double* neglog;
  const float* rowbuf;
  float* coef;
  double* lpart;
  const double* scalars;
};

__global__ void k_bs_loss(BsLossArgs a) {  // tb_loss objectives.cpp:120-142
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  double loss = 0.0, dlogz = 0.0;
  if (b < a.Bl) {
    const double w = 1.0 / a.B_global;
    double cum = 0.0;
    for (int t = 0; t < a.T; ++t) {
      const size_t r = (size_t)t * a.Bl + b;
      cum += (double)a.rowbuf[2 * r] - a.neglog[a.batch.nparents[(size_t)b * a.T + t]];
    }
    const double res = cum + a.scalars[0] - a.batch.log_rewards[b];
    loss = res * res * w;
    const double g = 2.0 * res * w;
    dlogz = g;
    for (int t = 0; t < a.T; ++t) a.coef[(size_t)t * a.Bl + b] = (float)g;
  }
  __shared__ double red[2][256];
  red[0][threadIdx.x] = loss;
  red[1][threadIdx.x] = dlogz;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if ((int)threadIdx.x < off) {
      red[0][threadIdx.x] += red[0][threadIdx.x + off];
      red[1][threadIdx.x] += red[1][threadIdx.x + off];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    a.lpart[2 * blockIdx.x] = red[0][0];
    a.lpart[2 * blockIdx.x + 1] = red[1][0];
  }
}

__global__ void k_bs_loss_finalize(const double* lpart, int n, double* scalars, int32_t* err) {
  if (threadIdx.x != 0) return;
  double l = 0.0, z = 0.0;
  for (int i = 0; i < n; ++i) {
    l += lpart[2 * i];
    z += lpart[2 * i + 1];
  }
  scalars[4] = l;
  scalars[3] = z;
  if (!isfinite(l)) atomicExch(err, GFNX_ERR_NUMERIC);
}

struct DlogEpi {  // recomputed logits -> dlogits image + per-tile column sums (bias grad)
  struct Args {
    EnvParams P;
    const float* bf;
    const float* rowbuf;
    const float* coef;
    const uint32_t* stst;
    const int16_t* actions;
    uint8_t* dlog;  // image with A/64 K-blocks per tile
    float* bpart;   // [tilesR][2H + A]
    int Bl, T, A, KBA;
  };
  static __device__ void finish(const Args& e, int m, int n, const float* scratch) {
    const int c = threadIdx.x;  // 256 threads, one output column each
    const float s = scratch[c] + scratch[256 + c] + scratch[512 + c] + scratch[768 + c];
    e.bpart[(size_t)m * (2 * kH + e.A) + 2 * kH + n * 256 + c] = s;
  }
  static __device__ void apply(const Args& e, int m, int n, int row, int col0, float (&v)[32],
                               float* scratch) {
    const size_t r = (size_t)m * kTile + row;
    const int t = (int)(r / e.Bl), b = (int)(r % e.Bl);
    const size_t bt = (size_t)b * e.T + t;
    const int V = e.P.bs_vocab;
    const int tw = (e.P.bs_slots + 3) / 4;
    uint32_t filled = e.stst[bt * e.P.SW + tw];  // slots <= 32 on this path
    const int act = e.actions[bt];
    const float lse = e.rowbuf[2 * r + 1], g = e.coef[r];
    const int c0 = n * 256 + col0;
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int c = c0 + i;
      const bool legal = !((filled >> (c / V)) & 1u);
      const float x = __bfloat162float(__float2bfloat16(v[i] + __ldg(e.bf + c)));
      float d = legal ? -g * __expf(x - lse) : 0.f;
      if (c == act) d += g;
      v[i] = d;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) pk[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
    // K-block (n*4 + col/64) of tile m in the wide dlogits image
    uint8_t* blk = e.dlog + ((size_t)m * e.KBA + n * 4 + col0 / 64) * (kTile * 128);
    st_row32(blk, row, col0 % 64, pk);
    const float s = warp_colsum32(v);  // this warp's 32 rows, lane = column
    scratch[((threadIdx.x >> 5) & 3) * 256 + col0 + (threadIdx.x & 31)] = s;
  }
};

struct DgradEpi {  // masked by ReLU bits -> dz image + bias column sums
  struct Args {
    const uint8_t* mask;
    uint8_t* dz;
    float* bpart;
    int boff;  // 0: db1, H: db2
    int A;
  };
  static __device__ void finish(const Args& e, int m, int, const float* scratch) {
    const int c = threadIdx.x;
    const float s = scratch[c] + scratch[256 + c] + scratch[512 + c] + scratch[768 + c];
    e.bpart[(size_t)m * (2 * kH + e.A) + e.boff + c] = s;
  }
  static __device__ void apply(const Args& e, int m, int, int row, int col0, float (&v)[32],
                               float* scratch) {
    const size_t r = (size_t)m * kTile + row;
    const uint32_t mk = *reinterpret_cast<const uint32_t*>(e.mask + r * (kH / 8) + col0 / 8);
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = ((mk >> i) & 1u) ? v[i] : 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) pk[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
    st_row32(e.dz + (size_t)m * (kTile * kH * 2), row, col0, pk);
    const float s = warp_colsum32(v);
    scratch[((threadIdx.x >> 5) & 3) * 256 + col0 + (threadIdx.x & 31)] = s;
  }
};


// ---------------------------------------------------------------------------
// weight gradients: per (task, row range) CTA, MN-major tcgen05 over 64-row stages
//   task 0            dW2     A' = h1 features (2 x 128),  B' = dz2
//   tasks 1..NT       dWf[n]  A' = h2 features (2 x 128),  B' = dlogits words [256n, 256n+256)
//   tasks NT+1..+S    dW1 token rows of slot p: A' = one-hot(token of slot p) (V <= 256)
//   task NT+S+1       dW1 "empty" rows of every slot + the filled/n feature (<= 128 rows)
// CTAs of one row range are adjacent in the grid so the shared operand (h2 or dz1) of a
// range is fetched from HBM once and re-served from L2.

constexpr int kWStage = 64;  // rows per stage
constexpr int kWStages = 3;

struct WgArgs {
  EnvParams P;
  const uint8_t *h1, *h2, *dz1, *dz2, *dlog;
  const uint32_t* stst;
  int Bl, T, R, tilesR, NT, KBA, nranges;
  float* wpart;  // [task][range][256][256]
};

GFNX_DEV void wg_copy_half(uint8_t* dst, const uint8_t* tile, int blk0, int nblk, int h, uint64_t* bar) {
  // rows [64h, 64h + 64) of feature blocks [blk0, blk0 + nblk) of a 128-row tile image
  for (int k = 0; k < nblk; ++k)
    bulk_g2s(dst + k * (kWStage * 128), tile + (size_t)(blk0 + k) * (kTile * 128) + h * (kWStage * 128),
             kWStage * 128, bar);
}

__global__ void __launch_bounds__(kThreads, 1) k_bs_wgrad(WgArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  constexpr int kA = kWStage * 256 * 2, kB = kWStage * 256 * 2;  // 32 KB each
  __shared__ uint64_t full[kWStages], empty[kWStages];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quarter = warp & 3, half = warp >> 2;
  const int task = blockIdx.x / a.nranges, range = blockIdx.x % a.nranges;
  const int NT = a.NT, S = a.P.bs_slots, V = a.P.bs_vocab;
  const bool built = task > NT;                 // dW1 tasks build the one-hot operand
  const int halves = (task == NT + S + 1) ? 1 : 2;  // M' = 256 (2 x 128) or 128
  const int per = (a.tilesR + a.nranges - 1) / a.nranges;
  const int t0 = range * per, t1 = min(a.tilesR, t0 + per);
  const int nq = t1 > t0 ? 2 * (t1 - t0) : 0;  // 64-row stages
  if (warp == 0) tmem_alloc<512>(&tbase);
  if (tid == 0) {
    for (int s2 = 0; s2 < kWStages; ++s2) {
      mbar_init(&full[s2], 1);
      mbar_init(&empty[s2], 1);
    }
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  auto issue_loads = [&](int q) {  // thread 0
    const int slot = q % kWStages, tile = t0 + q / 2, h = q % 2;
    uint8_t* sa = smem + slot * (kA + kB);
    uint8_t* sb = sa + kA;
    const size_t tb = (size_t)tile * (kTile * 256 * 2);
    const int bytes = (built ? 0 : kA) + kB;
    mbar_arrive_expect_tx(&full[slot], bytes);
    if (task == 0) {
      wg_copy_half(sa, a.h1 + tb, 0, 4, h, &full[slot]);
      wg_copy_half(sb, a.dz2 + tb, 0, 4, h, &full[slot]);
    } else if (!built) {
      wg_copy_half(sa, a.h2 + tb, 0, 4, h, &full[slot]);
      wg_copy_half(sb, a.dlog + (size_t)tile * a.KBA * (kTile * 128), 4 * (task - 1), 4, h, &full[slot]);
    } else {
      wg_copy_half(sb, a.dz1 + tb, 0, 4, h, &full[slot]);
    }
  };
  auto build = [&](int q) {  // all threads: one-hot operand rows for stage q
    const int slot = q % kWStages, tile = t0 + q / 2, h = q % 2;
    uint8_t* sa = smem + slot * (kA + kB);
    // zero 32 KB: 256 threads x 128 B
    uint4* z = reinterpret_cast<uint4*>(sa + tid * 128);
#pragma unroll
    for (int i = 0; i < 8; ++i) z[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    if (tid < kWStage) {
      const int r = tile * kTile + h * kWStage + tid;
      if (r < a.R) {
        const int t = r / a.Bl, b = r % a.Bl;
        BitseqEnv::State st;
        BitseqEnv::unpack(a.P, a.stst + ((size_t)b * a.T + t) * a.P.SW, st);
        auto put = [&](int f, float v) {  // feature f of this task's 256-wide operand
          *reinterpret_cast<__nv_bfloat16*>(sa + (f >> 6) * (kWStage * 128) +
                                            (sw128_offset(tid, f & 63, kWStage) & (kWStage * 128 - 1))) =
              __float2bfloat16(v);
        };
        if (task <= NT + S) {  // token of slot p
          const int p = task - NT - 1;
          if ((st.filled >> p) & 1) put(st.tok[p], 1.f);
        } else {  // empty indicators of every slot, then the filled/n count feature
          for (int p = 0; p < S; ++p)
            if (!((st.filled >> p) & 1)) put(p, 1.f);
          put(S, (float)st.count / S);
        }
      }
    }
    fence_proxy_async();
  };
  if (tid == 0)
    for (int q = 0; q < 2 && q < nq; ++q) issue_loads(q);
  if (built && nq > 0) build(0);
  for (int q = 0; q < nq; ++q) {
    const int slot = q % kWStages;
    __syncthreads();  // operand of stage q complete (built rows visible)
    if (tid == 0) {
      mbar_wait(&full[slot], (q / kWStages) & 1);
      tc_fence_after();
      const uint32_t a0 = smem_u32(smem + slot * (kA + kB)), b0 = a0 + kA;
      constexpr uint32_t idesc = umma_idesc_bf16(128, 256, true, true);
      for (int hh = 0; hh < halves; ++hh)
#pragma unroll
        for (int k = 0; k < kWStage / 16; ++k)
          umma_bf16(tmem + hh * 256,
                    umma_desc_sw128(a0 + hh * 2 * (kWStage * 128) + k * 2048, kWStage * 128, 1024),
                    umma_desc_sw128(b0 + k * 2048, kWStage * 128, 1024), idesc, (q > 0 || k > 0) ? 1u : 0u);
      umma_commit(&empty[slot]);
      if (q + 2 < nq) {  // refill the slot last used by stage q - 1
        if (q >= 1) mbar_wait(&empty[(q + 2) % kWStages], ((q - 1) / kWStages) & 1);
        issue_loads(q + 2);
      }
    }
    if (built && q + 1 < nq) {
      if (q >= 2) mbar_wait(&empty[(q + 1) % kWStages], ((q - 2) / kWStages) & 1);
      build(q + 1);
    }
  }
  if (tid == 0 && nq > 0) mbar_wait(&empty[(nq - 1) % kWStages], ((nq - 1) / kWStages) & 1);
  __syncthreads();
  tc_fence_after();
  // epilogue: lane quarter x column half, both M'-halves
  float* slab = a.wpart + ((size_t)task * a.nranges + range) * (256 * 256);
  for (int hh = 0; hh < 2; ++hh) {
    const int mrow = hh * 128 + quarter * 32 + lane;
    for (int q = 0; q < 4; ++q) {
      const int col = half * 128 + q * 32;
      uint32_t r32[32];
      tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + hh * 256 + col, r32);
      tmem_wait_ld();
      float* dst = slab + (size_t)mrow * 256 + col;
      const bool ok = nq > 0 && hh < halves;
#pragma unroll
      for (int i = 0; i < 32; ++i) dst[i] = ok ? __uint_as_float(r32[i]) : 0.f;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

// reductions (fixed order) of wgrad slabs and per-tile bias sums into the flat gradient
struct RedArgs {
  const float* wpart;
  const float* bpart;
  float* g;
  int nranges, NT, S, V, A, O, tilesR;
  MlpLayout L;
};

__global__ void k_bs_reduce(RedArgs a) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const MlpLayout& L = a.L;
  if (e >= L.n_params) return;
  auto slab_sum = [&](int task, int m, int n) {
    float s = 0.f;
    for (int r = 0; r < a.nranges; ++r)
      s += a.wpart[(((size_t)task * a.nranges + r) * 256 + m) * 256 + n];
    return s;
  };
  auto bias_sum = [&](int col) {
    float s = 0.f;
    for (int t = 0; t < a.tilesR; ++t) s += a.bpart[(size_t)t * (2 * kH + a.A) + col];
    return s;
  };
  float v = 0.f;
  if (e < L.off_b[0]) {  // W1 [O][H]
    const int f = (int)(e / kH), j = (int)(e % kH);
    const int W = a.V + 1;
    if (f == a.S * W) {
      v = slab_sum(a.NT + a.S + 1, a.S, j);
    } else {
      const int p = f / W, tok = f % W;
      v = tok == a.V ? slab_sum(a.NT + a.S + 1, p, j) : slab_sum(a.NT + 1 + p, tok, j);
    }
  } else if (e < L.off_w[1]) {
    v = bias_sum((int)(e - L.off_b[0]));
  } else if (e < L.off_b[1]) {
    const int64_t k = e - L.off_w[1];
    v = slab_sum(0, (int)(k / kH), (int)(k % kH));
  } else if (e < L.off_fw) {
    v = bias_sum(kH + (int)(e - L.off_b[1]));
  } else if (e < L.off_fb) {
    const int64_t k = e - L.off_fw;
    const int p = (int)(k / a.A), c = (int)(k % a.A);
    v = slab_sum(1 + c / 256, p, c % 256);
  } else if (e < L.off_bw) {
    v = bias_sum(2 * kH + (int)(e - L.off_fb));
  }
  a.g[e] = v;  // bwd / flow heads: unused by TB with uniform P_B -> 0
}

struct EmitArgs {
  const float* p;
  int64_t n;
  MlpLayout L;
  int A;
  __nv_bfloat16 *w1, *w2f, *w2d, *wff, *wfd;
};

__global__ void k_bs_emit(EmitArgs a) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.n) return;
  const MlpLayout& L = a.L;
  const __nv_bfloat16 v = __float2bfloat16(a.p[j]);
  if (j < L.off_b[0]) {
    a.w1[j] = v;
  } else if (j >= L.off_w[1] && j < L.off_b[1]) {
    const int64_t k = j - L.off_w[1];
    const int p = (int)(k / kH), q = (int)(k % kH);
    *reinterpret_cast<__nv_bfloat16*>((uint8_t*)a.w2f + sw128_offset(q, p, kH)) = v;
    *reinterpret_cast<__nv_bfloat16*>((uint8_t*)a.w2d + sw128_offset(p, q, kH)) = v;
  } else if (j >= L.off_fw && j < L.off_fb) {
    const int64_t k = j - L.off_fw;
    const int p = (int)(k / a.A), c = (int)(k % a.A);
    const int n = c / 256, cc = c % 256;
    *reinterpret_cast<__nv_bfloat16*>((uint8_t*)a.wff + (size_t)n * (256 * kH * 2) + sw128_offset(cc, p, 256)) = v;
    *reinterpret_cast<__nv_bfloat16*>((uint8_t*)a.wfd + sw128_offset(p, c, kH)) = v;
  }
}

EmitArgs emit_args(Ctx& c) {
  BsState& f = BS(c);
  EmitArgs a{};
  a.p = c.p32;
  a.n = c.L.n_params;
  a.L = c.L;
  a.A = f.A;
  a.w1 = f.w1;
  a.w2f = f.w2f;
  a.w2d = f.w2d;
  a.wff = f.wff;
  a.wfd = f.wfd;
  return a;
}

}  // namespace

// ---------------------------------------------------------------------------
// host side

bool bs_supported(const Ctx& c, std::string* why) {
  if (c.env.kind != GFNX_ENV_BITSEQ) return false;
  auto no = [&](const char* m) {
    *why = m;
    return false;
  };
  if (c.train.objective != GFNX_OBJ_TB) return no("bitseq fast path implements TB (BASELINE config #3)");
  if (c.L.n_trunk != 2 || c.L.dims[1] != kH || c.L.dims[2] != kH) return no("bitseq fast path needs a 2 x 256 MLP");
  if (c.P.bs_vocab != 256) return no("bitseq fast path needs k = 8 (256-word slots)");
  if (c.P.bs_slots > 32) return no("bitseq fast path supports <= 32 slots");
  if (c.Bl % kTile != 0) return no("bitseq fast path needs a per-rank batch that is a multiple of 128");
  return true;
}

void bs_init(Ctx& c) {
  auto* f = new BsState();
  c.fast = f;
  cudaDeviceGetAttribute(&f->num_sms, cudaDevAttrMultiProcessorCount, c.device);
  f->A = c.P.A;
  f->O = c.P.O;
  f->V = c.P.bs_vocab;
  f->S = c.P.bs_slots;
  f->T = c.P.T;
  f->NT = f->A / 256;
  f->KBA = f->A / 64;
  f->Bl = c.Bl;
  f->R = c.Bl * f->T;
  f->tilesB = c.Bl / kTile;
  f->tilesR = f->R / kTile;
  f->ntasks = 1 + f->NT + f->S + 1;
  f->nranges = std::max(1, f->num_sms / f->ntasks);
  f->loss_blocks = (c.Bl + 255) / 256;
  const size_t img = (size_t)f->tilesR * kTile * kH * 2;
  auto alloc = [&](auto** p, size_t bytes) { cuda_check(cudaMalloc((void**)p, bytes), "bitseq alloc"); };
  alloc(&f->w1, sizeof(__nv_bfloat16) * (size_t)f->O * kH);
  alloc(&f->w2f, sizeof(__nv_bfloat16) * kH * kH);
  alloc(&f->w2d, sizeof(__nv_bfloat16) * kH * kH);
  alloc(&f->wff, sizeof(__nv_bfloat16) * (size_t)f->A * kH);
  alloc(&f->wfd, sizeof(__nv_bfloat16) * (size_t)f->A * kH);
  alloc(&f->h1init, sizeof(float) * kH);
  alloc(&f->preact, sizeof(float) * (size_t)c.Bl * kH);
  alloc(&f->cur, sizeof(uint32_t) * (size_t)c.Bl * c.P.SW);
  alloc(&f->stst, sizeof(uint32_t) * (size_t)c.Bl * f->T * c.P.SW);
  alloc(&f->last_act, sizeof(int32_t) * c.Bl);
  alloc(&f->h1, img);
  alloc(&f->h2, img);
  alloc(&f->dz1, img);
  alloc(&f->dz2, img);
  alloc(&f->logits, sizeof(__nv_bfloat16) * (size_t)c.Bl * f->A);
  alloc(&f->dlog, (size_t)f->tilesR * f->KBA * (kTile * 128));
  alloc(&f->mask1, (size_t)f->R * (kH / 8));
  alloc(&f->mask2, (size_t)f->R * (kH / 8));
  alloc(&f->rowbuf, sizeof(float) * 2 * (size_t)f->R);
  alloc(&f->coef, sizeof(float) * (size_t)f->R);
  alloc(&f->bpart, sizeof(float) * (size_t)f->tilesR * (2 * kH + f->A));
  alloc(&f->wpart, sizeof(float) * (size_t)f->ntasks * f->nranges * 256 * 256);
  alloc(&f->lpart, sizeof(double) * 2 * f->loss_blocks);
  bs_sync_weights(c);
}

void bs_free(Ctx& c) {
  BsState* f = static_cast<BsState*>(c.fast);
  if (!f) return;
  void* ptrs[] = {f->w1, f->w2f, f->w2d, f->wff, f->wfd, f->h1init, f->preact, f->cur, f->stst,
                  f->last_act, f->h1, f->h2, f->dz1, f->dz2, f->logits, f->dlog, f->mask1,
                  f->mask2, f->rowbuf, f->coef, f->bpart, f->wpart, f->lpart};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete f;
  c.fast = nullptr;
}

void bs_sync_weights(Ctx& c) {
  EmitArgs a = emit_args(c);
  k_bs_emit<<<(unsigned)((a.n + 255) / 256), 256, 0, c.stream>>>(a);
  c.launches++;
}

void bs_rollout(Ctx& c, Key key, double eps) {
  BsState& f = BS(c);
  const int T = f.T, Bl = c.Bl;
  cudaMemsetAsync(c.batch.actions, 0xFF, sizeof(int16_t) * (size_t)Bl * T, c.stream);
  {
    ProfScope ps(c, "k_bs_init");
    k_bs_reset<<<(Bl * c.P.SW + 255) / 256, 256, 0, c.stream>>>(c.P, Bl, f.cur);
    k_bs_h1init<<<1, kH, 0, c.stream>>>(c.P, f.w1, c.p32 + c.L.off_b[0], f.h1init);
    c.launches += 2;
  }
  for (int t = 0; t < T; ++t) {
    {
      L1Args la{c.P, f.w1, f.h1init, f.preact, f.last_act, (uint8_t*)f.h1, f.mask1, Bl, t};
      ProfScope ps(c, "k_bs_layer1");
      k_bs_layer1<<<(Bl + 7) / 8, 256, 0, c.stream>>>(la);
      c.launches++;
    }
    GemmGeom g{};
    g.A = (const uint8_t*)f.h1;
    g.a_kb = 4;
    g.B = (const uint8_t*)f.w2f;
    g.b_kb = 4;
    g.m0 = t * f.tilesB;
    g.m_tiles = f.tilesB;
    g.n_tiles = 1;
    g.KB = 4;
    launch_gemm<256, HidEpi>(c, "k_gemm_hidden", g, HidEpi::Args{c.p32 + c.L.off_b[1], (uint8_t*)f.h2, f.mask2},
                             f.num_sms);
    GemmGeom g2 = g;
    g2.A = (const uint8_t*)f.h2;
    g2.B = (const uint8_t*)f.wff;
    g2.n_tiles = f.NT;
    launch_gemm<256, LogEpi>(c, "k_gemm_logits", g2, LogEpi::Args{c.p32 + c.L.off_fb, f.logits, f.A, t * Bl},
                             f.num_sms);
    SampleArgs sa{c.P, key, eps, c.b0, Bl, t, T, f.logits, f.cur, f.stst, f.last_act, f.rowbuf, c.batch};
    ProfScope ps(c, "k_bs_sample");
    k_bs_sample<<<(Bl + 7) / 8, 256, 0, c.stream>>>(sa);
    c.launches++;
  }
}

void bs_train(Ctx& c) {
  BsState& f = BS(c);
  const int Bl = c.Bl;
  {
    BsLossArgs la{c.batch, Bl, f.T, (double)c.B, c.d_neglog, f.rowbuf, f.coef, f.lpart, c.d_scalars};
    ProfScope ps(c, "k_bs_loss");
    k_bs_loss<<<f.loss_blocks, 256, 0, c.stream>>>(la);
    k_bs_loss_finalize<<<1, 32, 0, c.stream>>>(f.lpart, f.loss_blocks, c.d_scalars, c.batch.counters + 3);
    c.launches += 2;
  }
  GemmGeom g{};
  g.A = (const uint8_t*)f.h2;
  g.a_kb = 4;
  g.B = (const uint8_t*)f.wff;
  g.b_kb = 4;
  g.m0 = 0;
  g.m_tiles = f.tilesR;
  g.n_tiles = f.NT;
  g.KB = 4;
  DlogEpi::Args de{c.P, c.p32 + c.L.off_fb, f.rowbuf, f.coef, f.stst, c.batch.actions,
                   (uint8_t*)f.dlog, f.bpart, Bl, f.T, f.A, f.KBA};
  launch_gemm<256, DlogEpi>(c, "k_gemm_dlogits", g, de, f.num_sms);
  GemmGeom g2{};
  g2.A = (const uint8_t*)f.dlog;
  g2.a_kb = f.KBA;
  g2.B = (const uint8_t*)f.wfd;
  g2.b_kb = f.KBA;
  g2.m0 = 0;
  g2.m_tiles = f.tilesR;
  g2.n_tiles = 1;
  g2.KB = f.KBA;
  launch_gemm<256, DgradEpi>(c, "k_gemm_dgrad_head", g2, DgradEpi::Args{f.mask2, (uint8_t*)f.dz2, f.bpart, kH, f.A},
                             f.num_sms);
  GemmGeom g3{};
  g3.A = (const uint8_t*)f.dz2;
  g3.a_kb = 4;
  g3.B = (const uint8_t*)f.w2d;
  g3.b_kb = 4;
  g3.m0 = 0;
  g3.m_tiles = f.tilesR;
  g3.n_tiles = 1;
  g3.KB = 4;
  launch_gemm<256, DgradEpi>(c, "k_gemm_dgrad_hidden", g3, DgradEpi::Args{f.mask1, (uint8_t*)f.dz1, f.bpart, 0, f.A},
                             f.num_sms);
  {
    WgArgs wa{c.P, (const uint8_t*)f.h1, (const uint8_t*)f.h2, (const uint8_t*)f.dz1, (const uint8_t*)f.dz2,
              (const uint8_t*)f.dlog, f.stst, Bl, f.T, f.R, f.tilesR, f.NT, f.KBA, f.nranges, f.wpart};
    const int smem = kWStages * 2 * (kWStage * 256 * 2) + 1024;
    set_smem_once(k_bs_wgrad, smem);
    ProfScope ps(c, "k_bs_wgrad");
    k_bs_wgrad<<<f.ntasks * f.nranges, kThreads, smem, c.stream>>>(wa);
    c.launches++;
  }
  {
    RedArgs ra{f.wpart, f.bpart, c.g32, f.nranges, f.NT, f.S, f.V, f.A, f.O, f.tilesR, c.L};
    ProfScope ps(c, "k_bs_reduce");
    k_bs_reduce<<<(unsigned)((c.L.n_params + 255) / 256), 256, 0, c.stream>>>(ra);
    c.launches++;
  }
}

}  // namespace gfnx
