// lockstep.cu — bf16 tcgen05 fast path for the fixed-length environments:
//   bitseq NAR (SequenceEnv, proj/src/envs/sequences.cpp; BASELINE config #3:
//               n = 120, k = 8 -> 15 slots x 256 words, A = 3840, O = 3856, T = 15, MLP 2x256)
//   Ising      (IsingEnv, proj/src/envs/ising.cpp; config #4: 10x10, A = 200, O = 300,
//               T = 100, MLP 4x256)
// trained with trajectory balance (tb_loss objectives.cpp:120-142).
//
// Every trajectory takes exactly T steps, so the batch advances in lockstep and the rows of
// the training pass are laid out step-major: row r = t * Bl + b. The rollout's forward IS
// the training forward (parameters are fixed inside an iteration): the activation images,
// ReLU masks and per-row log-softmax statistics it produces feed the backward directly.
//
// Per rollout step t:
//   k_ls_layer1   warp per trajectory: incremental layer-1 pre-activation (fp32, resident)
//                 from the features the last action changed (Env::delta_features), coalesced
//                 W1 row reads; ReLU -> h1 tile image + mask
//   k_gemm<Hid>   h_{l-1} W_l^T (+b, ReLU) -> h_l image + mask, l = 2..NL   (tcgen05)
//   k_gemm<Log>   h_NL Wf^T (+bf) -> bf16 logits [Bl x Ap] and, per 128-column group, the
//                 masked (max, sum exp) over the legal columns               (tcgen05)
//   k_ls_sample   warp per trajectory: eps-uniform masked categorical with ONE uniform
//                 (eps_uniform objectives.cpp:242-264, categorical rng.cpp:87-100): group
//                 by cumulative group mass from the statistics, then the column inside the
//                 group from its 128 logits; env step; record
// Training:
//   k_ls_loss     per trajectory TB residual -> per-row coefficient g
//   k_gemm<Dlog>  recomputed logits -> dlogits = g (onehot - softmax) on legal columns
//   k_gemm<Dgrad> dlogits Wf (K = Ap) masked by h_NL > 0 -> dz_NL; then dz_l W_l -> dz_{l-1}
//   k_ls_wgrad    dW_l = h_{l-1}^T dz_l, dWf = h_NL^T dlogits (per 256 columns),
//                 dW1 = obs^T dz_1 (per 256 features, one-hot operand built in smem):
//                 MN-major tcgen05 over 64-row stages, warp-specialised
//   k_ls_colsum, k_ls_reduce   fixed-order reductions into the flat gradient; then Adam.
#include <math.h>
#include <string.h>

#include <type_traits>
#include <vector>

#include "engine.h"
#include "gemm.cuh"

namespace gfnx {

namespace {

constexpr int kH = 256;     // hidden width of this path
constexpr int kMaxNL = 4;   // hidden layers
constexpr int kMaxTasks = 48;

// ---------------------------------------------------------------------------
// env adapters: legality of 32 consecutive columns and the features of one 256-block,
// both straight from the packed state words.
template <class E>
struct Lock;

template <>
struct Lock<BitseqEnv> {  // k = 8 (256-word slots), <= 32 slots
  GFNX_DEV static uint32_t legal32(const EnvParams& P, const uint32_t* w, int c0) {
    if (c0 >= P.A) return 0u;
    if (P.bs_ar) return 0xffffffffu;  // AR fixed: every token (rows are never terminal here)
    const int tw = (P.bs_slots + 3) / 4;
    return ((w[tw] >> (c0 >> 8)) & 1u) ? 0u : 0xffffffffu;
  }
  // the state words legality depends on, cached in registers by the GEMM epilogues
  static constexpr int kLW = 1;
  // (AR fixed: no slot is ever blocked before the end, so the cached word is 0 and every
  //  column < A reads as legal, branch-free in the per-chunk test)
  GFNX_DEV static void load_lw(const EnvParams& P, const uint32_t* w, uint32_t (&lw)[kLW]) {
    lw[0] = P.bs_ar ? 0u : w[(P.bs_slots + 3) / 4];
  }
  GFNX_DEV static uint32_t legal32c(const EnvParams& P, const uint32_t (&lw)[kLW], int c0) {
    if (c0 >= P.A) return 0u;
    return ((lw[0] >> (c0 >> 8)) & 1u) ? 0u : 0xffffffffu;
  }
  // features with index in [f0, f0 + 256): put(f - f0, value); `part` of 4 splits the work
  template <class F>
  GFNX_DEV static void block_features(const EnvParams& P, const uint32_t* w, int f0, int part, F&& put) {
    const int V = P.bs_vocab, W = V + 1, S = P.bs_slots, tw = (S + 3) / 4;
    const uint32_t filled = w[tw];
    for (int p = part; p < S; p += 4) {
      const int f = p * W + (((filled >> p) & 1u) ? (int)((w[p >> 2] >> (8 * (p & 3))) & 0xffu) : V);
      if (f >= f0 && f < f0 + 256) put(f - f0, 1.f);
    }
    if (part == 0) {
      const int f = S * W;
      if (f >= f0 && f < f0 + 256) put(f - f0, (float)__popc(filled) / (float)S);
    }
  }
};

template <>
struct Lock<IsingEnv> {
  GFNX_DEV static uint32_t legal32(const EnvParams& P, const uint32_t* w, int c0) {
    if (c0 >= P.A) return 0u;
    const int site0 = c0 >> 1;  // 16 sites, inside one assigned-word
    uint32_t x = ~(w[site0 >> 5] >> (site0 & 31)) & 0xffffu;
    x = (x | (x << 8)) & 0x00FF00FFu;
    x = (x | (x << 4)) & 0x0F0F0F0Fu;
    x = (x | (x << 2)) & 0x33333333u;
    x = (x | (x << 1)) & 0x55555555u;
    x |= x << 1;
    const int left = P.A - c0;
    return left >= 32 ? x : (x & ((1u << left) - 1u));
  }
  static constexpr int kLW = 8;  // assigned-site words (<= 256 sites)
  GFNX_DEV static void load_lw(const EnvParams& P, const uint32_t* w, uint32_t (&lw)[kLW]) {
#pragma unroll
    for (int k = 0; k < kLW; ++k) lw[k] = k < P.SW / 2 ? w[k] : 0u;
  }
  GFNX_DEV static uint32_t legal32c(const EnvParams& P, const uint32_t (&lw)[kLW], int c0) {
    if (c0 >= P.A) return 0u;
    const int site0 = c0 >> 1, wi = site0 >> 5;
    uint32_t word = lw[0];
#pragma unroll
    for (int k = 1; k < kLW; ++k) word = wi == k ? lw[k] : word;
    uint32_t x = ~(word >> (site0 & 31)) & 0xffffu;
    x = (x | (x << 8)) & 0x00FF00FFu;
    x = (x | (x << 4)) & 0x0F0F0F0Fu;
    x = (x | (x << 2)) & 0x33333333u;
    x = (x | (x << 1)) & 0x55555555u;
    x |= x << 1;
    const int left = P.A - c0;
    return left >= 32 ? x : (x & ((1u << left) - 1u));
  }
  template <class F>
  GFNX_DEV static void block_features(const EnvParams& P, const uint32_t* w, int f0, int part, F&& put) {
    const int nw = P.SW / 2;
    const int i0 = f0 / 3, i1 = min(P.is_D, (f0 + 256 + 2) / 3);
    for (int i = i0 + part; i < i1; i += 4) {
      const uint32_t asg = (w[i >> 5] >> (i & 31)) & 1u, up = (w[nw + (i >> 5)] >> (i & 31)) & 1u;
      const int f = 3 * i + (asg ? (int)up : 2);
      if (f >= f0 && f < f0 + 256) put(f - f0, 1.f);
    }
  }
};

struct LsState {
  int num_sms = 0;
  int NL = 2, A = 0, Ap = 0, NT = 0, G = 0, O = 0, OB = 0, T = 0, KBA = 0;
  int Bl = 0, R = 0, tilesB = 0, tilesR = 0, SW = 0;
  int flow = 0;                              // DB / SubTB: log-flow head = head column A
  float* flowv = nullptr;                    // [R] log F(s) of every row (fp32, before rounding)
  float* gflow = nullptr;                    // [R] dL / dlog F(s)
  __nv_bfloat16* w1 = nullptr;               // [O][H] row-major
  __nv_bfloat16* wfw[kMaxNL] = {};           // layer l (1..NL-1): [H out][H in] image
  __nv_bfloat16* wdg[kMaxNL] = {};           // layer l: [H in][H out] image
  __nv_bfloat16* wff = nullptr;              // head fwd image: NT n-tiles x 4 K-blocks
  uint8_t* l1img = nullptr;                  // Ising layer-1 delta image (persistent rollout)
  __nv_bfloat16* wfd = nullptr;              // head dgrad image: 1 n-tile x KBA K-blocks
  float* bfp = nullptr;                      // head bias padded to Ap
  float* h1init = nullptr;                   // [H]
  float* preact = nullptr;                   // [Bl][H]
  uint32_t* cur = nullptr;                   // [Bl][SW] current packed state
  uint32_t* stst = nullptr;                  // [R][SW] state before the step of row r
  int32_t* last_act = nullptr;               // [Bl]
  __nv_bfloat16* h[kMaxNL] = {};             // [R] images, h[l] = output of hidden layer l+1
  __nv_bfloat16* dz[kMaxNL] = {};
  uint8_t* mask[kMaxNL] = {};                // [R][H/8]
  __nv_bfloat16* logits = nullptr;           // [Bl][Ap] row-major, per-step scratch
  float2* stats = nullptr;                   // [Bl][G] (max, sum exp) per 128-column group
  __nv_bfloat16* dlog = nullptr;             // [R] x Ap image
  float* rowbuf = nullptr;                   // [R][2]: logp(a), lse
  float* coef = nullptr;                     // [R]
  int bw = 0;                                // bias columns: NL*H + Ap
  float* bpart = nullptr;                    // [tilesR][bw] per-tile bias column sums
  int cgroups = 0;
  float* bpart2 = nullptr;                   // [cgroups][bw]
  float* wpart = nullptr;                    // [task][range][256][256]
  int ntasks = 0;
  int first[kMaxTasks + 1] = {};             // wgrad CTAs of task k: [first[k], first[k+1])
  int t_dense = 0, t_head = 0, t_w1 = 0;     // first task of each kind
  double* lpart = nullptr;
  double* lampow = nullptr;                  // SubTB: pow(lambda, k), k = 0..T
  int loss_blocks = 0;
};

LsState& LS(Ctx& c) { return *static_cast<LsState*>(c.fast); }

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
template <class E>
__global__ void __launch_bounds__(256) k_ls_layer1(L1Args a) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * 8 + warp;
  if (b >= a.Bl) return;
  float v[8];
  float* pre = a.preact + (size_t)b * kH + 8 * lane;
  if (a.t == 0) {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = a.h1init[8 * lane + j];
  } else {
    const float4 p0 = *reinterpret_cast<const float4*>(pre), p1 = *reinterpret_cast<const float4*>(pre + 4);
    v[0] = p0.x; v[1] = p0.y; v[2] = p0.z; v[3] = p0.w;
    v[4] = p1.x; v[5] = p1.y; v[6] = p1.z; v[7] = p1.w;
    auto add_row = [&](int f, float coef) {
      const uint4 q = __ldg(reinterpret_cast<const uint4*>(a.w1 + (size_t)f * kH) + lane);
      const uint32_t x[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        v[2 * e] += coef * bf16_lo(x[e]);
        v[2 * e + 1] += coef * bf16_hi(x[e]);
      }
    };
    if constexpr (std::is_same<E, BitseqEnv>::value) {
      // BitseqEnv::delta_features: the last action's slot leaves "empty" for its token
      // (NAR: slot act / V; AR fixed: slot t - 1, the token is the action), count feature + 1/S
      const int V = a.P.bs_vocab, W = V + 1, act = a.last_act[b];
      const int pos = a.P.bs_ar ? a.t - 1 : act / V, tok = a.P.bs_ar ? act : act - pos * V;
      add_row(pos * W + V, -1.0f);
      add_row(pos * W + tok, 1.0f);
      add_row(a.P.bs_slots * W, 1.0f / (float)a.P.bs_slots);
    } else {
      typename E::State dummy;
      E::delta_features(a.P, dummy, a.last_act[b], add_row);
    }
  }
  *reinterpret_cast<float4*>(pre) = make_float4(v[0], v[1], v[2], v[3]);
  *reinterpret_cast<float4*>(pre + 4) = make_float4(v[4], v[5], v[6], v[7]);
  uint32_t pk[4];
  uint32_t mb = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    pk[e] = pack_bf16x2_relu(v[2 * e], v[2 * e + 1]);
    mb |= (bf16_lo(pk[e]) > 0.f ? 1u : 0u) << (2 * e);
    mb |= (bf16_hi(pk[e]) > 0.f ? 1u : 0u) << (2 * e + 1);
  }
  const size_t r = (size_t)a.t * a.Bl + b;
  uint8_t* tile = a.h1 + (r / kTile) * (kTile * kH * 2);
  *reinterpret_cast<uint4*>(tile + sw128_offset((uint32_t)(r % kTile), 8 * lane, kTile)) =
      make_uint4(pk[0], pk[1], pk[2], pk[3]);
  a.mask1[r * (kH / 8) + lane] = (uint8_t)mb;
}

// ReLU mask of 32 consecutive bf16 columns (16 packed pairs, values >= 0 or +0), bit k <->
// column k (set when nonzero): the two flags of pair i land at bits i / 16 + i in 4
// instructions per pair, then one bit interleave of the two halves (Hacker's Delight 7-2)
GFNX_DEV uint32_t relu_mask32_seq(const uint32_t (&pk)[16]) {
  uint32_t x = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint32_t y = (pk[i] & 0x7FFF7FFFu) + 0x7FFF7FFFu;  // flags at bit 15 (column 2i), 31 (2i + 1)
    x |= (y >> (15 - i)) & (0x00010001u << i);
  }
  x = ((x & 0x0000FF00u) << 8) | ((x >> 8) & 0x0000FF00u) | (x & 0xFF0000FFu);
  x = ((x & 0x00F000F0u) << 4) | ((x >> 4) & 0x00F000F0u) | (x & 0xF00FF00Fu);
  x = ((x & 0x0C0C0C0Cu) << 2) | ((x >> 2) & 0x0C0C0C0Cu) | (x & 0xC3C3C3C3u);
  x = ((x & 0x22222222u) << 1) | ((x >> 1) & 0x22222222u) | (x & 0x99999999u);
  return x;
}

struct HidEpi : EpiBase {  // +b, ReLU -> h image + mask
  struct Args {
    const float* b;
    uint8_t* h;
    uint8_t* mask;
  };
  struct Local {};
  static __device__ const float* bias_src(const Args& e) { return e.b; }
  static __device__ void set_bias(Args& e, const float* b) { e.b = b; }
  static __device__ void apply(const Args& e, int m, int, int row, int col0, float (&v)[32], float*, Local&) {
    uint32_t pk[16];
    const float4* bb = reinterpret_cast<const float4*>(e.b + col0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float4 q = bb[i];
      pk[2 * i] = bias_relu_pack(__float_as_uint(v[4 * i]), __float_as_uint(v[4 * i + 1]), make_float2(q.x, q.y));
      pk[2 * i + 1] = bias_relu_pack(__float_as_uint(v[4 * i + 2]), __float_as_uint(v[4 * i + 3]), make_float2(q.z, q.w));
    }
    const uint32_t mb = relu_mask32_seq(pk);  // bit k <-> column col0 + k
    st_row32_g(e.h + (size_t)m * (kTile * kH * 2), row, col0, pk);
    const size_t r = (size_t)m * kTile + row;
    *reinterpret_cast<uint32_t*>(e.mask + r * (kH / 8) + col0 / 8) = mb;
  }
};

// +bf -> bf16 logits row-major [Bl][Ap] and masked (max, sum exp) per 128-column group
template <class E, bool FLOW = false>  // FLOW: DB / SubTB capture the log-flow column
struct LogEpi : EpiBase {
  struct Args {
    EnvParams P;
    const float* bf;  // padded to Ap
    const uint32_t* cur;
    __nv_bfloat16* logits;
    float2* stats;
    int Ap, G, row_base;  // global row of tile 0 of this step
    float* flowv;         // DB / SubTB: fp32 log F of the row (head column A), else null
  };
  struct Local {
    float mx, s;
    uint32_t lw[Lock<E>::kLW];
  };
  static __device__ const float* bias_src(const Args& e) { return e.bf; }
  static __device__ void set_bias(Args& e, const float* b) { e.bf = b; }
  static __device__ void begin(const Args& e, int m, int, int row, int, Local& l) {
    l.mx = -INFINITY;
    l.s = 0.f;
    const int b = m * kTile + row - e.row_base;
    Lock<E>::load_lw(e.P, e.cur + (size_t)b * e.P.SW, l.lw);
  }
  static __device__ void apply(const Args& e, int m, int n, int row, int col0, float (&v)[32], float*, Local& l) {
    const int b = m * kTile + row - e.row_base;
    const int c = n * 256 + col0;
    const uint32_t lm = Lock<E>::legal32c(e.P, l.lw, c);
    uint32_t pk[16];
    float cm = -INFINITY;
    const float4* bb = reinterpret_cast<const float4*>(e.bf + c);
    if (FLOW && e.P.A >= c && e.P.A < c + 32) {  // the log-flow column, before bf16 rounding
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (c + i == e.P.A) e.flowv[(size_t)m * kTile + row] = v[i] + e.bf[c + i];
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float4 bq = bb[i];
      pk[2 * i] = pack_bf16x2(v[4 * i] + bq.x, v[4 * i + 1] + bq.y);
      pk[2 * i + 1] = pack_bf16x2(v[4 * i + 2] + bq.z, v[4 * i + 3] + bq.w);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      v[2 * i] = bf16_lo(pk[i]);
      v[2 * i + 1] = bf16_hi(pk[i]);
    }
    if constexpr (std::is_same<E, BitseqEnv>::value) {  // legality is per 256-column slot
      if (lm) {
#pragma unroll
        for (int i = 0; i < 32; ++i) cm = fmaxf(cm, v[i]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if ((lm >> i) & 1u) cm = fmaxf(cm, v[i]);
    }
    uint8_t* dst = reinterpret_cast<uint8_t*>(e.logits + (size_t)b * e.Ap + c);
#pragma unroll
    for (int q = 0; q < 2; ++q)
      asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst + 32 * q), "r"(pk[8 * q]),
                   "r"(pk[8 * q + 1]), "r"(pk[8 * q + 2]), "r"(pk[8 * q + 3]), "r"(pk[8 * q + 4]),
                   "r"(pk[8 * q + 5]), "r"(pk[8 * q + 6]), "r"(pk[8 * q + 7])
                   : "memory");
    if (lm == 0u) return;
    const float nm = fmaxf(l.mx, cm), nm2 = -nm * kLog2e;
    float s = 0.f;
    if constexpr (std::is_same<E, BitseqEnv>::value) {  // all 32 columns legal here
#pragma unroll
      for (int i = 0; i < 32; ++i) s += ex2_ftz(fmaf(v[i], kLog2e, nm2));
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) s += ((lm >> i) & 1u) ? ex2_ftz(fmaf(v[i], kLog2e, nm2)) : 0.f;
    }
    l.s = l.s * ex2_ftz((l.mx - nm) * kLog2e) + s;  // l.mx = -inf -> factor 0
    l.mx = nm;
  }
  // the four 64-column parts of a row leave (max, sum exp) partials in scratch; finish()
  // merges the two parts of each 128-column group (online-softmax combine)
  static __device__ void row_done(const Args&, int, int, int row, int part, float* scratch, Local& l) {
    scratch[(row * 4 + part) * 2] = l.mx;
    scratch[(row * 4 + part) * 2 + 1] = l.s;
  }
  static __device__ void finish(const Args& e, int m, int n, const float* scratch) {
    const int c = threadIdx.x - 128;  // 256 of the 512 epilogue threads: (row, group)
    if (c >= 2 * kTile) return;
    const int row = c >> 1, g = c & 1;
    const float m0 = scratch[(row * 4 + 2 * g) * 2], s0 = scratch[(row * 4 + 2 * g) * 2 + 1];
    const float m1 = scratch[(row * 4 + 2 * g + 1) * 2], s1 = scratch[(row * 4 + 2 * g + 1) * 2 + 1];
    const float mx = fmaxf(m0, m1);
    const float sum = (m0 == -INFINITY ? 0.f : s0 * __expf(m0 - mx)) + (m1 == -INFINITY ? 0.f : s1 * __expf(m1 - mx));
    const int b = m * kTile + row - e.row_base;
    e.stats[(size_t)b * e.G + 2 * n + g] = make_float2(mx, sum);
  }
};

struct SampleArgs {
  EnvParams P;
  Key key;  // fold_in(rollout key, t)
  double eps;
  int b0, Bl, t, T, Ap, G;  // Bl: padded row stride (a multiple of 128)
  const __nv_bfloat16* logits;
  const float2* stats;
  uint32_t* cur;
  uint32_t* stst;
  int32_t* last_act;
  float* rowbuf;
  DeviceBatch batch;
  const int16_t* forced;  // [nreal * T] teacher-forced actions (rows starting with -1 are sampled) or null
  int nreal;              // real trajectories (rows >= nreal pad the batch to a multiple of 128)
};

GFNX_DEV double warp_sum_d(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// warp per trajectory: two-level inverse CDF with the reference's single uniform
template <class E>
GFNX_DEV void sample_one(const SampleArgs& a, int b, double u01) {
  const int lane = threadIdx.x & 31;
  const EnvParams& P = a.P;
  const uint32_t* w = a.cur + (size_t)b * P.SW;
  // ---- group level (lane g <-> 128-column group g; G <= 32)
  int lcount = 0;
  float gm = -INFINITY, gs = 0.f;
  if (lane < a.G) {
#pragma unroll
    for (int q = 0; q < 4; ++q) lcount += __popc(Lock<E>::legal32(P, w, lane * 128 + q * 32));
    const float2 st = a.stats[(size_t)b * a.G + lane];
    if (lcount > 0) {
      gm = st.x;
      gs = st.y;
    }
  }
  float hi = gm;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  const double gz = lcount > 0 ? (double)gs * (double)__expf(gm - hi) : 0.0;
  const double z = warp_sum_d(gz);
  int legal = lcount;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) legal += __shfl_xor_sync(0xffffffffu, legal, o);
  const double eps = a.eps;
  const double u_eps = legal > 0 ? eps / legal : 0.0;
  const double kz = (1.0 - eps) / z;  // policy weight scale (0 at eps = 1: bit-exact draws)
  const double mass = lcount > 0 ? kz * gz + u_eps * lcount : 0.0;
  double incl = mass;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const double total = __shfl_sync(0xffffffffu, incl, 31);
  double x = u01 * total;
  const unsigned pos = __ballot_sync(0xffffffffu, mass > 0.0);
  const unsigned hit = __ballot_sync(0xffffffffu, mass > 0.0 && x < incl);
  int grp = -1, act = -1;
  if (pos) {
    grp = hit ? __ffs(hit) - 1 : 31 - __clz(pos);  // rounding: last positive group
    x -= __shfl_sync(0xffffffffu, incl - mass, grp);
    // ---- column level: 4 consecutive columns per lane
    const int c = grp * 128 + lane * 4;
    const uint32_t lm = (Lock<E>::legal32(P, w, grp * 128 + (lane >> 3) * 32) >> ((lane & 7) * 4)) & 0xfu;
    const uint2 q = *reinterpret_cast<const uint2*>(a.logits + (size_t)b * a.Ap + c);
    const float xs[4] = {bf16_lo(q.x), bf16_hi(q.x), bf16_lo(q.y), bf16_hi(q.y)};
    double w4[4], ls = 0.0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      w4[e] = ((lm >> e) & 1u) ? kz * (double)__expf(xs[e] - hi) + u_eps : 0.0;
      ls += w4[e];
    }
    double ci = ls;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, ci, o);
      if (lane >= o) ci += y;
    }
    const unsigned h2 = __ballot_sync(0xffffffffu, ls > 0.0 && x < ci);
    int pick = -1;
    if (h2) {
      const int src = __ffs(h2) - 1;
      if (lane == src) {
        // first positive column whose running sum passes x, else the last positive one
        // (unrolled selects: w4 stays in registers)
        double acc = ci - ls;
        int first = -1, lastpos = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          acc += w4[e];
          if (w4[e] > 0.0) {
            if (first < 0 && x < acc) first = e;
            lastpos = e;
          }
        }
        pick = first >= 0 ? first : lastpos;
      }
      pick = __shfl_sync(0xffffffffu, pick, src);
      act = grp * 128 + src * 4 + pick;
    } else {  // rounding fallback: last legal column of the group
      const unsigned any = __ballot_sync(0xffffffffu, lm != 0u);
      const int src = 31 - __clz(any);
      const uint32_t ml = __shfl_sync(0xffffffffu, lm, src);
      act = grp * 128 + src * 4 + (31 - __clz(ml));
    }
  }
  // ---- record + env step (lane 0)
  bool fin = false;  // lane 0: the step entered a terminal state (its reward below, warp-wide)
  if (lane == 0) {
    const size_t bt = (size_t)b * a.T + a.t;
    const size_t r = (size_t)a.t * a.Bl + b;
    if (a.forced && b < a.nreal && a.forced[(size_t)b * a.T] >= 0) {  // rollout_from_actions (env_core.hpp:166-229)
      act = a.forced[bt];  // legality from the packed words (no unpacked State on the stack)
      if (act < 0 || act >= P.A || !((Lock<E>::legal32(P, w, act & ~31) >> (act & 31)) & 1u)) act = -1;
    }
    if (act < 0 || !(z > 0.0)) {
      atomicExch(a.batch.counters + 3, GFNX_ERR_CONTRACT);
      act = -1;
    }
  }
  if (__shfl_sync(0xffffffffu, act, 0) < 0) return;  // (warp-uniform)
  if (lane == 0) {
    const size_t bt = (size_t)b * a.T + a.t;
    const size_t r = (size_t)a.t * a.Bl + b;
    const float xa = __bfloat162float(a.logits[(size_t)b * a.Ap + act]);
    const float lse = hi + __logf((float)z);
    a.rowbuf[2 * r] = xa - lse;
    a.rowbuf[2 * r + 1] = lse;
    for (int i = 0; i < P.SW; ++i) a.stst[r * P.SW + i] = w[i];
    bool term;
    int nparents;
    uint32_t* cw = a.cur + (size_t)b * P.SW;
    if constexpr (std::is_same<E, BitseqEnv>::value) {
      // step in the packed domain (token byte + filled bit; sequences.cpp:257-267): no
      // per-token unpack / pack on the serial path, full state only at termination
      const int tw = (P.bs_slots + 3) / 4;
      const int pos = P.bs_ar ? __popc(w[tw]) : act / P.bs_vocab, sh = 8 * (pos & 3);  // AR: next slot
      cw[pos >> 2] = (w[pos >> 2] & ~(0xffu << sh)) | ((uint32_t)(P.bs_ar ? act : act % P.bs_vocab) << sh);
      const uint32_t filled = w[tw] | (1u << pos);
      cw[tw] = filled;
      nparents = P.bs_ar ? 1 : __popc(filled);
      term = __popc(filled) == P.bs_slots;
    } else {
      typename E::State s;
      E::unpack(P, w, s);
      term = E::step(P, s, act);
      E::pack(P, s, cw);
      nparents = E::num_parents(P, s);
    }
    a.batch.actions[bt] = (int16_t)act;
    a.batch.nparents[bt] = (uint16_t)nparents;
    a.last_act[b] = act;
    if (term) {
      a.batch.lengths[b] = a.t + 1;
      for (int i = 0; i < P.SW; ++i) a.batch.term_state[(size_t)b * P.SW + i] = cw[i];
      fin = true;
      if (!(std::is_same<E, BitseqEnv>::value && P.bs_words <= 2)) {
        typename E::State s;
        E::unpack(P, cw, s);
        a.batch.log_rewards[b] = E::log_reward(P, s);
      }
    }
    if (!isfinite(lse)) atomicExch(a.batch.counters + 3, GFNX_ERR_NUMERIC);
  }
  if constexpr (std::is_same<E, BitseqEnv>::value) {
    // ModeSet::log_reward (sequences.cpp:50-55) with the whole warp: lane s < slots places
    // token s's k bits (MSB first) into the <= 128-bit string, lane m takes modes m, m + 32,
    // ... (Hamming distance by popcount), warp min -> -beta * d / n (tabulated)
    if (P.bs_words <= 2 && __shfl_sync(0xffffffffu, fin ? 1 : 0, 0)) {
      __syncwarp();  // lane 0's new state words are visible to the warp
      const uint32_t* cw = a.cur + (size_t)b * P.SW;
      uint64_t lo = 0ull, hi = 0ull;
      if (lane < P.bs_slots) {
        const uint32_t tok = (cw[lane >> 2] >> (8 * (lane & 3))) & 0xffu;
        for (int j = 0; j < P.bs_k; ++j) {
          const int pos = lane * P.bs_k + j;  // string bit pos <- token bit k - 1 - j
          const uint64_t bit = (uint64_t)((tok >> (P.bs_k - 1 - j)) & 1u) << (63 - (pos & 63));
          if (pos < 64) lo |= bit;
          else hi |= bit;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lo |= __shfl_xor_sync(0xffffffffu, lo, o);
        hi |= __shfl_xor_sync(0xffffffffu, hi, o);
      }
      int best = P.bs_nbits + 1;
      for (int m = lane; m < P.n_modes; m += 32) {
        const uint64_t* md = P.modes + (size_t)m * P.bs_words;
        const int h = __popcll(lo ^ md[0]) + (P.bs_words > 1 ? __popcll(hi ^ md[1]) : 0);
        best = h < best ? h : best;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
      if (lane == 0) a.batch.log_rewards[b] = P.bs_logr[best];
    }
  }
}

constexpr int kSampleRows = 4;  // trajectories per warp (their uniforms drawn in parallel)

template <class E>
__global__ void __launch_bounds__(256) k_ls_sample(SampleArgs a) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bw = (blockIdx.x * 8 + warp) * kSampleRows;
  // rng.cpp:64-66 uniform of draw (t, b): lane j < kSampleRows draws row bw + j
  const double uj = (lane < kSampleRows && bw + lane < a.Bl)
                        ? uniform_scalar(fold_in(a.key, (uint64_t)(a.b0 + bw + lane)))
                        : 0.0;
#pragma unroll 1
  for (int j = 0; j < kSampleRows; ++j) {
    const double u01 = __shfl_sync(0xffffffffu, uj, j);
    if (bw + j < a.Bl) sample_one<E>(a, bw + j, u01);
  }
}

template <class E>
__global__ void k_ls_h1init(EnvParams P, const __nv_bfloat16* w1, const float* b1, float* h1init) {
  const int j = threadIdx.x;
  if (j >= kH) return;
  typename E::State s;
  E::reset(P, s);
  float v = b1[j];
  E::features(P, s, [&](int f, double val) { v += (float)val * __bfloat162float(w1[(size_t)f * kH + j]); });
  h1init[j] = v;
}

__global__ void k_ls_reset(int n, uint32_t* cur) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) cur[i] = 0;
}

// ---------------------------------------------------------------------------
// training kernels

struct LossArgs {
  DeviceBatch batch;
  int Bl, T;  // Bl: padded row stride; trajectories >= nreal are pad rows (coefficient 0)
  int nreal;
  double B_global;
  const double* neglog;
  const float* rowbuf;
  float* coef;
  double* lpart;
  const double* scalars;
};

__global__ void k_ls_loss(LossArgs a) {  // tb_loss objectives.cpp:120-142
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  double loss = 0.0, dlogz = 0.0;
  if (b >= a.nreal && b < a.Bl)
    for (int t = 0; t < a.T; ++t) a.coef[(size_t)t * a.Bl + b] = 0.f;
  if (b < a.nreal) {
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

// transition_loss (DB, objectives.cpp:94-118) and subtb_loss (:144-180) over the lockstep
// rows (every trajectory takes T steps): d_t = log pi(a_t|s_t) - log P_B, F(s_T) := log R,
// per-row dL/dlog pi(a) -> coef, dL/dlog F -> gflow; pad rows (b >= nreal) get zeros
struct FlowLossArgs {
  DeviceBatch batch;
  int Bl, T, nreal, subtb;
  double B_global, penalty, norm;  // norm: sum_{0<=j<k<=T} lambda^(k-j) (SubTB)
  const double* lampow;            // [T + 1] pow(lambda, k)
  const double* neglog;
  const float* rowbuf;
  const float* flowv;
  float* coef;
  float* gflow;
  double* lpart;
  const int32_t* nsteps;  // counters + 4: real transitions of the (global) batch
};

constexpr int kLsSubTBMaxT = 128;

__global__ void k_ls_loss_flow(FlowLossArgs a) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const int T = a.T;
  double loss = 0.0;
  if (b >= a.nreal && b < a.Bl)
    for (int t = 0; t < T; ++t) {
      a.coef[(size_t)t * a.Bl + b] = 0.f;
      a.gflow[(size_t)t * a.Bl + b] = 0.f;
    }
  if (b < a.nreal) {
    const double logR = a.batch.log_rewards[b];
    auto d_of = [&](int t) {
      const size_t r = (size_t)t * a.Bl + b;
      return (double)a.rowbuf[2 * r] - a.neglog[a.batch.nparents[(size_t)b * T + t]];
    };
    auto F_of = [&](int t) { return t < T ? (double)a.flowv[(size_t)t * a.Bl + b] : logR; };
    if (!a.subtb) {
      const double n = (double)*a.nsteps;
      double gprev = 0.0;
      for (int t = 0; t < T; ++t) {
        const size_t r = (size_t)t * a.Bl + b;
        const double res = F_of(t) - F_of(t + 1) + d_of(t);
        const double w = (t == T - 1 ? a.penalty : 1.0) / n;
        loss += w * (res * res);
        const double g = 2.0 * w * res;
        a.coef[r] = (float)g;
        a.gflow[r] = (float)(g - gprev);  // + from transition t, - from transition t - 1
        gprev = g;
      }
    } else {
      double cum[kLsSubTBMaxT + 1], F[kLsSubTBMaxT + 1], gF[kLsSubTBMaxT + 1], D[kLsSubTBMaxT + 1];
      cum[0] = 0.0;
      for (int t = 0; t < T; ++t) cum[t + 1] = cum[t] + d_of(t);
      for (int t = 0; t <= T; ++t) {
        F[t] = F_of(t);
        gF[t] = 0.0;
        D[t] = 0.0;
      }
      const double scale = 1.0 / a.norm / a.B_global;
      for (int j = 0; j < T; ++j)
        for (int k = j + 1; k <= T; ++k) {
          const double w = a.lampow[k - j] * scale;
          const double res = F[j] - F[k] + cum[k] - cum[j];
          loss += w * (res * res);
          const double g = 2.0 * w * res;
          gF[j] += g;
          gF[k] -= g;  // (k = T: the log-reward constant)
          D[j] += g;   // d_t for j <= t < k
          D[k] -= g;
        }
      double gd = 0.0;
      for (int t = 0; t < T; ++t) {
        const size_t r = (size_t)t * a.Bl + b;
        gd += D[t];
        a.coef[r] = (float)gd;
        a.gflow[r] = (float)gF[t];
      }
    }
  }
  __shared__ double red[256];
  red[threadIdx.x] = loss;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if ((int)threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    a.lpart[2 * blockIdx.x] = red[0];
    a.lpart[2 * blockIdx.x + 1] = 0.0;
  }
}

__global__ void k_ls_loss_finalize(const double* lpart, int n, double* scalars, int32_t* err) {
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

template <class E, bool FLOW = false>  // FLOW: DB / SubTB write the log-flow column's gradient
struct DlogEpi : EpiBase {  // recomputed logits -> dlogits image + per-tile column sums
  struct Args {
    EnvParams P;
    const float* bf;  // padded
    const float* rowbuf;
    const float* coef;
    const uint32_t* stst;
    const int16_t* actions;
    uint8_t* dlog;  // image with KBA K-blocks per tile
    float* bpart;   // [tilesR][bw]
    int Bl, T, KBA, bw, boff;
    const float* gflow;  // DB / SubTB: dL/dlog F per row -> head column A, else null
  };
  struct Local {
    float lse, g;
    int act;
    uint32_t lw[Lock<E>::kLW];
  };
  static __device__ const float* bias_src(const Args& e) { return e.bf; }
  static __device__ void set_bias(Args& e, const float* b) { e.bf = b; }
  static __device__ void begin(const Args& e, int m, int, int row, int, Local& l) {
    const size_t r = (size_t)m * kTile + row;
    const int t = (int)(r / e.Bl), b = (int)(r % e.Bl);
    l.lse = e.rowbuf[2 * r + 1];
    l.g = e.coef[r];
    l.act = e.actions[(size_t)b * e.T + t];
    Lock<E>::load_lw(e.P, e.stst + r * e.P.SW, l.lw);
  }
  static __device__ void finish(const Args& e, int m, int n, const float* scratch) {
    const int c = threadIdx.x - 128;  // the first 256 epilogue threads, one output column each
    if (c >= 256) return;
    const float s = scratch[c] + scratch[256 + c] + scratch[512 + c] + scratch[768 + c];
    e.bpart[(size_t)m * e.bw + e.boff + n * 256 + c] = s;
  }
  static __device__ void apply(const Args& e, int m, int n, int row, int col0, float (&v)[32], float* scratch,
                               Local& l) {
    const size_t r = (size_t)m * kTile + row;
    const int c0 = n * 256 + col0;
    const uint32_t lm = Lock<E>::legal32c(e.P, l.lw, c0);
    const float nl2 = -l.lse * kLog2e;
    uint32_t pk[16];
    const float4* bb = reinterpret_cast<const float4*>(e.bf + c0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {  // bf16 logits: FADD2 + one cvt per pair
      const float4 bq = bb[i];
      pk[2 * i] = add_pack_bf16x2(v[4 * i], v[4 * i + 1], bq.x, bq.y);
      pk[2 * i + 1] = add_pack_bf16x2(v[4 * i + 2], v[4 * i + 3], bq.z, bq.w);
    }
    // -g softmax = -g 2^(x log2e - lse log2e): FFMA2, two MUFU.EX2, FMUL2 per pair (the same
    // roundings as the scalar fmaf / multiply)
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float x0 = bf16_lo(pk[i]), x1 = bf16_hi(pk[i]);
      ffma2_st(x0, x1, kLog2e, nl2);
      x0 = ex2_ftz(x0);
      x1 = ex2_ftz(x1);
      fmul2_s(x0, x1, -l.g);
      float d0 = ((lm >> (2 * i)) & 1u) ? x0 : 0.f, d1 = ((lm >> (2 * i + 1)) & 1u) ? x1 : 0.f;
      if (c0 + 2 * i == l.act) d0 += l.g;
      if (c0 + 2 * i + 1 == l.act) d1 += l.g;
      v[2 * i] = d0;
      v[2 * i + 1] = d1;
    }
    if (FLOW && (unsigned)(e.P.A - c0) < 32u) {  // the log-flow column (warp-uniform test)
      const float gf = e.gflow[r];
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (c0 + i == e.P.A) v[i] = gf;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) pk[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
    uint8_t* blk = e.dlog + ((size_t)m * e.KBA + n * 4 + col0 / 64) * (kTile * 128);
    st_row32_g(blk, row, col0 % 64, pk);
    const float s = warp_colsum32(v);  // this warp's 32 rows, lane = column
    scratch[epi_quarter() * 256 + col0 + (threadIdx.x & 31)] = s;
  }
};

struct DgradEpi : EpiBase {  // masked by ReLU bits -> dz image + bias column sums
  struct Args {
    const uint8_t* mask;
    uint8_t* dz;
    float* bpart;
    int boff, bw;
  };
  struct Local {};
  static __device__ void finish(const Args& e, int m, int, const float* scratch) {
    const int c = threadIdx.x - 128;
    if (c >= 256) return;
    const float s = scratch[c] + scratch[256 + c] + scratch[512 + c] + scratch[768 + c];
    e.bpart[(size_t)m * e.bw + e.boff + c] = s;
  }
  static __device__ void apply(const Args& e, int m, int, int row, int col0, float (&v)[32], float* scratch,
                               Local&) {
    const size_t r = (size_t)m * kTile + row;
    const uint32_t mk = *reinterpret_cast<const uint32_t*>(e.mask + r * (kH / 8) + col0 / 8);
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = ((mk >> i) & 1u) ? v[i] : 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) pk[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
    st_row32_g(e.dz + (size_t)m * (kTile * kH * 2), row, col0, pk);
    const float s = warp_colsum32(v);
    scratch[epi_quarter() * 256 + col0 + (threadIdx.x & 31)] = s;
  }
};

// ---------------------------------------------------------------------------
// weight gradients: one CTA per (task, row range); per 64-row stage
//   dense task   A' = activation image (256 features, MN-major), B' = 256-column chunk of
//                a gradient image (dz_l or dlogits)
//   one-hot task A' = obs features [f0, f0 + 256) of the stage rows, built in smem from the
//                packed states (bulk-copied beside the operands), B' = dz_1
// Warp roles: warp 0 producer, warp 1 MMA issuer, warps 4..11 builders + epilogue.

constexpr int kWStage = 64;  // rows per stage
constexpr int kWStages = 3;
constexpr int kWOp = kWStage * 256 * 2;  // 32 KB operand per stage
constexpr int kWStBytes = kWStage * 16 * 4;  // packed states of a stage (SW <= 16)

struct WgTask {
  const uint8_t* a;  // dense: A' image (4 K-blocks per tile); one-hot: nullptr
  const uint8_t* b;  // B' image
  int b_kbs, b_kb0;  // K-blocks per tile of the B' image, first block used
  int f0, nf;        // one-hot: feature block [f0, f0 + nf)
};

struct WgArgs {
  EnvParams P;
  const uint32_t* stst;
  int tilesR, ntasks;
  int first[kMaxTasks + 1];  // CTAs [first[k], first[k+1]) split task k's rows into ranges
  float* wpart;
  long long* phase;  // optional diagnostics (gfnx_phase_timers)
  WgTask task[kMaxTasks];
};

GFNX_DEV void wg_copy_half(uint8_t* dst, const uint8_t* tile, int blk0, int h, uint64_t* bar) {
  // rows [64h, 64h + 64) of 4 feature blocks [blk0, blk0 + 4) of a 128-row tile image
  for (int k = 0; k < 4; ++k)
    bulk_g2s(dst + k * (kWStage * 128), tile + (size_t)(blk0 + k) * (kTile * 128) + h * (kWStage * 128),
             kWStage * 128, bar);
}

template <class E>
__global__ void __launch_bounds__(kGemmThreads, 1) k_ls_wgrad(const __grid_constant__ WgArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  constexpr int kSlot = 2 * kWOp + kWStBytes;
  __shared__ uint64_t full[kWStages], empty[kWStages], built[kWStages], done;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int task = 0;
  while (task + 1 < a.ntasks && (int)blockIdx.x >= a.first[task + 1]) ++task;
  const int nranges = a.first[task + 1] - a.first[task], range = blockIdx.x - a.first[task];
  const WgTask& tk = a.task[task];
  const bool onehot = tk.a == nullptr;
  const int halves = (onehot && tk.nf <= 128) ? 1 : 2;  // M' = 256 (2 x 128) or 128
  const int per = (a.tilesR + nranges - 1) / nranges;
  const int t0 = range * per, t1 = min(a.tilesR, t0 + per);
  const int nq = t1 > t0 ? 2 * (t1 - t0) : 0;  // 64-row stages
  const int SW = a.P.SW;
  if (warp == 0) tmem_alloc<512>(&tbase);
  if (tid == 32) {
    for (int s = 0; s < kWStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&built[s], 1);
    }
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  const long long tk0 = clock64();
  long long* ph = a.phase ? a.phase + (onehot ? 0 : 8) : nullptr;
  if (warp == 0) {
    if (lane == 0) {  // ---- producer
      long long tw = 0;
      for (int q = 0; q < nq; ++q) {
        const int slot = q % kWStages, tile = t0 + q / 2, h = q % 2;
        const long long t0w = clock64();
        if (q >= kWStages) mbar_wait(&empty[slot], ((q / kWStages) - 1) & 1);
        tw += clock64() - t0w;
        uint8_t* sa = smem + slot * kSlot;
        uint8_t* sb = sa + kWOp;
        const int st_bytes = kWStage * SW * 4;
        mbar_arrive_expect_tx(&full[slot], (onehot ? st_bytes : kWOp) + kWOp);
        if (onehot)
          bulk_g2s(sb + kWOp, a.stst + ((size_t)tile * kTile + h * kWStage) * SW, st_bytes, &full[slot]);
        else
          wg_copy_half(sa, tk.a + (size_t)tile * (4 * kTile * 128), 0, h, &full[slot]);
        wg_copy_half(sb, tk.b + (size_t)tile * tk.b_kbs * (kTile * 128), tk.b_kb0, h, &full[slot]);
      }
      if (ph) atomicAdd((unsigned long long*)ph + 4, (unsigned long long)tw);
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      constexpr uint32_t idesc = umma_idesc_bf16(128, 256, true, true);
      long long tf = 0, tb = 0;
      for (int q = 0; q < nq; ++q) {
        const int slot = q % kWStages;
        const long long t0w = clock64();
        mbar_wait(&full[slot], (q / kWStages) & 1);
        const long long t1w = clock64();
        if (onehot) mbar_wait(&built[slot], (q / kWStages) & 1);
        tf += t1w - t0w;
        tb += clock64() - t1w;
        tc_fence_after();
        const uint32_t a0 = smem_u32(smem + slot * kSlot), b0 = a0 + kWOp;
        for (int hh = 0; hh < halves; ++hh)
#pragma unroll
          for (int k = 0; k < kWStage / 16; ++k)
            umma_bf16(tmem + hh * 256, umma_desc_sw128(a0 + hh * 2 * (kWStage * 128) + k * 2048, kWStage * 128, 1024),
                      umma_desc_sw128(b0 + k * 2048, kWStage * 128, 1024), idesc, (q > 0 || k > 0) ? 1u : 0u);
        umma_commit(&empty[slot]);
      }
      umma_commit(&done);
      if (ph) {
        atomicAdd((unsigned long long*)ph + 2, (unsigned long long)tf);
        atomicAdd((unsigned long long*)ph + 3, (unsigned long long)tb);
        atomicAdd((unsigned long long*)ph + 5, (unsigned long long)nq);
      }
    }
  } else if (warp >= 4) {
    const int et = tid - 128;  // 0..255
    if (onehot) {  // ---- builders
      long long tf = 0, tbld = 0;
      for (int q = 0; q < nq; ++q) {
        const int slot = q % kWStages;
        uint8_t* sa = smem + slot * kSlot;
        const long long t0w = clock64();
        mbar_wait(&full[slot], (q / kWStages) & 1);  // slot free (producer waited) + states in
        const long long t1w = clock64();
        tf += t1w - t0w;
        uint4* z = reinterpret_cast<uint4*>(sa);  // lane-contiguous 16-byte stores (no bank conflicts)
#pragma unroll
        for (int i = 0; i < 8; ++i) z[i * 256 + et] = make_uint4(0, 0, 0, 0);
        epi_bar();
        const int row = et & 63, part = et >> 6;
        const uint32_t* w = reinterpret_cast<const uint32_t*>(sa + 2 * kWOp) + row * SW;
        uint8_t* rowp = sa + row * 128;
        const int rsw = row & 7;
        Lock<E>::block_features(a.P, w, tk.f0, part, [&](int f, float v) {
          const int c = f & 63;
          *reinterpret_cast<__nv_bfloat16*>(rowp + (f >> 6) * (kWStage * 128) + ((((c >> 3) ^ rsw)) << 4) +
                                            (c & 7) * 2) = __float2bfloat16(v);
        });
        fence_proxy_async();
        epi_bar();
        if (et == 0) mbar_arrive_local(&built[slot]);
        tbld += clock64() - t1w;
      }
      if (ph && et == 0) {
        atomicAdd((unsigned long long*)ph + 0, (unsigned long long)tf);
        atomicAdd((unsigned long long*)ph + 1, (unsigned long long)tbld);
      }
    }
    // ---- epilogue: lane quarter x column half, both M'-halves
    const int ew = warp - 4, quarter = ew & 3, half = ew >> 2;
    if (nq > 0) mbar_wait_sleep(&done, 0, 2000);
    tc_fence_after();
    float* slab = a.wpart + (size_t)blockIdx.x * (256 * 256);
    for (int hh = 0; hh < 2; ++hh) {
      const int mrow = hh * 128 + quarter * 32 + lane;
      for (int q = 0; q < 4; ++q) {
        const int col = half * 128 + q * 32;
        uint32_t r32[32];
        tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + hh * 256 + col, r32);
        tmem_wait_ld();
        float4* dst = reinterpret_cast<float4*>(slab + (size_t)mrow * 256 + col);
        const bool ok = nq > 0 && hh < halves;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          dst[i] = ok ? make_float4(__uint_as_float(r32[4 * i]), __uint_as_float(r32[4 * i + 1]),
                                    __uint_as_float(r32[4 * i + 2]), __uint_as_float(r32[4 * i + 3]))
                      : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (ph && tid == 0) {
    atomicAdd((unsigned long long*)ph + 6, (unsigned long long)(clock64() - tk0));
    atomicAdd((unsigned long long*)ph + 7, 1ull);
  }
  if (warp == 0) tmem_dealloc<512>(tmem);
}

// bias column sums: bpart [tilesR][bw] -> bpart2 [groups][bw] (fixed order)
__global__ void k_ls_colsum(const float* bpart, int tilesR, int bw, int groups, float* bpart2) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x, g = blockIdx.y;
  if (col >= bw) return;
  const int per = (tilesR + groups - 1) / groups;
  const int t0 = g * per, t1 = min(tilesR, t0 + per);
  float s = 0.f;
  for (int t = t0; t < t1; ++t) s += bpart[(size_t)t * bw + col];
  bpart2[(size_t)g * bw + col] = s;
}

struct RedArgs {
  const float* wpart;
  const float* bpart2;
  float* g;
  int groups, bw, A, O, NL, t_dense, t_head, t_w1;
  int first[kMaxTasks + 1];
  MlpLayout L;
  int flow;
};

__global__ void k_ls_reduce(RedArgs a) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const MlpLayout& L = a.L;
  if (e >= L.n_params) return;
  auto slab_sum = [&](int task, int m, int n) {
    float s = 0.f;
    for (int c = a.first[task]; c < a.first[task + 1]; ++c) s += a.wpart[((size_t)c * 256 + m) * 256 + n];
    return s;
  };
  auto bias_sum = [&](int col) {
    float s = 0.f;
    for (int g = 0; g < a.groups; ++g) s += a.bpart2[(size_t)g * a.bw + col];
    return s;
  };
  float v = 0.f;
  if (e < L.off_b[0]) {  // W1 [O][H]
    const int f = (int)(e / kH), j = (int)(e % kH);
    v = slab_sum(a.t_w1 + f / 256, f % 256, j);
  } else if (e >= L.off_fw && e < L.off_fb) {  // head [H][A]
    const int64_t k = e - L.off_fw;
    const int p = (int)(k / a.A), c = (int)(k % a.A);
    v = slab_sum(a.t_head + c / 256, p, c % 256);
  } else if (e >= L.off_fb && e < L.off_fb + a.A) {
    v = bias_sum(a.NL * kH + (int)(e - L.off_fb));
  } else if (a.flow && e >= L.off_flw && e < L.off_flb) {  // log-flow head [H][1] = head column A
    v = slab_sum(a.t_head + a.A / 256, (int)(e - L.off_flw), a.A % 256);
  } else if (a.flow && e == L.off_flb) {
    v = bias_sum(a.NL * kH + a.A);
  } else {
    for (int l = 0; l < a.NL; ++l) {
      if (e >= L.off_b[l] && e < L.off_b[l] + kH) {
        v = bias_sum(l * kH + (int)(e - L.off_b[l]));
        break;
      }
      if (l >= 1 && e >= L.off_w[l] && e < L.off_b[l]) {  // W_{l+1} [in][out]
        const int64_t k = e - L.off_w[l];
        v = slab_sum(a.t_dense + l - 1, (int)(k / kH), (int)(k % kH));
        break;
      }
    }
  }
  a.g[e] = v;  // bwd / flow heads: unused by TB with uniform P_B -> 0
}

struct EmitArgs {
  const float* p;
  int64_t n;
  MlpLayout L;
  int A, NL, flow;
  __nv_bfloat16 *w1, *wff, *wfd;
  __nv_bfloat16* wfw[kMaxNL];
  __nv_bfloat16* wdg[kMaxNL];
  float* bfp;
};

__global__ void k_ls_emit(EmitArgs a) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.n) return;
  const MlpLayout& L = a.L;
  const __nv_bfloat16 v = __float2bfloat16(a.p[j]);
  if (j < L.off_b[0]) {
    a.w1[j] = v;
  } else if (j >= L.off_fw && j < L.off_fb) {
    const int64_t k = j - L.off_fw;
    const int p = (int)(k / a.A), c = (int)(k % a.A);
    const int n = c / 256, cc = c % 256;
    *reinterpret_cast<__nv_bfloat16*>((uint8_t*)a.wff + (size_t)n * (256 * kH * 2) + sw128_offset(cc, p, 256)) = v;
    *reinterpret_cast<__nv_bfloat16*>((uint8_t*)a.wfd + sw128_offset(p, c, kH)) = v;
  } else if (j >= L.off_fb && j < L.off_fb + a.A) {
    a.bfp[j - L.off_fb] = a.p[j];
  } else if (a.flow && j >= L.off_flw && j < L.off_flb) {  // log-flow head as head column A
    const int p = (int)(j - L.off_flw), c = a.A, n = c / 256, cc = c % 256;
    *reinterpret_cast<__nv_bfloat16*>((uint8_t*)a.wff + (size_t)n * (256 * kH * 2) + sw128_offset(cc, p, 256)) = v;
    *reinterpret_cast<__nv_bfloat16*>((uint8_t*)a.wfd + sw128_offset(p, c, kH)) = v;
  } else if (a.flow && j == L.off_flb) {
    a.bfp[a.A] = a.p[j];
  } else {
    for (int l = 1; l < a.NL; ++l)
      if (j >= L.off_w[l] && j < L.off_b[l]) {
        const int64_t k = j - L.off_w[l];
        const int p = (int)(k / kH), q = (int)(k % kH);
        *reinterpret_cast<__nv_bfloat16*>((uint8_t*)a.wfw[l] + sw128_offset(q, p, kH)) = v;
        *reinterpret_cast<__nv_bfloat16*>((uint8_t*)a.wdg[l] + sw128_offset(p, q, kH)) = v;
      }
  }
}

EmitArgs emit_args(Ctx& c) {
  LsState& f = LS(c);
  EmitArgs a{};
  a.p = c.p32;
  a.n = c.L.n_params;
  a.L = c.L;
  a.A = f.A;
  a.NL = f.NL;
  a.flow = f.flow;
  a.w1 = f.w1;
  a.wff = f.wff;
  a.wfd = f.wfd;
  for (int l = 0; l < kMaxNL; ++l) {
    a.wfw[l] = f.wfw[l];
    a.wdg[l] = f.wdg[l];
  }
  a.bfp = f.bfp;
  return a;
}

// ---------------------------------------------------------------------------
// k_ls_persist: the whole lockstep rollout (all T steps) in one persistent kernel, for
// heads that fit one 256-column MMA (Ap <= 256: Ising, A = 2D). CTA k owns the 128-row
// trajectory tiles k and k + gridDim.x (<= 2 per CTA); per step and tile:
//   layer 1    incremental fp32 pre-activation (global, L2-resident) from the two
//              features the last action changed -> ReLU -> packed bf16 A operand in TMEM
//   layers 2.. tcgen05.mma with A from TMEM ("TS" form) against the layer's weight image,
//              streamed into shared memory once per step and shared by both tiles
//   head       same, logits in the accumulator; the row's two threads run the reference
//              eps-uniform mixture + categorical (rng.cpp:87-100) over their 128 columns
//              with the fp64 running sum carried from the first half to the second
// Every output of the per-step pipeline is produced the same way (activation images +
// ReLU masks of every layer, log pi(a)/lse record, states, actions), so training is shared.
constexpr int kPersistMaxTiles = 2;

struct PersistArgs {
  EnvParams P;
  Key key;
  double eps;
  int b0, Bl, T, NL, A, tilesB;
  const __nv_bfloat16* w1;    // [O][H]
  const float* h1init;        // [H]
  float* preact;              // [Bl][H]
  const uint8_t* wimg[kMaxNL + 1];  // [0] Ising layer-1 delta image, [1..NL-1] hidden, [NL] head
  const float* bias[kMaxNL];  // [l] bias of layer l (l = 1..NL-1)
  const float* bfp;           // head bias padded
  uint8_t* h[kMaxNL];
  uint8_t* mask[kMaxNL];
  uint32_t* cur;
  uint32_t* stst;
  int32_t* last_act;
  float* rowbuf;
  DeviceBatch batch;
  long long* phase;  // optional clocks (thread 0): [0] layer 1, [1] hidden layers, [2] head + sample
  // Ising: layer 1 as an MMA over the assigned-spin one-hot (feature 2 site + up) against
  // W1[3s + u] - W1[3s + 2] (wimg[0]), bias = h1init: no per-row fp32 state between steps
  int l1_mma;
  float* flowv;  // DB / SubTB: fp32 log F of every row (head column A), else null
  const int16_t* forced;  // [nreal * T] teacher-forced actions (rows starting with -1 are sampled) or null
  int nreal;              // real trajectories (the rest pad the batch to a multiple of 128)
};

// ReLU bit mask of 32 columns in the lockstep byte-mask order (bit i of the word <-> column i)

// (streaming store: evict-first in L2, so the activation images written once per step do
// not push the per-row layer-1 state out of L2)
GFNX_DEV void st_v8_words(uint8_t* dst, const uint32_t* r) {
  asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst), "r"(r[0]), "r"(r[1]), "r"(r[2]),
               "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}

// one 128-byte line of a 128B-swizzled tile image (logical chunk l at l ^ (row & 7))
GFNX_DEV void st_line_sw(uint8_t* line, int row, const uint32_t (&r)[32]) {
  const int x = row & 7;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int p = (2 * m) ^ x;
    uint32_t v[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[i] = (x & 1) ? r[8 * m + 4 + i] : r[8 * m + i];
      v[4 + i] = (x & 1) ? r[8 * m + i] : r[8 * m + 4 + i];
    }
    st_v8_words(line + (p & ~1) * 16, v);
  }
}

template <class E>
__global__ void __launch_bounds__(256, 1) k_ls_persist(PersistArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* wbuf = align1024(smem_raw);  // one 256 x 256 weight image (128 KB)
  __shared__ uint64_t mbar, wbar;
  __shared__ uint32_t tbase;
  __shared__ __align__(16) float h1i[kH];
  __shared__ __align__(16) float bias_s[kMaxNL][kH];
  __shared__ __align__(16) float bhead_s[kH];  // padded head bias (Ap <= 256)  // [0] = h1i's role for l1_mma; [l] = bias of layer l
  __shared__ Key skeys[256];
  __shared__ double row_u[kPersistMaxTiles][kTile];
  __shared__ float xf[kTile][2];
  __shared__ int xi[kTile][2];
  __shared__ double xd[kTile];
  __shared__ int xlast[kTile][2];
  __shared__ int s_lact[kPersistMaxTiles][kTile];  // last action of each row (layer-1 delta)
  const EnvParams& P = a.P;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quarter = warp & 3, half = warp >> 2;
  const int row = quarter * 32 + lane, c0 = half * 128;
  const int ntile = (a.tilesB - (int)blockIdx.x + gridDim.x - 1) / gridDim.x;  // 1 or 2
  if (warp == 0) tmem_alloc<512>(&tbase);
  if (tid == 0) {
    mbar_init(&mbar, 1);
    mbar_init(&wbar, 1);
    fence_mbar_init();
  }
  for (int j = tid; j < kH; j += 256) {
    h1i[j] = a.h1init[j];
    bias_s[0][j] = a.h1init[j];
    for (int l = 1; l < a.NL; ++l) bias_s[l][j] = a.bias[l][j];
    bhead_s[j] = a.bfp[j];
  }
  for (int t = tid; t < a.T && t < 256; t += 256) skeys[t] = fold_in(a.key, (uint64_t)t);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
  uint32_t mph = 0, wph = 0;
  auto load_w = [&](int l) {  // thread 0: weight image l into wbuf (previous users complete)
    mbar_arrive_expect_tx(&wbar, kH * kH * 2);
    bulk_g2s_big(wbuf, a.wimg[l], kH * kH * 2, &wbar);
  };
  auto mma_issue = [&](uint32_t d, uint32_t ta) {
    if (tid == 0) {
      tc_fence_after();
      mma_tk<kH, kH>(d, ta, wbuf, false);
      umma_commit(&mbar);
    }
  };
  // every thread waits on the MMA's mbarrier (no CTA barrier): a publish() barrier
  // separates consecutive commits, so no thread can miss a phase
  auto mma_wait = [&]() {
    mbar_wait(&mbar, mph);
    mph ^= 1;
    tc_fence_after();
  };
  auto publish = [&]() {
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
  };
  if (tid == 0) load_w(a.l1_mma ? 0 : 1);
  const int T = a.T, Bl = a.Bl;
  long long pc[3] = {0, 0, 0}, tclk = clock64();
  long long hs[3] = {0, 0, 0}, hclk = 0;  // hidden-layer sub-phases (image wait, MMA, epilogue)
  auto hmark = [&](int k) {
    if (a.phase && tid == 0) {
      const long long tn = clock64();
      if (k >= 0) hs[k] += tn - hclk;
      hclk = tn;
    }
  };
  auto pmark = [&](int k) {
    if (a.phase && tid == 0) {
      const long long tn = clock64();
      pc[k] += tn - tclk;
      tclk = tn;
    }
  };
  for (int t = 0; t < T; ++t) {
    if (!a.l1_mma) {
    // ---- layer 1 for every tile of this CTA
    for (int j = 0; j < ntile; ++j) {
      const int tile = blockIdx.x + j * gridDim.x;
      const int b = tile * kTile + row;
      float* pre = a.preact + (size_t)b * kH + c0;
      const size_t r = (size_t)t * Bl + b;
      int f2[2] = {0, 0};
      float cf[2] = {0.f, 0.f};
      int nf = 0;
      if (t > 0) {
        typename E::State dummy;
        E::delta_features(P, dummy, s_lact[j][row], [&](int f, float coef) {
          if (nf < 2) {
            f2[nf] = f;
            cf[nf] = coef;
          }
          ++nf;
        });
      }
      // 32-column chunks with the next chunk's pre-activation and W1 loads in flight
      float pv[2][32];
      uint4 wv[2][2][4];
      auto load_chunk = [&](int q, float (&p32)[32], uint4 (&w8)[2][4]) {
        const int col = q * 32;
        if (t == 0) {
#pragma unroll
          for (int i = 0; i < 32; ++i) p32[i] = h1i[c0 + col + i];
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 p4 = *reinterpret_cast<const float4*>(pre + col + 4 * i);
            p32[4 * i] = p4.x;
            p32[4 * i + 1] = p4.y;
            p32[4 * i + 2] = p4.z;
            p32[4 * i + 3] = p4.w;
          }
        }
#pragma unroll
        for (int d = 0; d < 2; ++d) {
          const uint4* wr = reinterpret_cast<const uint4*>(a.w1 + (size_t)f2[d] * kH + c0 + col);
#pragma unroll
          for (int c = 0; c < 4; ++c) w8[d][c] = d < nf ? __ldg(wr + c) : make_uint4(0, 0, 0, 0);
        }
      };
      uint32_t mw[4];
      load_chunk(0, pv[0], wv[0]);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int col = q * 32;
        if (q + 1 < 4) load_chunk(q + 1, pv[(q + 1) & 1], wv[(q + 1) & 1]);
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = pv[q & 1][i];
#pragma unroll
        for (int d = 0; d < 2; ++d)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint4 w4 = wv[q & 1][d][c];
            const uint32_t wq[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              v[8 * c + 2 * e] += cf[d] * bf16_lo(wq[e]);
              v[8 * c + 2 * e + 1] += cf[d] * bf16_hi(wq[e]);
            }
          }
#pragma unroll
        for (int i = 0; i < 8; ++i)
          *reinterpret_cast<float4*>(pre + col + 4 * i) = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) pk[i] = pack_bf16x2_relu(v[2 * i], v[2 * i + 1]);
        mw[q] = relu_mask32_seq(pk);
        tmem_st16(lane_base + kH + 128 * j + ((c0 + col) >> 1), pk);
      }
      __stcs(reinterpret_cast<uint4*>(a.mask[0] + r * (kH / 8) + half * 16), make_uint4(mw[0], mw[1], mw[2], mw[3]));
    }
    publish();
    // layer-1 images straight from TMEM (both halves, own 128 columns = two 64-col blocks)
    for (int j = 0; j < ntile; ++j) {
      const int tile = blockIdx.x + j * gridDim.x;
      const size_t m = (size_t)t * a.tilesB + tile;
#pragma unroll 1
      for (int blk = 0; blk < 2; ++blk) {
        uint32_t w32[32];
        tmem_ld32(lane_base + kH + 128 * j + (c0 >> 1) + 32 * blk, w32);
        tmem_wait_ld();
        st_line_sw(a.h[0] + m * (kTile * kH * 2) + ((c0 >> 6) + blk) * (kTile * 128) + row * 128, row, w32);
      }
    }
    }
    pmark(0);
    // activation image of (layer, tile) from its packed TMEM columns, deferred into the next
    // MMA's wait (the columns stay intact until the next epilogue of the same tile)
    int pend_l = -1, pend_j = 0;
    size_t pend_m = 0;
    auto emit_pending = [&]() {
      if (pend_l < 0) return;
#pragma unroll 1
      for (int blk = 0; blk < 2; ++blk) {
        uint32_t w32[32];
        tmem_ld32(lane_base + kH + 128 * pend_j + (c0 >> 1) + 32 * blk, w32);
        tmem_wait_ld();
        st_line_sw(a.h[pend_l] + pend_m * (kTile * kH * 2) + ((c0 >> 6) + blk) * (kTile * 128) + row * 128, row, w32);
      }
      pend_l = -1;
    };
    // ---- hidden layers 2..NL: MMA per tile (A from TMEM), epilogue back into the same columns
    const int l0 = a.l1_mma ? 0 : 1;
    for (int l = l0; l < a.NL; ++l) {
      hmark(-1);
      if (tid == 0) mbar_wait(&wbar, wph);
      wph ^= 1;
      hmark(0);
      for (int j = 0; j < ntile; ++j) {
        const int tile = blockIdx.x + j * gridDim.x;
        const int b = tile * kTile + row;
        const size_t r = (size_t)t * Bl + b;
        const size_t m = (size_t)t * a.tilesB + tile;
        if (l == 0) {  // assigned-spin one-hot of the row, features [128 half, +128): 64 packed columns
          const uint32_t* w = a.cur + (size_t)b * P.SW;
          const int nw = P.SW / 2;
          const int w0 = 2 * half;  // sites [64 half, 64 half + 64) = state words 2 half, 2 half + 1
          uint32_t asg[2], up[2];
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            asg[k] = w0 + k < nw ? w[w0 + k] : 0u;
            up[k] = w0 + k < nw ? w[nw + w0 + k] : 0u;
          }
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            uint32_t ob[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {  // site 64 half + 32 hh + i: (spin -1, spin +1) bf16 pair
              const uint32_t as = (asg[hh] >> i) & 1u, u1 = (up[hh] >> i) & 1u;
              ob[i] = (as & (u1 ^ 1u)) * 0x3F80u | (as & u1) * 0x3F800000u;
            }
            tmem_st32(lane_base + kH + 128 * j + 64 * half + 32 * hh, ob);
          }
          publish();
        }
        mma_issue(tmem, tmem + kH + 128 * j);
        if (half == 1 && l == l0 && j < kPersistMaxTiles)  // the row's uniform while the MMA runs
          row_u[j][row] = uniform_scalar(fold_in(skeys[t], (uint64_t)(a.b0 + b)));
        emit_pending();
        mma_wait();
        hmark(1);
        if (j == ntile - 1 && tid == 0) load_w(l + 1 < a.NL ? l + 1 : a.NL);  // wbuf free now
        uint32_t mw[4];
        const float* bl = bias_s[l];  // shared memory (a generic pointer into one array: LDS)
#pragma unroll 1
        for (int q = 0; q < 4; ++q) {
          const int col = c0 + q * 32;
          uint32_t rr[32];
          tmem_ld32(lane_base + col, rr);
          tmem_wait_ld();
          uint32_t pk[16];
          const float4* bb = reinterpret_cast<const float4*>(bl + col);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 bq = bb[i];
            pk[2 * i] = bias_relu_pack(rr[4 * i], rr[4 * i + 1], make_float2(bq.x, bq.y));
            pk[2 * i + 1] = bias_relu_pack(rr[4 * i + 2], rr[4 * i + 3], make_float2(bq.z, bq.w));
          }
          mw[q] = relu_mask32_seq(pk);
          tmem_st16(lane_base + kH + 128 * j + (col >> 1), pk);
        }
        __stcs(reinterpret_cast<uint4*>(a.mask[l] + r * (kH / 8) + half * 16), make_uint4(mw[0], mw[1], mw[2], mw[3]));
        pend_l = l;
        pend_j = j;
        pend_m = m;
        publish();
        hmark(2);
      }
    }
    pmark(1);
    // ---- head + sampling per tile. The row's two threads own 128 logit columns each.
    //   P1  fp32 logits + bias -> bf16-rounded x (the values the training pass recomputes),
    //       legality words, max over legal
    //   P2  e = exp(x - hi) over legal, bf16 into the tile's consumed A columns,
    //       z; then the mixture w = kz e + eps/legal summed in fp64 in column order:
    //       first half, carry, second half (the reference's sequential running sum)
    //   P3  search for the first column whose running sum exceeds u * total
    if (tid == 0) mbar_wait(&wbar, wph);
    wph ^= 1;
    for (int j = 0; j < ntile; ++j) {
      const int tile = blockIdx.x + j * gridDim.x;
      const int b = tile * kTile + row;
      const size_t r = (size_t)t * Bl + b;
      mma_issue(tmem, tmem + kH + 128 * j);
      const uint32_t* w = a.cur + (size_t)b * P.SW;
      uint32_t lw[Lock<E>::kLW];
      Lock<E>::load_lw(P, w, lw);
      emit_pending();  // the last hidden layer's last tile
      mma_wait();
      if (j == ntile - 1 && tid == 0) load_w(a.l1_mma ? 0 : 1);  // next step's first layer
      uint32_t lmw[4];
      float hi = -INFINITY;
      int lcount = 0;
#pragma unroll 1
      for (int q = 0; q < 4; ++q) {  // P1
        const int col = c0 + q * 32;
        uint32_t rr[32];
        tmem_ld32(lane_base + col, rr);
        tmem_wait_ld();
        const uint32_t lm = Lock<E>::legal32c(P, lw, col);
        lmw[q] = lm;
        lcount += __popc(lm);
        const float4* bb = reinterpret_cast<const float4*>(bhead_s + col);
        if (a.flowv && (unsigned)(P.A - col) < 32u) {  // log F (head column A), fp32, warp-uniform test
#pragma unroll
          for (int k = 0; k < 32; ++k)
            if (col + k == P.A) a.flowv[r] = __uint_as_float(rr[k]) + bhead_s[col + k];
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float4 bq = bb[i];
          const float bv[4] = {bq.x, bq.y, bq.z, bq.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int k = 4 * i + e;
            const float x = __bfloat162float(__float2bfloat16(__uint_as_float(rr[k]) + bv[e]));
            rr[k] = __float_as_uint(x);
            if ((lm >> k) & 1u) hi = fmaxf(hi, x);
          }
        }
        tmem_st32(lane_base + col, rr);  // x (fp32 of the bf16 value) in place
      }
      xf[row][half] = hi;
      xi[row][half] = lcount;
      tmem_wait_st();
      __syncthreads();
      hi = fmaxf(xf[row][0], xf[row][1]);
      const int legal = xi[row][0] + xi[row][1];
      __syncthreads();
      float zl = 0.f;
      const uint32_t ta_e = lane_base + kH + 128 * j + (c0 >> 1);  // consumed A columns of this tile
#pragma unroll 1
      for (int q = 0; q < 4; ++q) {  // P2: e (bf16) into the tile's consumed A columns
        const int col = c0 + q * 32;
        uint32_t rr[32];
        tmem_ld32(lane_base + col, rr);
        tmem_wait_ld();
        uint32_t pe[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const float e0 = ((lmw[q] >> (2 * k)) & 1u) ? __expf(__uint_as_float(rr[2 * k]) - hi) : 0.f;
          const float e1 = ((lmw[q] >> (2 * k + 1)) & 1u) ? __expf(__uint_as_float(rr[2 * k + 1]) - hi) : 0.f;
          zl += e0;
          zl += e1;
          pe[k] = pack_bf16x2(e0, e1);
        }
        tmem_st16(ta_e + 16 * q, pe);
      }
      xf[row][half] = zl;
      tmem_wait_st();
      __syncthreads();
      const float z = xf[row][0] + xf[row][1];
      const double u = legal > 0 ? a.eps / (double)legal : 0.0;
      const double kz = (double)((float)(1.0 - a.eps) * __frcp_rn(z));
      // fp64 running sum over this thread's legal columns from `acc`; optional search
      auto run = [&](double acc, double x_target, int& pick, int& lastc) {
        pick = -1;
        lastc = -1;
#pragma unroll 1
        for (int h2 = 0; h2 < 2; ++h2) {  // 32 packed words = 64 columns per load
          uint32_t rr[32];
          tmem_ld32(ta_e + 32 * h2, rr);
          tmem_wait_ld();
#pragma unroll
          for (int k = 0; k < 64; ++k) {
            const int cc = 64 * h2 + k;  // column offset within this thread's half
            if ((lmw[cc >> 5] >> (cc & 31)) & 1u) {
              const float e = (k & 1) ? bf16_hi(rr[k >> 1]) : bf16_lo(rr[k >> 1]);
              acc += kz * (double)e + u;
              if (pick < 0 && x_target < acc) pick = c0 + cc;
              lastc = c0 + cc;
            }
          }
        }
        return acc;
      };
      int pk_, lc_;
      if (half == 0) xd[row] = run(0.0, -1.0, pk_, lc_);  // first half's total
      __syncthreads();
      const double carry = xd[row];
      __syncthreads();
      if (half == 1) xd[row] = run(carry, -1.0, pk_, lc_);  // the row total
      __syncthreads();
      const double xt = row_u[j][row] * xd[row];
      int pick, lastc;
      run(half == 0 ? 0.0 : carry, xt, pick, lastc);
      xi[row][half] = pick;
      xlast[row][half] = lastc;
      __syncthreads();
      const int p0 = xi[row][0], p1 = xi[row][1];
      // rounding fallback: the last legal column (rng.cpp:97-99)
      int act = p0 >= 0 ? p0 : (p1 >= 0 ? p1 : (xlast[row][1] >= 0 ? xlast[row][1] : xlast[row][0]));
      bool forced_bad = false;
      if (a.forced && b < a.nreal && a.forced[(size_t)b * T] >= 0) {  // rollout_from_actions (env_core.hpp:166-229)
        act = a.forced[(size_t)b * T + t];
        forced_bad = act < 0 || act >= P.A || !((Lock<E>::legal32(P, w, act & ~31) >> (act & 31)) & 1u);
        if (forced_bad) act = 0;
      }
      const float lse = hi + __logf(z);
      {  // log pi(a) = x_a - lse, x_a (bf16-rounded logit) still in the accumulator columns
        float xa = 0.f;
        const int qa = act >= c0 && act < c0 + 128 ? ((act - c0) >> 5) : -1;
#pragma unroll 1
        for (int q = 0; q < 4; ++q) {  // warp-collective loads; the owner picks its column
          uint32_t rr[32];
          tmem_ld32(lane_base + c0 + q * 32, rr);
          tmem_wait_ld();
          if (q == qa) {
#pragma unroll
            for (int k = 0; k < 32; ++k)
              if (c0 + q * 32 + k == act) xa = __uint_as_float(rr[k]);
          }
        }
        if (qa >= 0) {
          a.rowbuf[2 * r] = xa - lse;
          a.rowbuf[2 * r + 1] = lse;
        }
      }
      tc_fence_before();
      if (half == 0) {  // record + env step
        const size_t bt = (size_t)b * T + t;
        if (act < 0 || forced_bad || legal == 0 || !(z > 0.f)) {
          atomicExch(a.batch.counters + 3, GFNX_ERR_CONTRACT);
        } else {
          for (int i = 0; i < P.SW; ++i) a.stst[r * P.SW + i] = w[i];
          uint32_t* cw = a.cur + (size_t)b * P.SW;
          bool term;
          int np;
          if constexpr (std::is_same<E, IsingEnv>::value) {
            // packed step (IsingEnv::step): assign site act / 2, spin up when act is odd;
            // every step assigns one site, so count = t + 1
            const int site = act >> 1, nw = P.SW / 2;
            const uint32_t bit = 1u << (site & 31);
            cw[site >> 5] = w[site >> 5] | bit;
            if (act & 1) cw[nw + (site >> 5)] = w[nw + (site >> 5)] | bit;
            np = t + 1;
            term = np == P.is_D;
          } else {
            typename E::State s;
            E::unpack(P, w, s);
            term = E::step(P, s, act);
            E::pack(P, s, cw);
            np = E::num_parents(P, s);
          }
          a.batch.actions[bt] = (int16_t)act;
          a.batch.nparents[bt] = (uint16_t)np;
          a.last_act[b] = act;
          s_lact[j][row] = act;
          if (term) {
            typename E::State s;
            E::unpack(P, cw, s);
            a.batch.lengths[b] = t + 1;
            a.batch.log_rewards[b] = E::log_reward(P, s);
            E::pack(P, s, a.batch.term_state + (size_t)b * P.SW);
          }
          if (!isfinite(lse)) atomicExch(a.batch.counters + 3, GFNX_ERR_NUMERIC);
        }
      }
      __syncthreads();
    }
    pmark(2);
  }
  if (a.phase && tid == 0)
    for (int k = 0; k < 3; ++k) atomicAdd((unsigned long long*)a.phase + k, (unsigned long long)pc[k]);
  if (a.phase && tid == 0)
    for (int k = 0; k < 3; ++k) atomicAdd((unsigned long long*)a.phase + 22 + k, (unsigned long long)hs[k]);
  if (tid == 0) mbar_wait(&wbar, wph);  // the prefetched image has landed before exit
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

// Ising layer-1 operand: K-major image of D(n, 2s + u) = W1[3s + u][n] - W1[3s + 2][n]
// (u = 0: spin -1, u = 1: spin +1; ising.cpp:122-129 feature order), zero beyond 2D
__global__ void k_ls_ising_l1img(const __nv_bfloat16* w1, int D, uint8_t* img) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= kH * kH) return;
  const int n = i / kH, k = i % kH, site = k >> 1, u = k & 1;
  float v = 0.f;
  if (site < D)
    v = __bfloat162float(w1[(size_t)(3 * site + u) * kH + n]) - __bfloat162float(w1[(size_t)(3 * site + 2) * kH + n]);
  *reinterpret_cast<__nv_bfloat16*>(img + sw128_offset(n, k, kH)) = __float2bfloat16(v);
}

template <class E>
void rollout_impl(Ctx& c, Key key, double eps, const int16_t* forced) {
  LsState& f = LS(c);
  const int T = f.T, Bl = f.Bl;  // padded batch (c.Bl real trajectories first)
  cudaMemsetAsync(c.batch.actions, 0xFF, sizeof(int16_t) * (size_t)Bl * T, c.stream);
  {
    ProfScope ps(c, "k_ls_init");
    k_ls_reset<<<(Bl * f.SW + 255) / 256, 256, 0, c.stream>>>(Bl * f.SW, f.cur);
    k_ls_h1init<E><<<1, kH, 0, c.stream>>>(c.P, f.w1, c.p32 + c.L.off_b[0], f.h1init);
    c.launches += 2;
  }
  // the whole rollout in one persistent kernel when the head fits one MMA and every CTA
  // holds at most two trajectory tiles (GFNX_LS_STEPWISE=1 forces the per-step kernels)
  const int grid = std::min(f.num_sms, f.tilesB);
  if (std::is_same<E, IsingEnv>::value && f.NT == 1 && Bl % kTile == 0 && f.tilesB <= kPersistMaxTiles * grid &&
      T <= 256) {
    PersistArgs pa{};
    pa.P = c.P;
    pa.key = key;
    pa.eps = eps;
    pa.b0 = c.b0;
    pa.Bl = Bl;
    pa.T = T;
    pa.NL = f.NL;
    pa.A = f.A;
    pa.tilesB = f.tilesB;
    pa.w1 = f.w1;
    pa.h1init = f.h1init;
    pa.preact = f.preact;
    for (int l = 1; l < f.NL; ++l) {
      pa.wimg[l] = (const uint8_t*)f.wfw[l];
      pa.bias[l] = c.p32 + c.L.off_b[l];
    }
    pa.wimg[f.NL] = (const uint8_t*)f.wff;
    if (std::is_same<E, IsingEnv>::value && 2 * c.P.is_D <= kH) {
      if (!f.l1img) cuda_check(cudaMalloc(&f.l1img, kH * kH * 2), "ising l1 image");
      k_ls_ising_l1img<<<kH * kH / 256, 256, 0, c.stream>>>(f.w1, c.P.is_D, f.l1img);
      c.launches++;
      pa.wimg[0] = f.l1img;
      pa.l1_mma = 1;
    }
    pa.bfp = f.bfp;
    for (int l = 0; l < f.NL; ++l) {
      pa.h[l] = (uint8_t*)f.h[l];
      pa.mask[l] = f.mask[l];
    }
    pa.cur = f.cur;
    pa.stst = f.stst;
    pa.last_act = f.last_act;
    pa.rowbuf = f.rowbuf;
    pa.batch = c.batch;
    pa.phase = c.phase;
    pa.forced = forced;
    pa.nreal = c.Bl;
    pa.flowv = f.flow ? f.flowv : nullptr;
    const int smem = kH * kH * 2 + 1024;
    set_smem_once(k_ls_persist<E>, smem);
    ProfScope ps(c, "k_ls_persist");
    k_ls_persist<E><<<grid, 256, smem, c.stream>>>(pa);
    c.launches++;
    return;
  }
  for (int t = 0; t < T; ++t) {
    {
      L1Args la{c.P, f.w1, f.h1init, f.preact, f.last_act, (uint8_t*)f.h[0], f.mask[0], Bl, t};
      ProfScope ps(c, "k_ls_layer1");
      k_ls_layer1<E><<<(Bl + 7) / 8, 256, 0, c.stream>>>(la);
      c.launches++;
    }
    GemmGeom g{};
    g.a_kb = 4;
    g.b_kb = 4;
    g.m0 = t * f.tilesB;
    g.m_tiles = f.tilesB;
    g.n_tiles = 1;
    g.KB = 4;
    for (int l = 1; l < f.NL; ++l) {
      g.A = (const uint8_t*)f.h[l - 1];
      g.B = (const uint8_t*)f.wfw[l];
      launch_gemm<256, HidEpi>(c, "k_gemm_hidden", g, HidEpi::Args{c.p32 + c.L.off_b[l], (uint8_t*)f.h[l], f.mask[l]},
                               f.num_sms);
    }
    g.A = (const uint8_t*)f.h[f.NL - 1];
    g.B = (const uint8_t*)f.wff;
    g.n_tiles = f.NT;
    if (f.flow) {
      typename LogEpi<E, true>::Args le{c.P, f.bfp, f.cur, f.logits, f.stats, f.Ap, f.G, t * Bl, f.flowv};
      launch_gemm<256, LogEpi<E, true>>(c, "k_gemm_logits", g, le, f.num_sms);
    } else {
      typename LogEpi<E, false>::Args le{c.P, f.bfp, f.cur, f.logits, f.stats, f.Ap, f.G, t * Bl, nullptr};
      launch_gemm<256, LogEpi<E, false>>(c, "k_gemm_logits", g, le, f.num_sms);
    }
    SampleArgs sa{c.P, fold_in(key, (uint64_t)t), eps, c.b0, Bl, t, T, f.Ap, f.G, f.logits, f.stats, f.cur, f.stst,
                  f.last_act, f.rowbuf, c.batch, forced, c.Bl};
    ProfScope ps(c, "k_ls_sample");
    k_ls_sample<E><<<(Bl + 8 * kSampleRows - 1) / (8 * kSampleRows), 256, 0, c.stream>>>(sa);
    c.launches++;
  }
}

template <class E>
void train_impl(Ctx& c) {
  LsState& f = LS(c);
  const int Bl = f.Bl, NL = f.NL;
  if (f.flow) {  // DB / SubTB
    const int T = f.T;
    double norm = 0.0;
    if (!f.lampow) {
      std::vector<double> lp(T + 1);
      for (int k = 0; k <= T; ++k) lp[k] = pow(c.train.subtb_lambda, (double)k);
      cuda_check(cudaMalloc(&f.lampow, sizeof(double) * (T + 1)), "lampow");
      cuda_check(cudaMemcpy(f.lampow, lp.data(), sizeof(double) * (T + 1), cudaMemcpyHostToDevice), "lampow");
    }
    for (int j = 0; j < T; ++j)  // subtb_loss's per-trajectory normaliser (every length is T)
      for (int k = j + 1; k <= T; ++k) norm += pow(c.train.subtb_lambda, (double)(k - j));
    FlowLossArgs la{c.batch, Bl, T, c.Bl, c.train.objective == GFNX_OBJ_SUBTB, (double)c.B,
                    c.train.terminal_penalty, norm, f.lampow, c.d_neglog, f.rowbuf, f.flowv, f.coef, f.gflow,
                    f.lpart, c.batch.counters + 4};
    ProfScope ps(c, "k_ls_loss");
    k_ls_loss_flow<<<f.loss_blocks, 256, 0, c.stream>>>(la);
    k_ls_loss_finalize<<<1, 32, 0, c.stream>>>(f.lpart, f.loss_blocks, c.d_scalars, c.batch.counters + 3);
    c.launches += 2;
  } else {
    LossArgs la{c.batch, Bl, f.T, c.Bl, (double)c.B, c.d_neglog, f.rowbuf, f.coef, f.lpart, c.d_scalars};
    ProfScope ps(c, "k_ls_loss");
    k_ls_loss<<<f.loss_blocks, 256, 0, c.stream>>>(la);
    k_ls_loss_finalize<<<1, 32, 0, c.stream>>>(f.lpart, f.loss_blocks, c.d_scalars, c.batch.counters + 3);
    c.launches += 2;
  }
  GemmGeom g{};
  g.A = (const uint8_t*)f.h[NL - 1];
  g.a_kb = 4;
  g.B = (const uint8_t*)f.wff;
  g.b_kb = 4;
  g.m0 = 0;
  g.m_tiles = f.tilesR;
  g.n_tiles = f.NT;
  g.KB = 4;
  auto dlog = [&](auto epi) {
    using Epi = decltype(epi);
    typename Epi::Args de{c.P, f.bfp, f.rowbuf, f.coef, f.stst, c.batch.actions, (uint8_t*)f.dlog, f.bpart,
                          Bl, f.T, f.KBA, f.bw, NL * kH, f.flow ? f.gflow : nullptr};
    launch_gemm<256, Epi>(c, "k_gemm_dlogits", g, de, f.num_sms);
  };
  if (f.flow) dlog(DlogEpi<E, true>{});
  else dlog(DlogEpi<E, false>{});
  GemmGeom g2{};
  g2.A = (const uint8_t*)f.dlog;
  g2.a_kb = f.KBA;
  g2.B = (const uint8_t*)f.wfd;
  g2.b_kb = f.KBA;
  g2.m0 = 0;
  g2.m_tiles = f.tilesR;
  g2.n_tiles = 1;
  g2.KB = f.KBA;
  launch_gemm<256, DgradEpi>(c, "k_gemm_dgrad_head", g2,
                             DgradEpi::Args{f.mask[NL - 1], (uint8_t*)f.dz[NL - 1], f.bpart, (NL - 1) * kH, f.bw},
                             f.num_sms);
  for (int l = NL - 1; l >= 1; --l) {  // dz_{l-1} = dz_l W_l, masked by h_{l-1} > 0
    GemmGeom g3{};
    g3.A = (const uint8_t*)f.dz[l];
    g3.a_kb = 4;
    g3.B = (const uint8_t*)f.wdg[l];
    g3.b_kb = 4;
    g3.m0 = 0;
    g3.m_tiles = f.tilesR;
    g3.n_tiles = 1;
    g3.KB = 4;
    launch_gemm<256, DgradEpi>(c, "k_gemm_dgrad_hidden", g3,
                               DgradEpi::Args{f.mask[l - 1], (uint8_t*)f.dz[l - 1], f.bpart, (l - 1) * kH, f.bw},
                               f.num_sms);
  }
  {
    WgArgs wa{};
    wa.P = c.P;
    wa.stst = f.stst;
    wa.tilesR = f.tilesR;
    wa.ntasks = f.ntasks;
    for (int k = 0; k <= f.ntasks; ++k) wa.first[k] = f.first[k];
    wa.wpart = f.wpart;
    wa.phase = c.phase;
    int k = 0;
    for (int l = 1; l < NL; ++l)  // dW_{l+1} = h_l^T dz_{l+1}
      wa.task[k++] = WgTask{(const uint8_t*)f.h[l - 1], (const uint8_t*)f.dz[l], 4, 0, 0, 256};
    for (int n = 0; n < f.NT; ++n)
      wa.task[k++] = WgTask{(const uint8_t*)f.h[NL - 1], (const uint8_t*)f.dlog, f.KBA, 4 * n, 0, 256};
    for (int j = 0; j < f.OB; ++j)
      wa.task[k++] = WgTask{nullptr, (const uint8_t*)f.dz[0], 4, 0, 256 * j, std::min(256, f.O - 256 * j)};
    const int smem = kWStages * (2 * kWOp + kWStBytes) + 1024;
    set_smem_once(k_ls_wgrad<E>, smem);
    ProfScope ps(c, "k_ls_wgrad");
    k_ls_wgrad<E><<<f.first[f.ntasks], kGemmThreads, smem, c.stream>>>(wa);
    c.launches++;
  }
  {
    ProfScope ps(c, "k_ls_reduce");
    k_ls_colsum<<<dim3((f.bw + 255) / 256, f.cgroups), 256, 0, c.stream>>>(f.bpart, f.tilesR, f.bw, f.cgroups,
                                                                           f.bpart2);
    RedArgs ra{f.wpart, f.bpart2, c.g32, f.cgroups, f.bw, f.A, f.O, NL, f.t_dense, f.t_head, f.t_w1, {}, c.L, f.flow};
    for (int k = 0; k <= f.ntasks; ++k) ra.first[k] = f.first[k];
    k_ls_reduce<<<(unsigned)((c.L.n_params + 255) / 256), 256, 0, c.stream>>>(ra);
    c.launches += 2;
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// host side

bool ls_supported(const Ctx& c, std::string* why) {
  const int kind = c.env.kind;
  if (kind != GFNX_ENV_BITSEQ && kind != GFNX_ENV_ISING) return false;
  auto no = [&](const char* m) {
    *why = m;
    return false;
  };
  if (c.train.objective != GFNX_OBJ_TB && c.train.objective != GFNX_OBJ_DB && c.train.objective != GFNX_OBJ_SUBTB)
    return no("bitseq/Ising fast path implements TB, DB and SubTB");
  if (c.train.objective == GFNX_OBJ_SUBTB && c.P.T > kLsSubTBMaxT) return no("bitseq/Ising SubTB supports T <= 128");
  if (c.L.n_trunk < 2 || c.L.n_trunk > kMaxNL) return no("bitseq/Ising fast path needs 2..4 hidden layers");
  for (int l = 1; l <= c.L.n_trunk; ++l)
    if (c.L.dims[l] != kH) return no("bitseq/Ising fast path needs hidden widths <= 256");
  if (kind == GFNX_ENV_BITSEQ) {
    if (c.P.bs_vocab != 256) return no("bitseq fast path needs k = 8 (256-word slots)");
    if (c.P.bs_slots > 32) return no("bitseq fast path supports <= 32 slots");
  } else {
    if (c.P.is_D > 128) return no("Ising fast path supports <= 128 sites");
  }
  if (c.P.SW > 16) return no("fast path supports <= 16 packed state words");
  if ((c.P.A + 255) / 256 * 2 > 32) return no("fast path supports <= 4096 actions");
  return true;
}

void ls_init(Ctx& c) {
  auto* f = new LsState();
  c.fast = f;
  cudaDeviceGetAttribute(&f->num_sms, cudaDevAttrMultiProcessorCount, c.device);
  f->NL = c.L.n_trunk;
  f->A = c.P.A;
  f->flow = c.train.objective == GFNX_OBJ_DB || c.train.objective == GFNX_OBJ_SUBTB;
  f->Ap = (f->A + f->flow + 255) / 256 * 256;  // the flow head rides along as column A
  f->NT = f->Ap / 256;
  f->G = f->Ap / 128;
  f->KBA = f->Ap / 64;
  f->O = c.P.O;
  f->OB = (f->O + 255) / 256;
  f->T = c.P.T;
  f->SW = c.P.SW;
  f->Bl = (c.Bl + kTile - 1) / kTile * kTile;  // lockstep rows pad the batch to whole 128-row tiles
  f->R = f->Bl * f->T;
  f->tilesB = f->Bl / kTile;
  f->tilesR = f->R / kTile;
  f->t_dense = 0;
  f->t_head = f->NL - 1;
  f->t_w1 = f->t_head + f->NT;
  f->ntasks = f->t_w1 + f->OB;
  if (f->ntasks > kMaxTasks) raise_error(GFNX_ERR_CONFIG, "fast path: too many weight-gradient tasks");
  {  // CTAs per task proportional to its per-stage cost (one-hot operands are built in smem;
     // their cost grows with the nonzeros per row inside the 256-feature block)
    auto weight = [&](int k) {
      if (k < f->t_w1) return 1.0;
      if (c.env.kind != GFNX_ENV_ISING) return 1.1;
      const int f0 = 256 * (k - f->t_w1);
      const int sites = std::max(0, std::min(c.P.is_D, (f0 + 256 + 2) / 3) - f0 / 3);
      return 1.0 + 3.0 * sites / 85.0;
    };
    double tot = 0.0;
    for (int k = 0; k < f->ntasks; ++k) tot += weight(k);
    int used = 0;
    for (int k = 0; k < f->ntasks; ++k) {
      f->first[k] = used;
      used += std::max(1, (int)(f->num_sms * weight(k) / tot));
    }
    f->first[f->ntasks] = used;
  }
  f->loss_blocks = (f->Bl + 255) / 256;
  f->bw = f->NL * kH + f->Ap;
  f->cgroups = std::min(256, std::max(1, f->tilesR / 16));
  const size_t img = (size_t)f->tilesR * kTile * kH * 2;
  auto alloc = [&](auto** p, size_t bytes) {
    cuda_check(cudaMalloc((void**)p, bytes), "lockstep alloc");
    cuda_check(cudaMemset(*p, 0, bytes), "lockstep alloc");
  };
  alloc(&f->w1, sizeof(__nv_bfloat16) * (size_t)f->O * kH);
  for (int l = 1; l < f->NL; ++l) {
    alloc(&f->wfw[l], sizeof(__nv_bfloat16) * kH * kH);
    alloc(&f->wdg[l], sizeof(__nv_bfloat16) * kH * kH);
  }
  alloc(&f->wff, sizeof(__nv_bfloat16) * (size_t)f->Ap * kH);
  alloc(&f->wfd, sizeof(__nv_bfloat16) * (size_t)f->Ap * kH);
  alloc(&f->bfp, sizeof(float) * f->Ap);
  alloc(&f->h1init, sizeof(float) * kH);
  alloc(&f->preact, sizeof(float) * (size_t)f->Bl * kH);
  alloc(&f->cur, sizeof(uint32_t) * (size_t)f->Bl * f->SW);
  alloc(&f->stst, sizeof(uint32_t) * (size_t)f->R * f->SW);
  alloc(&f->last_act, sizeof(int32_t) * f->Bl);
  for (int l = 0; l < f->NL; ++l) {
    alloc(&f->h[l], img);
    alloc(&f->dz[l], img);
    alloc(&f->mask[l], (size_t)f->R * (kH / 8));
  }
  alloc(&f->logits, sizeof(__nv_bfloat16) * (size_t)f->Bl * f->Ap);
  alloc(&f->stats, sizeof(float2) * (size_t)f->Bl * f->G);
  alloc(&f->dlog, (size_t)f->tilesR * f->KBA * (kTile * 128));
  alloc(&f->rowbuf, sizeof(float) * 2 * (size_t)f->R);
  alloc(&f->coef, sizeof(float) * (size_t)f->R);
  if (f->flow) {
    alloc(&f->flowv, sizeof(float) * (size_t)f->R);
    alloc(&f->gflow, sizeof(float) * (size_t)f->R);
  }
  alloc(&f->bpart, sizeof(float) * (size_t)f->tilesR * f->bw);
  alloc(&f->bpart2, sizeof(float) * (size_t)f->cgroups * f->bw);
  alloc(&f->wpart, sizeof(float) * (size_t)f->first[f->ntasks] * 256 * 256);
  alloc(&f->lpart, sizeof(double) * 2 * f->loss_blocks);
  ls_sync_weights(c);
}

void ls_free(Ctx& c) {
  LsState* f = static_cast<LsState*>(c.fast);
  if (!f) return;
  std::vector<void*> ptrs = {f->w1, f->wff, f->wfd, f->l1img, f->bfp, f->h1init, f->preact, f->cur, f->stst, f->last_act,
                             f->logits, f->stats, f->dlog, f->rowbuf, f->coef, f->bpart, f->bpart2, f->wpart,
                             f->lpart, f->flowv, f->gflow, f->lampow};
  for (int l = 0; l < kMaxNL; ++l) {
    ptrs.push_back(f->wfw[l]);
    ptrs.push_back(f->wdg[l]);
    ptrs.push_back(f->h[l]);
    ptrs.push_back(f->dz[l]);
    ptrs.push_back(f->mask[l]);
  }
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete f;
  c.fast = nullptr;
}

bool ls_debug_buffer(Ctx& c, const std::string& name, const void** ptr, size_t* bytes) {
  LsState& f = LS(c);
  const size_t img = (size_t)f.tilesR * kTile * kH * 2;
  auto layer = [&](const char* pre) { return name.size() == strlen(pre) + 1 && name.compare(0, strlen(pre), pre) == 0 ? name.back() - '0' : -1; };
  int l;
  if ((l = layer("h")) >= 0 && l < f.NL) { *ptr = f.h[l]; *bytes = img; return true; }
  if ((l = layer("dz")) >= 0 && l < f.NL) { *ptr = f.dz[l]; *bytes = img; return true; }
  if ((l = layer("mask")) >= 0 && l < f.NL) { *ptr = f.mask[l]; *bytes = (size_t)f.R * (kH / 8); return true; }
  if (name == "dlog") { *ptr = f.dlog; *bytes = (size_t)f.tilesR * f.KBA * (kTile * 128); return true; }
  if (name == "rowbuf") { *ptr = f.rowbuf; *bytes = sizeof(float) * 2 * (size_t)f.R; return true; }
  if (name == "coef") { *ptr = f.coef; *bytes = sizeof(float) * (size_t)f.R; return true; }
  return false;
}

void ls_sync_weights(Ctx& c) {
  EmitArgs a = emit_args(c);
  k_ls_emit<<<(unsigned)((a.n + 255) / 256), 256, 0, c.stream>>>(a);
  c.launches++;
}

namespace {
// rows are step-major (r = t * stride + b); rowbuf[2 r] = log pi(a | s)
__global__ void k_ls_row_logpf(const float* __restrict__ rowbuf, int Bl, int stride, int T, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= Bl * T) return;
  const int b = i / T, t = i % T;
  out[i] = (double)rowbuf[2 * ((size_t)t * stride + b)];
}
}  // namespace

void ls_row_logpf(Ctx& c, double* out) {
  const int n = c.Bl * LS(c).T;
  k_ls_row_logpf<<<(n + 255) / 256, 256, 0, c.stream>>>(LS(c).rowbuf, c.Bl, LS(c).Bl, LS(c).T, out);
  c.launches++;
}

void ls_rollout(Ctx& c, Key key, double eps, const int16_t* forced) {
  if (c.env.kind == GFNX_ENV_BITSEQ)
    rollout_impl<BitseqEnv>(c, key, eps, forced);
  else
    rollout_impl<IsingEnv>(c, key, eps, forced);
}

void ls_train(Ctx& c) {
  if (c.env.kind == GFNX_ENV_BITSEQ)
    train_impl<BitseqEnv>(c);
  else
    train_impl<IsingEnv>(c);
}

}  // namespace gfnx
