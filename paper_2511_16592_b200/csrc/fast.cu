// fast.cu — the bf16 tcgen05 fast path (sm_100a).
//
// One training iteration = 7 launches on one stream, no host synchronisation:
//   k_fast_rollout  persistent fused rollout: per 128-slot tile and env step, the layer-1
//                   pre-activation is updated incrementally in TMEM (only the features the
//                   last action changed), ReLU'd to a bf16 tile in smem, multiplied by the
//                   smem-resident hidden weight image on the tensor cores (tcgen05.mma,
//                   fp32 accumulator in TMEM), then the head, epsilon-uniform masked
//                   categorical (Threefry stream of the reference) and env step run per
//                   thread. Finished slots pull the next trajectory from a global counter,
//                   so geometric trajectory lengths do not idle the tile.
//                   (forward_rollout env_core.hpp:232-274 + rollout_from_actions :166-229)
//   k_fast_fwd      training forward over the Sum_b L_b real rows only (not B*(T+1) padded
//                   rows), layer-2 on tcgen05; stores bf16 activation tile images + per-row
//                   head statistics (mlp_forward_tape nn.cpp:91-126, masked_log_softmax
//                   tape.cpp:177-213)
//   k_fast_loss_warp TB/DB/SubTB/MDB residuals and their analytic backward, warp per trajectory
//                   (objectives.cpp:94-226), deterministic block partials
//   k_fast_bwd      head backward (SIMT), dgrad GEMMs on tcgen05, ReLU masks, bias grads, and
//                   [dW1 | db1] = [obs | 1]^T dz1 on tcgen05 while dz1 is in shared memory
//   k_fast_wgrad    dW2 / dWhead as tcgen05 GEMMs whose K dimension is the row count: the
//                   activation tile images are read MN-major straight from HBM
//   k_reduce        fixed-order reduction of per-CTA partial gradients (deterministic)
//   k_fast_adam     fused Adam over the flat fp32 parameters + logZ, re-emitting the bf16
//                   operand images (adam_step optim.cpp:19-43)
#include <math.h>

#include <algorithm>
#include <type_traits>
#include <vector>

#include "engine.h"
#include "fast_common.cuh"

namespace gfnx {

namespace {

constexpr int kHeadMax = 32;
constexpr int kGatherMax = 8;  // one-hot features gathered per row in the training forward

struct FastState {
  int num_sms = 0;
  int H = 0, A = 0, O = 0, Opad = 0;
  int64_t max_rows = 0, max_tiles = 0;
  __nv_bfloat16* w1 = nullptr;        // [O][H] row-major (layer-1 gathers)
  __nv_bfloat16* w2_fwd = nullptr;    // image [H out][H in] K-major
  __nv_bfloat16* w2_dgrad = nullptr;  // image [H in][H out] K-major
  __nv_bfloat16* whead_f = nullptr;   // image [NH][H] (head logits + flow)
  __nv_bfloat16* whead_d = nullptr;   // image [H][NH] non-swizzled (head dgrad)
  int NH = 16;
  uint32_t* stst = nullptr;           // [Bl*T][SW] state before each step
  __nv_bfloat16 *h1 = nullptr, *h2 = nullptr, *dz2 = nullptr;  // tile images
  __nv_bfloat16* dhead = nullptr;     // tile images [tiles][128][64]
  uint32_t *mask1 = nullptr, *mask2 = nullptr;  // ReLU bit masks [rows][H/32]
  float* rowbuf = nullptr;            // per row: probs[A], lpa, lps, flow, pad
  float* coef = nullptr;              // per row: ga, gs, gflow, pad
  float* wpart = nullptr;             // [num_sms][n_params] partial gradients
  double* lpart = nullptr;            // [blocks][2] loss / dlogz partials
  double* lampow = nullptr;           // pow(lambda, k)
  int32_t* work = nullptr;            // rollout work counter
  int32_t* frow_bt = nullptr;         // [max_tiles*128] row slot -> b*T + t (-1 = empty)
  uint32_t* slot_st = nullptr;        // [max_tiles*128][SW] packed state of each row slot
  int16_t* slot_act = nullptr;        // [max_tiles*128] its action (the training pass reads
                                      // both coalesced instead of through frow_bt)
  int32_t* bt_row = nullptr;          // [Bl*T] b*T + t -> row slot
  int32_t* tilectr = nullptr;         // number of 128-row tiles of row slots
  int32_t* det_used = nullptr;        // deterministic mode: filled tiles per rollout CTA
  int32_t* tile_list = nullptr;       // deterministic mode: training tile -> emission tile
  int det_per = 0, det_mt = 0, det_grid = 0;
  float* logits = nullptr;            // [slots][NH] rollout head outputs (fused forward)
  bool fused = false;                 // row slots hold the rollout's forward for the current weights
  int rs = 0;                         // rowbuf stride (floats)
  int loss_blocks = 0;                // per-thread loss (SubTB): 256 trajectories per block
  int loss_wblocks = 0;               // warp-per-trajectory loss: 8 trajectories per block
};

// legal forward actions among the first AMAX columns as a bit mask (hypergrid: SWAR)
template <class Env, int AMAX>
GFNX_DEV uint32_t legal_bits(const EnvParams& P, const typename Env::State& s, int A) {
  if constexpr (std::is_same<Env, HypergridEnv>::value) {
    return Env::legal_mask(P, s) & (A >= 32 ? 0xffffffffu : ((1u << A) - 1u)) &
           (AMAX >= 32 ? 0xffffffffu : ((1u << AMAX) - 1u));
  } else {
    uint32_t lm = 0;
#pragma unroll
    for (int c = 0; c < AMAX; ++c)
      if (c < A && Env::legal(P, s, c)) lm |= 1u << c;
    return lm;
  }
}

// training-forward record of every emitted row from the rollout's raw head outputs:
// masked log-softmax (tape.cpp:177-213) -> probs[A], log pi(a|s), log pi(stop|s), flow
template <class Env, int NH>
GFNX_DEV void row_stats_one(const EnvParams& P, const uint32_t* __restrict__ stst, const int16_t* __restrict__ actions,
                            const int32_t* __restrict__ frow_bt, const float* __restrict__ logits,
                            float* __restrict__ rowbuf, int rs, int flow, int32_t* err, int r) {
  const int bt = frow_bt[r];
  if (bt < 0) return;
  typename Env::State s;
  Env::unpack(P, stst + (size_t)r * P.SW, s);  // the slot-ordered copies (coalesced)
  const int act = actions[r];
  float lg[NH];
  const float4* src = reinterpret_cast<const float4*>(logits + (size_t)r * NH);
#pragma unroll
  for (int k = 0; k < NH / 4; ++k) {
    const float4 v = src[k];
    lg[4 * k] = v.x;
    lg[4 * k + 1] = v.y;
    lg[4 * k + 2] = v.z;
    lg[4 * k + 3] = v.w;
  }
  const int A = P.A;
  const uint32_t lm = legal_bits<Env, NH>(P, s, A);
  float hi = -INFINITY;
#pragma unroll
  for (int c = 0; c < NH; ++c)
    if ((lm >> c) & 1u) hi = fmaxf(hi, lg[c]);
  float e[NH], z = 0.f;
#pragma unroll
  for (int c = 0; c < NH; ++c) {
    e[c] = ((lm >> c) & 1u) ? __expf(lg[c] - hi) : 0.f;
    z += e[c];
  }
  const float lse = hi + __logf(z), rz = __frcp_rn(z);
  // the three picked columns straight from the (L1-resident) row: a select over lg[] by a
  // runtime column compiles to a local-memory array
  const float* lrow = logits + (size_t)r * NH;
  float la = (act >= 0 && act < NH) ? lrow[act] : 0.f;
  float ls = (P.stop >= 0 && P.stop < NH) ? lrow[P.stop] : 0.f;
  float fl = A < NH ? lrow[A] : 0.f;
  la -= lse;
  ls = P.stop >= 0 ? ls - lse : 0.f;
  fl = flow ? fl : 0.f;
  if (!isfinite(lse)) atomicExch(err, GFNX_ERR_NUMERIC);
  float4* out = reinterpret_cast<float4*>(rowbuf + (size_t)r * rs);
#pragma unroll
  for (int k = 0; k < NH + 4; k += 4)
    if (k < rs) {
      float q[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = k + j;
        q[j] = c < A ? (c < NH ? e[c < NH ? c : 0] * rz : 0.f) : c == A ? la : c == A + 1 ? ls : c == A + 2 ? fl : 0.f;
      }
      out[k >> 2] = make_float4(q[0], q[1], q[2], q[3]);
    }
}

// grid-stride over the used row slots (the slot count is known on the device only)
template <class Env, int NH>
__global__ void k_row_stats(EnvParams P, const uint32_t* __restrict__ stst, const int16_t* __restrict__ actions,
                            const int32_t* __restrict__ frow_bt, const int32_t* __restrict__ tilectr,
                            const float* __restrict__ logits, float* __restrict__ rowbuf, int rs, int flow,
                            int32_t* err, const int32_t* __restrict__ tile_list) {
  const int n = *tilectr * kTile;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    row_stats_one<Env, NH>(P, stst, actions, frow_bt, logits, rowbuf, rs, flow, err,
                           tile_list ? tile_list[r >> 7] * kTile + (r & (kTile - 1)) : r);
}

// deterministic mode: the filled tiles of every rollout CTA's region, in CTA order, as the
// training pass's tile list (the partially filled last tile's spare rows are empty slots)
__global__ void k_det_tiles(const int32_t* __restrict__ used, int nctas, int mt, int32_t* __restrict__ list,
                            int32_t* tilectr) {
  __shared__ int off[1025];
  if (threadIdx.x == 0) {
    int o = 0;
    for (int k = 0; k < nctas; ++k) {
      off[k] = o;
      o += used[k];
    }
    off[nctas] = o;
    *tilectr = o;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < nctas; k += blockDim.x)
    for (int i = 0; i < used[k]; ++i) list[off[k] + i] = k * mt + i;
}

// logical training tile i -> emission tile: the deterministic mode's list (LIST instantiations
// only, so the default kernels carry no list code), else the identity
template <bool LIST>
GFNX_DEV int phys_tile(const int32_t* list, int i) {
  if constexpr (LIST) return list[i];
  return i;
}

__global__ void k_rollout_reset(int32_t* tilectr, int32_t* counters, int32_t* work) {
  if (threadIdx.x == 0) {
    *tilectr = 0;
    *work = 0;
    counters[0] = 0;  // finish_counts
    counters[1] = 0;
  }
}

// row slots in trajectory order (row0[b] + t) when the training forward is recomputed
__global__ void k_linear_rows(const int32_t* __restrict__ lengths, const int32_t* __restrict__ row0, int Bl,
                              int T, const int32_t* counters, int32_t* frow_bt, int32_t* bt_row,
                              int32_t* tilectr, const uint32_t* __restrict__ stst, const int16_t* __restrict__ acts,
                              int SW, uint32_t* slot_st, int16_t* slot_act) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const int R = counters[0];
  const int tiles = (R + kTile - 1) / kTile;
  if (b < Bl) {
    const int L = lengths[b], r0 = row0[b];
    for (int t = 0; t < L; ++t) {
      const size_t bt = (size_t)b * T + t;
      frow_bt[r0 + t] = (int32_t)bt;
      bt_row[bt] = r0 + t;
      for (int i = 0; i < SW; ++i) slot_st[(size_t)(r0 + t) * SW + i] = stst[bt * SW + i];
      slot_act[r0 + t] = acts[bt];
    }
  }
  if (b < kTile && R + b < tiles * kTile) frow_bt[R + b] = -1;
  if (b == 0) *tilectr = tiles;
}

FastState& FS(Ctx& c) { return *static_cast<FastState*>(c.fast); }

struct Weights {
  const __nv_bfloat16* w1;
  const float* b1;
  const __nv_bfloat16* w2_fwd;
  const __nv_bfloat16* w2_dgrad;
  const float* b2;
  const float* wf;   // [H][A]
  const float* bf;   // [A]
  const float* wfl;  // [H]
  const float* bfl;  // [1]
  const __nv_bfloat16* whead_f;  // head image [NH][H] SW128 K-major (logits + flow rows)
  const __nv_bfloat16* whead_d;  // head dgrad image [H][NH] non-swizzled K-major
};

Weights weights_of(Ctx& c) {
  FastState& f = FS(c);
  const MlpLayout& L = c.L;
  Weights w;
  w.w1 = f.w1;
  w.b1 = c.p32 + L.off_b[0];
  w.w2_fwd = f.w2_fwd;
  w.w2_dgrad = f.w2_dgrad;
  w.b2 = c.p32 + L.off_b[1];
  w.wf = c.p32 + L.off_fw;
  w.bf = c.p32 + L.off_fb;
  w.wfl = c.p32 + L.off_flw;
  w.bfl = c.p32 + L.off_flb;
  w.whead_f = f.whead_f;
  w.whead_d = f.whead_d;
  return w;
}

// reference sampler (eps_uniform objectives.cpp:242-264 + categorical rng.cpp:87-100) on
// the fp32 logits of one row: exp in fp32, mixture weights / cumulative sum in fp64 in the
// reference's order (so eps = 1 draws are bit-exact), fully unrolled over AMAX (registers).
// On return e[c] = exp(logit[c] - hi) over legal c (0 elsewhere), z = sum e, rz = 1 / z:
// the masked log-softmax statistics of the row (lse = hi + log z) for the training record.
template <class Env, int AMAX>
GFNX_DEV int sample_row(const EnvParams& P, const typename Env::State& s, const float (&logit)[AMAX],
                        int A, double eps, double u01, const double* inv_legal, bool* bad,
                        float (&e)[AMAX], float& hi, float& z, float& rz) {
  const uint32_t lm = legal_bits<Env, AMAX>(P, s, A);
  const int legal = __popc(lm);
  hi = -INFINITY;
  z = 1.f;
  rz = 1.f;
#pragma unroll
  for (int c = 0; c < AMAX; ++c) e[c] = 0.f;
#pragma unroll
  for (int c = 0; c < AMAX; ++c)
    if ((lm >> c) & 1u) hi = fmaxf(hi, logit[c]);
  if (legal == 0 || !isfinite(hi)) {
    *bad = true;
    return -1;
  }
  z = 0.f;
#pragma unroll
  for (int c = 0; c < AMAX; ++c) {
    e[c] = ((lm >> c) & 1u) ? __expf(logit[c] - hi) : 0.f;
    z += e[c];
  }
  rz = __frcp_rn(z);
  // eps * (1/legal) from a table: exactly the reference's eps / legal at eps = 1 (where
  // the policy term vanishes and draws are bit-exact); policy weight in fp32
  const double u = eps * inv_legal[legal];
  const float kzf = (float)(1.0 - eps) * rz;
  const double kz = (double)kzf;
  double total = 0.0;
#pragma unroll
  for (int c = 0; c < AMAX; ++c)
    if ((lm >> c) & 1u) total += kz * (double)e[c] + u;
  const double x = u01 * total;
  double acc = 0.0;
  int pick = -1;
#pragma unroll
  for (int c = 0; c < AMAX; ++c)
    if ((lm >> c) & 1u) {
      acc += kz * (double)e[c] + u;
      if (pick < 0 && x < acc) pick = c;
    }
  return pick >= 0 ? pick : 31 - __clz(lm);
}

// ---------------------------------------------------------------------------
// k_fast_rollout
//
// 256 threads per CTA, two per trajectory slot: warp w serves TMEM lane quarter (w % 4)
// and column half (w / 4), so every slot's 256-wide hidden vector is split across two
// threads (tcgen05.ld lane-quarter rule). Per env step:
//   (1) layer-1 pre-activation updated in TMEM (fp32, columns [H, 2H)) from the features
//       the last action changed; ReLU -> bf16 A tile in smem
//   (2) tcgen05.mma 128 x H x H against the smem-resident W2 image
//   (3) ReLU(acc + b2) -> bf16 h2 tile in smem (half-1 threads also draw the row's uniform)
//   (4) tcgen05.mma 128 x NH x H head (logits + flow) -> TMEM, then half-0 threads sample,
//       step the env, record, and refill finished slots from the global work counter.


// 8 consecutive fp32 words (32-byte aligned) in one st.global.v8; zeros when !keep
GFNX_DEV void st_v8(float* dst, const uint32_t* r, bool keep) {
  const uint32_t m = keep ? 0xffffffffu : 0u;
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst), "r"(r[0] & m), "r"(r[1] & m),
               "r"(r[2] & m), "r"(r[3] & m), "r"(r[4] & m), "r"(r[5] & m), "r"(r[6] & m), "r"(r[7] & m)
               : "memory");
}

// one 128-byte row line (64 bf16 units = 16 packed words per 32 B pair... 32 words) of a
// 128B-swizzled tile image, row `prow`: logical 16-byte chunk l lands at chunk l ^ (prow & 7);
// stored as four 32-byte st.global.v8 (chunk pairs stay adjacent under the XOR)
GFNX_DEV void st_line_sw128(uint8_t* line, int prow, const uint32_t (&r)[32]) {
  const int x = prow & 7;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int p = (2 * m) ^ x;  // physical chunk of logical chunk 2m
    const uint32_t* lo = r + 8 * m;      // logical chunk 2m (words 0..3) and 2m+1 (words 4..7)
    uint32_t v[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[i] = (x & 1) ? lo[4 + i] : lo[i];
      v[4 + i] = (x & 1) ? lo[i] : lo[4 + i];
    }
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(line + (p & ~1) * 16), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
  }
}

// row counts of a fused rollout (what k_row_scan derives from the lengths otherwise):
// counters[0] = sum L, [1] = sum max(L - 1, 0), then the last CTA publishes [4], [5] and the
// int64 running totals [8..9]; counters[12] is the CTA ticket
GFNX_DEV void finish_counts(int32_t* counters, int rows, int rows_mdb) {
  atomicAdd(counters + 0, rows);
  atomicAdd(counters + 1, rows_mdb);
  __threadfence();
  if (atomicAdd(counters + 12, 1) == (int)gridDim.x - 1) {
    __threadfence();
    const int r0 = atomicAdd(counters + 0, 0), r1 = atomicAdd(counters + 1, 0);
    counters[4] = r0;
    counters[5] = r1;
    long long* acc = reinterpret_cast<long long*>(counters + 8);
    acc[0] += r0;
    acc[1] += 1;
    counters[12] = 0;
  }
}

struct RolloutArgs {
  EnvParams P;
  Weights W;
  Key key;
  double eps;
  int b0, Bl;
  DeviceBatch batch;
  uint32_t* stst;
  uint32_t* slot_st;  // the same state + action again at the row's emission slot
  int16_t* slot_act;
  int32_t* work;
  long long* phase;  // optional per-phase clock totals (gfnx_phase_timers), else nullptr
  // fused training forward: every sampled row's h1 / h2 (bf16 tile images), ReLU masks and
  // log-softmax statistics, in emission order; 128-row tiles are claimed from tilectr
  __nv_bfloat16 *h1, *h2;
  uint32_t *mask1, *mask2;
  float* rowbuf;
  int rs, flow;
  int32_t *frow_bt, *bt_row, *tilectr;
  float* logits;  // [slot][NH] head outputs (logits, flow at column A), bias included
  // deterministic mode: CTA k simulates trajectories [k per, (k+1) per) and emits into its
  // own tiles [k mt, (k+1) mt); det_used[k] = tiles it filled (k_det_tiles lists them)
  int det, per, mt;
  int32_t* det_used;
};

// H = 256 stages the A operand (h1, then h2) in two 128-column halves through one 32 KB
// buffer (split-K: the MMA over the first half runs while the second half is produced),
// which frees the shared memory that keeps W1 resident for the layer-1 row reads.
template <int H>
__host__ __device__ constexpr int rollout_acols() {
  return H == 256 ? H / 2 : H;
}
template <int H, int NH>
constexpr int rollout_smem_fixed() {
  return H * H * 2 + NH * H * 2 + kTile * rollout_acols<H>() * 2 + 1024;
}

template <class Env, int H, int NH, bool W1S, bool DET>
__global__ void __launch_bounds__(kThreads, 1) k_fast_rollout(RolloutArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  constexpr bool SPLIT = H == 256;
  constexpr int AK = rollout_acols<H>();  // columns of the staged A operand
  constexpr int HC = H / 2;               // columns owned by each thread of a row
  uint8_t* w2img = smem;                  // H x H bf16 (resident for the whole rollout)
  uint8_t* whimg = w2img + H * H * 2;     // head image [NH][H]
  uint8_t* atile = whimg + NH * H * 2;    // 128 x AK bf16 activations
  __nv_bfloat16* w1s = reinterpret_cast<__nv_bfloat16*>(atile + kTile * AK * 2);  // [O][H] if W1S
  const __nv_bfloat16* w1 = W1S ? w1s : a.W.w1;
  __shared__ __align__(16) float h1init[H];
  __shared__ __align__(16) float b2s[H];
  __shared__ float bhs[NH];
  __shared__ Key skeys[128];
  __shared__ double row_u[kTile];
  __shared__ int row_b[kTile], row_t[kTile];
  __shared__ int row_nd[kTile], row_df[kTile][4];
  __shared__ float row_dv[kTile][4];
  __shared__ uint8_t row_init[kTile];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  __shared__ unsigned long long smax;
  __shared__ double inv_legal[NH + 1];
  __shared__ int s_cur0, s_next;  // emission tiles: first claimed, next claimed
  __shared__ int s_pq[4];          // deterministic refills: finished rows per row quarter
  __shared__ int s_nterm;          // trajectories finished by this CTA
  __shared__ uint4 row_m1[kTile][H / 128], row_m2[kTile][H / 128];  // ReLU masks of the round

  const EnvParams& P = a.P;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quarter = warp & 3, half = warp >> 2;
  const int row = quarter * 32 + lane, c0 = half * HC;
  const int T = P.T, A = P.A;
  if (warp == 0) tmem_alloc<2 * H>(&tbase);  // [0, H) accumulator, [H, 2H) layer-1 pre-activation
  if (tid == 0) {
    mbar_init(&mbar, 1);
    fence_mbar_init();
    smax = 0;
    const int t0 = DET ? (int)blockIdx.x * a.mt : atomicAdd(a.tilectr, 2);
    for (int q = 0; q < 4; ++q) s_pq[q] = 0;
    s_cur0 = t0;
    s_next = t0 + 1;
    s_nterm = 0;
  }
  __syncthreads();
  // emission cursor (uniform over the CTA): rows of this CTA fill tile `cur` from `fill`,
  // overflowing into the pre-claimed tile s_next
  int cur = s_cur0, fill = 0, emitted = 0;
  int nclaim = s_cur0 + 2;  // deterministic mode: next tile of this CTA's region
  if (tid == 0) {
    mbar_arrive_expect_tx(&mbar, H * H * 2 + NH * H * 2);
    bulk_g2s_big(w2img, a.W.w2_fwd, H * H * 2, &mbar);
    bulk_g2s_big(whimg, a.W.whead_f, NH * H * 2, &mbar);
  }
  if (W1S) {  // W1 rows with 16-byte chunk c stored at c ^ (row & 7)
    const uint4* src = reinterpret_cast<const uint4*>(a.W.w1);
    uint4* dst = reinterpret_cast<uint4*>(w1s);
    constexpr int CPR = H / 8;  // chunks per row
    for (int i = tid; i < P.O * CPR; i += kThreads) {
      const int f = i / CPR, c = i % CPR;
      dst[f * CPR + (c ^ (f & 7))] = src[i];
    }
  }
  for (int t = tid; t < T && t < 128; t += kThreads) skeys[t] = fold_in(a.key, (uint64_t)t);
  for (int j = tid; j < H; j += kThreads) b2s[j] = a.W.b2[j];
  if (tid < NH) bhs[tid] = tid < A ? a.W.bf[tid] : (tid == A ? a.W.bfl[0] : 0.f);
  if (tid <= NH) inv_legal[tid] = tid ? 1.0 / tid : 0.0;
  {  // h1init = b1 + x(s0) W1 (layer-1 pre-activation of the initial state)
    typename Env::State s0;
    Env::reset(P, s0);
    for (int j = tid; j < H; j += kThreads) {
      float v = a.W.b1[j];
      Env::features(P, s0, [&](int f, double x) { v += (float)x * __bfloat162float(a.W.w1[(size_t)f * H + j]); });
      h1init[j] = v;
    }
  }
  mbar_wait(&mbar, 0);
  uint32_t phase = 1;
  tc_fence_after();
  __syncthreads();
  const uint32_t tmem = tbase;
  const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);

  // one MMA round: thread 0 issues `issue` and waits for completion; everyone re-syncs
  auto mma_round = [&](auto&& issue) {
    if (tid == 0) {
      tc_fence_after();
      issue();
      umma_commit(&mbar);
    }
  };
  // H = 128: every thread waits on the MMA mbarrier itself (a warp only re-stages the A-tile
  // rows it emitted, so a warp barrier orders them); the split-K H = 256 variant restages
  // rows another warp may still be emitting and keeps the CTA barrier
  auto mma_join = [&]() {
    if (SPLIT) {
      if (tid == 0) mbar_wait(&mbar, phase);
      __syncthreads();
    } else {
      mbar_wait(&mbar, phase);
      __syncwarp();
    }
    phase ^= 1;
    tc_fence_after();
  };
  auto publish = [&]() {  // generic-proxy smem writes -> visible to the tensor core
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
  };
  // ReLU(acc + bias) of TMEM columns [col0, col0 + 32) -> bf16 into the staged A tile
  auto stage32 = [&](uint32_t tcol, int acol, const float* bias, uint32_t* mword) {
    uint32_t r[32];
    tmem_ld32(lane_base + tcol, r);
    tmem_wait_ld();
    uint32_t pk[16];
    if (bias) {
      const float2* b2 = reinterpret_cast<const float2*>(bias);
#pragma unroll
      for (int i = 0; i < 16; ++i) pk[i] = bias_relu_pack(r[2 * i], r[2 * i + 1], b2[i]);
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) pk[i] = pack_bf16x2_relu(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
    }
    if (mword) *mword = relu_mask16(pk);
    st_row32(atile, row, acol, pk);
  };

  typename Env::State s;
  Env::reset(P, s);
  int b = -1, tstep = 0;
  bool active = false, bad = false, pending = false;
  int bnext = 0;
  // deterministic mode: a static trajectory range [beg, bend) per CTA, slot row r starts
  // with beg + r, finished rows refill in row order (ballot ranks), no work stealing
  const int beg = DET ? (int)blockIdx.x * a.per : 0;
  const int bend = DET ? min(a.Bl, beg + a.per) : a.Bl;
  int dbase = beg + kTile;
  unsigned pm_prev = 0u;
  if (half == 0) {
    b = DET ? beg + row : atomicAdd(a.work, 1);
    active = b < bend;
    row_init[row] = 1;
    row_nd[row] = 0;
    row_b[row] = b;
    row_t[row] = 0;
  }
  long long ph[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, tprev = clock64();
  auto mark = [&](int k) {
    if (a.phase && tid == 0) {
      const long long tnow = clock64();
      ph[k] += tnow - tprev;
      tprev = tnow;
    }
  };
  int nact;
  while ((nact = __syncthreads_count(active || pending)) > 0) {
    mark(0);
    if (a.phase && tid == 0) {
      ph[6] += 1;
      ph[7] += nact;
      ph[8] += smax;
      smax = 0;
    }
    // (1) layer-1 pre-activation (fp32 in TMEM columns [H, 2H)), own column half, updated
    //     from the W1 rows of the features the last action changed (smem-resident W1 is
    //     stored with its 16-byte chunks XOR-swizzled by row, so the 32 lanes of a warp -
    //     32 different rows - spread over the banks)
    const bool init = row_init[row];
    const int nd = init ? 0 : row_nd[row];
    int df[2] = {0, 0};
    float dv[2] = {0.f, 0.f};
#pragma unroll
    for (int d = 0; d < 2; ++d)
      if (d < nd) {
        df[d] = row_df[row][d];
        dv[d] = row_dv[row][d];
      }
#pragma unroll 1
    for (int q = 0; q < HC / 32; ++q) {
      const int col = c0 + q * 32;
      // W1 rows of the (at most 2) changed features, fetched before the TMEM round trip
      uint4 w[2][4];
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        const uint4* wr = reinterpret_cast<const uint4*>(w1 + (size_t)df[d] * H);
#pragma unroll
        for (int c = 0; c < 4; ++c)
          w[d][c] = d < nd ? (W1S ? wr[((col >> 3) + c) ^ (df[d] & 7)] : __ldg(wr + (col >> 3) + c))
                           : make_uint4(0, 0, 0, 0);
      }
      uint32_t r[32];
      tmem_ld32(lane_base + H + col, r);  // warp-collective: every lane executes it
      tmem_wait_ld();
      if (init) {
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(h1init[col + i]);
      } else {
#pragma unroll
        for (int d = 0; d < 2; ++d) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint32_t wv[4] = {w[d][c].x, w[d][c].y, w[d][c].z, w[d][c].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) fma2_bf16(r[8 * c + 2 * e], r[8 * c + 2 * e + 1], dv[d], wv[e]);
          }
        }
        // (more than 2 changed features: general path)
        for (int d = 2; d < nd; ++d) {
          const float dvx = row_dv[row][d];
          const int fx = row_df[row][d];
          const uint4* wr = reinterpret_cast<const uint4*>(w1 + (size_t)fx * H);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint4 x = W1S ? wr[((col >> 3) + c) ^ (fx & 7)] : __ldg(wr + (col >> 3) + c);
            const uint32_t wv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              r[8 * c + 2 * e] = __float_as_uint(__uint_as_float(r[8 * c + 2 * e]) + dvx * bf16_lo(wv[e]));
              r[8 * c + 2 * e + 1] = __float_as_uint(__uint_as_float(r[8 * c + 2 * e + 1]) + dvx * bf16_hi(wv[e]));
            }
          }
        }
      }
      tmem_st32(lane_base + H + col, r);
      if (!SPLIT || half == 0) {  // (split: half 1 stages its columns after the first K-half MMA)
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          pk[i] = pack_bf16x2_relu(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
        reinterpret_cast<uint32_t*>(row_m1[row])[col >> 5] = relu_mask16(pk);
        st_row32(atile, row, col, pk);
      }
    }
    tmem_wait_st();
    if constexpr (DET) {  // refill ranks: finished rows of the last step in row order
      const int tot = s_pq[0] + s_pq[1] + s_pq[2] + s_pq[3];
      if (pending) {
        int rank = __popc(pm_prev & ((1u << lane) - 1u));
        for (int q = 0; q < quarter; ++q) rank += s_pq[q];
        bnext = dbase + rank;
      }
      dbase += tot;
    }
    if (pending) {  // the refill claim issued at the last termination lands here
      b = bnext;
      active = b < bend;
      row_b[row] = active ? b : -1;
      pending = false;
    }
    publish();
    // emission slot of this row (identical in both threads of the row): ballots of the
    // four row quarters give the CTA-wide prefix without another barrier
    bool my_valid = false;
    int gslot = 0;
    bool crossed = false;
    int claim = 0;
    {
      int before = 0, n = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int rb = row_b[q * 32 + lane];
        const bool v = rb >= 0 && rb < a.Bl;
        const uint32_t m = __ballot_sync(0xffffffffu, v);
        n += __popc(m);
        if (q < quarter) before += __popc(m);
        if (q == quarter) {
          before += __popc(m & ((1u << lane) - 1u));
          my_valid = v;
        }
      }
      const int nxt = s_next;
      const int p = fill + before;
      gslot = (p < kTile ? cur : nxt) * kTile + (p & (kTile - 1));
      fill += n;
      emitted += n;
      if (fill >= kTile) {
        fill -= kTile;
        cur = nxt;
        crossed = true;
      }
      // the next tile is claimed now; s_next is rewritten in this round's sample phase,
      // after every thread has read it above
      if (crossed && tid == kThreads - 1) claim = DET ? nclaim++ : atomicAdd(a.tilectr, 1);
    }
    // copy the 64 staged columns [half*64, half*64+64) of the A tile (logical columns
    // col0 + ...) of this warp's 32 rows into their emission tile images + ReLU masks,
    // overlapping the MMA. Eight lanes move one row's 128-byte line, so each store
    // instruction writes four whole lines.
    auto emit = [&](__nv_bfloat16* img, int col0) {
      const int j = lane & 7;  // physical 16-byte chunk of the staged row
#pragma unroll 4
      for (int i = 0; i < 8; ++i) {
        const int rl = 4 * i + (lane >> 3);
        const int srow = quarter * 32 + rl;
        const int gs = __shfl_sync(0xffffffffu, my_valid ? gslot : -1, rl);
        const uint4 x = *reinterpret_cast<const uint4*>(atile + half * (kTile * 128) + srow * 128 + j * 16);
        if (gs >= 0) {
          const int prow = gs & (kTile - 1);
          uint8_t* dst = reinterpret_cast<uint8_t*>(img) + (size_t)(gs >> 7) * kTile * H * 2 +
                         ((col0 >> 6) + half) * (kTile * 128) + prow * 128;
          *reinterpret_cast<uint4*>(dst + (((j ^ (srow & 7)) ^ (prow & 7)) * 16)) = x;
        }
      }
    };
    mark(1);
    // (2) hidden layer on the tensor cores: acc[128 x H] = relu(h1) W2^T (split-K for H=256)
    mma_round([&] { mma_kk<H, AK>(tmem, atile, w2img, false); });
    if (half == 1) {  // draw the row's uniform while the MMA runs (rng.cpp:64-66)
      const int rb = row_b[row];
      row_u[row] = rb >= 0 && rb < a.Bl ? uniform_scalar(fold_in(skeys[row_t[row]], (uint64_t)(a.b0 + rb))) : 0.0;
    }
    emit(a.h1, 0);
    mma_join();
    if (SPLIT) {
      if (half == 1)
#pragma unroll 1
        for (int q = 0; q < HC / 32; ++q)
          stage32(H + c0 + q * 32, q * 32, nullptr, reinterpret_cast<uint32_t*>(row_m1[row]) + ((c0 >> 5) + q));
      publish();
      mma_round([&] { mma_kk<H, AK>(tmem, atile, w2img + (AK / 64) * (H * 128), true); });
      emit(a.h1, AK);
      mma_join();
    }
    mark(2);
    // (3) h2 = ReLU(acc + b2) -> staged bf16 tile, (4) head on the tensor cores
    if (!SPLIT || half == 0)
#pragma unroll 1
      for (int q = 0; q < HC / 32; ++q)
        stage32(c0 + q * 32, c0 + q * 32, b2s + c0 + q * 32, reinterpret_cast<uint32_t*>(row_m2[row]) + ((c0 >> 5) + q));
    publish();
    mark(3);
    mma_round([&] { mma_kk<NH, AK>(tmem, atile, whimg, false); });
    emit(a.h2, 0);
    mma_join();
    if (SPLIT) {  // head output sits in acc columns [0, NH): half 1 reads [HC, H)
      if (half == 1)
#pragma unroll 1
        for (int q = 0; q < HC / 32; ++q)
          stage32(c0 + q * 32, q * 32, b2s + c0 + q * 32, reinterpret_cast<uint32_t*>(row_m2[row]) + ((c0 >> 5) + q));
      publish();
      mma_round([&] { mma_kk<NH, AK>(tmem, atile, whimg + (AK / 64) * (NH * 128), true); });
      emit(a.h2, AK);
      mma_join();
    }
    mark(4);
    float logit[NH];
    {
      uint32_t r[16];
#pragma unroll
      for (int c0h = 0; c0h < NH; c0h += 16) {
        tmem_ld16(lane_base + c0h, r);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 16; ++c) logit[c0h + c] = __uint_as_float(r[c]) + bhs[c0h + c];
      }
    }
    tc_fence_before();
    const long long ts0 = a.phase ? clock64() : 0;
    if (half == 0 && active) {
      float ex[NH], hi, z, rz;
      const int act = sample_row<Env, NH>(P, s, logit, A, a.eps, row_u[row], inv_legal, &bad, ex, hi, z, rz);
      if (act < 0) {
        active = false;
        a.frow_bt[gslot] = -1;
      } else {
        const size_t bt = (size_t)b * T + tstep;
        {
          a.frow_bt[gslot] = (int32_t)bt;
          a.bt_row[bt] = gslot;
        }
        Env::pack(P, s, a.stst + bt * P.SW);
        Env::pack(P, s, a.slot_st + (size_t)gslot * P.SW);
        a.slot_act[gslot] = (int16_t)act;
        int n = 0;
        Env::delta_features(P, s, act, [&](int f, float v) {
          row_df[row][n] = f;
          row_dv[row][n] = v;
          ++n;
        });
        row_nd[row] = n;
        row_init[row] = 0;
        const double prev_r = P.mdb ? Env::log_reward(P, s) : 0.0;
        const bool term = Env::step(P, s, act);
        a.batch.actions[bt] = (int16_t)act;
        a.batch.nparents[bt] = (uint16_t)Env::num_parents(P, s);
        if (P.mdb && !term) a.batch.delta[bt] = Env::log_reward(P, s) - prev_r;
        ++tstep;
        if (term) {
          a.batch.lengths[b] = tstep;
          a.batch.log_rewards[b] = Env::log_reward(P, s);
          Env::pack(P, s, a.batch.term_state + (size_t)b * P.SW);
          if constexpr (!DET) bnext = atomicAdd(a.work, 1);  // consumed after the next layer-1 phase
          atomicAdd(&s_nterm, 1);
          pending = true;
          active = false;
          Env::reset(P, s);
          tstep = 0;
          row_init[row] = 1;
        } else if (tstep >= T) {
          bad = true;
          active = false;
        }
        row_b[row] = active ? b : -1;
        row_t[row] = tstep;
      }
    }
    if (crossed && tid == kThreads - 1) s_next = claim;
    if (half == 1 && my_valid) {  // raw logits + ReLU masks of the row (idle half)
      float4* lg = reinterpret_cast<float4*>(a.logits + (size_t)gslot * NH);
#pragma unroll
      for (int k = 0; k < NH / 4; ++k) lg[k] = make_float4(logit[4 * k], logit[4 * k + 1], logit[4 * k + 2], logit[4 * k + 3]);
      uint4* m1 = reinterpret_cast<uint4*>(a.mask1 + (size_t)gslot * (H / 32));
      uint4* m2 = reinterpret_cast<uint4*>(a.mask2 + (size_t)gslot * (H / 32));
#pragma unroll
      for (int k = 0; k < H / 128; ++k) {
        m1[k] = row_m1[row][k];
        m2[k] = row_m2[row][k];
      }
    }
    if (a.phase && half == 0) atomicMax(&smax, (unsigned long long)(clock64() - ts0));
    if constexpr (DET) {  // this step's finished rows, ranked at the next refill
      pm_prev = __ballot_sync(0xffffffffu, pending);
      if (lane == 0 && half == 0) s_pq[quarter] = __popc(pm_prev);
    }
    mark(5);
  }
  if (a.phase && tid == 0)
    for (int k = 0; k < 9; ++k) atomicAdd((unsigned long long*)a.phase + k, (unsigned long long)ph[k]);
  if (bad) atomicExch(a.batch.counters + 3, GFNX_ERR_CONTRACT);
  {  // unused emission rows: rows [fill, 128) of `cur` and the whole pre-claimed tile
    const int nxt = s_next;
    const int slot = tid < kTile ? cur * kTile + tid : nxt * kTile + (tid - kTile);
    if (tid >= fill) {
      a.frow_bt[slot] = -1;
      const int prow = slot & (kTile - 1);
#pragma unroll
      for (int blk = 0; blk < H / 64; ++blk) {
        const size_t off = (size_t)(slot >> 7) * kTile * H * 2 + blk * (kTile * 128) + prow * 128;
        uint4* d1 = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(a.h1) + off);
        uint4* d2 = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(a.h2) + off);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          d1[j] = make_uint4(0, 0, 0, 0);
          d2[j] = make_uint4(0, 0, 0, 0);
        }
      }
    }
  }
  __syncthreads();
  if (tid == 0 && DET) a.det_used[blockIdx.x] = cur - s_cur0 + (fill > 0 ? 1 : 0);
  if (tid == 0) finish_counts(a.batch.counters, emitted, emitted - s_nterm);
  if (warp == 0) tmem_dealloc<2 * H>(tmem);
}

// ---------------------------------------------------------------------------
// k_fast_rollout_ts: H = 256 rollout with every GEMM A operand in tensor memory.
//
// Layer 1 runs on the tensor cores as well: each row's observation (<= 128 features,
// one-hot / 0-1 for hypergrid and DAG) is written into TMEM as the bf16 A operand of
// obs W1 (W1^T resident in smem as a K-major image), so TMEM holds only the accumulator
// [0, H) (layer 1, then the hidden layer), the packed bf16 activations [H, H + H/2)
// (obs, then h1, then h2 - the A operand of the next MMA, "TS" form) and the head
// accumulator [H + H/2, H + H/2 + NH). No shared-memory A tile: one MMA round per layer
// (instead of two split-K halves), both threads of a row stage their column halves at once,
// and no layer-1 state survives between steps. h1 / h2 rows are copied from TMEM into the
// emission tiles while the next MMA runs.
template <int H, int NH>
constexpr int rollout_ts_smem_bytes() {
  return H * H * 2 + NH * H * 2 + H * 128 * 2 + 1024;
}

template <class Env, int H, int NH, int SA, bool DET>
__global__ void __launch_bounds__(kThreads, 1) k_fast_rollout_ts(RolloutArgs a) {
  static_assert(SA <= NH, "sampler width");
  static_assert(H == 256, "TS rollout is the H = 256 path");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  constexpr int HC = H / 2;              // columns owned by each thread of a row
  constexpr uint32_t TA = H;             // packed obs, then h1: columns [H, H + H/2)
  constexpr uint32_t TA2 = H + H / 2;    // packed h2: columns [H + H/2, 2H)
  constexpr uint32_t TH = 0;             // head accumulator: [0, NH) of the (consumed) accumulator
  uint8_t* w2img = smem;                 // H x H bf16 (resident)
  uint8_t* whimg = w2img + H * H * 2;    // head image [NH][H]
  uint8_t* w1img = whimg + NH * H * 2;   // W1^T image [H][128 features], K-major
  __shared__ __align__(16) float b1s[H];
  __shared__ __align__(16) float b2s[H];
  __shared__ float bhs[NH];
  __shared__ Key skeys[128];
  __shared__ double row_u[kTile];
  __shared__ int row_b[kTile], row_t[kTile];
  __shared__ uint2 row_fm[kTile][2];  // active 0/1 observation features (bit f), per column half
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  __shared__ unsigned long long smax;
  __shared__ double inv_legal[NH + 1];
  __shared__ int s_cur0, s_next;
  __shared__ int s_pq[4];  // deterministic refills: finished rows per row quarter
  __shared__ int s_nterm;

  const EnvParams& P = a.P;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quarter = warp & 3, half = warp >> 2;
  const int row = quarter * 32 + lane, c0 = half * HC;
  const int T = P.T, A = P.A;
  if (warp == 0) tmem_alloc<512>(&tbase);
  if (tid == 0) {
    mbar_init(&mbar, 1);
    fence_mbar_init();
    smax = 0;
    const int t0 = DET ? (int)blockIdx.x * a.mt : atomicAdd(a.tilectr, 2);
    for (int q = 0; q < 4; ++q) s_pq[q] = 0;
    s_cur0 = t0;
    s_next = t0 + 1;
    s_nterm = 0;
  }
  __syncthreads();
  int cur = s_cur0, fill = 0, emitted = 0;
  int nclaim = s_cur0 + 2;  // deterministic mode: next tile of this CTA's region
  if (tid == 0) {
    mbar_arrive_expect_tx(&mbar, H * H * 2 + NH * H * 2);
    bulk_g2s_big(w2img, a.W.w2_fwd, H * H * 2, &mbar);
    bulk_g2s_big(whimg, a.W.whead_f, NH * H * 2, &mbar);
  }
  // W1^T as the K-major B operand of obs W1: row n = hidden unit, K = 128 features (zero
  // beyond obs_dim); thread pairs build one 16-byte chunk (8 features) of a unit's row
  for (int i = tid; i < H * 16; i += kThreads) {
    const int n = i % H, c = i / H;
    uint32_t w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int f0 = 8 * c + 2 * e;
      const uint32_t lo = f0 < P.O ? __bfloat16_as_ushort(a.W.w1[(size_t)f0 * H + n]) : 0u;
      const uint32_t hi = f0 + 1 < P.O ? __bfloat16_as_ushort(a.W.w1[(size_t)(f0 + 1) * H + n]) : 0u;
      w[e] = lo | (hi << 16);
    }
    *reinterpret_cast<uint4*>(w1img + sw128_offset(n, 8 * c, H)) = make_uint4(w[0], w[1], w[2], w[3]);
  }
  fence_proxy_async();
  for (int t = tid; t < T && t < 128; t += kThreads) skeys[t] = fold_in(a.key, (uint64_t)t);
  for (int j = tid; j < H; j += kThreads) {
    b1s[j] = a.W.b1[j];
    b2s[j] = a.W.b2[j];
  }
  if (tid < NH) bhs[tid] = tid < A ? a.W.bf[tid] : (tid == A ? a.W.bfl[0] : 0.f);
  if (tid <= NH) inv_legal[tid] = tid ? 1.0 / tid : 0.0;
  mbar_wait(&mbar, 0);
  uint32_t phase = 1;
  tc_fence_after();
  __syncthreads();
  const uint32_t tmem = tbase;
  const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);

  // every thread waits on the MMA's mbarrier itself (no CTA barrier): the next commit can
  // only follow a publish() barrier, so no thread can miss a phase
  auto mma_join = [&]() {
    mbar_wait(&mbar, phase);
    phase ^= 1;
    tc_fence_after();
  };
  auto publish = [&]() {  // tcgen05.st of the A operand -> visible to the MMA issuer
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
  };
  bool bad = false;
  auto set_features = [&](const typename Env::State& st) {  // observation as a bit set
    // two scalar 64-bit halves (a 4-word array gets indexed by f >> 5 and lands in local memory)
    uint64_t lo = 0ull, hi = 0ull;
    Env::features(P, st, [&](int f, double x) {
      if (x != 1.0 || f >= 128) bad = true;  // this path takes 0/1 observations only
      const uint64_t bit = 1ull << (f & 63);
      lo |= f < 64 ? bit : 0ull;
      hi |= f >= 64 ? bit : 0ull;
    });
    row_fm[row][0] = make_uint2((uint32_t)lo, (uint32_t)(lo >> 32));
    row_fm[row][1] = make_uint2((uint32_t)hi, (uint32_t)(hi >> 32));
  };

  typename Env::State s;
  Env::reset(P, s);
  int b = -1, tstep = 0;
  bool active = false, pending = false;
  int bnext = 0;
  // deterministic mode: a static trajectory range [beg, bend) per CTA, slot row r starts
  // with beg + r, finished rows refill in row order (ballot ranks), no work stealing
  const int beg = DET ? (int)blockIdx.x * a.per : 0;
  const int bend = DET ? min(a.Bl, beg + a.per) : a.Bl;
  int dbase = beg + kTile;
  unsigned pm_prev = 0u;
  if (half == 0) {
    b = DET ? beg + row : atomicAdd(a.work, 1);
    active = b < bend;
    row_b[row] = b;
    row_t[row] = 0;
    set_features(s);
  }
  long long ph[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, tprev = clock64();
  auto sub = [&](int k, long long& t) {  // sub-phases of the sampling step (thread 0)
    if (a.phase && tid == 0) {
      const long long tn = clock64();
      ph[k] += tn - t;
      t = tn;
    }
  };
  auto mark = [&](int k) {
    if (a.phase && tid == 0) {
      const long long tnow = clock64();
      ph[k] += tnow - tprev;
      tprev = tnow;
    }
  };
  // copy this thread's 128 packed activation columns (two 64-feature blocks of its row)
  // from TMEM into the row's emission slot of `img`
  // The emission stores are spread over the MMA waits of the step chain: h1 block 0 of the
  // thread's half during the hidden MMA, block 1 during the head MMA; h2 blocks 0-1 by the
  // idle half while the row samples, blocks 2-3 during the next step's layer-1 MMA (TA2
  // holds h2 until the next hidden epilogue).
  // ... and the block's two ReLU mask words (units [64 blk, 64 blk + 64)) go out with it
  auto emit_block = [&](__nv_bfloat16* img, uint32_t* mask, uint32_t ta, int blk, bool valid, int gs) {
    uint32_t r[32];
    tmem_ld32(lane_base + ta + 32 * blk, r);
    tmem_wait_ld();
    if (valid) {
      const int prow = gs & (kTile - 1);
      uint8_t* dst = reinterpret_cast<uint8_t*>(img) + (size_t)(gs >> 7) * kTile * H * 2 + blk * (kTile * 128) +
                     prow * 128;
      st_line_sw128(dst, prow, r);
      uint32_t lo[16], hi[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        lo[i] = r[i];
        hi[i] = r[16 + i];
      }
      *reinterpret_cast<uint2*>(mask + (size_t)gs * (H / 32) + 2 * blk) = make_uint2(relu_mask16(lo), relu_mask16(hi));
    }
  };
  // ReLU(acc + bias) of the thread's HC accumulator columns -> packed bf16 at TMEM column
  // dst: two 32-column loads in flight per wait (the TMEM load latency is paid HC / 64 times)
  auto epilogue = [&](const float* bias, uint32_t dst) {
#pragma unroll 1
    for (int q = 0; q < HC / 64; ++q) {
      const int col = c0 + q * 64;
      uint32_t r0[32], r1[32];
      tmem_ld32(lane_base + col, r0);
      tmem_ld32(lane_base + col + 32, r1);
      tmem_wait_ld();
      const float2* b2 = reinterpret_cast<const float2*>(bias + col);
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) pk[i] = bias_relu_pack(r0[2 * i], r0[2 * i + 1], b2[i]);
      tmem_st16(lane_base + dst + (col >> 1), pk);
#pragma unroll
      for (int i = 0; i < 16; ++i) pk[i] = bias_relu_pack(r1[2 * i], r1[2 * i + 1], b2[16 + i]);
      tmem_st16(lane_base + dst + ((col + 32) >> 1), pk);
    }
  };
  bool h2_pend = false;  // h2 blocks 2-3 of the previous step's row slot still to emit
  int h2_gs = 0;
  int nact;
  while ((nact = __syncthreads_count(active || pending)) > 0) {
    mark(0);
    if (a.phase && tid == 0) {
      ph[6] += 1;
      ph[7] += nact;
      ph[8] += smax;
      smax = 0;
    }
    // (1) observation row (bf16, features [64*half, 64*half + 64) of this thread) into
    //     the TMEM A columns; layer 1 = obs W1 on the tensor cores
    {
      const uint2 fm = row_fm[row][half];
      uint32_t ob[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {  // bf16 1.0 = 0x3F80
        const uint32_t w = i < 16 ? fm.x : fm.y, sh = 2 * (i & 15);
        ob[i] = ((w >> sh) & 1u) * 0x3F80u | ((w >> (sh + 1)) & 1u) * 0x3F800000u;
      }
      tmem_st32(lane_base + TA + 32 * half, ob);
    }
    publish();
    if (tid == 0) {
      tc_fence_after();
      mma_tk_k<H>(tmem, tmem + TA, w1img, (P.O + 15) & ~15);
      umma_commit(&mbar);
    }
    emit_block(a.h2, a.mask2, TA2, 2 + half, h2_pend, h2_gs);  // (warp-collective TMEM load)
    h2_pend = false;
    mma_join();
    // h1 = ReLU(acc + b1) -> packed into TMEM (the hidden MMA's A operand) + ReLU mask
    epilogue(b1s, TA);
    if constexpr (DET) {  // refill ranks: finished rows of the last step in row order
      const int tot = s_pq[0] + s_pq[1] + s_pq[2] + s_pq[3];
      if (pending) {
        int rank = __popc(pm_prev & ((1u << lane) - 1u));
        for (int q = 0; q < quarter; ++q) rank += s_pq[q];
        bnext = dbase + rank;
      }
      dbase += tot;
    }
    if (pending) {  // the refill claim issued at the last termination lands here
      b = bnext;
      active = b < bend;
      row_b[row] = active ? b : -1;
      pending = false;
    }
    publish();
    // (2) hidden layer: acc[128 x H] = h1 W2^T, A from TMEM, one round (issued before the
    //     emission-slot bookkeeping, which overlaps it)
    if (tid == 0) {
      tc_fence_after();
      mma_tk<H, H>(tmem, tmem + TA, w2img, false);
      umma_commit(&mbar);
    }
    bool my_valid = false;
    int gslot = 0;
    bool crossed = false;
    int claim = 0;
    {
      int before = 0, n = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int rb = row_b[q * 32 + lane];
        const bool v = rb >= 0 && rb < a.Bl;
        const uint32_t m = __ballot_sync(0xffffffffu, v);
        n += __popc(m);
        if (q < quarter) before += __popc(m);
        if (q == quarter) {
          before += __popc(m & ((1u << lane) - 1u));
          my_valid = v;
        }
      }
      const int nxt = s_next;
      const int p = fill + before;
      gslot = (p < kTile ? cur : nxt) * kTile + (p & (kTile - 1));
      fill += n;
      emitted += n;
      if (fill >= kTile) {
        fill -= kTile;
        cur = nxt;
        crossed = true;
      }
      if (crossed && tid == kThreads - 1) claim = DET ? nclaim++ : atomicAdd(a.tilectr, 1);
    }
    mark(1);
    if (half == 1) {  // the row's uniform while the MMA runs (rng.cpp:64-66)
      const int rb = row_b[row];
      row_u[row] = rb >= 0 && rb < a.Bl ? uniform_scalar(fold_in(skeys[row_t[row]], (uint64_t)(a.b0 + rb))) : 0.0;
    }
    emit_block(a.h1, a.mask1, TA, (c0 >> 6), my_valid, gslot);
    mma_join();
    mark(2);
    // (3) h2 = ReLU(acc + b2) -> packed into TMEM (own columns: h1 stays for its mask)
    epilogue(b2s, TA2);
    publish();
    mark(3);
    // (4) head (logits + flow) on the tensor cores
    if (tid == 0) {
      tc_fence_after();
      mma_tk<NH, H>(tmem + TH, tmem + TA2, whimg, false);
      umma_commit(&mbar);
    }
    emit_block(a.h1, a.mask1, TA, (c0 >> 6) + 1, my_valid, gslot);
    mma_join();
    mark(4);
    float logit[NH];
    {
      uint32_t r[16];
      tmem_ld16(lane_base + TH, r);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < NH; ++c) logit[c] = __uint_as_float(r[c]) + bhs[c];
    }
    tc_fence_before();
    const long long ts0 = a.phase ? clock64() : 0;
    if (half == 0 && active) {
      // the sampler runs over SA >= A columns only (SA = 8 for A <= 8)
      float lgs[SA], ex[SA], hi, z, rz;
#pragma unroll
      for (int c = 0; c < SA; ++c) lgs[c] = logit[c];
      long long tsub = ts0;
      const int act = sample_row<Env, SA>(P, s, lgs, A, a.eps, row_u[row], inv_legal, &bad, ex, hi, z, rz);
      sub(9, tsub);
      if (act < 0) {
        active = false;
        a.frow_bt[gslot] = -1;
      } else {
        const size_t bt = (size_t)b * T + tstep;
        a.frow_bt[gslot] = (int32_t)bt;
        a.bt_row[bt] = gslot;
        Env::pack(P, s, a.stst + bt * P.SW);
        Env::pack(P, s, a.slot_st + (size_t)gslot * P.SW);
        a.slot_act[gslot] = (int16_t)act;
        const double prev_r = P.mdb ? Env::log_reward(P, s) : 0.0;
        const bool term = Env::step(P, s, act);
        a.batch.actions[bt] = (int16_t)act;
        a.batch.nparents[bt] = (uint16_t)Env::num_parents(P, s);
        if (P.mdb && !term) a.batch.delta[bt] = Env::log_reward(P, s) - prev_r;
        ++tstep;
        if (term) {
          a.batch.lengths[b] = tstep;
          a.batch.log_rewards[b] = Env::log_reward(P, s);
          Env::pack(P, s, a.batch.term_state + (size_t)b * P.SW);
          if constexpr (!DET) bnext = atomicAdd(a.work, 1);  // consumed after the next layer-1 phase
          atomicAdd(&s_nterm, 1);
          pending = true;
          active = false;
          Env::reset(P, s);
          tstep = 0;
        } else if (tstep >= T) {
          bad = true;
          active = false;
        }
        sub(10, tsub);
        set_features(s);
        sub(11, tsub);
        row_b[row] = active ? b : -1;
        row_t[row] = tstep;
      }
    }
    if (crossed && tid == kThreads - 1) s_next = claim;
    if (half == 1) {  // idle half while the row samples: raw head outputs, h2 blocks 0-1
      if (my_valid) {
        float4* lg = reinterpret_cast<float4*>(a.logits + (size_t)gslot * NH);
#pragma unroll
        for (int k = 0; k < NH / 4; ++k) lg[k] = make_float4(logit[4 * k], logit[4 * k + 1], logit[4 * k + 2], logit[4 * k + 3]);
      }
      emit_block(a.h2, a.mask2, TA2, 0, my_valid, gslot);  // h2 blocks 0-1 (2-3 follow next step)
      emit_block(a.h2, a.mask2, TA2, 1, my_valid, gslot);
    }
    h2_pend = my_valid;
    h2_gs = gslot;
    if (a.phase && half == 0) atomicMax(&smax, (unsigned long long)(clock64() - ts0));
    if constexpr (DET) {  // this step's finished rows, ranked at the next refill
      pm_prev = __ballot_sync(0xffffffffu, pending);
      if (lane == 0 && half == 0) s_pq[quarter] = __popc(pm_prev);
    }
    mark(5);
  }
  emit_block(a.h2, a.mask2, TA2, 2 + half, h2_pend, h2_gs);  // the last step's deferred h2 blocks
  if (a.phase && tid == 0)
    for (int k = 0; k < 12; ++k) atomicAdd((unsigned long long*)a.phase + (k < 9 ? k : k + 3), (unsigned long long)ph[k]);
  if (bad) atomicExch(a.batch.counters + 3, GFNX_ERR_CONTRACT);
  {  // unused emission rows: rows [fill, 128) of `cur` and the whole pre-claimed tile
    const int nxt = s_next;
    const int slot = tid < kTile ? cur * kTile + tid : nxt * kTile + (tid - kTile);
    if (tid >= fill) {
      a.frow_bt[slot] = -1;
      const int prow = slot & (kTile - 1);
#pragma unroll
      for (int blk = 0; blk < H / 64; ++blk) {
        const size_t off = (size_t)(slot >> 7) * kTile * H * 2 + blk * (kTile * 128) + prow * 128;
        uint4* d1 = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(a.h1) + off);
        uint4* d2 = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(a.h2) + off);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          d1[j] = make_uint4(0, 0, 0, 0);
          d2[j] = make_uint4(0, 0, 0, 0);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (tid == 0 && DET) a.det_used[blockIdx.x] = cur - s_cur0 + (fill > 0 ? 1 : 0);
  if (tid == 0) finish_counts(a.batch.counters, emitted, emitted - s_nterm);
  if (warp == 0) tmem_dealloc<512>(tmem);
}

// ---------------------------------------------------------------------------
// k_fast_fwd: forward over the real rows (2 threads per row, as in the rollout)

struct TrainArgs {
  EnvParams P;
  Weights W;
  DeviceBatch batch;
  int Bl;
  const uint32_t* stst;
  const int32_t* frow_bt;   // row slot -> b * T + t, -1 = empty slot
  const int32_t* tilectr;   // number of 128-row tiles of row slots
  const int32_t* tile_list; // deterministic mode: training tile -> emission tile, or null
  __nv_bfloat16 *h1, *h2, *dz2, *dhead;
  uint32_t *mask1, *mask2;  // ReLU masks of h1 / h2, [rows][H/32]
  const uint32_t* slot_st;  // slot-ordered packed states / actions (training path only)
  const int16_t* slot_act;
  float* rowbuf;
  int rs;
  float* coef;
  float* wpart;
  int64_t n_params;
  int64_t pstride;  // per-CTA partial slab stride (n_params rounded up to 8 floats: 32-byte stores)
  MlpLayout L;
  int objective;
  long long* phase;  // optional diagnostics: [9..11] wgrad pass clocks (thread 0, summed over CTAs)
};

// smem: W2 image | head image | staged A (split-K for H = 256, as in the rollout) | W1 (opt.)
template <int H, int NH>
constexpr int fwd_smem_fixed() {
  return H * H * 2 + NH * H * 2 + kTile * rollout_acols<H>() * 2 + 1024;
}

constexpr int kMaxSWFwd = 4;  // packed state words prefetched per row

template <class Env, int H, int NH, bool W1S>
__global__ void __launch_bounds__(kThreads, 1) k_fast_fwd(TrainArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  constexpr bool SPLIT = H == 256;
  constexpr int AK = rollout_acols<H>();
  constexpr int HC = H / 2;
  uint8_t* w2img = smem;
  uint8_t* whimg = w2img + H * H * 2;
  uint8_t* atile = whimg + NH * H * 2;
  __nv_bfloat16* w1s = reinterpret_cast<__nv_bfloat16*>(atile + kTile * AK * 2);
  const __nv_bfloat16* w1 = W1S ? w1s : a.W.w1;
  __shared__ float b1s[H], b2s[H];
  __shared__ float bhs[NH];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  const EnvParams& P = a.P;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quarter = warp & 3, half = warp >> 2;
  const int row = quarter * 32 + lane, c0 = half * HC;
  const int A = P.A;
  const int tiles = *a.tilectr;
  const int R = tiles * kTile;
  if ((int)blockIdx.x >= tiles) return;
  if (warp == 0) tmem_alloc<H>(&tbase);
  if (tid == 0) {
    mbar_init(&mbar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    mbar_arrive_expect_tx(&mbar, H * H * 2 + NH * H * 2);
    bulk_g2s_big(w2img, a.W.w2_fwd, H * H * 2, &mbar);
    bulk_g2s_big(whimg, a.W.whead_f, NH * H * 2, &mbar);
  }
  if (W1S) {  // 16-byte chunk c of W1 row f stored at c ^ (f & 7) (bank spread, as the rollout)
    const uint4* src = reinterpret_cast<const uint4*>(a.W.w1);
    uint4* dst = reinterpret_cast<uint4*>(w1s);
    constexpr int CPR = H / 8;
    for (int i = tid; i < P.O * CPR; i += kThreads) {
      const int f = i / CPR, c = i % CPR;
      dst[f * CPR + (c ^ (f & 7))] = src[i];
    }
  }
  for (int j = tid; j < H; j += kThreads) {
    b1s[j] = a.W.b1[j];
    b2s[j] = a.W.b2[j];
  }
  if (tid < NH) bhs[tid] = tid < A ? a.W.bf[tid] : (tid == A ? a.W.bfl[0] : 0.f);
  mbar_wait(&mbar, 0);
  uint32_t phase = 1;
  tc_fence_after();
  __syncthreads();
  const uint32_t tmem = tbase;
  const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
  const bool flow = a.objective == GFNX_OBJ_DB || a.objective == GFNX_OBJ_SUBTB;
  auto mma_join = [&]() {
    if (tid == 0) mbar_wait(&mbar, phase);
    phase ^= 1;
    __syncthreads();
    tc_fence_after();
  };
  auto publish = [&]() {
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
  };
  // row record of a tile, fetched one tile ahead (row -> (b, t) -> packed state, action)
  auto fetch = [&](int tile, uint32_t (&w)[kMaxSWFwd], int& act) {
    const int r = tile * kTile + row;
    act = 0;
#pragma unroll
    for (int i = 0; i < kMaxSWFwd; ++i) w[i] = 0;
    if (r < R && tile < tiles && a.frow_bt[r] >= 0) {
      const size_t bt = (size_t)a.frow_bt[r];
#pragma unroll
      for (int i = 0; i < kMaxSWFwd; ++i)
        if (i < P.SW) w[i] = a.stst[bt * P.SW + i];
      act = a.batch.actions[bt];
    }
  };
  uint32_t wn[kMaxSWFwd];
  int actn;
  fetch(blockIdx.x, wn, actn);
  for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int r = tile * kTile + row;
    const bool valid = r < R && a.frow_bt[r] >= 0;
    uint32_t wc[kMaxSWFwd];
#pragma unroll
    for (int i = 0; i < kMaxSWFwd; ++i) wc[i] = wn[i];
    const int act = actn;
    fetch(tile + gridDim.x, wn, actn);  // in flight during this tile
    typename Env::State s;
    Env::unpack(P, wc, s);
    // layer 1: sparse one-hot gather (fp32) -> bf16 ReLU; own column half. With split-K,
    // half 1 keeps its packed values until the first K-half MMA has read the staged tile.
    int nf = 0;
    int fidx[kGatherMax];
    float fval[kGatherMax];
    if (valid)
      Env::features(P, s, [&](int f, double x) {
        if (nf < kGatherMax) {
          fidx[nf] = f;
          fval[nf] = (float)x;
          ++nf;
        }
      });
    uint32_t keep[SPLIT ? HC / 2 : 1];
    if (tid == 0) bulk_wait_read0();  // previous tile's h2 stores have left smem
    __syncthreads();
#pragma unroll
    for (int q = 0; q < HC / 32; ++q) {
      const int col = c0 + q * 32;
      float v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = b1s[col + i];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint4 w[kGatherMax];
#pragma unroll
        for (int k = 0; k < kGatherMax; ++k)
          if (k < nf) {
            const uint4* wr = reinterpret_cast<const uint4*>(w1 + (size_t)fidx[k] * H);
            w[k] = W1S ? wr[((col >> 3) + c) ^ (fidx[k] & 7)] : __ldg(wr + (col >> 3) + c);
          }
#pragma unroll
        for (int k = 0; k < kGatherMax; ++k)
          if (k < nf) {
            const uint32_t wv[4] = {w[k].x, w[k].y, w[k].z, w[k].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              v[8 * c + 2 * e] += fval[k] * bf16_lo(wv[e]);
              v[8 * c + 2 * e + 1] += fval[k] * bf16_hi(wv[e]);
            }
          }
      }
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) pk[i] = valid ? pack_bf16x2_relu(v[2 * i], v[2 * i + 1]) : 0u;
      const uint32_t mb = relu_mask16(pk);
      if (valid) a.mask1[(size_t)r * (H / 32) + half * (HC / 32) + q] = mb;
      if (!SPLIT || half == 0) {
        st_row32(atile, row, col, pk);
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) keep[(q * 16 + i) % (SPLIT ? HC / 2 : 1)] = pk[i];
      }
    }
    publish();
    // hidden layer, K-half 0 (or all of K): h1 image out + MMA
    if (tid == 0) {
      tc_fence_after();
      bulk_s2g(a.h1 + (size_t)tile * kTile * H, atile, kTile * AK * 2);
      bulk_commit();
      mma_kk<H, AK>(tmem, atile, w2img, false);
      umma_commit(&mbar);
    }
    mma_join();
    if (SPLIT) {
      if (tid == 0) bulk_wait_read0();
      __syncthreads();
      if (half == 1)
#pragma unroll
        for (int q = 0; q < HC / 32; ++q) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) pk[i] = keep[(q * 16 + i) % (SPLIT ? HC / 2 : 1)];
          st_row32(atile, row, q * 32, pk);
        }
      publish();
      if (tid == 0) {
        tc_fence_after();
        bulk_s2g(a.h1 + (size_t)tile * kTile * H + kTile * AK, atile, kTile * AK * 2);
        bulk_commit();
        mma_kk<H, AK>(tmem, atile, w2img + (AK / 64) * (H * 128), true);
        umma_commit(&mbar);
      }
      mma_join();
    }
    if (tid == 0) bulk_wait_read0();
    __syncthreads();
    // epilogue: h2 (bf16-rounded) -> staged tile + ReLU mask; head GEMM per K-half
    auto h2_stage = [&](int q, int acol) {
      const int col = c0 + q * 32;
      uint32_t r32[32];
      tmem_ld32(lane_base + col, r32);
      tmem_wait_ld();
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float x0 = fmaxf(__uint_as_float(r32[2 * i]) + b2s[col + 2 * i], 0.f);
        const float x1 = fmaxf(__uint_as_float(r32[2 * i + 1]) + b2s[col + 2 * i + 1], 0.f);
        pk[i] = valid ? pack_bf16x2(x0, x1) : 0u;
      }
      const uint32_t mb = relu_mask16(pk);
      if (valid) a.mask2[(size_t)r * (H / 32) + half * (HC / 32) + q] = mb;
      st_row32(atile, row, acol, pk);
    };
    if (!SPLIT || half == 0)
#pragma unroll 1
      for (int q = 0; q < HC / 32; ++q) h2_stage(q, c0 + q * 32);
    publish();
    if (tid == 0) {
      tc_fence_after();
      bulk_s2g(a.h2 + (size_t)tile * kTile * H, atile, kTile * AK * 2);
      bulk_commit();
      mma_kk<NH, AK>(tmem, atile, whimg, false);
      umma_commit(&mbar);
    }
    mma_join();
    if (SPLIT) {  // head output sits in acc columns [0, NH): half 1 reads [HC, H)
      if (tid == 0) bulk_wait_read0();
      __syncthreads();
      if (half == 1)
#pragma unroll 1
        for (int q = 0; q < HC / 32; ++q) h2_stage(q, q * 32);
      publish();
      if (tid == 0) {
        tc_fence_after();
        bulk_s2g(a.h2 + (size_t)tile * kTile * H + kTile * AK, atile, kTile * AK * 2);
        bulk_commit();
        mma_kk<NH, AK>(tmem, atile, whimg + (AK / 64) * (NH * 128), true);
        umma_commit(&mbar);
      }
      mma_join();
    }
    float logit[NH];
    {
      uint32_t r16[16];
#pragma unroll
      for (int c0h = 0; c0h < NH; c0h += 16) {
        tmem_ld16(lane_base + c0h, r16);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 16; ++c) logit[c0h + c] = __uint_as_float(r16[c]) + bhs[c0h + c];
      }
    }
    tc_fence_before();
    if (half == 0 && valid) {  // masked log-softmax statistics of the row
      float hi = -INFINITY;
#pragma unroll
      for (int c = 0; c < NH; ++c)
        if (c < A && Env::legal(P, s, c)) hi = fmaxf(hi, logit[c]);
      float z = 0.f;
#pragma unroll
      for (int c = 0; c < NH; ++c)
        if (c < A && Env::legal(P, s, c)) z += __expf(logit[c] - hi);
      const float lse = hi + __logf(z);
      float* out = a.rowbuf + (size_t)r * a.rs;
      float la = 0.f, ls = 0.f, fl = 0.f;
#pragma unroll
      for (int c = 0; c < NH; ++c) {
        if (c < A) out[c] = Env::legal(P, s, c) ? __expf(logit[c] - lse) : 0.f;
        if (c == act) la = logit[c];
        if (c == P.stop) ls = logit[c];
        if (c == A) fl = logit[c];
      }
      out[A] = la - lse;
      out[A + 1] = P.stop >= 0 ? ls - lse : 0.f;
      out[A + 2] = flow ? fl : 0.f;
      if (!isfinite(lse)) atomicExch(a.batch.counters + 3, GFNX_ERR_NUMERIC);
    }
  }
  if (tid == 0) bulk_wait0();
  __syncthreads();
  if (warp == 0) tmem_dealloc<H>(tmem);
}

// ---------------------------------------------------------------------------
// k_fast_loss_warp: residuals of every objective and their analytic backward

struct LossArgs {
  DeviceBatch batch;
  int Bl, T, A, stop, objective, B_global;
  double terminal_penalty;
  const double* lampow;
  const double* neglog;
  const float* rowbuf;
  int rs;
  const int32_t* bt_row;  // b * T + t -> row slot
  float* coef;
  double* lpart;
  const double* scalars;
};

// TB / DB / SubTB / MDB with one warp per trajectory (lanes over the steps, SubTB lanes over
// the sub-trajectory starts then ends): the per-step loads are independent, so a trajectory
// costs two dependent loads instead of 2 L (objectives.cpp:94-226); partial sums in a fixed
// tree order.
GFNX_DEV double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

constexpr int kSubTBMaxT = 128;  // supported() caps max_traj_len at 128 on this path

// SUBTB: the only objective with per-warp shared scratch (34 KB per block); the others run
// 8 blocks per SM (register-bound at 32 registers)
template <bool SUBTB>
__global__ void __launch_bounds__(256, SUBTB ? 4 : 8) k_fast_loss_warp(LossArgs a) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int nw = gridDim.x * (blockDim.x >> 5);
  const int* cnt = a.batch.counters;
  double norm = (double)a.B_global;
  if (a.objective == GFNX_OBJ_DB) norm = (double)cnt[4];
  if (a.objective == GFNX_OBJ_MDB) norm = (double)cnt[5];
  double loss = 0.0, dlogz = 0.0;  // lane 0
  for (int b = blockIdx.x * (blockDim.x >> 5) + wib; b < a.Bl; b += nw) {
    const int L = a.batch.lengths[b];
    const int32_t* rows = a.bt_row + (size_t)b * a.T;
    const uint16_t* np = a.batch.nparents + (size_t)b * a.T;
    const double logr = a.batch.log_rewards[b];
    auto rec = [&](int t, int k) { return (double)a.rowbuf[(size_t)rows[t] * a.rs + a.A + k]; };
    auto C = [&](int t) { return reinterpret_cast<float4*>(a.coef + (size_t)rows[t] * 4); };
    if (a.objective == GFNX_OBJ_TB) {  // tb_loss objectives.cpp:120-142
      const double w = 1.0 / norm;
      double sd = 0.0;
      for (int t = lane; t < L; t += 32) sd += rec(t, 0) - a.neglog[np[t]];
      sd = warp_sum_d(sd);
      const double res = sd + a.scalars[0] - logr;
      const double g = 2.0 * res * w;
      for (int t = lane; t < L; t += 32) *C(t) = make_float4((float)g, 0.f, 0.f, 0.f);
      if (lane == 0) {
        loss += res * res * w;
        dlogz += g;
      }
    } else if (a.objective == GFNX_OBJ_DB) {  // transition_loss :94-118
      double carry = 0.0, ls = 0.0;
      for (int k0 = 0; k0 < L; k0 += 32) {
        const int t = k0 + lane;
        double g = 0.0;
        if (t < L) {
          const double d = rec(t, 0) - a.neglog[np[t]];
          const double f1 = t + 1 < L ? rec(t + 1, 2) : logr;
          const double res = rec(t, 2) - f1 + d;
          const double w = (t == L - 1 ? a.terminal_penalty : 1.0) / norm;
          ls += res * res * w;
          g = 2.0 * res * w;
        }
        double gp = __shfl_up_sync(0xffffffffu, g, 1);
        if (lane == 0) gp = carry;
        if (t < L) *C(t) = make_float4((float)g, 0.f, (float)(g - gp), 0.f);
        carry = __shfl_sync(0xffffffffu, g, 31);
      }
      ls = warp_sum_d(ls);
      if (lane == 0) loss += ls;
    } else if constexpr (SUBTB) {  // subtb_loss :144-180, lanes over j then k
      __shared__ double sub_F[8][kSubTBMaxT + 1], sub_c[8][kSubTBMaxT + 1], sub_S[8][kSubTBMaxT + 1],
          sub_T[8][kSubTBMaxT + 1];
      double* F = sub_F[wib];
      double* cum = sub_c[wib];
      double* Sg = sub_S[wib];
      double* Tg = sub_T[wib];
      double carry = 0.0;
      for (int k0 = 0; k0 < L; k0 += 32) {  // F(s_t), cum = exclusive prefix of d
        const int t = k0 + lane;
        const double d = t < L ? rec(t, 0) - a.neglog[np[t]] : 0.0;
        if (t < L) F[t] = rec(t, 2);
        double incl = d;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        if (t < L) cum[t + 1] = carry + incl;
        carry += __shfl_sync(0xffffffffu, incl, 31);
      }
      if (lane == 0) {
        F[L] = logr;
        cum[0] = 0.0;
      }
      double nl = 0.0;  // norm_b = sum_{j<k<=L} lambda^(k-j) = sum_m (L+1-m) lambda^m
      for (int m = 1 + lane; m <= L; m += 32) nl += (double)(L + 1 - m) * a.lampow[m];
      const double nrm = warp_sum_d(nl);
      __syncwarp();
      double ls = 0.0;
      for (int j = lane; j < L; j += 32) {  // S_j = sum_k g_jk (loss terms counted here)
        double sj = 0.0;
        for (int k = j + 1; k <= L; ++k) {
          const double w = a.lampow[k - j] / nrm / norm;
          const double res = (F[j] - F[k]) + (cum[k] - cum[j]);
          ls += res * res * w;
          sj += 2.0 * res * w;
        }
        Sg[j] = sj;
      }
      for (int k = lane; k <= L; k += 32) {  // T_k = sum_j g_jk
        double tk = 0.0;
        for (int j = 0; j < k; ++j) {
          const double w = a.lampow[k - j] / nrm / norm;
          const double res = (F[j] - F[k]) + (cum[k] - cum[j]);
          tk += 2.0 * res * w;
        }
        Tg[k] = tk;
      }
      if (lane == 0) Sg[L] = 0.0;
      __syncwarp();
      // gF[c] = S_c - T_c, gc[c] = T_c - S_c; coefficient of log pi at step c: sum_{c' > c} gc[c']
      double suf = 0.0;
      for (int k0 = 0; k0 <= L; k0 += 32) {
        const int c = L - k0 - lane;
        const double v = c >= 0 ? Tg[c] - Sg[c] : 0.0;
        double incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        if (c >= 0 && c < L) *C(c) = make_float4((float)(suf + incl - v), 0.f, (float)(Sg[c] - Tg[c]), 0.f);
        suf += __shfl_sync(0xffffffffu, incl, 31);
      }
      ls = warp_sum_d(ls);
      if (lane == 0) loss += ls;
      __syncwarp();
    } else {  // mdb_loss :186-226
      const double w = 1.0 / norm;
      double carry = 0.0, ls = 0.0;
      for (int k0 = 0; k0 < L; k0 += 32) {
        const int t = k0 + lane;
        double g = 0.0;
        if (t + 1 < L) {
          const double res = rec(t, 0) + (rec(t + 1, 1) - rec(t, 1)) - a.neglog[np[t]] -
                             a.batch.delta[(size_t)b * a.T + t];
          ls += res * res * w;
          g = 2.0 * res * w;
        }
        double gp = __shfl_up_sync(0xffffffffu, g, 1);
        if (lane == 0) gp = carry;
        if (t < L) *C(t) = make_float4((float)g, (float)(gp - g), 0.f, 0.f);
        carry = __shfl_sync(0xffffffffu, g, 31);
      }
      ls = warp_sum_d(ls);
      if (lane == 0) loss += ls;
    }
  }
  __shared__ double red[2][32];
  if (lane == 0) {
    red[0][wib] = loss;
    red[1][wib] = dlogz;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double l = 0.0, z = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      l += red[0][i];
      z += red[1][i];
    }
    a.lpart[2 * blockIdx.x] = l;
    a.lpart[2 * blockIdx.x + 1] = z;
  }
}

// fixed-order two-level sum of the block partials (256 threads: strided, then a tree)
__global__ void k_loss_finalize(const double* lpart, int nblocks, double* scalars, int tb,
                                int32_t* err) {
  __shared__ double red[2][256];
  double l = 0.0, z = 0.0;
  const double2* lp = reinterpret_cast<const double2*>(lpart);
  int i = threadIdx.x;
  for (; i + 7 * (int)blockDim.x < nblocks; i += 8 * blockDim.x) {  // 8 loads in flight
    double2 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = lp[i + k * blockDim.x];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      l += v[k].x;
      z += v[k].y;
    }
  }
  for (; i < nblocks; i += blockDim.x) {
    l += lp[i].x;
    z += lp[i].y;
  }
  red[0][threadIdx.x] = l;
  red[1][threadIdx.x] = z;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if ((int)threadIdx.x < off) {
      red[0][threadIdx.x] += red[0][threadIdx.x + off];
      red[1][threadIdx.x] += red[1][threadIdx.x + off];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    scalars[4] = red[0][0];
    scalars[3] = tb ? red[1][0] : 0.0;
    if (!isfinite(red[0][0])) atomicExch(err, GFNX_ERR_NUMERIC);
  }
}

// ---------------------------------------------------------------------------
// k_fast_bwd: dlogits, head dgrad and W2 dgrad on the tensor cores, ReLU masks, bias grads,
// and [dW1 | db1] = [obs | 1]^T dz1 while dz1 is still in shared memory (dz1 never goes to
// HBM): the one-hot observation rows of the two 64-row units are built in the dhead tile
// (free once the head MMA and the dhead store are done) and in the first 16 KB of the W2
// dgrad image (re-fetched from L2 during the next tile's dlogits / head MMA), and multiplied
// against the dz tile in place

// D[128 features x N] (+)= obs_u^T dz[rows 64u .. 64u + 63]: obs unit image [2 feature
// blocks][64 rows][128 B] (MN-major, LBO 8 KB), dz tile [N / 64 blocks][128 rows][128 B]
// (MN-major, LBO 16 KB), K = 64 rows in four K = 16 steps
template <int N>
GFNX_DEV void mma_obs_dz(uint32_t d_tmem, const void* obs_img, const void* dz_img, int u, bool acc) {
  constexpr uint32_t idesc = umma_idesc_bf16(128, N, true, true);
  const uint32_t a0 = smem_u32(obs_img), b0 = smem_u32(dz_img) + u * 64 * 128;
#pragma unroll
  for (int s = 0; s < 4; ++s)
    umma_bf16(d_tmem, umma_desc_sw128(a0 + s * 2048, 64 * 128, 1024), umma_desc_sw128(b0 + s * 2048, kTile * 128, 1024),
              idesc, (acc || s > 0) ? 1u : 0u);
}

template <int H, int NH>
constexpr int bwd_smem_bytes() {
  return H * H * 2 + kTile * H * 2 + kTile * 64 * 2 + H * NH * 2 + kThreads * 8 * 4 + kThreads * 4 + 1024;
}

template <class Env, int H, int NH, bool LIST>
__global__ void __launch_bounds__(kThreads, 1) k_fast_bwd(TrainArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* wdimg = smem;                     // W2 dgrad image [H in][H out]
  uint8_t* atile = wdimg + H * H * 2;        // dz tile
  uint8_t* htile = atile + kTile * H * 2;    // dhead tile [128][64]
  uint8_t* whd = htile + kTile * 64 * 2;     // head dgrad image [H][NH], non-swizzled
  float* red = reinterpret_cast<float*>(whd + H * NH * 2);  // [kThreads * 8 / H][H] bias partials
  float* redh = red + kThreads * 8;                           // [kThreads / NH][NH] head bias partials
  constexpr int HC = H / 2;
  __shared__ uint64_t mbar, mbar1, mbar2, mbarw;  // mbar1 / mbar2: the dW1 MMAs of the htile /
                                                  // W2-window obs units; mbarw: the W2 patch
  __shared__ uint32_t tbase;
  const EnvParams& P = a.P;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quarter = warp & 3, half = warp >> 2;
  const int row = quarter * 32 + lane, c0 = half * HC;
  const int A = P.A;
  const int tiles = *a.tilectr;
  const int R = tiles * kTile;
  float* part = a.wpart + (size_t)blockIdx.x * a.pstride;
  float acc_b2 = 0.f, acc_bh = 0.f;  // thread j owns bias column j (db1: the dW1 GEMM's feature O)
  if ((int)blockIdx.x < tiles) {
    if (warp == 0) tmem_alloc<2 * H>(&tbase);  // [0, H): dgrad accumulators, [H, 2H): dW1 | db1
    if (tid == 0) {
      mbar_init(&mbar, 1);
      mbar_init(&mbar1, 1);
      mbar_init(&mbar2, 1);
      mbar_init(&mbarw, 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
      mbar_arrive_expect_tx(&mbar, H * H * 2 + H * NH * 2);
      bulk_g2s_big(wdimg, a.W.w2_dgrad, H * H * 2, &mbar);
      bulk_g2s_big(whd, a.W.whead_d, H * NH * 2, &mbar);
    }
    mbar_wait(&mbar, 0);
    uint32_t phase = 1;
    tc_fence_after();
    __syncthreads();
    const uint32_t tmem = tbase;
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    const bool flow = a.objective == GFNX_OBJ_DB || a.objective == GFNX_OBJ_SUBTB;
    // per-row inputs of a tile, prefetched one tile ahead (the slot map two tiles ahead, so
    // no load in flight depends on another): masks (both halves), and for half 0 the packed
    // state, action, loss coefficients and softmax record
    struct RowIn {
      uint32_t mk2[HC / 32], mk1[HC / 32];
      uint32_t mk1x;  // half 1: h1 mask word of the last chunk of half 0 (its extra dz1 chunk)
      uint32_t sw[kMaxSWFwd];
      int act;
      float ga, gs, gf;
      float pr[NH];
    };
    auto slot_of = [&](int tile) { return tile < tiles ? a.frow_bt[phys_tile<LIST>(a.tile_list, tile) * kTile + row] : -1; };
    // vector loads only: these rows are strided, so every load instruction of a warp touches
    // 32 lines and the load/store unit, not the latency, bounds the prefetch
    auto load_row = [&](int tile, int rbt, RowIn& x) {
      const int r = (tile < tiles ? phys_tile<LIST>(a.tile_list, tile) : 0) * kTile + row;
      const bool v = rbt >= 0, v0 = v && half == 0;
      const size_t mo = (size_t)r * (H / 32) + half * (HC / 32);
      if constexpr (HC / 32 == 4) {
        const uint4 z = make_uint4(0u, 0u, 0u, 0u);
        const uint4 m2 = v ? *reinterpret_cast<const uint4*>(a.mask2 + mo) : z;
        const uint4 m1 = v ? *reinterpret_cast<const uint4*>(a.mask1 + mo) : z;
        x.mk2[0] = m2.x; x.mk2[1] = m2.y; x.mk2[2] = m2.z; x.mk2[3] = m2.w;
        x.mk1[0] = m1.x; x.mk1[1] = m1.y; x.mk1[2] = m1.z; x.mk1[3] = m1.w;
      } else {
        static_assert(HC / 32 == 2, "mask words per thread");
        const uint2 z = make_uint2(0u, 0u);
        const uint2 m2 = v ? *reinterpret_cast<const uint2*>(a.mask2 + mo) : z;
        const uint2 m1 = v ? *reinterpret_cast<const uint2*>(a.mask1 + mo) : z;
        x.mk2[0] = m2.x; x.mk2[1] = m2.y;
        x.mk1[0] = m1.x; x.mk1[1] = m1.y;
      }
      x.mk1x = (v && half == 1) ? a.mask1[(size_t)r * (H / 32) + HC / 32 - 1] : 0u;
#pragma unroll
      for (int i = 0; i < kMaxSWFwd; ++i) x.sw[i] = (v0 && i < P.SW) ? a.slot_st[(size_t)r * P.SW + i] : 0u;
      x.act = v0 ? a.slot_act[r] : 0;
      const float4 cf = v0 ? *reinterpret_cast<const float4*>(a.coef + (size_t)r * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
      x.ga = cf.x;
      x.gs = cf.y;
      x.gf = flow ? cf.z : 0.f;
      const float4* pr4 = reinterpret_cast<const float4*>(a.rowbuf + (size_t)r * a.rs);
#pragma unroll
      for (int c4 = 0; c4 < NH / 4; ++c4) {
        const float4 q = (v0 && 4 * c4 < A) ? pr4[c4] : make_float4(0.f, 0.f, 0.f, 0.f);
        x.pr[4 * c4] = q.x;
        x.pr[4 * c4 + 1] = q.y;
        x.pr[4 * c4 + 2] = q.z;
        x.pr[4 * c4 + 3] = q.w;
      }
    };
    int rbt_cur = slot_of(blockIdx.x), rbt_next = slot_of(blockIdx.x + gridDim.x);
    RowIn nx;
    load_row(blockIdx.x, rbt_cur, nx);
    long long pc[7] = {0, 0, 0, 0, 0, 0, 0}, tclk = clock64();
    auto pmark = [&](int k) {  // phase clocks (thread 0): slots 15..19, tiles in 20
      if (a.phase && tid == 0) {
        const long long tn = clock64();
        pc[k] += tn - tclk;
        tclk = tn;
      }
    };
    // one-hot observation row rl of a 64-row unit image x (+ constant feature O: its output
    // row is db1 = sum_r dz1[r]); the row's own thread zeroes it (chunks rotated by row, no
    // bank conflicts) and writes its features
    auto build_obs_row = [&](uint8_t* x, int rl, bool v, const uint32_t (&w)[kMaxSWFwd]) {
#pragma unroll
      for (int blk = 0; blk < 2; ++blk)
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<uint4*>(x + blk * (64 * 128) + rl * 128 + ((c + rl) & 7) * 16) = make_uint4(0, 0, 0, 0);
      if (v) {
        typename Env::State s;
        Env::unpack(P, w, s);
        auto put = [&](int f, float y) {
          *reinterpret_cast<__nv_bfloat16*>(x + sw128_offset(rl, f, 64)) = __float2bfloat16(y);
        };
        Env::features(P, s, [&](int f, double val) { put(f, (float)val); });
        put(P.O, 1.f);
      }
    };
    bool w1_pending = false, w1_acc = false, w2_patch = false;
    uint32_t phase1 = 0, phase2 = 0, phasew = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
      const int pt = phys_tile<LIST>(a.tile_list, tile);  // emission tile of this training tile
      const int rbt = rbt_cur;
      const bool valid = rbt >= 0;
      const RowIn cx = nx;
      rbt_cur = rbt_next;
      rbt_next = slot_of(tile + 2 * gridDim.x);
      load_row(tile + gridDim.x, rbt_cur, nx);  // in flight during this tile
      pmark(6);
      // the previous tile's dW1 MMA groups may still run: htile is rewritten (dlogits) after the
      // first group's mbarrier, the W2 window after the second's; atile only after this tile's
      // head MMA, whose commit covers every earlier MMA
      const bool prev_w1 = w1_pending;
      w1_pending = false;
      uint32_t mk2[HC / 32], mk1[HC / 32];
#pragma unroll
      for (int q = 0; q < HC / 32; ++q) {
        mk2[q] = cx.mk2[q];
        mk1[q] = cx.mk1[q];
      }
      const uint32_t mk1x = cx.mk1x;
      if (half == 0) {
        // dlogits (masked log-softmax backward, tape.cpp:413-434): g_c - p_c * sum(g)
        typename Env::State s;
        Env::reset(P, s);
        if (valid) Env::unpack(P, cx.sw, s);
        const int act = cx.act;
        const float g_a = cx.ga, g_s = cx.gs, g_f = cx.gf;
        const float gsum = g_a + g_s;
        const float* pr = cx.pr;
        // only the NH head columns are written: the head dgrad MMA reads K = NH, and the
        // wgrad pass C output columns >= NH (from stale smem) are never read back
        uint32_t pk[NH / 2];
#pragma unroll
        for (int i = 0; i < NH / 2; ++i) {
          float x[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int c = 2 * i + e;
            float v = 0.f;
            if (valid && c < A && Env::legal(P, s, c)) {
              v = -pr[c] * gsum;
              if (c == act) v += g_a;
              if (c == P.stop) v += g_s;
            }
            if (c == A) v = g_f;
            x[e] = v;
          }
          pk[i] = pack_bf16x2(x[0], x[1]);
        }
        // htile is free once the previous tile's first dW1 MMA group has read its obs unit
        if (prev_w1) mbar_wait(&mbar1, phase1);
#pragma unroll
        for (int c8 = 0; c8 < NH / 8; ++c8)
          *reinterpret_cast<uint4*>(htile + sw128_offset(row, 8 * c8, kTile)) =
              make_uint4(pk[4 * c8], pk[4 * c8 + 1], pk[4 * c8 + 2], pk[4 * c8 + 3]);
      }
      if (prev_w1) {
        phase1 ^= 1;
        w2_patch = true;
      }
      fence_proxy_async();
      tc_fence_before();
      __syncthreads();
      pmark(0);
      if (tid == 0) {  // dh2 = dhead Wf^T (+ dflow wfl^T): 128 x H x NH on the tensor cores
        tc_fence_after();
        bulk_s2g(a.dhead + (size_t)pt * kTile * 64, htile, kTile * 64 * 2);
        bulk_commit();
        mma_k_sw128_none<H, NH>(tmem, htile, whd);
        umma_commit(&mbar);
        if (prev_w1) {  // restore the W2 image's first 16 KB once the second dW1 group has read it
          mbar_wait(&mbar2, phase2);
          mbar_arrive_expect_tx(&mbarw, 16384);
          bulk_g2s(wdimg, a.W.w2_dgrad, 16384, &mbarw);
        }
      }
      if (prev_w1) phase2 ^= 1;
      mbar_wait(&mbar, phase);
      phase ^= 1;
      tc_fence_after();
      __syncthreads();
      pmark(1);
#pragma unroll
      for (int q = 0; q < HC / 32; ++q) {
        const int col = c0 + q * 32;
        uint32_t r32[32];
        tmem_ld32(lane_base + col, r32);
        tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          pk[i] = pack_bf16x2(((mk2[q] >> i) & 1u) ? __uint_as_float(r32[2 * i]) : 0.f,
                              ((mk2[q] >> (16 + i)) & 1u) ? __uint_as_float(r32[2 * i + 1]) : 0.f);
        st_row32(atile, row, col, pk);
      }
      fence_proxy_async();
      tc_fence_before();
      __syncthreads();
      pmark(2);
      if (tid == 0) {
        tc_fence_after();
        bulk_s2g(a.dz2 + (size_t)pt * kTile * H, atile, kTile * H * 2);
        bulk_commit();
        if (w2_patch) {
          mbar_wait(&mbarw, phasew);
          phasew ^= 1;
        }
        mma_kk<H, H>(tmem, atile, wdimg, false);  // dh1 = dz2 W2^T
        umma_commit(&mbar);
      }
      // db2 of this tile (deterministic, overlaps the MMA): thread = (row group, 8 columns)
      // sums its rows with 16-byte loads, then a fixed-order sum over the row groups
      {
        constexpr int CG = H / 8, RG = kThreads / CG, RPG = kTile / RG;
        const int cg = tid % CG, rg = tid / CG;
        float sv[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
        for (int i = 0; i < RPG; ++i) {
          const uint4 q = *reinterpret_cast<const uint4*>(atile + sw128_offset(rg * RPG + i, 8 * cg, kTile));
          const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            sv[2 * e] += bf16_lo(w[e]);
            sv[2 * e + 1] += bf16_hi(w[e]);
          }
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) red[rg * H + 8 * cg + e] = sv[e];
        // head bias: thread = (16-row group, head column), fixed order
        constexpr int HG = kThreads / NH, HR = kTile / HG;
        const int hc = tid % NH, hg = tid / NH;
        float hs = 0.f;
#pragma unroll
        for (int i = 0; i < HR; ++i)
          hs += __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(htile + sw128_offset(hg * HR + i, hc, kTile)));
        redh[hg * NH + hc] = hs;
        __syncthreads();
        if (tid < H) {
          float t = 0.f;
#pragma unroll
          for (int g = 0; g < RG; ++g) t += red[g * H + tid];
          acc_b2 += t;
        }
        if (tid <= A) {
          float t = 0.f;
#pragma unroll
          for (int g = 0; g < HG; ++g) t += redh[g * NH + tid];
          acc_bh += t;
        }
      }
      mbar_wait(&mbar, phase);
      phase ^= 1;
      tc_fence_after();
      if (tid == 0) bulk_wait_read0();
      __syncthreads();
      pmark(3);
      // dz1 = dh1 masked by ReLU(h1) -> atile: half 0 takes one 32-column chunk fewer than
      // half 1 (it also builds the obs rows)
      auto dz1_chunk = [&](int col, uint32_t mw) {
        uint32_t r32[32];
        tmem_ld32(lane_base + col, r32);
        tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          pk[i] = pack_bf16x2(((mw >> i) & 1u) ? __uint_as_float(r32[2 * i]) : 0.f,
                              ((mw >> (16 + i)) & 1u) ? __uint_as_float(r32[2 * i + 1]) : 0.f);
        st_row32(atile, row, col, pk);
      };
      if (half == 0) {
#pragma unroll
        for (int q = 0; q < HC / 32 - 1; ++q) dz1_chunk(q * 32, mk1[q]);
      } else {
        dz1_chunk(HC - 32, mk1x);
#pragma unroll
        for (int q = 0; q < HC / 32; ++q) dz1_chunk(HC + q * 32, mk1[q]);
      }
      // obs units: rows 0..63 in htile, rows 64..127 in the W2 image's first 16 KB (its W2
      // MMA has completed)
      if (half == 0) build_obs_row(quarter < 2 ? htile : wdimg, row & 63, valid, cx.sw);
      tc_fence_before();
      fence_proxy_async();
      __syncthreads();
      if (tid == 0) {  // [dW1 | db1] += [obs | 1]^T dz1; completion waited before htile / the
                       // W2 image / atile are rewritten
        tc_fence_after();
        mma_obs_dz<H>(tmem + H, htile, atile, 0, w1_acc);
        umma_commit(&mbar1);  // htile free (the next tile's dlogits wait on it)
        mma_obs_dz<H>(tmem + H, wdimg, atile, 1, true);
        umma_commit(&mbar2);  // W2 window free (and every earlier MMA complete)
      }
      w1_pending = true;
      w1_acc = true;
      pmark(4);
      pc[5] += 1;
    }
    if (a.phase && tid == 0)
      for (int k = 0; k < 7; ++k) atomicAdd((unsigned long long*)a.phase + 15 + k, (unsigned long long)pc[k]);
    if (w1_pending) mbar_wait(&mbar2, phase2);  // covers both dW1 groups
    tc_fence_after();
    // [dW1 | db1] of this CTA -> its partial slab: TMEM lane = input feature f (<= O), the two
    // halves read their column halves
#pragma unroll 1
    for (int q = 0; q < HC / 32; ++q) {
      const int col = c0 + q * 32;
      uint32_t r32[32];
      tmem_ld32(lane_base + H + col, r32);
      tmem_wait_ld();
      if (row <= P.O) {
        float* dst = row < P.O ? part + a.L.off_w[0] + (size_t)row * H + col : part + a.L.off_b[0] + col;
#pragma unroll
        for (int i = 0; i < 32; i += 8) st_v8(dst + i, r32 + i, true);
      }
    }
    if (tid == 0) bulk_wait0();
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<2 * H>(tmem);
  } else {  // no tile: zero [dW1 | db1] partials
    for (int i = tid; i < (P.O + 1) * H; i += kThreads) {
      const int f = i / H, j = i % H;
      part[f < P.O ? a.L.off_w[0] + (size_t)f * H + j : a.L.off_b[0] + j] = 0.f;
    }
  }
  // bias partials of this CTA (every CTA writes its slots, zeros when it had no tile)
  if (tid < H) part[a.L.off_b[1] + tid] = acc_b2;
  if (tid < A) part[a.L.off_fb + tid] = acc_bh;
  if (tid == A) part[a.L.off_flb] = acc_bh;
}

// ---------------------------------------------------------------------------
// k_fast_wgrad: dW2 = h1^T dz2, dWhead = h2^T dhead (K = rows; [dW1 | db1] is k_fast_bwd's)
//
// The activation tile images are streamed as 64-row units through a 3-stage ring of
// shared-memory stages (bulk copies on mbarriers, "full"), consumed by tcgen05.mma with
// MN-major descriptors (LBO = 64 rows x 128 B between 64-feature blocks), and released by
// the MMA's commit ("empty"): the loads of unit q + 2 are in flight while unit q multiplies.
// One sequence runs through the two passes (A: h1/dz2, C: h2/dhead); TMEM holds one pass's
// accumulators, read back into the CTA's partial slab between passes.
constexpr int kWgStages = 3;
constexpr int kWgRows = 64;           // rows per unit
constexpr int kWgStage = 65536;       // X operand [0, 32 KB), Y operand [32 KB, 64 KB)

template <int H>
constexpr int wgrad_smem_bytes() {
  return kWgStages * kWgStage + 1024;
}

// D[128 x N] (+)= X'^T Y' over one 64-row unit: X' = features [m0, m0 + 128) of X, Y' = N
// features of Y, both MN-major with 64-feature blocks of 64 rows x 128 B.
template <int N>
GFNX_DEV void mma_mn64(uint32_t d_tmem, const void* x_img, int m0, const void* y_img, bool acc) {
  constexpr uint32_t idesc = umma_idesc_bf16(128, N, true, true);
  constexpr uint32_t LBO = kWgRows * 128;
  const uint32_t x0 = smem_u32(x_img) + (m0 >> 6) * LBO, y0 = smem_u32(y_img);
#pragma unroll
  for (int s = 0; s < kWgRows / 16; ++s)
    umma_bf16(d_tmem, umma_desc_sw128(x0 + s * 2048, LBO, 1024), umma_desc_sw128(y0 + s * 2048, LBO, 1024),
              idesc, (acc || s > 0) ? 1u : 0u);
}

template <class Env, int H, bool LIST>
__global__ void __launch_bounds__(kTile, 1) k_fast_wgrad(TrainArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* ring = align1024(smem_raw);
  __shared__ uint64_t full[kWgStages], empty[kWgStages];
  __shared__ uint32_t tbase;
  const EnvParams& P = a.P;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int A = P.A;
  const int tiles = *a.tilectr;
  const int R = tiles * kTile;
  const int per = (tiles + gridDim.x - 1) / gridDim.x;
  const int t0 = blockIdx.x * per, t1 = min(tiles, t0 + per);
  const int nu = t1 > t0 ? 2 * (t1 - t0) : 0;  // units per pass
  const int NQ = 2 * nu;
  float* part = a.wpart + (size_t)blockIdx.x * a.pstride;
  const MlpLayout& L = a.L;
  constexpr int KH = H / 128;  // 128-feature M blocks of the h operands
  if (warp == 0) tmem_alloc<512>(&tbase);
  if (tid == 0) {
    for (int i = 0; i < kWgStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
  auto X = [&](int st) { return ring + st * kWgStage; };
  auto Y = [&](int st) { return ring + st * kWgStage + 32768; };
  auto src = [&](const void* img, int u, int blk, int width) {  // 64-row unit u, 64-feature block blk
    const int tile = phys_tile<LIST>(a.tile_list, t0 + (u >> 1)), hh = u & 1;
    return reinterpret_cast<const uint8_t*>(img) + (size_t)tile * kTile * width * 2 + blk * (kTile * 128) +
           hh * (kWgRows * 128);
  };
  auto issue_load = [&](int q) {  // thread 0
    const int st = q % kWgStages, p = 2 * (q / nu), u = q % nu;
    if (q >= kWgStages) mbar_wait(&empty[st], ((q / kWgStages) - 1) & 1);
    constexpr uint32_t ub = kWgRows * 128;  // one 64-feature block of a unit
    if (p == 0) {
      mbar_arrive_expect_tx(&full[st], 2 * (H / 64) * ub);
      for (int k = 0; k < H / 64; ++k) {
        bulk_g2s(X(st) + k * ub, src(a.h1, u, k, H), ub, &full[st]);
        bulk_g2s(Y(st) + k * ub, src(a.dz2, u, k, H), ub, &full[st]);
      }
    } else {
      mbar_arrive_expect_tx(&full[st], (H / 64) * ub + ub);
      for (int k = 0; k < H / 64; ++k) bulk_g2s(X(st) + k * ub, src(a.h2, u, k, H), ub, &full[st]);
      bulk_g2s(Y(st), src(a.dhead, u, 0, 64), ub, &full[st]);
    }
  };
  // TMEM accumulators of pass p -> this CTA's partial slab (zeros when it had no rows)
  auto readout = [&](int p) {
    const bool any = nu > 0;
    if (p == 0) {
      for (int h = 0; h < KH; ++h) {
        const int pr = 128 * h + tid;  // input feature of layer 2
        for (int q = 0; q < H / 32; ++q) {
          uint32_t r32[32];
          tmem_ld32(lane_base + h * H + q * 32, r32);
          tmem_wait_ld();
          float* dst = part + L.off_w[1] + (size_t)pr * H + q * 32;
#pragma unroll
          for (int i = 0; i < 32; i += 8) st_v8(dst + i, r32 + i, any);
        }
      }
    } else {
      for (int h = 0; h < KH; ++h) {
        const int pr = 128 * h + tid;
        for (int q = 0; q < 2; ++q) {
          uint32_t r32[32];
          tmem_ld32(lane_base + h * 64 + q * 32, r32);
          tmem_wait_ld();
          for (int i = 0; i < 32; ++i) {
            const int c = q * 32 + i;
            const float v = any ? __uint_as_float(r32[i]) : 0.f;
            if (c < A) part[L.off_fw + (size_t)pr * A + c] = v;
            else if (c == A) part[L.off_flw + pr] = v;
          }
        }
      }
    }
  };
  long long tclk = clock64();
  auto pclock = [&](int k) {
    if (a.phase && tid == 0) {
      const long long t = clock64();
      atomicAdd((unsigned long long*)a.phase + 9 + k, (unsigned long long)(t - tclk));
      tclk = t;
    }
  };
  if (tid == 0)
    for (int q = 0; q < kWgStages - 1 && q < NQ; ++q) issue_load(q);
  for (int q = 0; q < NQ; ++q) {
    const int st = q % kWgStages, p = 2 * (q / nu), u = q % nu;
    if (u == 0 && q > 0) {  // pass boundary: accumulators of pass A -> slab
      pclock(0);
      if (tid == 0) mbar_wait(&empty[(q - 1) % kWgStages], ((q - 1) / kWgStages) & 1);
      __syncthreads();
      tc_fence_after();
      readout(0);
      tc_fence_before();
      __syncthreads();
    }
    if (tid == 0) {
      mbar_wait(&full[st], (q / kWgStages) & 1);
      tc_fence_after();
      if (p == 0) {
#pragma unroll
        for (int h = 0; h < KH; ++h) mma_mn64<H>(tmem + h * H, X(st), 128 * h, Y(st), u > 0);
      } else {
#pragma unroll
        for (int h = 0; h < KH; ++h) mma_mn64<64>(tmem + h * 64, X(st), 128 * h, Y(st), u > 0);
      }
      umma_commit(&empty[st]);
      if (q + kWgStages - 1 < NQ) issue_load(q + kWgStages - 1);
    }
  }
  if (NQ > 0 && tid == 0) mbar_wait(&empty[(NQ - 1) % kWgStages], ((NQ - 1) / kWgStages) & 1);
  pclock(2);
  __syncthreads();
  tc_fence_after();
  if (NQ == 0) readout(0);
  readout(2);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

// fixed-order reduction over CTAs (deterministic)
// block = 32 consecutive parameters x 8 partial groups: warp q sums partial slabs q, q + 8, ...
// (four loads in flight, coalesced across the 32 parameters), then a fixed-order sum of the
// 8 group totals (deterministic); the short per-thread chains keep the loads latency-hidden
constexpr int kRedE = 32, kRedG = 8;
__global__ void __launch_bounds__(kRedE * kRedG) k_reduce(const float* __restrict__ wpart, int nparts, int64_t n,
                                                          int64_t stride, float* g) {
  __shared__ float sg[kRedG][kRedE];
  const int el = threadIdx.x % kRedE, grp = threadIdx.x / kRedE;
  const int64_t e = (int64_t)blockIdx.x * kRedE + el;
  float s4[4] = {0.f, 0.f, 0.f, 0.f};
  if (e < n) {
    int c = grp;
    for (; c + 3 * kRedG < nparts; c += 4 * kRedG) {
#pragma unroll
      for (int k = 0; k < 4; ++k) s4[k] += wpart[(size_t)(c + k * kRedG) * stride + e];
    }
    for (; c < nparts; c += kRedG) s4[0] += wpart[(size_t)c * stride + e];
  }
  sg[grp][el] = (s4[0] + s4[1]) + (s4[2] + s4[3]);
  __syncthreads();
  if (grp == 0 && e < n) {
    float t = 0.f;
#pragma unroll
    for (int q = 0; q < kRedG; ++q) t += sg[q][el];
    g[e] = t;
  }
}

// ---------------------------------------------------------------------------
// Adam (optim.cpp:19-43) over fp32 params + bf16 operand images; logZ (TB) on thread 0

struct AdamArgs {
  float *p, *m, *v;
  const float* g;
  int64_t n;
  float lr, b1, b2, eps, wd;
  double beta1, beta2;      // bias corrections 1 - beta^t in fp64 (std::pow, optim.cpp:27-28)
  double* scalars;
  int do_z;
  double z_lr, zeps;
  // device-owned step counters [adam_t, z_t, ticket]: a step is taken and counted only when
  // the iteration's error word is clear, so a failed batch never reaches the parameters
  // (the reference throws before adam_step, train.cpp:174-183)
  int64_t* steps;
  const int32_t* err;
  MlpLayout L;
  __nv_bfloat16 *w1, *w2f, *w2d, *whf, *whd;
  int H, O, A, NH;
};

__device__ __forceinline__ void emit_images(const AdamArgs& a, int64_t j, float pj) {
  const MlpLayout& L = a.L;
  if (!a.w1) return;  // env paths that emit their own images (lockstep.cu)
  if (j < L.off_b[0]) {  // W1 [O][H] row-major bf16
    a.w1[j] = __float2bfloat16(pj);
  } else if (j >= L.off_w[1] && j < L.off_b[1]) {  // W2 [in p][out q]
    const int64_t k = j - L.off_w[1];
    const int p = (int)(k / a.H), q = (int)(k % a.H);
    const __nv_bfloat16 v = __float2bfloat16(pj);
    *reinterpret_cast<__nv_bfloat16*>((uint8_t*)a.w2f + sw128_offset(q, p, a.H)) = v;
    *reinterpret_cast<__nv_bfloat16*>((uint8_t*)a.w2d + sw128_offset(p, q, a.H)) = v;
  } else if ((j >= L.off_fw && j < L.off_fb) || (j >= L.off_flw && j < L.off_flb)) {
    // head weights: Wf [H p][A c] and the flow column (c = A) into both head images
    int p, c;
    if (j < L.off_fb) {
      p = (int)((j - L.off_fw) / a.A);
      c = (int)((j - L.off_fw) % a.A);
    } else {
      p = (int)(j - L.off_flw);
      c = a.A;
    }
    const __nv_bfloat16 v = __float2bfloat16(pj);
    *reinterpret_cast<__nv_bfloat16*>((uint8_t*)a.whf + sw128_offset(c, p, a.NH)) = v;
    *reinterpret_cast<__nv_bfloat16*>((uint8_t*)a.whd + nsw_offset(p, c, a.NH)) = v;
  }
}

__global__ void k_fast_adam(AdamArgs a) {
  __shared__ int skip;
  __shared__ float bc[2];
  __shared__ double zbc[2];
  if (threadIdx.x == 0) {
    skip = *a.err != 0;
    const double t = (double)(a.steps[0] + 1), zt = (double)(a.steps[1] + 1);
    bc[0] = (float)(1.0 - pow(a.beta1, t));
    bc[1] = (float)(1.0 - pow(a.beta2, t));
    zbc[0] = 1.0 - pow(a.beta1, zt);
    zbc[1] = 1.0 - pow(a.beta2, zt);
  }
  __syncthreads();
  if (skip) return;
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < a.n) {
    const float gj = a.g[j];
    const float m = a.b1 * a.m[j] + (1.f - a.b1) * gj;
    const float v = a.b2 * a.v[j] + (1.f - a.b2) * gj * gj;
    a.m[j] = m;
    a.v[j] = v;
    const float mhat = m / bc[0], vhat = v / bc[1];
    const float pj = a.p[j] - a.lr * (mhat / (sqrtf(vhat) + a.eps) + a.wd * a.p[j]);
    a.p[j] = pj;
    emit_images(a, j, pj);
  }
  if (a.do_z && j == 0) {  // logZ keeps fp64 state (train.cpp:186-190)
    const double gj = a.scalars[3];
    a.scalars[1] = a.beta1 * a.scalars[1] + (1.0 - a.beta1) * gj;
    a.scalars[2] = a.beta2 * a.scalars[2] + (1.0 - a.beta2) * gj * gj;
    const double mhat = a.scalars[1] / zbc[0], vhat = a.scalars[2] / zbc[1];
    a.scalars[0] -= a.z_lr * (mhat / (sqrt(vhat) + a.zeps));
  }
  adam_commit(a.steps, a.do_z);
}

__global__ void k_emit_images(AdamArgs a) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < a.n) emit_images(a, j, a.p[j]);
}

AdamArgs adam_args(Ctx& c) {
  FastState& f = FS(c);
  AdamArgs a{};
  a.p = c.p32;
  a.m = c.m32;
  a.v = c.v32;
  a.g = c.g32;
  a.n = c.L.n_params;
  a.L = c.L;
  a.w1 = f.w1;
  a.w2f = f.w2_fwd;
  a.w2d = f.w2_dgrad;
  a.whf = f.whead_f;
  a.whd = f.whead_d;
  a.H = f.H;
  a.O = f.O;
  a.A = f.A;
  a.NH = f.NH;
  a.scalars = c.d_scalars;
  return a;
}

// exact terminal marginal of the policy on the hypergrid (exact.hpp:76-113 restated for the
// grid DAG): states in level order (level = sum of coordinates); P(s) = sum over the
// parents s - e_i of P(s - e_i) pi(i | s - e_i) (a fixed-order gather, no atomics),
// P_T(s) = P(s) pi(stop | s)
__global__ void k_hg_marginal_level(int r0, int r1, const int32_t* __restrict__ parents, int dim,
                                    const float* __restrict__ probs, int rs, int stop, double* P, double* PT) {
  const int r = r0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= r1) return;
  double p = r == 0 ? 1.0 : 0.0;
  for (int i = 0; i < dim; ++i) {
    const int q = parents[(size_t)r * dim + i];
    if (q >= 0) p += P[q] * (double)probs[(size_t)q * rs + i];
  }
  P[r] = p;
  PT[r] = p * (double)probs[(size_t)r * rs + stop];
}

// the deterministic / work-stealing instantiation of a rollout kernel
template <void (*KD)(RolloutArgs), void (*KN)(RolloutArgs)>
void launch_det(const RolloutArgs& a, int grid, int smem, cudaStream_t st) {
  if (a.det) {
    set_smem_once(KD, smem);
    KD<<<grid, kThreads, smem, st>>>(a);
  } else {
    set_smem_once(KN, smem);
    KN<<<grid, kThreads, smem, st>>>(a);
  }
}

template <class Env, int H, int NH>
struct Kernels {
  static void rollout(Ctx& c, Key key, double eps) {
    FastState& f = FS(c);
    RolloutArgs a{};
    a.P = c.P;
    a.W = weights_of(c);
    a.key = key;
    a.eps = eps;
    a.b0 = c.b0;
    a.Bl = c.Bl;
    a.batch = c.batch;
    a.stst = f.stst;
    a.work = f.work;
    a.phase = c.phase;
    a.h1 = f.h1;
    a.h2 = f.h2;
    a.mask1 = f.mask1;
    a.mask2 = f.mask2;
    a.rowbuf = f.rowbuf;
    a.rs = f.rs;
    a.flow = c.train.objective == GFNX_OBJ_DB || c.train.objective == GFNX_OBJ_SUBTB;
    a.frow_bt = f.frow_bt;
    a.bt_row = f.bt_row;
    a.slot_st = f.slot_st;
    a.slot_act = f.slot_act;
    a.tilectr = f.tilectr;
    a.logits = f.logits;
    a.det = c.train.deterministic ? 1 : 0;
    // counters only: the per-step arrays beyond each trajectory's length are never read on
    // the device (gfnx_export_batch pads them from the lengths)
    k_rollout_reset<<<1, 32, 0, c.stream>>>(f.tilectr, c.batch.counters, f.work);
    c.launches++;
    const int grid = std::min(f.num_sms, (c.Bl + kTile - 1) / kTile);
    if (a.det) {  // static ranges and regions (fast_init sized the slots for grid * mt tiles)
      a.per = f.det_per;
      a.mt = f.det_mt;
      a.det_used = f.det_used;
      if (grid != f.det_grid) raise_error(GFNX_ERR_CONFIG, "deterministic rollout: grid mismatch");
    }
    const int fixed = rollout_smem_fixed<H, NH>();
    const int w1b = c.P.O * H * 2;
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, k_fast_rollout<Env, H, NH, true, false>);
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c.device);
    ProfScope ps(c, "k_fast_rollout");
    if constexpr (H == 256) {
      const int tsb = rollout_ts_smem_bytes<H, NH>();
      cudaFuncAttributes ft{};
      cudaFuncGetAttributes(&ft, k_fast_rollout_ts<Env, H, NH, NH, false>);
      if (tsb + (int)ft.sharedSizeBytes <= optin) {
        if (c.P.A <= 8) {
          launch_det<k_fast_rollout_ts<Env, H, NH, 8, true>, k_fast_rollout_ts<Env, H, NH, 8, false>>(
              a, grid, tsb, c.stream);
        } else {
          launch_det<k_fast_rollout_ts<Env, H, NH, NH, true>, k_fast_rollout_ts<Env, H, NH, NH, false>>(
              a, grid, tsb, c.stream);
        }
        c.launches++;
        f.fused = true;
        det_list(c, grid);
        return;
      }
    }
    if (fixed + w1b + (int)fa.sharedSizeBytes <= optin) {  // W1 resident in smem
      launch_det<k_fast_rollout<Env, H, NH, true, true>, k_fast_rollout<Env, H, NH, true, false>>(a, grid, fixed + w1b,
                                                                                               c.stream);
    } else {
      launch_det<k_fast_rollout<Env, H, NH, false, true>, k_fast_rollout<Env, H, NH, false, false>>(a, grid, fixed,
                                                                                                 c.stream);
    }
    c.launches++;
    f.fused = true;
    det_list(c, grid);
  }
  static void det_list(Ctx& c, int grid) {
    FastState& f = FS(c);
    if (!c.train.deterministic) return;
    k_det_tiles<<<1, 256, 0, c.stream>>>(f.det_used, grid, f.det_mt, f.tile_list, f.tilectr);
    c.launches++;
  }
  // policy forward (masked softmax record) over `n` explicit packed states (eval buffers)
  static void eval_forward(Ctx& c, const uint32_t* stst, const int32_t* rows, const int32_t* tiles,
                           const int16_t* acts, __nv_bfloat16* h1, __nv_bfloat16* h2, uint32_t* m1,
                           uint32_t* m2, float* rowbuf) {
    FastState& f = FS(c);
    TrainArgs ta{};
    ta.P = c.P;
    ta.W = weights_of(c);
    ta.batch = c.batch;
    ta.batch.actions = const_cast<int16_t*>(acts);
    ta.Bl = c.Bl;
    ta.stst = stst;
    ta.frow_bt = rows;
    ta.tilectr = tiles;
    ta.h1 = h1;
    ta.h2 = h2;
    ta.mask1 = m1;
    ta.mask2 = m2;
    ta.rowbuf = rowbuf;
    ta.rs = f.rs;
    ta.L = c.L;
    ta.objective = c.train.objective;
    const int fixed = fwd_smem_fixed<H, NH>();
    const int w1b = c.P.O * H * 2;
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, k_fast_fwd<Env, H, NH, true>);
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c.device);
    if (fixed + w1b + (int)fa.sharedSizeBytes <= optin && c.P.SW <= kMaxSWFwd) {
      set_smem_once(k_fast_fwd<Env, H, NH, true>, fixed + w1b);
      k_fast_fwd<Env, H, NH, true><<<f.num_sms, kThreads, fixed + w1b, c.stream>>>(ta);
    } else {
      set_smem_once(k_fast_fwd<Env, H, NH, false>, fixed);
      k_fast_fwd<Env, H, NH, false><<<f.num_sms, kThreads, fixed, c.stream>>>(ta);
    }
    c.launches++;
  }
  static void train(Ctx& c, bool apply, double lr) {
    FastState& f = FS(c);
    TrainArgs ta{};
    ta.P = c.P;
    ta.W = weights_of(c);
    ta.batch = c.batch;
    ta.Bl = c.Bl;
    ta.stst = f.stst;
    ta.frow_bt = f.frow_bt;
    ta.tilectr = f.tilectr;
    ta.tile_list = (f.fused && c.train.deterministic) ? f.tile_list : nullptr;
    ta.h1 = f.h1;
    ta.h2 = f.h2;
    ta.dz2 = f.dz2;
    ta.dhead = f.dhead;
    ta.mask1 = f.mask1;
    ta.mask2 = f.mask2;
    ta.slot_st = f.slot_st;
    ta.slot_act = f.slot_act;
    ta.rowbuf = f.rowbuf;
    ta.rs = f.rs;
    ta.coef = f.coef;
    ta.wpart = f.wpart;
    ta.n_params = c.L.n_params;
    ta.pstride = (c.L.n_params + 7) & ~(int64_t)7;
    ta.L = c.L;
    ta.objective = c.train.objective;
    ta.phase = c.phase;
    // CTAs of the training kernels: one per SM, but never more than the row tiles can
    // occupy (emission tiles <= Bl*T/128 + 2 per rollout CTA); small batches (config #1,
    // B = 16) then write and reduce only a few partial gradient slabs
    const int64_t tiles_max = ((int64_t)c.Bl * c.P.T + kTile - 1) / kTile +
                              2 * std::min(f.num_sms, (c.Bl + kTile - 1) / kTile);
    const int grid = (int)std::min<int64_t>(f.num_sms, tiles_max);
    if (!f.fused) {  // weights changed since the rollout: recompute the forward over the rows
      ensure_row0(c);
      k_linear_rows<<<(std::max(c.Bl, kTile) + 255) / 256, 256, 0, c.stream>>>(
          c.batch.lengths, c.batch.row0, c.Bl, c.P.T, c.batch.counters, f.frow_bt, f.bt_row, f.tilectr,
          f.stst, c.batch.actions, c.P.SW, f.slot_st, f.slot_act);
      c.launches++;
      const int fixed = fwd_smem_fixed<H, NH>();
      const int w1b = c.P.O * H * 2;
      cudaFuncAttributes fa{};
      cudaFuncGetAttributes(&fa, k_fast_fwd<Env, H, NH, true>);
      int optin = 0;
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c.device);
      ProfScope ps(c, "k_fast_fwd");
      if (fixed + w1b + (int)fa.sharedSizeBytes <= optin && c.P.SW <= kMaxSWFwd) {
        set_smem_once(k_fast_fwd<Env, H, NH, true>, fixed + w1b);
        k_fast_fwd<Env, H, NH, true><<<grid, kThreads, fixed + w1b, c.stream>>>(ta);
      } else {
        set_smem_once(k_fast_fwd<Env, H, NH, false>, fixed);
        k_fast_fwd<Env, H, NH, false><<<grid, kThreads, fixed, c.stream>>>(ta);
      }
      c.launches++;
    } else {
      ProfScope ps(c, "k_row_stats");
      const int nslots = (int)(f.max_tiles * kTile);
      k_row_stats<Env, NH><<<std::min((nslots + 255) / 256, f.num_sms * 32), 256, 0, c.stream>>>(
          c.P, f.slot_st, f.slot_act, f.frow_bt, f.tilectr, f.logits, f.rowbuf, f.rs,
          c.train.objective == GFNX_OBJ_DB || c.train.objective == GFNX_OBJ_SUBTB, c.batch.counters + 3,
          ta.tile_list);
      c.launches++;
    }
    LossArgs la{};
    la.batch = c.batch;
    la.Bl = c.Bl;
    la.T = c.P.T;
    la.A = c.P.A;
    la.stop = c.P.stop;
    la.objective = c.train.objective;
    la.B_global = c.B;
    la.terminal_penalty = c.train.terminal_penalty;
    la.lampow = f.lampow;
    la.neglog = c.d_neglog;
    la.rowbuf = f.rowbuf;
    la.rs = f.rs;
    la.bt_row = f.bt_row;
    la.coef = f.coef;
    la.lpart = f.lpart;
    la.scalars = c.d_scalars;
    {
      ProfScope ps(c, "k_fast_loss");
      if (c.train.objective == GFNX_OBJ_SUBTB) k_fast_loss_warp<true><<<f.loss_wblocks, 256, 0, c.stream>>>(la);
      else k_fast_loss_warp<false><<<f.loss_wblocks, 256, 0, c.stream>>>(la);
    }
    k_loss_finalize<<<1, 256, 0, c.stream>>>(f.lpart, f.loss_wblocks, c.d_scalars,
                                             c.train.objective == GFNX_OBJ_TB, c.batch.counters + 3);
    int smem = bwd_smem_bytes<H, NH>();
    const bool list = ta.tile_list != nullptr;
    if (list) set_smem_once(k_fast_bwd<Env, H, NH, true>, smem);
    else set_smem_once(k_fast_bwd<Env, H, NH, false>, smem);
    {
      ProfScope ps(c, "k_fast_bwd");
      if (list) k_fast_bwd<Env, H, NH, true><<<grid, kThreads, smem, c.stream>>>(ta);
      else k_fast_bwd<Env, H, NH, false><<<grid, kThreads, smem, c.stream>>>(ta);
    }
    const int64_t n = c.L.n_params;
    // world > 1: [dW1 | db1] (the parameters before W2) is final after k_fast_bwd — reduce it
    // and start its all-reduce on the comm stream while k_fast_wgrad runs
    const int64_t nA = c.world > 1 ? c.L.off_w[1] : 0;
    if (nA > 0) {
      ProfScope ps(c, "k_reduce");
      k_reduce<<<(unsigned)((nA + kRedE - 1) / kRedE), kRedE * kRedG, 0, c.stream>>>(f.wpart, grid, nA, ta.pstride,
                                                                                     c.g32);
      c.launches++;
      grad_bucket_async(c, c.g32, nA);
    }
    smem = wgrad_smem_bytes<H>();
    if (list) set_smem_once(k_fast_wgrad<Env, H, true>, smem);
    else set_smem_once(k_fast_wgrad<Env, H, false>, smem);
    {
      ProfScope ps(c, "k_fast_wgrad");
      if (list) k_fast_wgrad<Env, H, true><<<grid, kTile, smem, c.stream>>>(ta);
      else k_fast_wgrad<Env, H, false><<<grid, kTile, smem, c.stream>>>(ta);
    }
    {
      ProfScope ps(c, "k_reduce");
      k_reduce<<<(unsigned)((n - nA + kRedE - 1) / kRedE), kRedE * kRedG, 0, c.stream>>>(
          f.wpart + nA, grid, n - nA, ta.pstride, c.g32 + nA);
    }
    c.launches += 5;
    (void)apply;
    (void)lr;
  }
};



bool supported(const Ctx& c, int* H) {
  *H = c.L.H();
  if (c.L.n_trunk != 2) return false;
  if (c.L.dims[1] != c.L.dims[2]) return false;
  if (*H != 256 && *H != 128) return false;
  if (c.shape.num_actions + 1 > (c.env.kind == GFNX_ENV_HYPERGRID ? 16 : 32)) return false;
  if (c.shape.obs_dim >= 128) return false;  // feature obs_dim carries db1 in the bwd dW1 GEMM
  if (c.shape.max_traj_len > 128) return false;
  if (c.env.kind == GFNX_ENV_DAG) return *H == 128;
  return c.env.kind == GFNX_ENV_HYPERGRID;
}

template <class F>
void with_kernels(Ctx& c, F&& fn) {
  int H = 0;
  if (!supported(c, &H))
    raise_error(GFNX_ERR_CONFIG,
                "bf16 fast path supports 2-hidden-layer MLPs on hypergrid (widths <= 256) and DAG "
                "(widths <= 128); use precision=GFNX_PREC_FP64_CHECK for other configurations");
  if (c.env.kind == GFNX_ENV_HYPERGRID) {
    if (H == 256) fn(Kernels<HypergridEnv, 256, 16>{});
    else fn(Kernels<HypergridEnv, 128, 16>{});
  } else {
    fn(Kernels<DagEnv, 128, 32>{});
  }
}

bool lockstep(const Ctx& c) { return c.env.kind == GFNX_ENV_BITSEQ || c.env.kind == GFNX_ENV_ISING; }

// per-row log pi_F(a_t | s_t) of the training record, (b, t) order (0 past each end)
__global__ void k_fast_row_logpf(const int32_t* __restrict__ lengths, const int32_t* __restrict__ bt_row,
                                 const float* __restrict__ rowbuf, int rs, int A, int Bl, int T, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= Bl * T) return;
  const int b = i / T, t = i % T;
  out[i] = t < lengths[b] ? (double)rowbuf[(size_t)bt_row[i] * rs + A] : 0.0;
}

}  // namespace

void fast_row_logpf(Ctx& c, double* out) {
  if (lockstep(c)) {
    ls_row_logpf(c, out);
    return;
  }
  FastState& f = FS(c);
  const int n = c.Bl * c.P.T;
  k_fast_row_logpf<<<(n + 255) / 256, 256, 0, c.stream>>>(c.batch.lengths, f.bt_row, f.rowbuf, f.rs, c.P.A, c.Bl,
                                                          c.P.T, out);
  c.launches++;
}

bool fast_rollout_counts(const Ctx& c) { return !lockstep(c); }

void fast_hg_marginal(Ctx& c, std::vector<double>* pt) {
  if (c.env.kind != GFNX_ENV_HYPERGRID || lockstep(c))
    raise_error(GFNX_ERR_CONFIG, "exact terminal marginal: hypergrid fast path only");
  const int d = c.env.hg_dim, side = c.env.hg_side;
  int64_t n = 1;
  for (int i = 0; i < d; ++i) n *= side;
  if (n > (1 << 24)) raise_error(GFNX_ERR_CONFIG, "exact terminal marginal: grid too large");
  // cells in level order (sum of coordinates), packed states, parents per dimension
  std::vector<int64_t> cells(n);
  std::vector<int> lvl(n);
  for (int64_t x = 0; x < n; ++x) {
    int64_t y = x;
    int sum = 0;
    for (int i = 0; i < d; ++i) {
      sum += (int)(y % side);
      y /= side;
    }
    cells[x] = x;
    lvl[x] = sum;
  }
  std::stable_sort(cells.begin(), cells.end(), [&](int64_t a, int64_t b) { return lvl[a] < lvl[b]; });
  std::vector<int32_t> pos(n);
  for (int64_t r = 0; r < n; ++r) pos[cells[r]] = (int32_t)r;
  const int SW = c.P.SW;
  std::vector<uint32_t> st((size_t)n * SW, 0u);
  std::vector<int32_t> par((size_t)n * d, -1);
  std::vector<int> level_start;
  int64_t stride[8];
  stride[0] = 1;
  for (int i = 1; i < d; ++i) stride[i] = stride[i - 1] * side;
  for (int64_t r = 0; r < n; ++r) {
    const int64_t x = cells[r];
    uint64_t cw = 0;
    for (int i = 0; i < d; ++i) {
      const int ci = (int)((x / stride[i]) % side);
      cw |= (uint64_t)ci << (8 * i);
      if (ci > 0) par[(size_t)r * d + i] = pos[x - stride[i]];
    }
    st[(size_t)r * SW] = (uint32_t)cw;
    if (SW > 1) st[(size_t)r * SW + 1] = (uint32_t)(cw >> 32);
    if (r == 0 || lvl[cells[r]] != lvl[cells[r - 1]]) level_start.push_back((int)r);
  }
  level_start.push_back((int)n);
  FastState& f = FS(c);
  const int64_t tiles = (n + kTile - 1) / kTile, slots = tiles * kTile;
  std::vector<int32_t> rows(slots, -1);
  for (int64_t r = 0; r < n; ++r) rows[r] = (int32_t)r;
  const int32_t ntiles = (int32_t)tiles;
  uint32_t* d_st;
  int32_t *d_rows, *d_tiles, *d_par;
  int16_t* d_act;
  __nv_bfloat16 *d_h1, *d_h2;
  uint32_t *d_m1, *d_m2;
  float* d_rb;
  double *d_P, *d_PT;
  const int H = f.H;
  cuda_check(cudaMalloc(&d_st, sizeof(uint32_t) * st.size()), "eval");
  cuda_check(cudaMalloc(&d_rows, sizeof(int32_t) * slots), "eval");
  cuda_check(cudaMalloc(&d_tiles, sizeof(int32_t)), "eval");
  cuda_check(cudaMalloc(&d_par, sizeof(int32_t) * par.size()), "eval");
  cuda_check(cudaMalloc(&d_act, sizeof(int16_t) * n), "eval");
  cuda_check(cudaMalloc(&d_h1, sizeof(__nv_bfloat16) * slots * H), "eval");
  cuda_check(cudaMalloc(&d_h2, sizeof(__nv_bfloat16) * slots * H), "eval");
  cuda_check(cudaMalloc(&d_m1, sizeof(uint32_t) * slots * (H / 32)), "eval");
  cuda_check(cudaMalloc(&d_m2, sizeof(uint32_t) * slots * (H / 32)), "eval");
  cuda_check(cudaMalloc(&d_rb, sizeof(float) * slots * f.rs), "eval");
  cuda_check(cudaMalloc(&d_P, sizeof(double) * n), "eval");
  cuda_check(cudaMalloc(&d_PT, sizeof(double) * n), "eval");
  cudaMemcpyAsync(d_st, st.data(), sizeof(uint32_t) * st.size(), cudaMemcpyHostToDevice, c.stream);
  cudaMemcpyAsync(d_rows, rows.data(), sizeof(int32_t) * slots, cudaMemcpyHostToDevice, c.stream);
  cudaMemcpyAsync(d_tiles, &ntiles, sizeof(int32_t), cudaMemcpyHostToDevice, c.stream);
  cudaMemcpyAsync(d_par, par.data(), sizeof(int32_t) * par.size(), cudaMemcpyHostToDevice, c.stream);
  cudaMemsetAsync(d_act, 0, sizeof(int16_t) * n, c.stream);
  with_kernels(c, [&](auto k) {
    decltype(k)::eval_forward(c, d_st, d_rows, d_tiles, d_act, d_h1, d_h2, d_m1, d_m2, d_rb);
  });
  for (size_t l = 0; l + 1 < level_start.size(); ++l) {
    const int r0 = level_start[l], r1 = level_start[l + 1];
    k_hg_marginal_level<<<(r1 - r0 + 255) / 256, 256, 0, c.stream>>>(r0, r1, d_par, d, d_rb, f.rs, c.P.stop, d_P, d_PT);
  }
  c.launches += (int64_t)level_start.size() - 1;
  std::vector<double> ptr(n);
  cuda_check(cudaMemcpyAsync(ptr.data(), d_PT, sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream), "eval");
  cuda_check(cudaStreamSynchronize(c.stream), "eval");
  void* bufs[] = {d_st, d_rows, d_tiles, d_par, d_act, d_h1, d_h2, d_m1, d_m2, d_rb, d_P, d_PT};
  for (void* b : bufs) cudaFree(b);
  pt->assign(n, 0.0);
  for (int64_t r = 0; r < n; ++r) (*pt)[cells[r]] = ptr[r];  // back to row-major cell order
}

// mc_terminal_logprob (exact.hpp:229-241) on the fast path (hypergrid, DAG): the N = n K
// uniform backward walks run on the device (k_bwd_walk: the reference's Threefry draws,
// env_core.hpp:314-370), laid out as explicit state rows; ONE batched policy forward over
// every transition (the training-forward kernel on eval buffers) gives log pi(a|s); per walk
// log P_F - log P_B in forward order, then the per-terminal logsumexp (k_mc_terms_rows,
// k_mc_lse). The only host sync reads the row count to size the activation buffers.
void fast_mc_terminal_logprob(Ctx& c, const uint32_t* d_terms_in, int64_t n, int K, const uint64_t* d_keys,
                              double* d_out) {
  if ((c.env.kind != GFNX_ENV_HYPERGRID && c.env.kind != GFNX_ENV_DAG) || lockstep(c))
    raise_error(GFNX_ERR_CONFIG, "mc terminal log-prob (fast rows): hypergrid / DAG fast path only");
  const int64_t N = n * K;
  if (N > (1 << 24)) raise_error(GFNX_ERR_CONFIG, "mc terminal log-prob: too many walks");
  const int T = c.P.T, SW = c.P.SW;
  FastState& f = FS(c);
  int16_t* d_act;
  uint16_t* d_np;
  int32_t *d_len, *d_row0, *d_tiles, *d_rows;
  uint32_t* d_st;
  double* d_terms;
  auto alloc = [&](auto** p, size_t bytes) { cuda_check(cudaMallocAsync((void**)p, bytes, c.stream), "mc"); };
  alloc(&d_act, sizeof(int16_t) * N * T);
  alloc(&d_np, sizeof(uint16_t) * N * T);
  alloc(&d_len, sizeof(int32_t) * N);
  alloc(&d_row0, sizeof(int32_t) * (N + 1));
  alloc(&d_tiles, sizeof(int32_t));
  alloc(&d_st, sizeof(uint32_t) * N * T * SW);
  alloc(&d_terms, sizeof(double) * N);
  launch_bwd_walk(c, d_terms_in, (int)N, 0, N, K, d_keys, Key{0, 0}, 0, d_act, d_np, d_len, d_st);
  exclusive_scan_i32(c, d_len, d_row0, (int)N);
  int32_t R = 0;
  cuda_check(cudaMemcpyAsync(&R, d_row0 + N, sizeof R, cudaMemcpyDeviceToHost, c.stream), "mc");
  cuda_check(cudaStreamSynchronize(c.stream), "mc");
  const int64_t tiles = (R + kTile - 1) / kTile, slots = std::max<int64_t>(tiles, 1) * kTile;
  const int H = f.H;
  __nv_bfloat16 *d_h1, *d_h2;
  uint32_t *d_m1, *d_m2;
  float* d_rb;
  alloc(&d_rows, sizeof(int32_t) * slots);
  alloc(&d_h1, sizeof(__nv_bfloat16) * slots * H);
  alloc(&d_h2, sizeof(__nv_bfloat16) * slots * H);
  alloc(&d_m1, sizeof(uint32_t) * slots * (H / 32));
  alloc(&d_m2, sizeof(uint32_t) * slots * (H / 32));
  alloc(&d_rb, sizeof(float) * slots * f.rs);
  launch_walk_rows(c, d_len, d_row0, (int)N, d_rows, d_tiles, kTile);
  with_kernels(c, [&](auto kk) {
    decltype(kk)::eval_forward(c, d_st, d_rows, d_tiles, d_act, d_h1, d_h2, d_m1, d_m2, d_rb);
  });
  launch_mc_terms_rows(c, d_rb, f.rs, d_row0, d_np, d_len, (int)N, d_terms);
  launch_mc_lse(c, d_terms, (int)n, K, d_out);
  void* bufs[] = {d_act, d_np, d_len, d_row0, d_tiles, d_st, d_terms, d_rows, d_h1, d_h2, d_m1, d_m2, d_rb};
  for (void* p : bufs) cudaFreeAsync(p, c.stream);
}

// rollout_from_actions (env_core.hpp:166-229) into the resident batch: lockstep paths take
// the actions inside their rollout kernels; hypergrid / DAG replay the env (k_replay) and the
// training pass recomputes the forward over the rows (the weights did not produce them)
void fast_forced_rollout(Ctx& c, const int16_t* d_forced) {
  if (lockstep(c)) {
    ls_rollout(c, Key{0, 0}, 0.0, d_forced);
    return;
  }
  int H = 0;
  if (!supported(c, &H)) with_kernels(c, [](auto) {});  // raises config_error
  launch_replay(c, d_forced, FS(c).stst);
  FS(c).fused = false;
}

// ---------------------------------------------------------------------------
// tv_buffer (metrics.cpp:35-48 over the FifoBuffer of train.cpp:231, hypergrid)

// append terminal states b in [b_lo, Bl) of the resident batch at ring positions
// (head + b) % cap, evicting what those positions held (oldest-first, buffer.hpp:24-28); the
// positions of one push are distinct, the counts are integer atomics (order-independent)
__global__ void k_hg_buffer_push(const uint32_t* __restrict__ term, int SW, int dim, int side, int Bl, int b_lo,
                                 int64_t head, int64_t cap, int64_t size, int32_t* fifo, int32_t* hist) {
  const int b = b_lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= Bl) return;
  int64_t cell = 0, stride = 1;
  for (int i = 0; i < dim; ++i) {  // packed state: byte i = coordinate i
    cell += (int64_t)((term[(size_t)b * SW + (i >> 2)] >> (8 * (i & 3))) & 0xffu) * stride;
    stride *= side;
  }
  const int64_t pos = (head + b) % cap;
  if (size == cap || pos < size) atomicSub(hist + fifo[pos], 1);
  fifo[pos] = (int32_t)cell;
  atomicAdd(hist + cell, 1);
}

// tv_distance(empirical, exact) (metrics.cpp:35-48): 0.5 * (sum_x |phat_x - p_x| + 1 - covered),
// fixed-order block reduction in fp64
__global__ void __launch_bounds__(1024) k_hg_buffer_tv(const int32_t* __restrict__ hist, const double* __restrict__ p,
                                                       int64_t cells, int64_t size, double* out) {
  __shared__ double sa[1024], sc[1024];
  double acc = 0.0, cov = 0.0;
  for (int64_t x = threadIdx.x; x < cells; x += 1024) {
    const int h = hist[x];
    const double ph = h > 0 ? (double)h / (double)size : 0.0;
    if (h > 0) cov += ph;
    acc += fabs(ph - p[x]);
  }
  sa[threadIdx.x] = acc;
  sc[threadIdx.x] = cov;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) {
      sa[threadIdx.x] += sa[threadIdx.x + w];
      sc[threadIdx.x] += sc[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = 0.5 * (sa[0] + (1.0 - sc[0]));
}

void hg_buffer_free(Ctx& c) {
  Ctx::TermBuffer& t = c.tbuf;
  for (void* q : {(void*)t.fifo, (void*)t.hist, (void*)t.p, (void*)t.out})
    if (q) cudaFree(q);
  t = Ctx::TermBuffer{};
}

void hg_buffer_reset(Ctx& c, int64_t capacity) {
  if (c.env.kind != GFNX_ENV_HYPERGRID) raise_error(GFNX_ERR_CONFIG, "tv_buffer: hypergrid only");
  if (capacity < 1) raise_error(GFNX_ERR_CONFIG, "FifoBuffer: capacity must be >= 1");
  const int d = c.env.hg_dim, side = c.env.hg_side;
  int64_t cells = 1;
  for (int i = 0; i < d; ++i) cells *= side;
  if (cells > (1 << 26) || capacity > (int64_t)1 << 31) raise_error(GFNX_ERR_CONFIG, "tv_buffer: too large");
  hg_buffer_free(c);
  Ctx::TermBuffer& t = c.tbuf;
  t.cap = capacity;
  t.cells = cells;
  // grid_exact_distribution (hypergrid.cpp:121-140): exp(log reward) in the reference's
  // enumeration order (last coordinate fastest), normalised by their running sum
  std::vector<double> v(cells), p(cells);
  std::vector<int> co(d, 0);
  double z = 0.0;
  for (int64_t n = 0; n < cells; ++n) {
    uint32_t p1 = 1, p2 = 1;
    int64_t x = 0, st = 1;
    for (int i = 0; i < d; ++i) {
      p1 &= (c.P.hg_f1[co[i] >> 5] >> (co[i] & 31)) & 1u;
      p2 &= (c.P.hg_f2[co[i] >> 5] >> (co[i] & 31)) & 1u;
      x += co[i] * st;
      st *= side;
    }
    v[n] = exp(c.P.hg_logr[p1 | (p2 << 1)]);
    z += v[n];
    p[x] = v[n];
    for (int i = d - 1; i >= 0; --i) {
      if (++co[i] < side) break;
      co[i] = 0;
    }
  }
  for (double& q : p) q /= z;
  cuda_check(cudaMalloc(&t.fifo, sizeof(int32_t) * capacity), "tv_buffer");
  cuda_check(cudaMalloc(&t.hist, sizeof(int32_t) * cells), "tv_buffer");
  cuda_check(cudaMalloc(&t.p, sizeof(double) * cells), "tv_buffer");
  cuda_check(cudaMalloc(&t.out, sizeof(double)), "tv_buffer");
  cuda_check(cudaMemsetAsync(t.hist, 0, sizeof(int32_t) * cells, c.stream), "tv_buffer");
  cuda_check(cudaMemcpyAsync(t.p, p.data(), sizeof(double) * cells, cudaMemcpyHostToDevice, c.stream), "tv_buffer");
  cuda_check(cudaStreamSynchronize(c.stream), "tv_buffer");
}

void hg_buffer_push(Ctx& c) {
  Ctx::TermBuffer& t = c.tbuf;
  if (!t.fifo) raise_error(GFNX_ERR_CONTRACT, "tv_buffer: gfnx_buffer_reset first");
  if (!c.has_batch) raise_error(GFNX_ERR_CONTRACT, "tv_buffer: no resident batch");
  const int Bl = c.Bl;
  const int b_lo = (int64_t)Bl > t.cap ? Bl - (int)t.cap : 0;  // earlier items of the batch are overwritten
  k_hg_buffer_push<<<(Bl - b_lo + 255) / 256, 256, 0, c.stream>>>(c.batch.term_state, c.P.SW, c.env.hg_dim,
                                                                   c.env.hg_side, Bl, b_lo, t.head, t.cap, t.size,
                                                                   t.fifo, t.hist);
  c.launches++;
  cuda_check(cudaGetLastError(), "tv_buffer push");
  t.head = (t.head + Bl) % t.cap;
  t.size = std::min(t.cap, t.size + Bl);
}

double hg_buffer_tv(Ctx& c) {
  Ctx::TermBuffer& t = c.tbuf;
  if (!t.fifo) raise_error(GFNX_ERR_CONTRACT, "tv_buffer: gfnx_buffer_reset first");
  if (t.size == 0) raise_error(GFNX_ERR_CONTRACT, "FifoBuffer: empirical of empty buffer");
  k_hg_buffer_tv<<<1, 1024, 0, c.stream>>>(t.hist, t.p, t.cells, t.size, t.out);
  c.launches++;
  double tv = 0.0;
  cuda_check(cudaMemcpyAsync(&tv, t.out, sizeof(double), cudaMemcpyDeviceToHost, c.stream), "tv_buffer");
  cuda_check(cudaStreamSynchronize(c.stream), "tv_buffer");
  return tv;
}

void fast_init(Ctx& c) {
  if (lockstep(c)) {
    std::string why;
    if (!ls_supported(c, &why))
      raise_error(GFNX_ERR_CONFIG, why + "; use precision=GFNX_PREC_FP64_CHECK for this configuration");
    ls_init(c);
    return;
  }
  int H = 0;
  if (!supported(c, &H))
    raise_error(GFNX_ERR_CONFIG,
                "bf16 fast path supports 2-hidden-layer MLPs on hypergrid (widths <= 256) and DAG "
                "(widths <= 128); use precision=GFNX_PREC_FP64_CHECK for other configurations");
  auto* f = new FastState();
  c.fast = f;
  cudaDeviceGetAttribute(&f->num_sms, cudaDevAttrMultiProcessorCount, c.device);
  f->H = H;
  f->A = c.shape.num_actions;
  f->O = c.shape.obs_dim;
  const int T = c.P.T;
  f->max_rows = (int64_t)c.Bl * T;
  // + 2 tiles per rollout CTA: partially filled / pre-claimed emission tiles
  f->max_tiles = (f->max_rows + kTile - 1) / kTile + 2 * f->num_sms;
  if (c.train.deterministic) {  // static per-CTA regions: per trajectories of <= T rows each
    f->det_grid = std::min(f->num_sms, (c.Bl + kTile - 1) / kTile);
    f->det_per = (c.Bl + f->det_grid - 1) / f->det_grid;
    f->det_mt = (int)(((int64_t)f->det_per * T + kTile - 1) / kTile) + 2;
    f->max_tiles = std::max<int64_t>(f->max_tiles, (int64_t)f->det_grid * f->det_mt);
    cuda_check(cudaMalloc(&f->det_used, sizeof(int32_t) * f->det_grid), "fast det");
    cuda_check(cudaMalloc(&f->tile_list, sizeof(int32_t) * f->max_tiles), "fast det");
  }
  const int64_t slots = f->max_tiles * kTile;
  f->rs = (f->A + 3 + 3) & ~3;  // probs[A], lpa, lps, flow, padded to 16 bytes
  f->loss_blocks = (c.Bl + 255) / 256;
  f->loss_wblocks = (c.Bl + 7) / 8;
  const size_t img = (size_t)f->max_tiles * kTile * H * 2;
  cuda_check(cudaMalloc(&f->w1, sizeof(__nv_bfloat16) * (size_t)f->O * H), "fast w1");
  cuda_check(cudaMalloc(&f->w2_fwd, sizeof(__nv_bfloat16) * H * H), "fast w2");
  cuda_check(cudaMalloc(&f->w2_dgrad, sizeof(__nv_bfloat16) * H * H), "fast w2");
  f->NH = c.env.kind == GFNX_ENV_HYPERGRID ? 16 : 32;
  cuda_check(cudaMalloc(&f->whead_f, sizeof(__nv_bfloat16) * f->NH * H), "fast whead");
  cuda_check(cudaMalloc(&f->whead_d, sizeof(__nv_bfloat16) * f->NH * H), "fast whead");
  cuda_check(cudaMemset(f->whead_f, 0, sizeof(__nv_bfloat16) * f->NH * H), "fast whead");
  cuda_check(cudaMemset(f->whead_d, 0, sizeof(__nv_bfloat16) * f->NH * H), "fast whead");
  cuda_check(cudaMalloc(&f->stst, sizeof(uint32_t) * (size_t)c.Bl * T * c.P.SW), "fast stst");
  cuda_check(cudaMalloc(&f->h1, img), "fast h1");
  cuda_check(cudaMalloc(&f->h2, img), "fast h2");
  cuda_check(cudaMalloc(&f->dz2, img), "fast dz2");
  cuda_check(cudaMalloc(&f->dhead, (size_t)f->max_tiles * kTile * 64 * 2), "fast dhead");
  cuda_check(cudaMalloc(&f->mask1, sizeof(uint32_t) * (size_t)slots * (H / 32)), "fast masks");
  cuda_check(cudaMalloc(&f->mask2, sizeof(uint32_t) * (size_t)slots * (H / 32)), "fast masks");
  cuda_check(cudaMalloc(&f->rowbuf, sizeof(float) * (size_t)slots * f->rs), "fast rowbuf");
  cuda_check(cudaMalloc(&f->coef, sizeof(float) * (size_t)slots * 4), "fast coef");
  cuda_check(cudaMalloc(&f->frow_bt, sizeof(int32_t) * (size_t)slots), "fast rows");
  cuda_check(cudaMalloc(&f->slot_st, sizeof(uint32_t) * (size_t)slots * c.P.SW), "fast rows");
  cuda_check(cudaMalloc(&f->slot_act, sizeof(int16_t) * (size_t)slots), "fast rows");
  cuda_check(cudaMalloc(&f->bt_row, sizeof(int32_t) * (size_t)f->max_rows), "fast rows");
  cuda_check(cudaMalloc(&f->tilectr, sizeof(int32_t)), "fast rows");
  cuda_check(cudaMalloc(&f->logits, sizeof(float) * (size_t)slots * f->NH), "fast logits");
  cuda_check(cudaMemset(f->tilectr, 0, sizeof(int32_t)), "fast rows");
  const size_t pstride = (size_t)((c.L.n_params + 7) & ~(int64_t)7);
  cuda_check(cudaMalloc(&f->wpart, sizeof(float) * (size_t)f->num_sms * pstride), "fast wpart");
  cuda_check(cudaMemset(f->wpart, 0, sizeof(float) * (size_t)f->num_sms * pstride), "fast wpart");
  cuda_check(cudaMalloc(&f->lpart, sizeof(double) * 2 * std::max(f->loss_blocks, f->loss_wblocks)), "fast lpart");
  cuda_check(cudaMalloc(&f->work, sizeof(int32_t)), "fast work");
  std::vector<double> lp(T + 1);
  for (int k = 0; k <= T; ++k) lp[k] = pow(c.train.subtb_lambda, (double)k);
  cuda_check(cudaMalloc(&f->lampow, sizeof(double) * (T + 1)), "fast lampow");
  cuda_check(cudaMemcpy(f->lampow, lp.data(), sizeof(double) * (T + 1), cudaMemcpyHostToDevice), "lampow");
  fast_sync_weights(c);
}

void fast_free(Ctx& c) {
  if (lockstep(c)) {
    ls_free(c);
    return;
  }
  FastState* f = static_cast<FastState*>(c.fast);
  if (!f) return;
  void* ptrs[] = {f->w1, f->w2_fwd, f->w2_dgrad, f->whead_f, f->whead_d, f->stst, f->h1, f->h2, f->dz2, f->dhead,
                  f->mask1, f->mask2,
                  f->rowbuf, f->coef, f->wpart, f->lpart, f->lampow, f->work,
                  f->frow_bt, f->slot_st, f->slot_act, f->bt_row, f->tilectr, f->logits, f->det_used, f->tile_list};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete f;
  c.fast = nullptr;
}

void fast_sync_weights(Ctx& c) {
  if (lockstep(c)) {
    ls_sync_weights(c);
    return;
  }
  FS(c).fused = false;
  AdamArgs a = adam_args(c);
  k_emit_images<<<(unsigned)((a.n + 255) / 256), 256, 0, c.stream>>>(a);
  c.launches++;
  cuda_check(cudaGetLastError(), "emit images");
}

void fast_rollout(Ctx& c, Key key, double eps) {
  if (lockstep(c)) {
    ls_rollout(c, key, eps);
    return;
  }
  with_kernels(c, [&](auto k) { decltype(k)::rollout(c, key, eps); });
}

void fast_train(Ctx& c, bool apply, double lr, double* /*loss*/) {
  if (lockstep(c)) {
    ls_train(c);
    return;
  }
  with_kernels(c, [&](auto k) { decltype(k)::train(c, apply, lr); });
}

void fast_adam(Ctx& c, double lr) {
  const int64_t n = c.L.n_params;
  const gfnx_train_desc& s = c.train;
  const bool bitseq = lockstep(c);
  AdamArgs a{};
  if (!bitseq) {
    a = adam_args(c);
    FS(c).fused = false;
  }
  a.p = c.p32;
  a.m = c.m32;
  a.v = c.v32;
  a.g = c.g32;
  a.n = n;
  a.L = c.L;
  a.scalars = c.d_scalars;
  a.lr = (float)lr;
  a.b1 = (float)s.beta1;
  a.b2 = (float)s.beta2;
  a.beta1 = s.beta1;
  a.beta2 = s.beta2;
  a.eps = (float)s.adam_eps;
  a.wd = (float)s.weight_decay;
  a.do_z = s.objective == GFNX_OBJ_TB;
  a.z_lr = s.z_lr;
  a.zeps = s.adam_eps;
  a.steps = c.d_steps;
  a.err = c.batch.counters + 3;
  {
    ProfScope ps(c, "k_fast_adam");
    k_fast_adam<<<(unsigned)((n + 255) / 256), 256, 0, c.stream>>>(a);
    c.launches++;
  }
  if (bitseq) ls_sync_weights(c);
}

}  // namespace gfnx

// ---------------------------------------------------------------------------
// micro-benchmark hook: tcgen05.mma issue-to-completion rate on one SM (diagnostics)
namespace gfnx {
namespace {
template <int N>
__global__ void __launch_bounds__(128, 1) k_mma_rate(int reps, int mode, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* aimg = smem;                 // 128 x 256 bf16
  uint8_t* bimg = smem + 128 * 256 * 2;  // N x 256 bf16
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  for (int i = tid; i < (128 + N) * 256 * 2 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3c003c00u, 0x3c003c00u, 0, 0);
  if (tid < 32) tmem_alloc<512>(&tbase);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    uint32_t ph = 0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (mode == 0) {  // 128 x N x 256 from K-major SW128 images
        mma_kk<N, 256>(tbase + (r & 1) * 256, aimg, bimg, false);
      } else if (mode == 5) {  // A from TMEM (the rollout's TS form), D in [0, N)
        mma_tk<N, 256>(tbase, tbase + 256, bimg, false);

      } else if (mode >= 3) {  // MN-major operands (weight-gradient shape), K = 256 rows
        constexpr uint32_t idesc = umma_idesc_bf16(128, N, true, true);
        const uint32_t a0 = smem_u32(aimg), b0 = smem_u32(bimg);
        const uint32_t lbo = mode == 3 ? 64 * 128 : 128 * 128;  // 64- or 128-row MN blocks
        for (int k = 0; k < 16; ++k)
          umma_bf16(tbase, umma_desc_sw128(a0 + (k & 3) * 2048, lbo, 1024),
                    umma_desc_sw128(b0 + (k & 3) * 2048, lbo, 1024), idesc, k > 0);
      } else {  // same FLOPs as 16 separate K=16 issues with commits in between
        constexpr uint32_t idesc = umma_idesc_bf16(128, N, false, false);
        const uint32_t a0 = smem_u32(aimg), b0 = smem_u32(bimg);
        for (int s = 0; s < 16; ++s) {
          umma_bf16(tbase, umma_desc_sw128(a0 + (s >> 2) * (128 * 128) + (s & 3) * 32, 16, 1024),
                    umma_desc_sw128(b0 + (s >> 2) * (N * 128) + (s & 3) * 32, 16, 1024), idesc, s > 0);
        }
      }
      if ((mode != 2 && mode != 4) || r == reps - 1) {
        umma_commit(&bar);
        mbar_wait(&bar, ph);
        ph ^= 1;
      }
    }
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_dealloc<512>(tbase);
}
}  // namespace

namespace {
// D[128 x 256] = A[128 x 256] B[256 x 256]^T with A staged in TMEM (bf16 pairs per column):
// checks the TS operand layout the rollout relies on
__global__ void __launch_bounds__(128, 1) k_test_ts(const uint32_t* A, const __nv_bfloat16* B, float* D) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* bimg = align1024(smem_raw);
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 256 * 256; i += 128) {
    const int n = i / 256, k = i % 256;
    *reinterpret_cast<__nv_bfloat16*>(bimg + sw128_offset(n, k, 256)) = B[i];
  }
  if (warp == 0) tmem_alloc<512>(&tbase);
  if (tid == 0) {
    mbar_init(&mbar, 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase, lb = tmem + ((uint32_t)(warp * 32) << 16);
  for (int q = 0; q < 4; ++q) {  // row tid: 128 packed columns
    uint32_t r[32];
    for (int i = 0; i < 32; ++i) r[i] = A[tid * 128 + q * 32 + i];
    tmem_st32(lb + 256 + q * 32, r);
  }
  tmem_wait_st();
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  if (tid == 0) {
    tc_fence_after();
    mma_tk<256, 256>(tmem, tmem + 256, bimg, false);
    umma_commit(&mbar);
    mbar_wait(&mbar, 0);
  }
  __syncthreads();
  tc_fence_after();
  for (int q = 0; q < 8; ++q) {
    uint32_t r[32];
    tmem_ld32(lb + q * 32, r);
    tmem_wait_ld();
    for (int i = 0; i < 32; ++i) D[tid * 256 + q * 32 + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}
}  // namespace

void test_ts_mma(const uint16_t* a, const uint16_t* b, float* d) {
  uint32_t* da;
  __nv_bfloat16* db;
  float* dd;
  cudaMalloc(&da, 128 * 256 * 2);
  cudaMalloc(&db, 256 * 256 * 2);
  cudaMalloc(&dd, 128 * 256 * 4);
  cudaMemcpy(da, a, 128 * 256 * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b, 256 * 256 * 2, cudaMemcpyHostToDevice);
  const int smem = 256 * 256 * 2 + 1024;
  cudaFuncSetAttribute(k_test_ts, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_test_ts<<<1, 128, smem>>>(da, db, dd);
  cudaMemcpy(d, dd, 128 * 256 * 4, cudaMemcpyDeviceToHost);
  cudaFree(da);
  cudaFree(db);
  cudaFree(dd);
}

void test_mma_rate(int n, int reps, int mode, int grid, long long* host_out) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * grid);
  const int smem = (128 + 256) * 256 * 2 + 1024;
  if (n == 256) {
    cudaFuncSetAttribute(k_mma_rate<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_mma_rate<256><<<grid, 128, smem>>>(reps, mode, d);
  } else if (n == 16) {
    cudaFuncSetAttribute(k_mma_rate<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_mma_rate<16><<<grid, 128, smem>>>(reps, mode, d);
  } else if (n == 32) {
    cudaFuncSetAttribute(k_mma_rate<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_mma_rate<32><<<grid, 128, smem>>>(reps, mode, d);
  } else {
    cudaFuncSetAttribute(k_mma_rate<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_mma_rate<128><<<grid, 128, smem>>>(reps, mode, d);
  }
  cudaMemcpy(host_out, d, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
  cudaFree(d);
}
}  // namespace gfnx
