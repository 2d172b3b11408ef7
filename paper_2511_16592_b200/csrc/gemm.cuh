// gemm.cuh — pipelined tcgen05 GEMM over tile images, with pluggable epilogues.
//
//   C[m][n] = sum_k A[m][k] * B[n][k]
//
// A: activation tile images (128-row tiles; per tile `a_kb` K-blocks of 64 columns, each a
//    16 KB 128B-swizzled block) — the layout every fast-path kernel writes.
// B: weight images, N-tiles of BN rows; per N-tile `b_kb` K-blocks of BN x 128 B.
// One CTA (256 threads) per work item (m_tile, n_tile), persistent over items. Thread 0
// streams K-blocks through a 4-stage smem ring with 1-D bulk copies (TMA engine) and
// issues tcgen05.mma into a TMEM accumulator; all 8 warps run the epilogue (two threads
// per row, tcgen05.ld lane quarters), while thread 0 already prefetches the next item.
#pragma once

#include "fast_common.cuh"

namespace gfnx {
namespace {

constexpr int kStages = 4;

template <int BN>
constexpr int gemm_smem_bytes() {
  return kStages * (kTile * 128 + BN * 128) + 1024;
}

struct GemmGeom {
  const uint8_t* A;
  int a_kb;        // K-blocks per A tile (row stride of the A image in 16 KB blocks)
  int a_kb0;       // first K-block of A used (e.g. a head chunk inside a wide image)
  const uint8_t* B;
  int b_kb;        // K-blocks per B n-tile
  int m0, m_tiles;  // A tiles [m0, m0 + m_tiles)
  int n_tiles;
  int KB;           // K-blocks to accumulate
};

// Warp-level transpose-sum: on return lane l holds sum over the warp's 32 rows of v[l].
GFNX_DEV float warp_colsum32(float (&v)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool upper = lane & s;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const float send = upper ? v[i] : v[i + s];
      const float keep = upper ? v[i + s] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return v[0];
}

// Epi must provide:
//   struct Args;
//   static __device__ void apply(const Args&, int m_tile, int n_tile, int row, int col0,
//                                float (&v)[32], float* scratch);  // 32 output columns
//   static __device__ void finish(const Args&, int m_tile, int n_tile, const float* scratch);
// `scratch` is a [4][BN] smem array (per lane-quarter column partials) that finish()
// reads after a CTA barrier — used for deterministic per-tile column sums.
template <int BN, class Epi>
__global__ void __launch_bounds__(kThreads, 1) k_gemm(GemmGeom g, typename Epi::Args e) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  constexpr int kStageA = kTile * 128, kStageB = BN * 128;
  __shared__ uint64_t full[kStages], empty[kStages], accb;
  __shared__ uint32_t tbase;
  __shared__ float scratch[4 * BN];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quarter = warp & 3, half = warp >> 2;
  const int row = quarter * 32 + lane;
  const int items = g.m_tiles * g.n_tiles;
  if ((int)blockIdx.x >= items) return;
  if (warp == 0) tmem_alloc<BN>(&tbase);
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&accb, 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
  constexpr uint32_t idesc = umma_idesc_bf16(128, BN, false, false);
  // producer/consumer state lives in thread 0 only. K-blocks are loaded and consumed in
  // one global order (item-major); a stage is refilled one block after it was consumed,
  // so one MMA is always queued behind the one the refill waits for.
  uint32_t loaded = 0, consumed = 0;
  uint32_t acc_phase = 0;
  int pre_item = blockIdx.x, pre_kb = 0;
  auto next_load = [&]() {
    if (pre_item >= items) return;
    const int m = g.m0 + pre_item / g.n_tiles, n = pre_item % g.n_tiles;
    const uint32_t st = loaded % kStages;
    if (loaded >= kStages) mbar_wait(&empty[st], ((loaded / kStages) - 1) & 1);
    uint8_t* sa = smem + st * (kStageA + kStageB);
    uint8_t* sb = sa + kStageA;
    mbar_arrive_expect_tx(&full[st], kStageA + kStageB);
    bulk_g2s(sa, g.A + ((size_t)m * g.a_kb + g.a_kb0 + pre_kb) * kStageA, kStageA, &full[st]);
    bulk_g2s_big(sb, g.B + ((size_t)n * g.b_kb + pre_kb) * kStageB, kStageB, &full[st]);
    ++loaded;
    if (++pre_kb == g.KB) {
      pre_kb = 0;
      pre_item += gridDim.x;
    }
  };
  if (tid == 0)
    for (int i = 0; i < kStages; ++i) next_load();
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    const int m = g.m0 + item / g.n_tiles, n = item % g.n_tiles;
    if (tid == 0) {
      tc_fence_after();
      for (int kb = 0; kb < g.KB; ++kb) {
        const uint32_t st = consumed % kStages;
        mbar_wait(&full[st], (consumed / kStages) & 1);
        tc_fence_after();
        const uint32_t a0 = smem_u32(smem + st * (kStageA + kStageB));
        const uint32_t b0 = a0 + kStageA;
#pragma unroll
        for (int s = 0; s < 4; ++s)
          umma_bf16(tmem, umma_desc_sw128(a0 + s * 32, 16, 1024),
                    umma_desc_sw128(b0 + s * 32, 16, 1024), idesc, (kb > 0 || s > 0) ? 1u : 0u);
        umma_commit(&empty[st]);
        ++consumed;
        if (consumed >= 2) next_load();
      }
      umma_commit(&accb);
    }
    mbar_wait(&accb, acc_phase);
    acc_phase ^= 1;
    tc_fence_after();
#pragma unroll 1
    for (int q = 0; q < BN / 64; ++q) {
      const int col0 = half * (BN / 2) + q * 32;
      uint32_t r[32];
      tmem_ld32(lane_base + col0, r);
      tmem_wait_ld();
      float v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
      Epi::apply(e, m, n, row, col0, v, scratch);
    }
    tc_fence_before();
    __syncthreads();  // accumulator drained before the next item's MMAs
    Epi::finish(e, m, n, scratch);
    __syncthreads();
  }
  __syncthreads();
  if (warp == 0) tmem_dealloc<BN>(tmem);
}

template <int BN, class Epi>
void launch_gemm(Ctx& c, const char* name, const GemmGeom& g, const typename Epi::Args& e, int num_sms) {
  const int smem = gemm_smem_bytes<BN>();
  set_smem_once(k_gemm<BN, Epi>, smem);
  const int items = g.m_tiles * g.n_tiles;
  const int grid = items < num_sms ? items : num_sms;
  ProfScope ps(c, name);
  k_gemm<BN, Epi><<<grid, kThreads, smem, c.stream>>>(g, e);
  c.launches++;
}

}  // namespace
}  // namespace gfnx
