// gemm.cuh — warp-specialised tcgen05 GEMM over tile images, with pluggable epilogues.
//
//   C[m][n] = sum_k A[m][k] * B[n][k]
//
// A: activation tile images (128-row tiles; per tile `a_kb` K-blocks of 64 columns, each a
//    16 KB 128B-swizzled block) — the layout every fast-path kernel writes.
// B: weight images, N-tiles of BN rows; per N-tile `b_kb` K-blocks of BN x 128 B.
//
// Persistent CTAs over work items (m_tile, n_tile). Warp roles (12 warps):
//   warp 0      bulk-copy producer (TMA engine, 1-D cp.async.bulk) into a smem ring
//   warp 1      single-thread tcgen05.mma issuer into one of two TMEM accumulators
//   warps 4..11 epilogue: tcgen05.ld, two threads per accumulator row (warp w reads TMEM
//               lane quarter w % 4, column half (w - 4) / 4), Epi callbacks
// The two accumulators let the MMAs of item i+1 run while the epilogue drains item i.
//
// Two B policies:
//   resident B (KB <= 4): the whole B n-tile (<= 128 KB) stays in smem across consecutive
//     items of the same n; only A K-blocks stream through a 4-deep ring. Items are handed
//     out in contiguous n-major chunks so a CTA sees at most a couple of distinct n.
//   streamed B: A and B K-blocks stream together through a 4-deep ring (K up to A = 3840).
#pragma once

#include "fast_common.cuh"

namespace gfnx {
namespace {

constexpr int kStages = 4;
constexpr int kGemmThreads = 384;   // k_ls_wgrad (8 epilogue warps)
constexpr int kEpiThreads = 256;
constexpr int kGemmEpiParts = 4;    // k_gemm: 16 epilogue warps = lane quarter x column quarter
constexpr int kGemmKThreads = 128 + 128 * kGemmEpiParts;

template <int BN, bool kResB>
constexpr int gemm_smem_bytes() {
  return kResB ? 4 * BN * 128 + kStages * kTile * 128 + 1024 : kStages * (kTile * 128 + BN * 128) + 1024;
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

// Epilogue interface (derive from EpiBase and hide what you need):
//   struct Args; struct Local;
//   begin(e, m, n, row, half, loc)                  once per (item, thread) before the chunks
//   apply(e, m, n, row, col0, v[32], scratch, loc)  32 accumulator columns [col0, col0 + 32)
//   row_done(e, m, n, row, part, scratch, loc)      after the thread's BN/4 columns (part 0..3)
//   finish(e, m, n, scratch)                        after an epilogue barrier (all rows done);
// `scratch` is a [4][BN] smem array of per-lane-quarter column partials for finish().
struct EpiBase {
  struct Local {};
  template <class Args, class Loc>
  static __device__ void begin(const Args&, int, int, int, int, Loc&) {}
  template <class Args, class Loc>
  static __device__ void row_done(const Args&, int, int, int, int, float*, Loc&) {}
  template <class Args>
  static __device__ void finish(const Args&, int, int, const float*) {}
  // per-column bias the epilogue reads (nullptr: none); k_gemm stages it in shared memory
  template <class Args>
  static __device__ const float* bias_src(const Args&) { return nullptr; }
  template <class Args>
  static __device__ void set_bias(Args&, const float*) {}
};
constexpr int kGemmBiasMax = 4096;  // columns of bias staged per CTA (bitseq: 3840)

// column-partial slot of the calling epilogue thread
GFNX_DEV int epi_quarter() { return ((threadIdx.x >> 5) - 4) & 3; }

GFNX_DEV void epi_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
GFNX_DEV void gemm_epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(128 * kGemmEpiParts) : "memory"); }

struct ItemSeq {  // the items a CTA processes, in order
  int first, count, stride;
  GFNX_DEV int item(int j) const { return first + j * stride; }
};

template <bool kResB>
GFNX_DEV ItemSeq item_seq(int items) {
  if (kResB) {  // contiguous chunk (n-major order keeps the resident B tile)
    const int per = (items + gridDim.x - 1) / gridDim.x;
    const int first = blockIdx.x * per;
    return ItemSeq{first, max(0, min(per, items - first)), 1};
  }
  const int c = items > (int)blockIdx.x ? (items - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  return ItemSeq{(int)blockIdx.x, c, (int)gridDim.x};
}

template <bool kResB>
GFNX_DEV void item_mn(const GemmGeom& g, int item, int& m, int& n) {
  if (kResB) {
    n = item / g.m_tiles;
    m = g.m0 + item % g.m_tiles;
  } else {
    m = g.m0 + item / g.n_tiles;
    n = item % g.n_tiles;
  }
}

template <int BN, bool kResB, class Epi>
__global__ void __launch_bounds__(kGemmKThreads, 1) k_gemm(GemmGeom g, typename Epi::Args e) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  constexpr int kStageA = kTile * 128, kStageB = BN * 128;
  constexpr int kRing = kResB ? kStageA : kStageA + kStageB;
  uint8_t* ring = kResB ? smem + 4 * kStageB : smem;  // resident B occupies the front
  __shared__ uint64_t full[kStages], empty[kStages], tfull[2], tempty[2], bfull;
  __shared__ uint32_t tbase;
  __shared__ float scratch[4 * BN];
  __shared__ __align__(16) float bias_s[kGemmBiasMax];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const ItemSeq seq = item_seq<kResB>(g.m_tiles * g.n_tiles);
  if (seq.count == 0) return;
  // the epilogue's bias columns from shared memory (the epilogue's streaming stores would
  // otherwise keep evicting them from L1)
  typename Epi::Args el = e;
  if (const float* bsrc = Epi::bias_src(e)) {
    const int nb = g.n_tiles * BN;
    if (nb <= kGemmBiasMax) {
      for (int i = tid; i < nb; i += blockDim.x) bias_s[i] = bsrc[i];
      Epi::set_bias(el, bias_s);
    }
  }
  if (warp == 0) tmem_alloc<2 * BN>(&tbase);
  if (tid == 32) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 1);
    }
    mbar_init(&bfull, 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (warp == 0) {
    if (lane == 0) {  // ---- producer
      uint32_t L = 0;
      int cur_n = -1;
      for (int j = 0; j < seq.count; ++j) {
        int m, n;
        item_mn<kResB>(g, seq.item(j), m, n);
        if (kResB && n != cur_n) {
          // all MMAs reading the old B tile have completed once the newest A stage is free
          if (L > 0) mbar_wait(&empty[(L - 1) % kStages], ((L - 1) / kStages) & 1);
          mbar_arrive_expect_tx(&bfull, g.KB * kStageB);
          for (int kb = 0; kb < g.KB; ++kb)
            bulk_g2s_big(smem + kb * kStageB, g.B + ((size_t)n * g.b_kb + kb) * kStageB, kStageB, &bfull);
          cur_n = n;
        }
        for (int kb = 0; kb < g.KB; ++kb, ++L) {
          const uint32_t st = L % kStages;
          if (L >= kStages) mbar_wait(&empty[st], ((L / kStages) - 1) & 1);
          uint8_t* sa = ring + st * kRing;
          mbar_arrive_expect_tx(&full[st], kResB ? kStageA : kStageA + kStageB);
          bulk_g2s(sa, g.A + ((size_t)m * g.a_kb + g.a_kb0 + kb) * kStageA, kStageA, &full[st]);
          if (!kResB)
            bulk_g2s_big(sa + kStageA, g.B + ((size_t)n * g.b_kb + kb) * kStageB, kStageB, &full[st]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      constexpr uint32_t idesc = umma_idesc_bf16(128, BN, false, false);
      uint32_t C = 0, nb = 0;
      int cur_n = -1;
      for (int j = 0; j < seq.count; ++j) {
        int m, n;
        item_mn<kResB>(g, seq.item(j), m, n);
        if (kResB && n != cur_n) {
          mbar_wait(&bfull, nb & 1);
          ++nb;
          cur_n = n;
        }
        const uint32_t buf = j & 1, use = j >> 1;
        if (use >= 1) mbar_wait(&tempty[buf], (use - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + buf * BN;
        for (int kb = 0; kb < g.KB; ++kb, ++C) {
          const uint32_t st = C % kStages;
          mbar_wait(&full[st], (C / kStages) & 1);
          tc_fence_after();
          const uint32_t a0 = smem_u32(ring + st * kRing);
          const uint32_t b0 = kResB ? smem_u32(smem + kb * kStageB) : a0 + kStageA;
#pragma unroll
          for (int s = 0; s < 4; ++s)
            umma_bf16(d, umma_desc_sw128(a0 + s * 32, 16, 1024), umma_desc_sw128(b0 + s * 32, 16, 1024),
                      idesc, (kb > 0 || s > 0) ? 1u : 0u);
          umma_commit(&empty[st]);
        }
        umma_commit(&tfull[buf]);
      }
    }
  } else if (warp >= 4) {  // ---- epilogue: 16 warps = TMEM lane quarter x column quarter
    const int ew = warp - 4, quarter = ew & 3, part = ew >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    for (int j = 0; j < seq.count; ++j) {
      int m, n;
      item_mn<kResB>(g, seq.item(j), m, n);
      const uint32_t buf = j & 1;
      typename Epi::Local loc;
      Epi::begin(el, m, n, row, part, loc);
      mbar_wait(&tfull[buf], (j >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int q = 0; q < BN / (32 * kGemmEpiParts); ++q) {
        const int col0 = part * (BN / kGemmEpiParts) + q * 32;
        uint32_t r[32];
        tmem_ld32(lane_base + buf * BN + col0, r);
        tmem_wait_ld();
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
        Epi::apply(el, m, n, row, col0, v, scratch, loc);
      }
      tc_fence_before();
      Epi::row_done(el, m, n, row, part, scratch, loc);
      gemm_epi_bar();
      if (tid == 128) mbar_arrive_local(&tempty[buf]);
      Epi::finish(el, m, n, scratch);
      gemm_epi_bar();
    }
  }
  __syncthreads();
  if (warp == 0) tmem_dealloc<2 * BN>(tmem);
}

template <int BN, class Epi>
void launch_gemm(Ctx& c, const char* name, const GemmGeom& g, const typename Epi::Args& e, int num_sms) {
  const int items = g.m_tiles * g.n_tiles;
  const int grid = items < num_sms ? items : num_sms;
  ProfScope ps(c, name);
  if (g.KB <= 4) {
    constexpr int smem = gemm_smem_bytes<BN, true>();
    set_smem_once(k_gemm<BN, true, Epi>, smem);
    k_gemm<BN, true, Epi><<<grid, kGemmKThreads, smem, c.stream>>>(g, e);
  } else {
    constexpr int smem = gemm_smem_bytes<BN, false>();
    set_smem_once(k_gemm<BN, false, Epi>, smem);
    k_gemm<BN, false, Epi><<<grid, kGemmKThreads, smem, c.stream>>>(g, e);
  }
  c.launches++;
}

}  // namespace
}  // namespace gfnx
