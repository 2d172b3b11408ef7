// common.cuh — shared device primitives for libgfnx (sm_100a only).
//
//  * Threefry-2x64-20, fold_in, uniform (proj/src/rng.cpp:19-66), bit-exact with the host.
//  * PTX wrappers: mbarrier, TMEM alloc/ld/st, tcgen05.mma (kind::f16, cta_group::1),
//    tcgen05.commit, async-proxy fences and 1-D bulk copies (TMA engine).
//  * UMMA shared-memory / instruction descriptors for 128B-swizzled bf16 tiles.
#pragma once

#include <cuda_runtime.h>
#if defined(__CUDACC__)
#include <cuda_bf16.h>
#endif
#include <stdint.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libgfnx targets sm_100a only"
#endif

#define GFNX_DEV __device__ __forceinline__

namespace gfnx {

// ---------------------------------------------------------------------------
// Threefry-2x64-20 (rng.cpp:19-34) — integer only, so device == host bit for bit.
struct Key {
  uint64_t hi, lo;
};

__host__ __device__ __forceinline__ uint64_t rotl64(uint64_t x, int r) {
  return (x << r) | (x >> (64 - r));
}

__host__ __device__ __forceinline__ void threefry2x64(Key k, uint64_t c0, uint64_t c1,
                                                      uint64_t& o0, uint64_t& o1) {
  const uint64_t ks0 = k.hi, ks1 = k.lo, ks2 = k.hi ^ k.lo ^ 0x1BD11BDAA9FC1A22ULL;
  uint64_t x0 = c0 + ks0, x1 = c1 + ks1;
  // 5 groups of 4 rounds, rotations {16,42,12,31},{16,32,24,21} alternate (kRot, rng.cpp:13)
#define GFNX_TF_ROUND(r) \
  x0 += x1;              \
  x1 = rotl64(x1, r);    \
  x1 ^= x0;
  GFNX_TF_ROUND(16) GFNX_TF_ROUND(42) GFNX_TF_ROUND(12) GFNX_TF_ROUND(31)
  x0 += ks1; x1 += ks2 + 1;
  GFNX_TF_ROUND(16) GFNX_TF_ROUND(32) GFNX_TF_ROUND(24) GFNX_TF_ROUND(21)
  x0 += ks2; x1 += ks0 + 2;
  GFNX_TF_ROUND(16) GFNX_TF_ROUND(42) GFNX_TF_ROUND(12) GFNX_TF_ROUND(31)
  x0 += ks0; x1 += ks1 + 3;
  GFNX_TF_ROUND(16) GFNX_TF_ROUND(32) GFNX_TF_ROUND(24) GFNX_TF_ROUND(21)
  x0 += ks1; x1 += ks2 + 4;
  GFNX_TF_ROUND(16) GFNX_TF_ROUND(42) GFNX_TF_ROUND(12) GFNX_TF_ROUND(31)
  x0 += ks2; x1 += ks0 + 5;
#undef GFNX_TF_ROUND
  o0 = x0;
  o1 = x1;
}

__host__ __device__ __forceinline__ Key make_key(uint64_t seed) {  // rng.cpp:17
  return Key{0x9E3779B97F4A7C15ULL, seed};
}

__host__ __device__ __forceinline__ Key fold_in(Key k, uint64_t idx) {  // rng.cpp:36-39
  Key o;
  threefry2x64(k, idx, 0x3C6EF372FE94F82BULL, o.hi, o.lo);
  return o;
}

__host__ __device__ __forceinline__ double to_unit(uint64_t w) {  // rng.cpp:47-50
  return (double)(w >> 11) * 0x1.0p-53;
}

__host__ __device__ __forceinline__ double uniform_scalar(Key k) {  // rng.cpp:64-66
  uint64_t a, b;
  threefry2x64(k, 0, 0, a, b);
  return to_unit(a);
}

#if defined(__CUDACC__)
// ---------------------------------------------------------------------------
// Small helpers
GFNX_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

GFNX_DEV uint32_t lane_id() { return threadIdx.x & 31; }

// 2^x on the SFU with flush-to-zero (one MUFU.EX2, no subnormal range fix-ups); results
// below 2^-126 become 0 — for softmax terms exp(x - lse) that never matter
GFNX_DEV float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
constexpr float kLog2e = 1.4426950408889634f;

GFNX_DEV uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// ReLU + round-to-nearest bf16 pair in one cvt (cvt.rn.relu clamps negatives to +0):
// the same bits as pack_bf16x2(fmaxf(lo, 0), fmaxf(hi, 0)) for every non-NaN input
GFNX_DEV uint32_t pack_bf16x2_relu(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// (a0, a1) += s * (the two bf16 halves of w) as one FFMA2 (fma.rn.f32x2: per lane the same
// single rounding as FFMA)
GFNX_DEV void fma2_bf16(uint32_t& a0, uint32_t& a1, float s, uint32_t w) {
  unsigned long long acc, m, sv;
  asm("mov.b64 %0, {%1, %2};" : "=l"(acc) : "r"(a0), "r"(a1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(m) : "r"(w << 16), "r"(w & 0xffff0000u));
  asm("mov.b64 %0, {%1, %1};" : "=l"(sv) : "f"(s));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(sv), "l"(m));
  asm("mov.b64 {%0, %1}, %2;" : "=r"(a0), "=r"(a1) : "l"(acc));
}
// ReLU(acc + bias) of an fp32 accumulator pair (raw TMEM words) as one packed bf16 pair:
// one FADD2 (add.rn.f32x2, IEEE fp32 per lane like FADD) + one cvt
GFNX_DEV uint32_t bias_relu_pack(uint32_t a_lo, uint32_t a_hi, float2 b) {
  unsigned long long x, y;
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "r"(a_lo), "r"(a_hi));
  asm("mov.b64 %0, {%1, %2};" : "=l"(y) : "f"(b.x), "f"(b.y));
  asm("add.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(y));
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x));
  return pack_bf16x2_relu(lo, hi);
}

// (a + b) of an fp32 pair rounded to a packed bf16 pair: one FADD2 + one cvt, the same bits
// as pack_bf16x2(a.x + b.x, a.y + b.y)
GFNX_DEV uint32_t add_pack_bf16x2(float a_lo, float a_hi, float b_lo, float b_hi) {
  unsigned long long x, y;
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a_lo), "f"(a_hi));
  asm("mov.b64 %0, {%1, %2};" : "=l"(y) : "f"(b_lo), "f"(b_hi));
  asm("add.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(y));
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x));
  return pack_bf16x2(lo, hi);
}
// (x0 s + t, x1 s + t) as one FFMA2 and (x0 s, x1 s) as one FMUL2: per lane the same single
// rounding as fmaf / an fp32 multiply
GFNX_DEV void ffma2_st(float& x0, float& x1, float s, float t) {
  unsigned long long x, sv, tv;
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(x0), "f"(x1));
  asm("mov.b64 %0, {%1, %1};" : "=l"(sv) : "f"(s));
  asm("mov.b64 %0, {%1, %1};" : "=l"(tv) : "f"(t));
  asm("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x) : "l"(sv), "l"(tv));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x0), "=f"(x1) : "l"(x));
}
GFNX_DEV void fmul2_s(float& x0, float& x1, float s) {
  unsigned long long x, sv;
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(x0), "f"(x1));
  asm("mov.b64 %0, {%1, %1};" : "=l"(sv) : "f"(s));
  asm("mul.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(sv));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x0), "=f"(x1) : "l"(x));
}

GFNX_DEV float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
GFNX_DEV float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }

// ---------------------------------------------------------------------------
// mbarrier
GFNX_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
GFNX_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

GFNX_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

// wait with a back-off sleep between polls: for warps that idle through a long phase, so
// their polling does not steal issue slots from the producer / MMA warps
GFNX_DEV void mbar_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t ns) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  while (true) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (done) break;
    __nanosleep(ns);
  }
}

GFNX_DEV void mbar_arrive_local(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

GFNX_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// 1-D bulk copy global -> shared through the TMA engine (SASS: UBLKCP), completes on bar.
GFNX_DEV void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// 1-D bulk copy shared -> global (bulk_group completion).
GFNX_DEV void bulk_s2g(void* dst_gmem, const void* src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst_gmem),
               "r"(smem_u32(src_smem)), "r"(bytes)
               : "memory");
}
GFNX_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
GFNX_DEV void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
GFNX_DEV void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// generic-proxy smem writes -> visible to the async proxy (UMMA operand reads, bulk copies)
GFNX_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ---------------------------------------------------------------------------
// TMEM
template <uint32_t kCols>
GFNX_DEV void tmem_alloc(uint32_t* dst_smem) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
template <uint32_t kCols>
GFNX_DEV void tmem_dealloc(uint32_t taddr) {  // same warp that allocated
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols));
}
GFNX_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
GFNX_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 32 lanes x 32 consecutive fp32 columns; thread i of the warp gets lane (base_lane + i).
GFNX_DEV void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
GFNX_DEV void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
GFNX_DEV void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31]));
}
GFNX_DEV void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]));
}
GFNX_DEV void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
GFNX_DEV void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ---------------------------------------------------------------------------
// UMMA (tcgen05.mma kind::f16, bf16 x bf16 -> fp32, single CTA)
//
// Operand tiles use the canonical 128B-swizzled layouts (cute mma_sm100_desc.hpp):
//   K-major : rows of 64 bf16 (128 B), 8-row groups of 1024 B (SBO = 1024), XOR swizzle of
//             the 16-byte chunk index with (row & 7). A 64-wide K block of an R-row tile
//             is R*128 bytes; the next K block follows.
//   MN-major: the same bytes read transposed: 64 MN-contiguous elements per 128 B row,
//             8 K-rows per 1024 B atom (SBO = 1024), next 64-wide MN block at LBO.
// Our activation "tile image" (rows x features, 64-feature blocks of rows*128 B) is thus
// the K-major A operand of the forward GEMM AND the MN-major operand of the weight
// gradient GEMM, with no transposition.
GFNX_DEV uint64_t umma_desc_sw128(uint32_t smem_addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm100)
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

#endif  // __CUDACC__

// Non-swizzled K-major operand: 8-row x 16-byte core matrices, LBO = stride between core
// matrices along K, SBO = stride between 8-row groups along M/N.
GFNX_DEV uint64_t umma_desc_none(uint32_t smem_addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version; layout type 0 = SWIZZLE_NONE
  return d;
}

__host__ __device__ constexpr uint32_t umma_idesc_bf16(uint32_t M, uint32_t N, bool a_mn,
                                                       bool b_mn) {
  return (1u << 4)                   // D fp32
         | (1u << 7)                 // A bf16
         | (1u << 10)                // B bf16
         | ((a_mn ? 1u : 0u) << 15)  // A major
         | ((b_mn ? 1u : 0u) << 16)  // B major
         | ((N >> 3) << 17) | ((M >> 4) << 24);
}

#if defined(__CUDACC__)
GFNX_DEV void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                        uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// A operand from tensor memory ("TS" form): 128 lanes = rows of A, K packed along the
// columns (two bf16 per 32-bit column); a K = 16 step reads 8 columns at tmem_a.
GFNX_DEV void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                           uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

GFNX_DEV void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

#endif  // __CUDACC__

// Byte offset of element (row n, k) of a non-swizzled K-major bf16 operand with K columns.
__host__ __device__ __forceinline__ uint32_t nsw_offset(uint32_t n, uint32_t k, uint32_t K) {
  return (n >> 3) * (K / 8) * 128u + (k >> 3) * 128u + (n & 7) * 16u + (k & 7) * 2u;
}

// Byte offset of element (row, col) in a 128B-swizzled bf16 tile image with `rows` rows.
__host__ __device__ __forceinline__ uint32_t sw128_offset(uint32_t row, uint32_t col,
                                                          uint32_t rows) {
  const uint32_t blk = col >> 6, c = col & 63;
  const uint32_t chunk = (c >> 3) ^ (row & 7);
  return blk * rows * 128u + row * 128u + chunk * 16u + (c & 7) * 2u;
}

}  // namespace gfnx
