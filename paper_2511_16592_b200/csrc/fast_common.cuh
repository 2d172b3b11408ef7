// fast_common.cuh — tensor-core / bulk-copy helpers shared by the fast-path TUs.
#pragma once

#include <mutex>
#include <tuple>

#include <vector>

#include "engine.h"

namespace gfnx {
namespace {

constexpr int kTile = 128;     // rows per CTA tile = TMEM lanes
constexpr int kThreads = 256;  // two threads per tile row

// ---------------------------------------------------------------------------
// tensor-core helpers (single elected thread issues, accumulator in TMEM)

// D[128 x N] (+)= A[128 x K] * B[N x K]^T, both K-major 128B-swizzled tile images in smem.
template <int N, int K>
GFNX_DEV void mma_kk(uint32_t d_tmem, const void* a_img, const void* b_img, bool acc) {
  constexpr uint32_t idesc = umma_idesc_bf16(128, N, false, false);
  const uint32_t a0 = smem_u32(a_img), b0 = smem_u32(b_img);
#pragma unroll
  for (int s = 0; s < K / 16; ++s) {
    const uint32_t ao = a0 + (s >> 2) * (128 * 128) + (s & 3) * 32;
    const uint32_t bo = b0 + (s >> 2) * (N * 128) + (s & 3) * 32;
    umma_bf16(d_tmem, umma_desc_sw128(ao, 16, 1024), umma_desc_sw128(bo, 16, 1024), idesc,
              (acc || s > 0) ? 1u : 0u);
  }
}

// D[128 x N] (+)= A'[128 x 128] * B'[N x 128]^T with A' = act^T, B' = dz^T read MN-major
// from 128-row tile images: a_img holds features [m0, m0+128) of a tile with 128 rows.
template <int N>
GFNX_DEV void mma_mn(uint32_t d_tmem, const void* a_img, int m0, const void* b_img, bool acc) {
  constexpr uint32_t idesc = umma_idesc_bf16(128, N, true, true);
  const uint32_t a0 = smem_u32(a_img) + (m0 >> 6) * (128 * 128), b0 = smem_u32(b_img);
#pragma unroll
  for (int s = 0; s < kTile / 16; ++s) {
    const uint32_t ao = a0 + s * 2048, bo = b0 + s * 2048;
    umma_bf16(d_tmem, umma_desc_sw128(ao, 128 * 128, 1024), umma_desc_sw128(bo, 128 * 128, 1024),
              idesc, (acc || s > 0) ? 1u : 0u);
  }
}

// ReLU mask of 32 consecutive bf16 columns packed as 16 bf16x2 words (values >= 0 or -0):
// bit i <-> column 2i, bit 16 + i <-> column 2i + 1 (set when the value is nonzero).
GFNX_DEV uint32_t relu_mask16(const uint32_t (&pk)[16]) {
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) m |= ((((pk[i] & 0x7FFF7FFFu) + 0x7FFF7FFFu) >> 15) & 0x00010001u) << i;
  return m;
}

// D[128 x N] (+)= A[128 x K] * B[N x K]^T with A in TMEM (columns a_col.., K/2 of them)
// and B a K-major 128B-swizzled image in smem.
template <int N, int K>
GFNX_DEV void mma_tk(uint32_t d_tmem, uint32_t a_tmem, const void* b_img, bool acc) {
  constexpr uint32_t idesc = umma_idesc_bf16(128, N, false, false);
  const uint32_t b0 = smem_u32(b_img);
#pragma unroll
  for (int s = 0; s < K / 16; ++s) {
    const uint32_t bo = b0 + (s >> 2) * (N * 128) + (s & 3) * 32;
    umma_bf16_ts(d_tmem, a_tmem + s * 8, umma_desc_sw128(bo, 16, 1024), idesc, (acc || s > 0) ? 1u : 0u);
  }
}

// the same with a runtime K (multiple of 16, <= the image's K): layer 1 reads only the
// obs_dim features that exist (hypergrid 4x20: K = 80, 5 instead of 8 K-steps)
template <int N>
GFNX_DEV void mma_tk_k(uint32_t d_tmem, uint32_t a_tmem, const void* b_img, int k) {
  constexpr uint32_t idesc = umma_idesc_bf16(128, N, false, false);
  const uint32_t b0 = smem_u32(b_img);
#pragma unroll 1
  for (int s = 0; s < k / 16; ++s) {
    const uint32_t bo = b0 + (s >> 2) * (N * 128) + (s & 3) * 32;
    umma_bf16_ts(d_tmem, a_tmem + s * 8, umma_desc_sw128(bo, 16, 1024), idesc, s > 0 ? 1u : 0u);
  }
}

// store 32 consecutive bf16 columns [c0, c0+32) of row `row` into a 128-row tile image
GFNX_DEV void st_row32(uint8_t* img, int row, int c0, const uint32_t (&pk)[16]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint4 v = make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
    *reinterpret_cast<uint4*>(img + sw128_offset(row, c0 + 8 * c, kTile)) = v;
  }
}
// the same 32 columns into a tile image in GLOBAL memory with two 32-byte stores (the chunk
// pairs (2m, 2m+1) of a 64-column block stay adjacent under the XOR swizzle, halves swapped
// when row & 1)
GFNX_DEV void st_row32_g(uint8_t* img, int row, int c0, const uint32_t (&pk)[16]) {
  const int x = row & 7;
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    const int l0 = ((c0 & 63) >> 3) + 2 * m;  // logical chunk (even)
    const int p = l0 ^ x;
    uint32_t v[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[i] = (x & 1) ? pk[8 * m + 4 + i] : pk[8 * m + i];
      v[4 + i] = (x & 1) ? pk[8 * m + i] : pk[8 * m + 4 + i];
    }
    uint8_t* dst = img + (c0 >> 6) * (kTile * 128) + row * 128 + (p & ~1) * 16;
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst), "r"(v[0]), "r"(v[1]), "r"(v[2]),
                 "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
  }
}

GFNX_DEV void ld_row32(const uint8_t* img, int row, int c0, float (&v)[32]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint4 q = *reinterpret_cast<const uint4*>(img + sw128_offset(row, c0 + 8 * c, kTile));
    v[8 * c + 0] = bf16_lo(q.x); v[8 * c + 1] = bf16_hi(q.x);
    v[8 * c + 2] = bf16_lo(q.y); v[8 * c + 3] = bf16_hi(q.y);
    v[8 * c + 4] = bf16_lo(q.z); v[8 * c + 5] = bf16_hi(q.z);
    v[8 * c + 6] = bf16_lo(q.w); v[8 * c + 7] = bf16_hi(q.w);
  }
}

GFNX_DEV void bulk_g2s_big(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  for (uint32_t off = 0; off < bytes; off += 32768) {
    const uint32_t n = bytes - off < 32768 ? bytes - off : 32768;
    bulk_g2s((uint8_t*)dst + off, (const uint8_t*)src + off, n, bar);
  }
}

GFNX_DEV uint8_t* align1024(uint8_t* p) {
  return (uint8_t*)(((uintptr_t)p + 1023) & ~(uintptr_t)1023);
}

// D[128 x N] = A[128 x K] (SW128 tile image) * B[N x K]^T with B non-swizzled (K small)
template <int N, int K>
GFNX_DEV void mma_k_sw128_none(uint32_t d_tmem, const void* a_img, const void* b_img) {
  constexpr uint32_t idesc = umma_idesc_bf16(128, N, false, false);
  const uint32_t a0 = smem_u32(a_img), b0 = smem_u32(b_img);
#pragma unroll
  for (int s = 0; s < K / 16; ++s)
    umma_bf16(d_tmem, umma_desc_sw128(a0 + s * 32, 16, 1024),
              umma_desc_none(b0 + s * 256, 128, (K / 8) * 128), idesc, s > 0 ? 1u : 0u);
}

template <class K>
void set_smem_once(K kernel, int smem) {
  // (kernel, device, bytes) already applied; ctxs may run on several host threads / GPUs
  static std::mutex mu;
  static std::vector<std::tuple<const void*, int, int>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  for (auto& d : done)
    if (std::get<0>(d) == (const void*)kernel && std::get<1>(d) == dev && std::get<2>(d) >= smem) return;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  done.emplace_back((const void*)kernel, dev, smem);
}


}  // namespace
}  // namespace gfnx
