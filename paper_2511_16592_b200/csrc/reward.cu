// reward.cu — batched terminal log-reward kernels over structure-of-arrays packed states.
//
// The reward of a batch of terminal states (log_reward_of of every env: hypergrid.cpp:111-119,
// ModeSet::log_reward sequences.cpp:50-55, ising_energy ising.cpp:40-51 / :143-145,
// graph_log_reward dag.cpp:313-322) as a standalone, HBM-streaming kernel: the packed state
// words are stored word-major ([SW][n], so a warp's loads of word w are one coalesced 128-byte
// line per 32 states), one fp64 out per state. Bit-exact with the reference by construction
// (envs.cuh: tables built on the host with the reference's expressions, fp64 additions in the
// reference's order). The rollout computes the same rewards at termination inside its step;
// these kernels serve callers that score states they hold (and the SURVEY §8(d)(ii) B sweep).
//
//   hypergrid, DAG : the generic kernel (a few table lookups per state: HBM-bound)
//   Ising          : per-site tables of the reference's row sum sum_b J_ab s_b for each
//                    pattern of the site's (ascending) neighbour spins, so a state costs one
//                    table lookup and one fp64 add per site, in the reference's site order
//                    (the D dependent fp64 adds are the floor of a bit-exact energy)
//   bitseq         : the string as big-endian 32-bit chunks (token bytes byte-swapped), min
//                    over the modes of XOR + popcount, modes in shared memory
#include <algorithm>
#include <vector>

#include "engine.h"

namespace gfnx {

namespace {

template <class Env>
__device__ __forceinline__ double reward_one(const EnvParams& P, const uint32_t (&w)[16], int32_t* err) {
  typename Env::State s;
  Env::unpack(P, w, s);
  if constexpr (std::is_same<Env, IsingEnv>::value) {
    if (s.count != P.is_D) atomicExch(err, GFNX_ERR_CONTRACT);  // ising_energy: incomplete
  }
  if constexpr (std::is_same<Env, BitseqEnv>::value) {
    if (s.count != P.bs_slots) atomicExch(err, GFNX_ERR_CONTRACT);
  }
  return Env::log_reward(P, s);
}

// Each thread scores 4 consecutive terminals per pass: one 16-byte streaming load per state
// word (SW x 16 B in flight per thread), two 16-byte stores of the fp64 results.
template <class Env, int SWM>
__global__ void __launch_bounds__(256) k_reward_soa(EnvParams P, const uint32_t* __restrict__ st, int64_t n,
                                                    double* __restrict__ out, int32_t* err) {
  const int64_t n4 = (n % 4 == 0) ? n / 4 : 0;  // vector path needs 16-byte aligned word rows
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += (int64_t)gridDim.x * blockDim.x) {
    uint4 v[SWM];
#pragma unroll
    for (int k = 0; k < SWM; ++k)
      v[k] = k < P.SW ? __ldcs(reinterpret_cast<const uint4*>(st + (size_t)k * n) + q) : make_uint4(0u, 0u, 0u, 0u);
    double r[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t w[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const uint4 x = k < SWM ? v[k < SWM ? k : 0] : make_uint4(0u, 0u, 0u, 0u);
        w[k] = j == 0 ? x.x : j == 1 ? x.y : j == 2 ? x.z : x.w;
      }
      r[j] = reward_one<Env>(P, w, err);
    }
    __stcs(reinterpret_cast<double2*>(out) + 2 * q, make_double2(r[0], r[1]));
    __stcs(reinterpret_cast<double2*>(out) + 2 * q + 1, make_double2(r[2], r[3]));
  }
  for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t w[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) w[k] = k < P.SW ? __ldcs(st + (size_t)k * n + i) : 0u;
    __stcs(out + i, reward_one<Env>(P, w, err));
  }
}

// Ising on a side x side torus (D <= 128 sites): tab[a][p] = the reference's row sum for the
// neighbour-spin pattern p (bit q = spin of the q-th ascending neighbour is +1), then
// quad = sum_a s_a * row_a in site order. SIDE is a compile-time constant so every neighbour
// bit position folds to an immediate.
template <int SIDE>
__device__ __forceinline__ int ising_nbr(int a, int q) {  // ascending distinct neighbours of a
  const int r = a / SIDE, c = a % SIDE;
  int v[4] = {((r + SIDE - 1) % SIDE) * SIDE + c, ((r + 1) % SIDE) * SIDE + c, r * SIDE + (c + SIDE - 1) % SIDE,
              r * SIDE + (c + 1) % SIDE};
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 3 - i; ++j)
      if (v[j] > v[j + 1]) {
        const int t = v[j];
        v[j] = v[j + 1];
        v[j + 1] = t;
      }
  return v[q];
}

template <int SIDE>
__global__ void __launch_bounds__(256) k_reward_ising(int64_t n, int SW, const uint32_t* __restrict__ st,
                                                      const double* __restrict__ tab_g, double* __restrict__ out,
                                                      int32_t* err) {
  constexpr int D = SIDE * SIDE;
  static_assert(D <= 128 && SIDE >= 3, "torus with 4 distinct neighbours, <= 128 sites");
  __shared__ double tab[D * 16];
  for (int i = threadIdx.x; i < D * 16; i += blockDim.x) tab[i] = tab_g[i];
  __syncthreads();
  constexpr int NW = (D + 31) / 32;
  const int nw = SW / 2;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t up[NW];
    bool full = true;
#pragma unroll
    for (int k = 0; k < NW; ++k) {
      const uint32_t asg = __ldcs(st + (size_t)k * n + i);
      up[k] = __ldcs(st + (size_t)(nw + k) * n + i);
      const uint32_t want = (k == NW - 1 && D % 32) ? (1u << (D % 32)) - 1u : 0xffffffffu;
      full &= asg == want;
    }
    if (!full) atomicExch(err, GFNX_ERR_CONTRACT);
    double quad = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      uint32_t p = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int b = ising_nbr<SIDE>(a, q);
        p |= ((up[b >> 5] >> (b & 31)) & 1u) << q;
      }
      const double row = tab[a * 16 + p];
      quad += ((up[a >> 5] >> (a & 31)) & 1u) ? row : -row;  // spins[a] * row, exact
    }
    __stcs(out + i, quad);  // log_reward = -energy = quad (ising.cpp:143-145)
  }
}

// bitseq ModeSet: best = min_m hamming(x, mode_m); log_reward = bs_logr[best]
template <int NW>
__global__ void __launch_bounds__(256) k_reward_bitseq(EnvParams P, int64_t n, const uint32_t* __restrict__ st,
                                                       double* __restrict__ out, int32_t* err) {
  extern __shared__ uint32_t modes[];  // [n_modes][NW] big-endian 32-bit chunks
  for (int i = threadIdx.x; i < P.n_modes * NW; i += blockDim.x) {
    const int m = i / NW, k = i % NW;
    const uint64_t w = P.modes[m * P.bs_words + (k >> 1)];
    modes[i] = (k & 1) ? (uint32_t)w : (uint32_t)(w >> 32);
  }
  __syncthreads();
  const int tw = (P.bs_slots + 3) / 4;
  const uint32_t all = P.bs_slots == 32 ? 0xffffffffu : (1u << P.bs_slots) - 1u;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t x[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) {  // tokens 4k..4k+3, MSB-first bits: byte-swapped token word
      const uint32_t v = k < tw ? __ldcs(st + (size_t)k * n + i) : 0u;
      x[k] = __byte_perm(v, 0, 0x0123);
    }
    if (__ldcs(st + (size_t)tw * n + i) != all) atomicExch(err, GFNX_ERR_CONTRACT);
    int best = P.bs_nbits + 1;
    for (int m = 0; m < P.n_modes; ++m) {
      int h = 0;
#pragma unroll
      for (int k = 0; k < NW; ++k) h += __popc(x[k] ^ modes[m * NW + k]);
      best = min(best, h);
    }
    __stcs(out + i, P.bs_logr[best]);
  }
}

// hypergrid, one packed word (dim <= 4, side <= 32): 8 terminals per thread per pass (two
// 16-byte loads in flight), p1 / p2 = AND over the coordinates of the tabulated predicates
__global__ void __launch_bounds__(256) k_reward_hg(EnvParams P, const uint32_t* __restrict__ st, int64_t n8,
                                                   double* __restrict__ out) {
  const uint32_t f1 = P.hg_f1[0], f2 = P.hg_f2[0];
  const double r0 = P.hg_logr[0], r1 = P.hg_logr[1], r2 = P.hg_logr[2], r3 = P.hg_logr[3];
  const int dim = P.hg_dim;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n8; q += (int64_t)gridDim.x * blockDim.x) {
    const uint4 a = __ldcs(reinterpret_cast<const uint4*>(st) + 2 * q);
    const uint4 b = __ldcs(reinterpret_cast<const uint4*>(st) + 2 * q + 1);
    const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t p1 = 1u, p2 = 1u;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (i < dim) {
          const uint32_t c = (w[j] >> (8 * i)) & 0xffu;
          p1 &= f1 >> c;
          p2 &= f2 >> c;
        }
      const uint32_t k = (p1 & 1u) | ((p2 & 1u) << 1);
      r[j] = k == 0 ? r0 : k == 1 ? r1 : k == 2 ? r2 : r3;  // hg_logr[p1 | 2 p2]
    }
    double2* o = reinterpret_cast<double2*>(out) + 4 * q;
#pragma unroll
    for (int j = 0; j < 4; ++j) __stcs(o + j, make_double2(r[2 * j], r[2 * j + 1]));
  }
}

// DAG (d <= 8): graph_log_reward = sum_j cache[j][parents_j] in j order (dag.cpp:313-322), the
// cache in shared memory; 4 terminals per thread per pass (16-byte loads of each word)
template <int SWM>
__global__ void __launch_bounds__(256) k_reward_dag(EnvParams P, const uint32_t* __restrict__ st, int64_t n4,
                                                    double* __restrict__ out) {
  __shared__ double cache[kMaxDagD << kMaxDagD];
  const int d = P.dag_d;
  for (int i = threadIdx.x; i < (d << d); i += blockDim.x) cache[i] = P.dag_cache[i];
  __syncthreads();
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += (int64_t)gridDim.x * blockDim.x) {
    uint4 v[SWM];
#pragma unroll
    for (int k = 0; k < SWM; ++k) v[k] = __ldcs(reinterpret_cast<const uint4*>(st + (size_t)k * 4 * n4) + q);
    double r[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t rows[2 * SWM];
#pragma unroll
      for (int k = 0; k < SWM; ++k) {
        const uint32_t x = j == 0 ? v[k].x : j == 1 ? v[k].y : j == 2 ? v[k].z : v[k].w;
        rows[2 * k] = x & 0xffffu;
        rows[2 * k + 1] = x >> 16;
      }
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < 2 * SWM; ++c) {
        if (c >= d) break;
        uint32_t par = 0;
#pragma unroll
        for (int u = 0; u < 2 * SWM; ++u)
          if (u < d) par |= ((rows[u] >> c) & 1u) << u;
        acc += cache[(c << d) + par];
      }
      r[j] = acc;
    }
    __stcs(reinterpret_cast<double2*>(out) + 2 * q, make_double2(r[0], r[1]));
    __stcs(reinterpret_cast<double2*>(out) + 2 * q + 1, make_double2(r[2], r[3]));
  }
}

int reward_grid(const Ctx& c, int64_t n, int per_thread) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
  const int64_t threads = (n + per_thread - 1) / per_thread;
  return (int)std::max<int64_t>(1, std::min<int64_t>((threads + 255) / 256, (int64_t)sms * 8));
}

}  // namespace

void reward_free(Ctx& c) {
  if (c.d_is_rowtab) cudaFree(c.d_is_rowtab);
  c.d_is_rowtab = nullptr;
}

// out[i] = log R of packed terminal state i (word-major SoA [SW][n]); device pointers,
// stream-ordered on the ctx stream; contract violations (not a terminal state) raise the
// ctx error word
void reward_soa(Ctx& c, const uint32_t* st, int64_t n, double* out) {
  if (n <= 0) return;
  const EnvParams& P = c.P;
  int32_t* err = c.batch.counters + 3;
  const int grid = reward_grid(c, n, 4);
  const int grid1 = reward_grid(c, n, 1);
  ProfScope ps(c, "k_reward");
  switch (c.env.kind) {
    case GFNX_ENV_HYPERGRID:
      if (P.SW == 1 && P.hg_dim <= 4 && P.hg_side <= 32 && n % 8 == 0)
        k_reward_hg<<<reward_grid(c, n, 8), 256, 0, c.stream>>>(P, st, n / 8, out);
      else
        k_reward_soa<HypergridEnv, 16><<<grid, 256, 0, c.stream>>>(P, st, n, out, err);
      break;
    case GFNX_ENV_DAG:
      if (P.SW == 3 && n % 4 == 0)  // d = 5, 6
        k_reward_dag<3><<<grid, 256, 0, c.stream>>>(P, st, n / 4, out);
      else if (P.SW == 4 && n % 4 == 0)  // d = 7, 8
        k_reward_dag<4><<<grid, 256, 0, c.stream>>>(P, st, n / 4, out);
      else
        k_reward_soa<DagEnv, 16><<<grid, 256, 0, c.stream>>>(P, st, n, out, err);
      break;
    case GFNX_ENV_ISING:
      if (c.env.is_side == 10) {
        if (!c.d_is_rowtab) {  // the reference's row sums per site and neighbour pattern
          const int D = P.is_D;
          std::vector<double> tab((size_t)D * 16, 0.0);
          for (int a = 0; a < D; ++a)
            for (int p = 0; p < 16; ++p) {
              double row = 0.0;
              for (int q = 0; q < 4; ++q) {
                if (c.h_is_nbr[(size_t)a * 4 + q] < 0) continue;
                row += c.h_is_J[(size_t)a * 4 + q] * (((p >> q) & 1) ? 1.0 : -1.0);
              }
              tab[(size_t)a * 16 + p] = row;
            }
          cuda_check(cudaMalloc(&c.d_is_rowtab, sizeof(double) * tab.size()), "ising row table");
          cuda_check(cudaMemcpy(c.d_is_rowtab, tab.data(), sizeof(double) * tab.size(), cudaMemcpyHostToDevice),
                     "ising row table");
        }
        k_reward_ising<10><<<grid1, 256, 0, c.stream>>>(n, P.SW, st, c.d_is_rowtab, out, err);
      } else {
        k_reward_soa<IsingEnv, 16><<<grid, 256, 0, c.stream>>>(P, st, n, out, err);
      }
      break;
    case GFNX_ENV_BITSEQ:
      if ((P.bs_nbits + 31) / 32 == 4 && P.bs_k == 8) {
        k_reward_bitseq<4><<<grid1, 256, P.n_modes * 4 * 4, c.stream>>>(P, n, st, out, err);
      } else {
        k_reward_soa<BitseqEnv, 16><<<grid, 256, 0, c.stream>>>(P, st, n, out, err);
      }
      break;
  }
  c.launches++;
  cuda_check(cudaGetLastError(), "reward launch");
}

}  // namespace gfnx
