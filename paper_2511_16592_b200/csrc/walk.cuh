// walk.cuh — backward moves of the four device environments, for the uniform backward
// walks of backward_rollout (env_core.hpp:314-370), mc_terminal_logprob (exact.hpp:229-241)
// and the EB-GFN back-and-forth proposal (ising.cpp:252-360).
//
//   bwd_count(P, s)        #legal backward actions = count_legal(backward_action_mask)
//   bwd_pick(P, s, q)      the q-th legal backward action in index order
//   bwd_apply(P, s, ab)    backward_step_instance, returning get_forward_action(s', ab, s)
//
// Reference masks / steps / forward actions (file:line):
//   hypergrid hypergrid.cpp:34-41 (step), :52-61 (mask), get_forward_action = same index
//   bitseq NAR sequences.cpp:348-350 (mask), :375-376 (forward action pos * vocab + token)
//   Ising      ising.cpp:104-107 (mask = assigned sites), :118-121 (2 site + [spin > 0])
//   DAG        dag.cpp:407-417 (step, closure rebuilt), :433-443 (mask), same index
#pragma once

#include <type_traits>

#include "envs.cuh"

namespace gfnx {

__host__ __device__ __forceinline__ int popc32(uint32_t x) {
#ifdef __CUDA_ARCH__
  return __popc(x);
#else
  return __builtin_popcount(x);
#endif
}
__host__ __device__ __forceinline__ int popc64(uint64_t x) {
#ifdef __CUDA_ARCH__
  return __popcll(x);
#else
  return __builtin_popcountll(x);
#endif
}
// index of the q-th set bit (q < popc(x))
__host__ __device__ __forceinline__ int nth_bit64(uint64_t x, int q) {
  for (int i = 0; i < q; ++i) x &= x - 1;
#ifdef __CUDA_ARCH__
  return __ffsll((long long)x) - 1;
#else
  return __builtin_ctzll(x);
#endif
}

template <class Env>
__host__ __device__ inline int bwd_count(const EnvParams& P, const typename Env::State& s) {
  if constexpr (std::is_same<Env, HypergridEnv>::value) {
    if (s.term) return 1;
    int n = 0;
    for (int j = 0; j < P.hg_dim; ++j) n += s.c(j) > 0;
    return n;
  } else if constexpr (std::is_same<Env, DagEnv>::value) {
    if (s.term) return 1;
    int n = 0;
    for (int u = 0; u < P.dag_d; ++u) n += popc32(s.adj.get(u));
    return n;
  } else if constexpr (std::is_same<Env, BitseqEnv>::value) {
    return P.bs_ar ? (s.count > 0 ? 1 : 0) : popc64(s.filled);
  } else {
    int n = 0;
    for (int w = 0; w < (P.is_D + 31) / 32; ++w) n += popc32(s.asg[w]);
    return n;
  }
}

template <class Env>
__host__ __device__ inline int bwd_pick(const EnvParams& P, const typename Env::State& s, int q) {
  if constexpr (std::is_same<Env, HypergridEnv>::value) {
    if (s.term) return P.stop;
    for (int j = 0; j < P.hg_dim; ++j)
      if (s.c(j) > 0 && q-- == 0) return j;
    return -1;
  } else if constexpr (std::is_same<Env, DagEnv>::value) {
    if (s.term) return P.stop;
    // edge actions in index order a = u (d - 1) + (v < u ? v : v - 1): row u ascending, v ascending
    for (int u = 0; u < P.dag_d; ++u) {
      const uint32_t row = s.adj.get(u);
      const int n = popc32(row);
      if (q < n) {
        const int v = nth_bit64(row, q);
        return u * (P.dag_d - 1) + (v < u ? v : v - 1);
      }
      q -= n;
    }
    return -1;
  } else if constexpr (std::is_same<Env, BitseqEnv>::value) {
    return P.bs_ar ? 0 : nth_bit64(s.filled, q);
  } else {
    for (int w = 0; w < (P.is_D + 31) / 32; ++w) {
      const int n = popc32(s.asg[w]);
      if (q < n) return 32 * w + nth_bit64(s.asg[w], q);
      q -= n;
    }
    return -1;
  }
}

// backward_action_mask entry ab at s (hypergrid.cpp:52-61, dag.cpp:433-443,
// sequences.cpp:348-350, ising.cpp:104-107)
template <class Env>
__host__ __device__ inline bool bwd_legal(const EnvParams& P, const typename Env::State& s, int ab) {
  if constexpr (std::is_same<Env, HypergridEnv>::value) {
    if (s.term) return ab == P.stop;
    return ab >= 0 && ab < P.hg_dim && s.c(ab) > 0;
  } else if constexpr (std::is_same<Env, DagEnv>::value) {
    if (s.term) return ab == P.stop;
    if (ab < 0 || ab >= P.stop) return false;
    int u, v;
    DagEnv::edge(ab, P.dag_d, u, v);
    return (s.adj.get(u) >> v) & 1;
  } else if constexpr (std::is_same<Env, BitseqEnv>::value) {
    if (P.bs_ar) return ab == 0 && s.count > 0;
    return ab >= 0 && ab < P.bs_slots && ((s.filled >> ab) & 1);
  } else {
    return ab >= 0 && ab < P.is_D && ((s.asg[ab >> 5] >> (ab & 31)) & 1);
  }
}

// one backward step s -> s' under backward action ab; returns the forward action s' -> s
template <class Env>
__host__ __device__ inline int bwd_apply(const EnvParams& P, typename Env::State& s, int ab) {
  s.step -= 1;
  if constexpr (std::is_same<Env, HypergridEnv>::value) {
    if (ab == P.stop) {
      s.term = false;
      return ab;
    }
    s.cw -= 1ull << (8 * ab);
    return ab;
  } else if constexpr (std::is_same<Env, DagEnv>::value) {
    if (ab == P.stop) {
      s.term = false;
      return ab;
    }
    int u, v;
    DagEnv::edge(ab, P.dag_d, u, v);
    uint32_t w[4] = {0u, 0u, 0u, 0u};
    const int sw = P.SW;
    EnvParams Q = P;
    Q.SW = sw < 4 ? sw : 4;
    DagEnv::pack(Q, s, w);
    w[u >> 1] &= ~(1u << (v + 16 * (u & 1)));
    DagEnv::unpack(Q, w, s);  // closure_from_adjacency
    return ab;
  } else if constexpr (std::is_same<Env, BitseqEnv>::value) {
    const int pos = P.bs_ar ? s.count - 1 : ab;  // AR: remove-last (get_forward_action = the token)
    const int tok = s.tok[pos];
    s.filled &= ~(1ull << pos);
    s.tok[pos] = 0;
    s.count -= 1;
    s.term = false;
    return P.bs_ar ? tok : pos * P.bs_vocab + tok;
  } else {
    const uint32_t bit = 1u << (ab & 31);
    const int up = (s.up[ab >> 5] & bit) ? 1 : 0;
    s.asg[ab >> 5] &= ~bit;
    s.up[ab >> 5] &= ~bit;
    s.count -= 1;
    s.term = false;
    return 2 * ab + up;
  }
}

// a packed terminal state as the env's terminal instance (hypergrid / DAG: the stop flag is
// not in the packed words; bitseq / Ising terminals are the fully assigned states)
template <class Env>
__host__ __device__ inline void unpack_terminal(const EnvParams& P, const uint32_t* w, typename Env::State& s) {
  Env::unpack(P, w, s);
  s.term = true;
  if constexpr (std::is_same<Env, HypergridEnv>::value) {
    int sum = 0;
    for (int j = 0; j < P.hg_dim; ++j) sum += s.c(j);
    s.step = sum + 1;
  } else if constexpr (std::is_same<Env, DagEnv>::value) {
    s.step = s.count + 1;
  } else {
    s.step = s.count;
  }
}

// is the packed state a valid terminal of the env? (contract_violation otherwise:
// backward_rollout's "non-terminal input", ising terminal_from_spins, sequence terminals)
template <class Env>
__host__ __device__ inline bool terminal_ok(const EnvParams& P, const typename Env::State& s) {
  if constexpr (std::is_same<Env, HypergridEnv>::value) {
    for (int j = 0; j < P.hg_dim; ++j)
      if (s.c(j) > P.hg_side - 1) return false;
    return true;
  } else if constexpr (std::is_same<Env, DagEnv>::value) {
    for (int u = 0; u < P.dag_d; ++u)  // acyclic: no vertex reaches itself through another
      if ((s.adj.get(u) >> u) & 1) return false;
    for (int u = 0; u < P.dag_d; ++u)
      for (int v = 0; v < P.dag_d; ++v)
        if (u != v && ((s.adj.get(u) >> v) & 1) && ((s.cl.get(u) >> v) & 1)) return false;
    return true;
  } else if constexpr (std::is_same<Env, BitseqEnv>::value) {
    return s.count == P.bs_slots;
  } else {
    return s.count == P.is_D;
  }
}

// length of the forward trajectory that ends in terminal s (all backward walks reach s0 in
// exactly this many steps)
template <class Env>
__host__ __device__ inline int walk_length(const EnvParams& P, const typename Env::State& s) {
  if constexpr (std::is_same<Env, HypergridEnv>::value || std::is_same<Env, DagEnv>::value) {
    return s.step;  // unpack_terminal: increments + un-stop
  } else {
    return s.count;
  }
}

}  // namespace gfnx
