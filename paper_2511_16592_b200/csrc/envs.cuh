// envs.cuh — device implementations of the four hot-path environments.
//
// Each env is a struct of static __host__ __device__ functions over a small
// register-resident State (SoA across trajectories, one State per thread):
//   reset, step (returns true on entering a terminal state), legal(a), num_parents,
//   backward_action, log_reward (fp64, reference operation order), pack (to the
//   packed state words shared with the oracle), and obs features (sparse one-hot).
//
// Reference methods followed (file:line):
//   hypergrid  proj/src/envs/hypergrid.cpp:17-119
//   bitseq NAR proj/src/envs/sequences.cpp:50-55, 236-300, 302-327, 354-373, 396-409, 427-443
//   ising      proj/src/envs/ising.cpp:40-51, 72-145
//   dag        proj/src/envs/dag.cpp:313-329, 373-466
//
// Rewards are bit-exact by construction: everything that goes through libm (log) is
// tabulated on the host with the reference expression; the device only selects table
// entries or performs the same fp64 additions in the same order.
#pragma once

#include "common.cuh"

namespace gfnx {

constexpr int kMaxHgDim = 8;
constexpr int kMaxSlots = 64;    // bitseq slots (n_bits / k)
constexpr int kMaxModeWords = 8; // 512 bits per mode
constexpr int kMaxIsingD = 256;
constexpr int kMaxDagD = 8;
constexpr int kMaxParents = 512;

struct EnvParams {
  int kind, A, Ab, O, T, stop, SW;
  int mdb;  // record delta log-reward
  // hypergrid
  int hg_dim, hg_side;
  uint32_t hg_f1[8], hg_f2[8];  // bit c: coordinate value c satisfies 0.25 < x  /  0.3 < x < 0.4
  double hg_logr[4];            // log(r0 + r1*p1 + r2*p2) for (p1, p2) in {0,1}^2, index p1 | 2 p2
  // bitseq (non-autoregressive, k-bit words)
  int bs_slots, bs_vocab, bs_k, bs_nbits, bs_words, n_modes;
  int bs_ar;                    // SeqScheme::kAutoregressiveFixed: tokens appended left to right
  const uint64_t* modes;        // [n_modes][bs_words], string bit i -> word i/64, bit 63 - i%64
  const double* bs_logr;        // [n_bits + 1]: -beta * d / n_bits
  // ising
  int is_D;
  const int16_t* is_nbr;        // [D][4] ascending neighbour indices (-1 pad)
  const double* is_J;           // [D][4] coupling values
  const double* is_Jd;          // [D][D] dense coupling (EB-GFN's learned model) or null
  // dag
  int dag_d;
  const double* dag_cache;      // [d][2^d]
  // -log(k), k = 0..kMaxParents (entry 0 unused)
  const double* neglog;
};

// ---------------------------------------------------------------------------
struct HypergridEnv {
  struct State {  // coordinate i in bits [8i, 8i + 8) of cw (register-resident: no local memory)
    uint64_t cw;
    int step;
    bool term;
    __host__ __device__ int c(int i) const { return (int)((cw >> (8 * i)) & 0xffu); }
  };
  __host__ __device__ static void reset(const EnvParams&, State& s) {
    s.cw = 0;
    s.step = 0;
    s.term = false;
  }
  __host__ __device__ static bool legal(const EnvParams& P, const State& s, int a) {
    if (s.term) return false;
    if (a == P.stop) return true;
    return s.c(a) < P.hg_side - 1;
  }
  __host__ __device__ static bool step(const EnvParams& P, State& s, int a) {
    s.step += 1;
    if (a == P.stop) {
      s.term = true;
      return true;
    }
    s.cw += 1ull << (8 * a);
    return false;
  }
  __host__ __device__ static int num_parents(const EnvParams& P, const State& s) {
    if (s.term) return 1;
    // nonzero coordinate bytes (bytes >= hg_dim are 0): high bit of ((b & 0x7f) + 0x7f) | b
    const uint64_t L7 = 0x7f7f7f7f7f7f7f7full;
    const uint64_t nz = (((s.cw & L7) + L7) | s.cw) & 0x8080808080808080ull;
#ifdef __CUDA_ARCH__
    return __popcll(nz);
#else
    return __builtin_popcountll(nz);
#endif
  }
  // every legal forward action as a bit mask (bit a <-> action a), SWAR over the coordinate
  // bytes: for c < 128 and side - 1 <= 128 the byte (c | 0x80) - (side - 1) keeps its high bit
  // iff c >= side - 1; the multiply gathers the per-byte flags into bits 0..7
  __host__ __device__ static uint32_t legal_mask(const EnvParams& P, const State& s) {
    if (s.term) return 0u;
    uint32_t m = 0;
    if (P.hg_side <= 128) {
      const uint64_t H = 0x8080808080808080ull;
      const uint64_t ge = ((s.cw | H) - 0x0101010101010101ull * (uint64_t)(P.hg_side - 1)) & H;
      m = (uint32_t)((((~ge & H) >> 7) * 0x0102040810204080ull) >> 56) & ((1u << P.hg_dim) - 1u);
    } else {
      for (int i = 0; i < P.hg_dim; ++i) m |= (s.c(i) < P.hg_side - 1 ? 1u : 0u) << i;
    }
    return m | (1u << P.stop);
  }
  __host__ __device__ static int backward_action(const EnvParams&, int a) { return a; }
  __host__ __device__ static double log_reward(const EnvParams& P, const State& s) {
    uint32_t p1 = 1, p2 = 1;
    for (int i = 0; i < P.hg_dim; ++i) {
      const int c = s.c(i);
      p1 &= (P.hg_f1[c >> 5] >> (c & 31)) & 1;
      p2 &= (P.hg_f2[c >> 5] >> (c & 31)) & 1;
    }
    return P.hg_logr[p1 | (p2 << 1)];
  }
  __host__ __device__ static void pack(const EnvParams& P, const State& s, uint32_t* w) {
    // byte i = coordinate i: the packed words are the little-endian bytes of cw
    w[0] = (uint32_t)s.cw;
    if (P.SW > 1) w[1] = (uint32_t)(s.cw >> 32);
    for (int i = 2; i < P.SW; ++i) w[i] = 0;
  }
  __host__ __device__ static void unpack(const EnvParams& P, const uint32_t* w, State& s) {
    reset(P, s);
    s.cw = (uint64_t)w[0] | (P.SW > 1 ? (uint64_t)w[1] << 32 : 0ull);
    if (P.hg_dim < 8) s.cw &= (1ull << (8 * P.hg_dim)) - 1ull;
  }
  // active one-hot features (value 1.0): i * side + c_i   (hypergrid.cpp:82-85)
  template <class F>
  __host__ __device__ static void features(const EnvParams& P, const State& s, F&& f) {
    for (int i = 0; i < P.hg_dim; ++i) f(i * P.hg_side + s.c(i), 1.0);
  }
  // change of the observation caused by action a taken in s (for incremental layer 1)
  template <class F>
  __host__ __device__ static void delta_features(const EnvParams& P, const State& s, int a, F&& f) {
    if (a == P.stop) return;
    f(a * P.hg_side + s.c(a), -1.0f);
    f(a * P.hg_side + s.c(a) + 1, 1.0f);
  }
};

// ---------------------------------------------------------------------------
struct BitseqEnv {
  struct State {
    uint8_t tok[kMaxSlots];
    uint64_t filled;
    int count;
    int step;
    bool term;
  };
  __host__ __device__ static void reset(const EnvParams&, State& s) {
    for (int i = 0; i < kMaxSlots; ++i) s.tok[i] = 0;
    s.filled = 0;
    s.count = 0;
    s.step = 0;
    s.term = false;
  }
  // action_mask (sequences.cpp:302-327): NAR every word of every empty slot; AR fixed every
  // token until terminal
  __host__ __device__ static bool legal(const EnvParams& P, const State& s, int a) {
    if (s.term) return false;
    if (P.bs_ar) return a >= 0 && a < P.bs_vocab;
    return !((s.filled >> (a / P.bs_vocab)) & 1);
  }
  __host__ __device__ static bool step(const EnvParams& P, State& s, int a) {  // sequences.cpp:236-267
    s.step += 1;
    const int pos = P.bs_ar ? s.count : a / P.bs_vocab;
    s.tok[pos] = (uint8_t)(P.bs_ar ? a : a % P.bs_vocab);
    s.filled |= 1ull << pos;
    s.count += 1;
    if (s.count == P.bs_slots) {
      s.term = true;
      return true;
    }
    return false;
  }
  // #legal backward actions (sequences.cpp:329-352): NAR the filled slots, AR remove-last
  __host__ __device__ static int num_parents(const EnvParams& P, const State& s) {
    return P.bs_ar ? (s.count > 0 ? 1 : 0) : s.count;
  }
  __host__ __device__ static int backward_action(const EnvParams& P, int a) { return P.bs_ar ? 0 : a / P.bs_vocab; }
  // min Hamming distance to the mode set (ModeSet::log_reward sequences.cpp:50-55)
  __host__ __device__ static int best_distance(const EnvParams& P, const State& s) {
    uint64_t bits[kMaxModeWords];
    for (int w = 0; w < kMaxModeWords; ++w) bits[w] = 0;
    int pos = 0;
    for (int i = 0; i < P.bs_slots; ++i)
      for (int b = P.bs_k - 1; b >= 0; --b, ++pos)
        if ((s.tok[i] >> b) & 1) bits[pos >> 6] |= 1ull << (63 - (pos & 63));
    int best = P.bs_nbits + 1;
    for (int m = 0; m < P.n_modes; ++m) {
      int h = 0;
      for (int w = 0; w < P.bs_words; ++w) {
#ifdef __CUDA_ARCH__
        h += __popcll(bits[w] ^ P.modes[m * P.bs_words + w]);
#else
        h += __builtin_popcountll(bits[w] ^ P.modes[m * P.bs_words + w]);
#endif
      }
      best = h < best ? h : best;
    }
    return best;
  }
  __host__ __device__ static double log_reward(const EnvParams& P, const State& s) {
    return P.bs_logr[best_distance(P, s)];
  }
  __host__ __device__ static void pack(const EnvParams& P, const State& s, uint32_t* w) {
    for (int i = 0; i < P.SW; ++i) w[i] = 0;
    const int tw = (P.bs_slots + 3) / 4;
    for (int i = 0; i < P.bs_slots; ++i)
      if ((s.filled >> i) & 1) {
        w[i >> 2] |= (uint32_t)s.tok[i] << (8 * (i & 3));
        w[tw + (i >> 5)] |= 1u << (i & 31);
      }
  }
  __host__ __device__ static void unpack(const EnvParams& P, const uint32_t* w, State& s) {
    reset(P, s);
    const int tw = (P.bs_slots + 3) / 4;
    for (int i = 0; i < P.bs_slots; ++i)
      if ((w[tw + (i >> 5)] >> (i & 31)) & 1) {
        s.tok[i] = (uint8_t)(w[i >> 2] >> (8 * (i & 3)));
        s.filled |= 1ull << i;
        s.count += 1;
      }
  }
  // sequences.cpp:396-409: slot i one-hot over vocab+1 (empty -> vocab), then filled/n
  template <class F>
  __host__ __device__ static void features(const EnvParams& P, const State& s, F&& f) {
    const int width = P.bs_vocab + 1;
    for (int i = 0; i < P.bs_slots; ++i)
      f(i * width + (((s.filled >> i) & 1) ? s.tok[i] : P.bs_vocab), 1.0);
    f(P.bs_slots * width, (double)s.count / P.bs_slots);
  }
  // (AR: the action fills slot s.count of the state it is taken in)
  template <class F>
  __host__ __device__ static void delta_features(const EnvParams& P, const State& s, int a, F&& f) {
    const int width = P.bs_vocab + 1, pos = P.bs_ar ? s.count : a / P.bs_vocab;
    f(pos * width + P.bs_vocab, -1.0f);
    f(pos * width + (P.bs_ar ? a : a % P.bs_vocab), 1.0f);
    f(P.bs_slots * width, 1.0f / (float)P.bs_slots);
  }
};

// ---------------------------------------------------------------------------
struct IsingEnv {
  static constexpr int kW = kMaxIsingD / 32;
  struct State {
    uint32_t asg[kW], up[kW];
    int count;
    int step;
    bool term;
  };
  __host__ __device__ static void reset(const EnvParams&, State& s) {
    for (int i = 0; i < kW; ++i) s.asg[i] = s.up[i] = 0;
    s.count = 0;
    s.step = 0;
    s.term = false;
  }
  __host__ __device__ static bool legal(const EnvParams&, const State& s, int a) {
    if (s.term) return false;
    const int site = a >> 1;
    return !((s.asg[site >> 5] >> (site & 31)) & 1);
  }
  __host__ __device__ static bool step(const EnvParams& P, State& s, int a) {
    s.step += 1;
    const int site = a >> 1;
    s.asg[site >> 5] |= 1u << (site & 31);
    if (a & 1) s.up[site >> 5] |= 1u << (site & 31);
    s.count += 1;
    if (s.count == P.is_D) {
      s.term = true;
      return true;
    }
    return false;
  }
  __host__ __device__ static int num_parents(const EnvParams&, const State& s) { return s.count; }
  __host__ __device__ static int backward_action(const EnvParams&, int a) { return a >> 1; }
  __host__ __device__ static int spin(const State& s, int i) {
    if (!((s.asg[i >> 5] >> (i & 31)) & 1)) return 0;
    return ((s.up[i >> 5] >> (i & 31)) & 1) ? 1 : -1;
  }
  // -E = quad = sum_a s_a * (sum_b J_ab s_b), dense row sums reduce to the ascending
  // neighbour list since the remaining terms are exact zeros (ising.cpp:40-51).
  __host__ __device__ static double log_reward(const EnvParams& P, const State& s) {
    double quad = 0.0;
    if (P.is_Jd) {  // dense ising_energy (ising.cpp:40-51): the EB-GFN model coupling
      for (int a = 0; a < P.is_D; ++a) {
        double row = 0.0;
        for (int b = 0; b < P.is_D; ++b) row += P.is_Jd[(size_t)a * P.is_D + b] * (double)spin(s, b);
        quad += (double)spin(s, a) * row;
      }
      return -(-quad);
    }
    for (int a = 0; a < P.is_D; ++a) {
      double row = 0.0;
      for (int q = 0; q < 4; ++q) {
        const int b = P.is_nbr[a * 4 + q];
        if (b >= 0) row += P.is_J[a * 4 + q] * (double)spin(s, b);
      }
      quad += (double)spin(s, a) * row;
    }
    const double energy = -quad;
    return -energy;
  }
  __host__ __device__ static void pack(const EnvParams& P, const State& s, uint32_t* w) {
    const int nw = P.SW / 2;
    for (int i = 0; i < nw; ++i) {
      w[i] = s.asg[i];
      w[nw + i] = s.up[i];
    }
  }
  __host__ __device__ static void unpack(const EnvParams& P, const uint32_t* w, State& s) {
    reset(P, s);
    const int nw = P.SW / 2;
    for (int i = 0; i < nw; ++i) {
      s.asg[i] = w[i];
      s.up[i] = w[nw + i];
#ifdef __CUDA_ARCH__
      s.count += __popc(w[i]);
#else
      s.count += __builtin_popcount(w[i]);
#endif
    }
  }
  // ising.cpp:122-129: 3 * site + {-1 -> 0, +1 -> 1, unassigned -> 2}
  template <class F>
  __host__ __device__ static void features(const EnvParams& P, const State& s, F&& f) {
    for (int i = 0; i < P.is_D; ++i) {
      const int v = spin(s, i);
      f(3 * i + (v == 0 ? 2 : (v > 0 ? 1 : 0)), 1.0);
    }
  }
  template <class F>
  __host__ __device__ static void delta_features(const EnvParams&, const State&, int a, F&& f) {
    const int site = a >> 1;
    f(3 * site + 2, -1.0f);
    f(3 * site + (a & 1), 1.0f);
  }
};

// ---------------------------------------------------------------------------
// eight 16-bit rows in two registers (dynamic row index without local memory)
struct U16x8 {
  uint64_t lo, hi;
  __host__ __device__ uint32_t get(int i) const {
    return (uint32_t)((((i & 4) ? hi : lo) >> (16 * (i & 3))) & 0xffffu);
  }
  __host__ __device__ void orv(int i, uint32_t v) {
    const uint64_t m = (uint64_t)(v & 0xffffu) << (16 * (i & 3));
    if (i & 4)
      hi |= m;
    else
      lo |= m;
  }
};

struct DagEnv {
  struct State {
    U16x8 adj, cl;  // adj row u bit v: u->v ; cl row a bit b: b ~> a
    int count;
    int step;
    bool term;
  };
  __host__ __device__ static void reset(const EnvParams&, State& s) {
    s.adj.lo = s.adj.hi = 0;
    // cl[a] = 1 << a
    s.cl.lo = 0x0008000400020001ull;
    s.cl.hi = 0x0080004000200010ull;
    s.count = 0;
    s.step = 0;
    s.term = false;
  }
  __host__ __device__ static void edge(int a, int d, int& u, int& v) {  // dag.cpp:379-383
    u = a / (d - 1);
    const int r = a % (d - 1);
    v = r < u ? r : r + 1;
  }
  __host__ __device__ static bool legal(const EnvParams& P, const State& s, int a) {
    if (s.term) return false;
    if (a == P.stop) return true;
    int u, v;
    edge(a, P.dag_d, u, v);
    return !((s.adj.get(u) >> v) & 1) && !((s.cl.get(u) >> v) & 1);
  }
  __host__ __device__ static bool step(const EnvParams& P, State& s, int a) {
    s.step += 1;
    if (a == P.stop) {
      s.term = true;
      return true;
    }
    int u, v;
    edge(a, P.dag_d, u, v);
    s.adj.orv(u, 1u << v);
    const uint32_t row_u = s.cl.get(u);  // closure_update dag.cpp:324-329
    for (int q = 0; q < P.dag_d; ++q)
      if ((s.cl.get(q) >> v) & 1) s.cl.orv(q, row_u);
    s.count += 1;
    return false;
  }
  __host__ __device__ static int num_parents(const EnvParams&, const State& s) {
    return s.term ? 1 : s.count;
  }
  __host__ __device__ static int backward_action(const EnvParams&, int a) { return a; }
  __host__ __device__ static double log_reward(const EnvParams& P, const State& s) {
    const int d = P.dag_d;
    double acc = 0.0;
    for (int j = 0; j < d; ++j) {
      uint32_t parents = 0;
      for (int u = 0; u < d; ++u)
        if ((s.adj.get(u) >> j) & 1) parents |= 1u << u;
      acc += P.dag_cache[j * (1 << d) + parents];
    }
    return acc;
  }
  __host__ __device__ static void pack(const EnvParams& P, const State& s, uint32_t* w) {
    // row u in 16-bit half (u & 1) of word u >> 1: the words are the halves of adj.lo/hi
    const uint32_t x[4] = {(uint32_t)s.adj.lo, (uint32_t)(s.adj.lo >> 32), (uint32_t)s.adj.hi,
                           (uint32_t)(s.adj.hi >> 32)};
#pragma unroll
    for (int i = 0; i < 4; ++i)  // (constant indices: x stays in registers)
      if (i < P.SW) w[i] = x[i];
    for (int i = 4; i < P.SW; ++i) w[i] = 0u;
  }
  // adjacency only; the transpose closure is rebuilt (closure_from_adjacency dag.cpp:331-346)
  __host__ __device__ static void unpack(const EnvParams& P, const uint32_t* w, State& s) {
    reset(P, s);
    const int d = P.dag_d;
#pragma unroll
    for (int u = 0; u < kMaxDagD; ++u) {  // constant word indices: the caller's w stays in registers
      if (u >= d) break;
      const uint32_t row = (w[u >> 1] >> (16 * (u & 1))) & 0xffffu;
      s.adj.orv(u, row);
#ifdef __CUDA_ARCH__
      s.count += __popc(row);
#else
      s.count += __builtin_popcount(row);
#endif
    }
    U16x8 cl{0, 0};
    for (int a = 0; a < d; ++a) {
      uint32_t c = 1u << a;
      for (int b = 0; b < d; ++b)
        if ((s.adj.get(b) >> a) & 1) c |= 1u << b;
      cl.orv(a, c);
    }
    for (int k = 0; k < d; ++k)
      for (int a = 0; a < d; ++a)
        if ((cl.get(a) >> k) & 1) cl.orv(a, cl.get(k));
    for (int a = d; a < kMaxDagD; ++a) cl.orv(a, 1u << a);
    s.cl = cl;
  }
  template <class F>
  __host__ __device__ static void features(const EnvParams& P, const State& s, F&& f) {
    for (int u = 0; u < P.dag_d; ++u)
      for (int v = 0; v < P.dag_d; ++v)
        if ((s.adj.get(u) >> v) & 1) f(u * P.dag_d + v, 1.0);
  }
  template <class F>
  __host__ __device__ static void delta_features(const EnvParams& P, const State&, int a, F&& f) {
    if (a == P.stop) return;
    int u, v;
    edge(a, P.dag_d, u, v);
    f(u * P.dag_d + v, 1.0f);
  }
};

}  // namespace gfnx
