/*
 * gfn_oracle.c — CPU oracle (TEST INFRASTRUCTURE ONLY; see gfn_oracle.h).
 *
 * fp64 restatement of the reference hot path with the reference's operation
 * order. Built with -ffp-contract=off (oracle/Makefile) so that, like the
 * "portable" reference build in oracle/_ref, no FMA contraction happens; the
 * two then agree bit for bit on rollouts, rewards, losses and parameters.
 */
#include "gfn_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ====================================================================== */
/* RNG — proj/src/rng.cpp                                                  */
/* ====================================================================== */

static const uint64_t kParity = 0x1BD11BDAA9FC1A22ULL; /* rng.cpp:12 */
static const int kRot[8] = {16, 42, 12, 31, 16, 32, 24, 21}; /* rng.cpp:13 */

static inline uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

void orc_make_key(uint64_t seed, uint64_t out[2]) { /* rng.cpp:17 */
  out[0] = 0x9E3779B97F4A7C15ULL;
  out[1] = seed;
}

void orc_threefry2x64(const uint64_t key[2], uint64_t c0, uint64_t c1, uint64_t out[2]) {
  /* rng.cpp:19-34: 20 rounds, key injection every 4 rounds */
  const uint64_t ks[3] = {key[0], key[1], key[0] ^ key[1] ^ kParity};
  uint64_t x0 = c0 + ks[0];
  uint64_t x1 = c1 + ks[1];
  for (int round = 0; round < 20; ++round) {
    x0 += x1;
    x1 = rotl64(x1, kRot[round % 8]);
    x1 ^= x0;
    if (round % 4 == 3) {
      const int s = round / 4 + 1;
      x0 += ks[s % 3];
      x1 += ks[(s + 1) % 3] + (uint64_t)s;
    }
  }
  out[0] = x0;
  out[1] = x1;
}

void orc_fold_in(const uint64_t key[2], uint64_t index, uint64_t out[2]) { /* rng.cpp:36-39 */
  orc_threefry2x64(key, index, 0x3C6EF372FE94F82BULL, out);
}

static inline double to_unit(uint64_t w) { return (double)(w >> 11) * 0x1.0p-53; } /* :47-50 */

double orc_uniform_scalar(const uint64_t key[2]) { /* rng.cpp:64-66 */
  uint64_t w[2];
  orc_threefry2x64(key, 0, 0, w);
  return to_unit(w[0]);
}

static void random_uniform(const uint64_t key[2], size_t n, double* out) { /* rng.cpp:52-62 */
  for (size_t i = 0; i < n; i += 2) {
    uint64_t w[2];
    orc_threefry2x64(key, i / 2, 0, w);
    out[i] = to_unit(w[0]);
    if (i + 1 < n) out[i + 1] = to_unit(w[1]);
  }
}

static void random_normal(const uint64_t key[2], size_t n, double* out) { /* rng.cpp:68-80 */
  for (size_t i = 0; i < n; i += 2) {
    uint64_t w[2];
    orc_threefry2x64(key, i / 2, 1, w);
    double u1 = to_unit(w[0]);
    double u2 = to_unit(w[1]);
    if (u1 <= 0.0) u1 = 0x1.0p-53;
    const double r = sqrt(-2.0 * log(u1));
    out[i] = r * cos(2.0 * M_PI * u2);
    if (i + 1 < n) out[i + 1] = r * sin(2.0 * M_PI * u2);
  }
}

static int random_range(const uint64_t key[2], int n) { /* rng.cpp:82-85 */
  return (int)(orc_uniform_scalar(key) * n) % n;
}

int32_t orc_categorical(const uint64_t key[2], const double* w, int32_t n) { /* rng.cpp:87-100 */
  double total = 0.0;
  for (int i = 0; i < n; ++i) total += w[i];
  if (!(total > 0.0)) return -1;
  const double u = orc_uniform_scalar(key) * total;
  double acc = 0.0;
  for (int i = 0; i < n; ++i) {
    acc += w[i];
    if (u < acc) return i;
  }
  for (int i = n - 1; i >= 0; --i)
    if (w[i] > 0.0) return i;
  return n - 1;
}

int32_t orc_eps_uniform(const double* logits, const uint8_t* mask, int32_t n, double eps,
                        double* probs) { /* objectives.cpp:242-264 */
  int legal = 0;
  double hi = -INFINITY;
  for (int i = 0; i < n; ++i)
    if (mask[i]) {
      ++legal;
      if (logits[i] > hi) hi = logits[i];
    }
  if (legal == 0) return 0;
  if (!isfinite(hi)) return -1;
  double z = 0.0;
  for (int i = 0; i < n; ++i) {
    probs[i] = 0.0;
    if (mask[i]) {
      probs[i] = exp(logits[i] - hi);
      z += probs[i];
    }
  }
  const double u = eps / legal;
  for (int i = 0; i < n; ++i)
    if (mask[i]) probs[i] = (1.0 - eps) * probs[i] / z + u;
  return legal;
}

double orc_schedule_value(const gfnx_schedule* s, int64_t step) { /* optim.cpp:45-66 */
  if (s->warmup > 0 && step < s->warmup)
    return s->start_value * (double)step / (double)s->warmup;
  switch (s->kind) {
    case 0:
      return s->start_value;
    case 1: {
      if (s->horizon <= 0) return s->end_value;
      double prog = (double)(step - s->warmup) / (double)s->horizon;
      if (prog > 1.0) prog = 1.0;
      return s->start_value + (s->end_value - s->start_value) * prog;
    }
    case 2: {
      if (s->horizon <= 0) return s->end_value;
      double prog = (double)(step - s->warmup) / (double)s->horizon;
      if (prog > 1.0) prog = 1.0;
      return s->end_value + 0.5 * (s->start_value - s->end_value) * (1.0 + cos(M_PI * prog));
    }
  }
  return s->start_value;
}

/* ====================================================================== */
/* Environment state                                                        */
/* ====================================================================== */

#define ORC_MAX_SLOTS 256

typedef struct orc_state {
  int32_t is_terminal;
  int32_t step_count;
  int32_t count;               /* filled (bitseq) / assigned (ising) / num_edges (dag) */
  int32_t v[ORC_MAX_SLOTS];    /* coords / tokens (-1 empty) / spins (0,+1,-1) */
  uint32_t adj[16];            /* dag adjacency rows (bit v = edge u->v) */
  uint32_t closure_t[16];      /* dag transpose closure, reflexive */
} orc_state;

struct orc_trainer {
  gfnx_env_desc env;
  gfnx_train_desc tr;
  char err[256];
  /* shape */
  int A, Ab, O, T, stop, state_words;
  /* bitseq */
  int bs_slots, bs_vocab, n_modes;
  uint8_t* modes; /* [n_modes x n_bits] of 0/1 */
  /* ising */
  int is_D;
  double* J; /* D x D */
  /* dag */
  int dag_d;
  double* dag_cache; /* [d][2^d] */
  uint32_t dag_true_adj[16];
  /* mlp */
  int n_trunk;
  int dims[10]; /* dims[0] = O, dims[1..n_trunk] hidden */
  int64_t off_w[10], off_b[10];
  int64_t off_fw, off_fb, off_bw, off_bb, off_flw, off_flb;
  int64_t n_params;
  double* params;
  double log_z;
  double* grads;
  double dlogz;
  double* adam_m;
  double* adam_v;
  int64_t adam_t;
  double z_m, z_v;
  int64_t z_t;
  /* batch slice */
  int B, b0, nb;
  int32_t* lengths;
  int32_t* fwd_actions;
  int32_t* bwd_actions;
  double* log_rewards;
  double* log_pb;
  double* delta;
  uint32_t* terminal_state;
  orc_state* states; /* [nb * (T+1)] visited states */
  int has_batch;
};

static int fail(orc_trainer* tr, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(tr->err, sizeof tr->err, fmt, ap);
  va_end(ap);
  return -1;
}

/* ---------------- hypergrid (hypergrid.cpp) ---------------- */

static double grid_log_reward(const orc_trainer* tr, const int32_t* coords) { /* :111-119 */
  double prod1 = 1.0, prod2 = 1.0;
  const int side = tr->env.hg_side;
  for (int i = 0; i < tr->env.hg_dim; ++i) {
    const double x = fabs((double)coords[i] / (side - 1) - 0.5);
    if (!(0.25 < x)) prod1 = 0.0;
    if (!(0.3 < x && x < 0.4)) prod2 = 0.0;
  }
  return log(tr->env.hg_r0 + tr->env.hg_r1 * prod1 + tr->env.hg_r2 * prod2);
}

/* ---------------- bitseq NAR + ModeSet (sequences.cpp) ---------------- */

static int bitseq_log_reward_best(const orc_trainer* tr, const orc_state* s) {
  /* ModeSet::log_reward (sequences.cpp:50-55) over encode_terminal bits (:427-443) */
  const int n = tr->env.bs_n_bits, k = tr->env.bs_k;
  uint8_t bits[2048];
  for (int i = 0; i < tr->bs_slots; ++i)
    for (int b = k - 1, j = 0; b >= 0; --b, ++j) bits[i * k + j] = (uint8_t)((s->v[i] >> b) & 1);
  int best = n + 1;
  for (int m = 0; m < tr->n_modes; ++m) {
    const uint8_t* mode = tr->modes + (size_t)m * n;
    int h = 0;
    for (int i = 0; i < n; ++i) h += bits[i] != mode[i];
    if (h < best) best = h;
  }
  return best;
}

static double bitseq_log_reward(const orc_trainer* tr, const orc_state* s) {
  const int best = bitseq_log_reward_best(tr, s);
  return -tr->env.bs_beta * (double)best / (double)tr->env.bs_n_bits;
}

static int generate_modes(orc_trainer* tr) { /* sequences.cpp:72-98 */
  static const char* words[5] = {"00000000", "11111111", "11110000", "00001111", "00111100"};
  const int n = tr->env.bs_n_bits;
  if (n <= 0 || n % 8 != 0) return fail(tr, "generate_modes: need 8 | n");
  const int target = tr->env.bs_num_modes;
  if (target < 1) return fail(tr, "generate_modes: target_count must be positive");
  const int blocks = n / 8;
  double distinct = 1.0;
  for (int i = 0; i < blocks; ++i) distinct *= 5.0;
  const int cap = distinct < (double)target ? (int)distinct : target;
  tr->modes = (uint8_t*)calloc((size_t)cap * n, 1);
  uint64_t key[2], mkey[2];
  orc_make_key(tr->env.bs_modes_seed, key);
  orc_fold_in(key, 0x30DE, mkey); /* train.cpp:417-420 */
  uint64_t draw = 0;
  int count = 0;
  uint8_t* cand = (uint8_t*)malloc(n);
  while (count < cap) {
    for (int b = 0; b < blocks; ++b) {
      uint64_t k2[2];
      orc_fold_in(mkey, draw++, k2);
      const int w = random_range(k2, 5);
      for (int j = 0; j < 8; ++j) cand[b * 8 + j] = (uint8_t)(words[w][j] - '0');
    }
    /* std::set<std::string> insert: sorted, unique ('0' < '1' like 0 < 1) */
    int lo = 0, hi = count, found = 0;
    while (lo < hi) {
      const int mid = (lo + hi) / 2;
      const int c = memcmp(tr->modes + (size_t)mid * n, cand, n);
      if (c == 0) {
        found = 1;
        break;
      }
      if (c < 0) lo = mid + 1; else hi = mid;
    }
    if (found) continue;
    memmove(tr->modes + (size_t)(lo + 1) * n, tr->modes + (size_t)lo * n, (size_t)(count - lo) * n);
    memcpy(tr->modes + (size_t)lo * n, cand, n);
    ++count;
  }
  free(cand);
  tr->n_modes = count;
  return 0;
}

/* ---------------- ising (ising.cpp) ---------------- */

static void toroidal_coupling(orc_trainer* tr) { /* ising.cpp:15-31 */
  const int side = tr->env.is_side, d = side * side;
  tr->J = (double*)calloc((size_t)d * d, sizeof(double));
  static const int dr[4] = {1, -1, 0, 0}, dc[4] = {0, 0, 1, -1};
  for (int r = 0; r < side; ++r)
    for (int c = 0; c < side; ++c) {
      const int a = ((r + side) % side) * side + (c + side) % side;
      for (int q = 0; q < 4; ++q) {
        const int rr = r + dr[q], cc = c + dc[q];
        const int b = ((rr + side) % side) * side + (cc + side) % side;
        if (a != b) tr->J[(size_t)a * d + b] = tr->env.is_sigma;
      }
    }
}

static double ising_log_reward(const orc_trainer* tr, const orc_state* s) { /* :40-51,143-145 */
  const int d = tr->is_D;
  double quad = 0.0;
  for (int a = 0; a < d; ++a) {
    double row = 0.0;
    for (int b = 0; b < d; ++b) row += tr->J[(size_t)a * d + b] * s->v[b];
    quad += s->v[a] * row;
  }
  const double energy = -quad;
  return -energy;
}

/* ---------------- dag (dag.cpp) ---------------- */

static double cholesky_logdet(double* a, int n, int* ok) { /* dag.cpp:20-38 */
  double logdet = 0.0;
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j <= i; ++j) {
      double s = a[(size_t)i * n + j];
      for (int k = 0; k < j; ++k) s -= a[(size_t)i * n + k] * a[(size_t)j * n + k];
      if (i == j) {
        if (!(s > 0.0)) *ok = 0;
        a[(size_t)i * n + j] = sqrt(s);
        logdet += 2.0 * log(a[(size_t)i * n + j]);
      } else {
        a[(size_t)i * n + j] = s / a[(size_t)j * n + j];
      }
    }
  }
  return logdet;
}

static void cholesky_solve(const double* l, int n, double* b) { /* dag.cpp:41-54 */
  for (int i = 0; i < n; ++i) {
    double s = b[i];
    for (int k = 0; k < i; ++k) s -= l[(size_t)i * n + k] * b[k];
    b[i] = s / l[(size_t)i * n + i];
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = b[i];
    for (int k = i + 1; k < n; ++k) s -= l[(size_t)k * n + i] * b[k];
    b[i] = s / l[(size_t)i * n + i];
  }
}

static double log_multivariate_gamma(int ell, double a) { /* dag.cpp:56-60 */
  double v = 0.25 * ell * (ell - 1) * log(M_PI);
  for (int i = 1; i <= ell; ++i) v += lgamma(a + 0.5 * (1.0 - i));
  return v;
}

static int dag_build(orc_trainer* tr) {
  const int d = tr->env.dag_d, n = tr->env.dag_data_n;
  if (d < 1 || d > 16) return fail(tr, "dag env: d must lie in [1, 16]");
  if (n < 1) return fail(tr, "er dataset: n must be >= 1");
  /* generate_er_dataset (dag.cpp:70-119) with key fold_in(make_key(data_seed), 0xDA7A) */
  uint64_t root[2], key[2];
  orc_make_key(tr->env.dag_data_seed, root);
  orc_fold_in(root, 0xDA7A, key);
  int order[16];
  for (int i = 0; i < d; ++i) order[i] = i;
  for (int i = d - 1; i > 0; --i) {
    uint64_t k2[2];
    orc_fold_in(key, 1000 + (uint64_t)i, k2);
    const int j = random_range(k2, i + 1);
    const int t = order[i];
    order[i] = order[j];
    order[j] = t;
  }
  double p = 0.0;
  if (d > 1) {
    p = 2.0 * tr->env.dag_expected_in_degree / (d - 1);
    if (p > 1.0) p = 1.0;
  }
  uint64_t edge_key[2], weight_key[2], eps_key[2];
  orc_fold_in(key, 1, edge_key);
  orc_fold_in(key, 2, weight_key);
  orc_fold_in(key, 3, eps_key);
  double* weights = (double*)malloc(sizeof(double) * d * d);
  random_normal(weight_key, (size_t)d * d, weights);
  double tw[256] = {0};
  uint32_t adj[16] = {0};
  uint64_t draw = 0;
  for (int i = 0; i < d; ++i)
    for (int j = i + 1; j < d; ++j) {
      const int u = order[i], v = order[j];
      uint64_t k2[2];
      orc_fold_in(edge_key, draw++, k2);
      if (orc_uniform_scalar(k2) < p) {
        adj[u] |= 1u << v;
        tw[u * d + v] = weights[u * d + v];
      }
    }
  const double noise_sd = sqrt(0.1);
  double* eps = (double*)malloc(sizeof(double) * n * d);
  random_normal(eps_key, (size_t)n * d, eps);
  double* x = (double*)calloc((size_t)n * d, sizeof(double));
  for (int row = 0; row < n; ++row)
    for (int pos = 0; pos < d; ++pos) {
      const int j = order[pos];
      double mean = 0.0;
      for (int u = 0; u < d; ++u)
        if (adj[u] & (1u << j)) mean += tw[u * d + j] * x[(size_t)row * d + u];
      x[(size_t)row * d + j] = mean + noise_sd * eps[(size_t)row * d + j];
    }
  memcpy(tr->dag_true_adj, adj, sizeof adj);
  const uint32_t nmask = 1u << d;
  tr->dag_cache = (double*)calloc((size_t)d * nmask, sizeof(double));
  const double nn = (double)n;
  int ok = 1;
  if (tr->env.dag_score == GFNX_DAG_LINGAUSS) { /* LocalScoreCache::lingauss dag.cpp:163-212 */
    const double s2 = tr->env.dag_noise_var, w2 = tr->env.dag_weight_var;
    if (!(s2 > 0.0) || !(w2 > 0.0)) return fail(tr, "score cache: variances must be positive");
    double gram[256] = {0};
    for (int i = 0; i < n; ++i)
      for (int a = 0; a < d; ++a)
        for (int b = 0; b <= a; ++b) {
          const double v = x[(size_t)i * d + a] * x[(size_t)i * d + b];
          gram[a * d + b] += v;
          if (a != b) gram[b * d + a] += v;
        }
    for (int j = 0; j < d; ++j) {
      const double yy = gram[j * d + j];
      for (uint32_t mask = 0; mask < nmask; ++mask) {
        if (mask & (1u << j)) continue;
        int pa[16], np = 0;
        for (int i = 0; i < d; ++i)
          if (mask & (1u << i)) pa[np++] = i;
        double quad = yy / s2;
        double logdet = nn * log(s2);
        if (np > 0) {
          double bm[256], v[16];
          for (int a = 0; a < np; ++a) {
            v[a] = gram[pa[a] * d + j];
            for (int c = 0; c < np; ++c)
              bm[a * np + c] = gram[pa[a] * d + pa[c]] / s2 + (a == c ? 1.0 / w2 : 0.0);
          }
          const double logdet_b = cholesky_logdet(bm, np, &ok);
          double xs[16];
          memcpy(xs, v, sizeof(double) * np);
          cholesky_solve(bm, np, xs);
          double vx = 0.0;
          for (int a = 0; a < np; ++a) vx += v[a] * xs[a];
          quad -= vx / (s2 * s2);
          logdet += np * log(w2) + logdet_b;
        }
        tr->dag_cache[(size_t)j * nmask + mask] = -0.5 * (nn * log(2.0 * M_PI) + logdet + quad);
      }
    }
  } else { /* LocalScoreCache::bge dag.cpp:236-298 */
    const double alpha_mu = tr->env.dag_alpha_mu;
    const double alpha_w = tr->env.dag_alpha_w > 0.0 ? tr->env.dag_alpha_w : d + 2.0;
    if (!(alpha_mu > 0.0)) return fail(tr, "bge: alpha_mu must be positive");
    if (!(alpha_w > d - 1)) return fail(tr, "bge: alpha_w must exceed d - 1");
    double xbar[16] = {0};
    for (int i = 0; i < n; ++i)
      for (int a = 0; a < d; ++a) xbar[a] += x[(size_t)i * d + a];
    for (int a = 0; a < d; ++a) xbar[a] /= nn;
    double r[256] = {0};
    for (int i = 0; i < n; ++i)
      for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b)
          r[a * d + b] += (x[(size_t)i * d + a] - xbar[a]) * (x[(size_t)i * d + b] - xbar[b]);
    const double shrink = nn * alpha_mu / (nn + alpha_mu);
    for (int a = 0; a < d; ++a) {
      for (int b = 0; b < d; ++b) r[a * d + b] += shrink * xbar[a] * xbar[b];
      r[a * d + a] += 1.0;
    }
    double* logdet_r = (double*)calloc(nmask, sizeof(double));
    double* subset_ml = (double*)calloc(nmask, sizeof(double));
    for (uint32_t mask = 1; mask < nmask; ++mask) {
      int mem[16], ell = 0;
      for (int i = 0; i < d; ++i)
        if (mask & (1u << i)) mem[ell++] = i;
      double sub[256];
      for (int a = 0; a < ell; ++a)
        for (int b = 0; b < ell; ++b) sub[a * ell + b] = r[mem[a] * d + mem[b]];
      logdet_r[mask] = cholesky_logdet(sub, ell, &ok);
    }
    for (uint32_t mask = 1; mask < nmask; ++mask) {
      const int ell = __builtin_popcount(mask);
      const double dof = alpha_w - d + ell;
      double v = -0.5 * nn * ell * log(M_PI);
      v += 0.5 * ell * log(alpha_mu / (nn + alpha_mu));
      v += log_multivariate_gamma(ell, 0.5 * (nn + dof));
      v -= log_multivariate_gamma(ell, 0.5 * dof);
      v -= 0.5 * (nn + dof) * logdet_r[mask];
      subset_ml[mask] = v;
    }
    for (int j = 0; j < d; ++j)
      for (uint32_t mask = 0; mask < nmask; ++mask) {
        if (mask & (1u << j)) continue;
        tr->dag_cache[(size_t)j * nmask + mask] = subset_ml[mask | (1u << j)] - subset_ml[mask];
      }
    free(logdet_r);
    free(subset_ml);
  }
  free(weights);
  free(eps);
  free(x);
  if (!ok) return fail(tr, "cholesky: matrix not positive definite");
  return 0;
}

static double dag_graph_log_reward(const orc_trainer* tr, const uint32_t* adj) { /* :313-322 */
  const int d = tr->dag_d;
  double acc = 0.0;
  for (int j = 0; j < d; ++j) {
    uint32_t parents = 0;
    for (int u = 0; u < d; ++u)
      if (adj[u] & (1u << j)) parents |= 1u << u;
    acc += tr->dag_cache[(size_t)j * (1u << d) + parents];
  }
  return acc;
}

static void dag_edge_from_action(int action, int d, int* u, int* v) { /* dag.cpp:379-383 */
  *u = action / (d - 1);
  const int r = action % (d - 1);
  *v = r < *u ? r : r + 1;
}

/* ---------------- generic env dispatch ---------------- */

static void env_reset(const orc_trainer* tr, orc_state* s) {
  memset(s, 0, sizeof *s);
  switch (tr->env.kind) {
    case GFNX_ENV_BITSEQ:
      for (int i = 0; i < tr->bs_slots; ++i) s->v[i] = -1;
      break;
    case GFNX_ENV_DAG:
      for (int a = 0; a < tr->dag_d; ++a) s->closure_t[a] = 1u << a;
      break;
    default:
      break;
  }
}

static double state_log_reward(const orc_trainer* tr, const orc_state* s) {
  switch (tr->env.kind) {
    case GFNX_ENV_HYPERGRID: return grid_log_reward(tr, s->v);
    case GFNX_ENV_BITSEQ: return bitseq_log_reward(tr, s);
    case GFNX_ENV_ISING: return ising_log_reward(tr, s);
    case GFNX_ENV_DAG: return dag_graph_log_reward(tr, s->adj);
  }
  return 0.0;
}

/* step_instance of each env; returns log R on entering a terminal state, else 0 */
static double env_step(const orc_trainer* tr, orc_state* s, int a) {
  s->step_count += 1;
  switch (tr->env.kind) {
    case GFNX_ENV_HYPERGRID: /* hypergrid.cpp:24-32 */
      if (a == tr->stop) {
        s->is_terminal = 1;
        return grid_log_reward(tr, s->v);
      }
      s->v[a] += 1;
      return 0.0;
    case GFNX_ENV_BITSEQ: { /* sequences.cpp:236-267: non-autoregressive or AR fixed */
      const int pos = tr->env.bs_scheme ? s->count : a / tr->bs_vocab;
      s->v[pos] = tr->env.bs_scheme ? a : a % tr->bs_vocab;
      s->count += 1;
      if (s->count == tr->bs_slots) {
        s->is_terminal = 1;
        return bitseq_log_reward(tr, s);
      }
      return 0.0;
    }
    case GFNX_ENV_ISING: { /* ising.cpp:72-82 */
      const int site = a / 2;
      s->v[site] = (a & 1) ? 1 : -1;
      s->count += 1;
      if (s->count == tr->is_D) {
        s->is_terminal = 1;
        return ising_log_reward(tr, s);
      }
      return 0.0;
    }
    case GFNX_ENV_DAG: { /* dag.cpp:385-398 */
      if (a == tr->stop) {
        s->is_terminal = 1;
        return dag_graph_log_reward(tr, s->adj);
      }
      int u, v;
      dag_edge_from_action(a, tr->dag_d, &u, &v);
      s->adj[u] |= 1u << v;
      const uint32_t row_u = s->closure_t[u]; /* closure_update dag.cpp:324-329 */
      for (int q = 0; q < tr->dag_d; ++q)
        if (s->closure_t[q] & (1u << v)) s->closure_t[q] |= row_u;
      s->count += 1;
      return 0.0;
    }
  }
  return 0.0;
}

static void env_action_mask(const orc_trainer* tr, const orc_state* s, uint8_t* out) {
  memset(out, 0, tr->A);
  if (s->is_terminal) return;
  switch (tr->env.kind) {
    case GFNX_ENV_HYPERGRID: /* hypergrid.cpp:43-50 */
      for (int i = 0; i < tr->env.hg_dim; ++i) out[i] = s->v[i] < tr->env.hg_side - 1;
      out[tr->stop] = 1;
      break;
    case GFNX_ENV_BITSEQ: /* sequences.cpp:302-327 */
      if (tr->env.bs_scheme) {
        if (!s->is_terminal) memset(out, 1, tr->bs_vocab);
        break;
      }
      for (int p = 0; p < tr->bs_slots; ++p)
        if (s->v[p] < 0) memset(out + p * tr->bs_vocab, 1, tr->bs_vocab);
      break;
    case GFNX_ENV_ISING: /* ising.cpp:91-102 */
      for (int site = 0; site < tr->is_D; ++site) {
        const uint8_t f = s->v[site] == 0;
        out[2 * site] = f;
        out[2 * site + 1] = f;
      }
      break;
    case GFNX_ENV_DAG: { /* dag.cpp:419-431 */
      const int d = tr->dag_d;
      for (int u = 0; u < d; ++u)
        for (int v = 0; v < d; ++v) {
          if (u == v) continue;
          const int present = (s->adj[u] >> v) & 1;
          const int cycle = (s->closure_t[u] >> v) & 1;
          if (!present && !cycle) out[u * (d - 1) + (v < u ? v : v - 1)] = 1;
        }
      out[tr->stop] = 1;
      break;
    }
  }
}

/* number of legal backward actions (count_legal of backward_action_mask) */
static int env_num_parents(const orc_trainer* tr, const orc_state* s) {
  switch (tr->env.kind) {
    case GFNX_ENV_HYPERGRID: { /* hypergrid.cpp:52-61 */
      if (s->is_terminal) return 1;
      int c = 0;
      for (int i = 0; i < tr->env.hg_dim; ++i) c += s->v[i] > 0;
      return c;
    }
    case GFNX_ENV_BITSEQ: /* sequences.cpp:329-352: NAR filled slots, AR fixed remove-last */
      return tr->env.bs_scheme ? (s->count > 0) : s->count;
    case GFNX_ENV_ISING: return s->count;   /* ising.cpp:104-107 */
    case GFNX_ENV_DAG: {                    /* dag.cpp:433-443 */
      if (s->is_terminal) return 1;
      int c = 0;
      for (int u = 0; u < tr->dag_d; ++u) c += __builtin_popcount(s->adj[u]);
      return c;
    }
  }
  return 0;
}

static int env_backward_action(const orc_trainer* tr, int a) {
  switch (tr->env.kind) {
    case GFNX_ENV_HYPERGRID: return a;                   /* hypergrid.cpp:63-73 */
    case GFNX_ENV_BITSEQ: return tr->env.bs_scheme ? 0 : a / tr->bs_vocab; /* sequences.cpp:354-373 */
    case GFNX_ENV_ISING: return a / 2;                   /* ising.cpp:109-114 */
    case GFNX_ENV_DAG: return a;                         /* dag.cpp:445-455 */
  }
  return a;
}

static void env_encode_obs(const orc_trainer* tr, const orc_state* s, double* out) {
  memset(out, 0, sizeof(double) * tr->O);
  switch (tr->env.kind) {
    case GFNX_ENV_HYPERGRID: /* hypergrid.cpp:82-85 */
      for (int i = 0; i < tr->env.hg_dim; ++i) out[i * tr->env.hg_side + s->v[i]] = 1.0;
      break;
    case GFNX_ENV_BITSEQ: { /* sequences.cpp:396-409 */
      const int width = tr->bs_vocab + 1;
      for (int i = 0; i < tr->bs_slots; ++i) {
        const int tok = s->v[i];
        out[i * width + (tok < 0 ? tr->bs_vocab : tok)] = 1.0;
      }
      out[tr->bs_slots * width] = (double)s->count / tr->bs_slots;
      break;
    }
    case GFNX_ENV_ISING: /* ising.cpp:122-129 */
      for (int site = 0; site < tr->is_D; ++site) {
        const int v = s->v[site] == 0 ? 2 : (s->v[site] > 0 ? 1 : 0);
        out[3 * site + v] = 1.0;
      }
      break;
    case GFNX_ENV_DAG: /* dag.cpp:462-466 */
      for (int u = 0; u < tr->dag_d; ++u)
        for (int v = 0; v < tr->dag_d; ++v)
          out[u * tr->dag_d + v] = ((s->adj[u] >> v) & 1) ? 1.0 : 0.0;
      break;
  }
}

/* Packed state (shared with the device engine). */
static int env_state_words(const orc_trainer* tr) {
  switch (tr->env.kind) {
    case GFNX_ENV_HYPERGRID: return (tr->env.hg_dim + 3) / 4;
    case GFNX_ENV_BITSEQ: return (tr->bs_slots + 3) / 4 + (tr->bs_slots + 31) / 32;
    case GFNX_ENV_ISING: return 2 * ((tr->is_D + 31) / 32);
    case GFNX_ENV_DAG: return (tr->dag_d + 1) / 2;
  }
  return 0;
}

static void env_pack(const orc_trainer* tr, const orc_state* s, uint32_t* w) {
  const int nw = tr->state_words;
  memset(w, 0, sizeof(uint32_t) * nw);
  switch (tr->env.kind) {
    case GFNX_ENV_HYPERGRID:
      for (int i = 0; i < tr->env.hg_dim; ++i) w[i / 4] |= (uint32_t)(s->v[i] & 0xFF) << (8 * (i % 4));
      break;
    case GFNX_ENV_BITSEQ: { /* token bytes, then the filled-slot bitmask */
      const int tw = (tr->bs_slots + 3) / 4;
      for (int i = 0; i < tr->bs_slots; ++i)
        if (s->v[i] >= 0) {
          w[i / 4] |= (uint32_t)s->v[i] << (8 * (i % 4));
          w[tw + i / 32] |= 1u << (i % 32);
        }
      break;
    }
    case GFNX_ENV_ISING: {
      const int nwh = nw / 2;
      for (int i = 0; i < tr->is_D; ++i) {
        if (s->v[i] != 0) w[i / 32] |= 1u << (i % 32);
        if (s->v[i] > 0) w[nwh + i / 32] |= 1u << (i % 32);
      }
      break;
    }
    case GFNX_ENV_DAG:
      for (int u = 0; u < tr->dag_d; ++u) w[u / 2] |= (s->adj[u] & 0xFFFF) << (16 * (u % 2));
      break;
  }
}

static void env_unpack(const orc_trainer* tr, const uint32_t* w, orc_state* s) {
  env_reset(tr, s);
  s->is_terminal = 1;
  switch (tr->env.kind) {
    case GFNX_ENV_HYPERGRID:
      for (int i = 0; i < tr->env.hg_dim; ++i) s->v[i] = (w[i / 4] >> (8 * (i % 4))) & 0xFF;
      break;
    case GFNX_ENV_BITSEQ: {
      const int tw = (tr->bs_slots + 3) / 4;
      for (int i = 0; i < tr->bs_slots; ++i) {
        const int filled = (w[tw + i / 32] >> (i % 32)) & 1;
        s->v[i] = filled ? (int)((w[i / 4] >> (8 * (i % 4))) & 0xFF) : -1;
        s->count += filled;
      }
      break;
    }
    case GFNX_ENV_ISING: {
      const int nwh = tr->state_words / 2;
      for (int i = 0; i < tr->is_D; ++i) {
        const int asg = (w[i / 32] >> (i % 32)) & 1, up = (w[nwh + i / 32] >> (i % 32)) & 1;
        s->v[i] = asg ? (up ? 1 : -1) : 0;
        s->count += asg;
      }
      break;
    }
    case GFNX_ENV_DAG:
      for (int u = 0; u < tr->dag_d; ++u) s->adj[u] = (w[u / 2] >> (16 * (u % 2))) & 0xFFFF;
      break;
  }
}

double orc_log_reward_of_state(const orc_trainer* tr, const uint32_t* packed) {
  orc_state s;
  env_unpack(tr, packed, &s);
  return state_log_reward(tr, &s);
}

/* ====================================================================== */
/* MLP — proj/src/nn.cpp                                                   */
/* ====================================================================== */

static void dense_init(double* w, int in, int out, const uint64_t key[2]) { /* nn.cpp:28-39 */
  const double bound = 1.0 / sqrt((double)in);
  const size_t n = (size_t)in * out;
  double* u = (double*)malloc(sizeof(double) * n);
  random_uniform(key, n, u);
  for (size_t i = 0; i < n; ++i) w[i] = (2.0 * u[i] - 1.0) * bound;
  free(u);
}

static void mlp_layout(orc_trainer* tr) { /* MlpParams::tensors order, nn.cpp:8-19 */
  int64_t off = 0;
  for (int l = 0; l < tr->n_trunk; ++l) {
    tr->off_w[l] = off;
    off += (int64_t)tr->dims[l] * tr->dims[l + 1];
    tr->off_b[l] = off;
    off += tr->dims[l + 1];
  }
  const int H = tr->dims[tr->n_trunk];
  tr->off_fw = off; off += (int64_t)H * tr->A;
  tr->off_fb = off; off += tr->A;
  tr->off_bw = off; off += (int64_t)H * tr->Ab;
  tr->off_bb = off; off += tr->Ab;
  tr->off_flw = off; off += H;
  tr->off_flb = off; off += 1;
  tr->n_params = off;
}

static void mlp_init(orc_trainer* tr) { /* nn.cpp:41-58, key fold_in(root, 0) (train.cpp:204) */
  uint64_t root[2], key[2];
  orc_make_key(tr->tr.seed, root);
  orc_fold_in(root, 0, key);
  int k = 0;
  uint64_t lk[2];
  for (int l = 0; l < tr->n_trunk; ++l) {
    orc_fold_in(key, k++, lk);
    dense_init(tr->params + tr->off_w[l], tr->dims[l], tr->dims[l + 1], lk);
  }
  const int H = tr->dims[tr->n_trunk];
  orc_fold_in(key, k++, lk);
  dense_init(tr->params + tr->off_fw, H, tr->A, lk);
  orc_fold_in(key, k++, lk);
  dense_init(tr->params + tr->off_bw, H, tr->Ab, lk);
  orc_fold_in(key, k++, lk);
  dense_init(tr->params + tr->off_flw, H, 1, lk);
  tr->log_z = tr->tr.logz_init;
}

/* Dense layer of mlp_forward for one row: z = matmul(h, W) then += bias (nn.cpp:63-86,
 * matmul_acc tensor.cpp:67-77: c starts at 0, c[j] += a[p] * W[p][j] for p in order). */
static void dense_row(const double* h, int in, const double* W, const double* b, int out,
                      double* z, int relu) {
  for (int j = 0; j < out; ++j) z[j] = 0.0;
  for (int p = 0; p < in; ++p) {
    const double av = h[p];
    const double* wr = W + (size_t)p * out;
    for (int j = 0; j < out; ++j) z[j] += av * wr[j];
  }
  for (int j = 0; j < out; ++j) {
    z[j] += b[j];
    if (relu && z[j] < 0.0) z[j] = 0.0;
  }
}

/* Forward of one row through the trunk; acts[l] receives layer outputs (post-ReLU). */
static void trunk_row(const orc_trainer* tr, const double* obs, double** acts) {
  const double* h = obs;
  for (int l = 0; l < tr->n_trunk; ++l) {
    dense_row(h, tr->dims[l], tr->params + tr->off_w[l], tr->params + tr->off_b[l],
              tr->dims[l + 1], acts[l], 1);
    h = acts[l];
  }
}

int32_t orc_mlp_forward(const orc_trainer* tr, const double* obs, int32_t n, double* fwd_logits,
                        double* flow) {
  double* acts[10];
  for (int l = 0; l < tr->n_trunk; ++l) acts[l] = (double*)malloc(sizeof(double) * tr->dims[l + 1]);
  const int H = tr->dims[tr->n_trunk];
  for (int r = 0; r < n; ++r) {
    trunk_row(tr, obs + (size_t)r * tr->O, acts);
    const double* h = acts[tr->n_trunk - 1];
    if (fwd_logits)
      dense_row(h, H, tr->params + tr->off_fw, tr->params + tr->off_fb, tr->A,
                fwd_logits + (size_t)r * tr->A, 0);
    if (flow) dense_row(h, H, tr->params + tr->off_flw, tr->params + tr->off_flb, 1, flow + r, 0);
  }
  for (int l = 0; l < tr->n_trunk; ++l) free(acts[l]);
  return 0;
}

/* ====================================================================== */
/* Trainer lifecycle                                                       */
/* ====================================================================== */

static int resolve_horizon(gfnx_schedule* s, int64_t iterations) { /* train.cpp:98-101 */
  if (s->horizon < 0) s->horizon = iterations / 2 > 1 ? iterations / 2 : 1;
  if (s->horizon == 0) s->horizon = iterations - s->warmup > 1 ? iterations - s->warmup : 1;
  return 0;
}

orc_trainer* orc_create(const gfnx_env_desc* env, const gfnx_train_desc* train, int32_t b0,
                        int32_t nb, char* err, int32_t errlen) {
  orc_trainer* tr = (orc_trainer*)calloc(1, sizeof(orc_trainer));
  tr->env = *env;
  tr->tr = *train;
  resolve_horizon(&tr->tr.lr, tr->tr.iterations);
  resolve_horizon(&tr->tr.explore, tr->tr.iterations);
  int rc = 0;
  switch (env->kind) {
    case GFNX_ENV_HYPERGRID: /* HypergridEnv::validate hypergrid.cpp:9-15 */
      if (env->hg_dim < 1 || env->hg_dim > ORC_MAX_SLOTS) rc = fail(tr, "hypergrid: dim must be >= 1");
      else if (env->hg_side < 2 || env->hg_side > 255) rc = fail(tr, "hypergrid: side must be in [2, 255]");
      else if (env->hg_r0 <= 0.0) rc = fail(tr, "hypergrid: r0 must be positive for log rewards");
      tr->A = env->hg_dim + 1;
      tr->Ab = env->hg_dim + 1;
      tr->O = env->hg_dim * env->hg_side;
      tr->T = env->hg_dim * (env->hg_side - 1) + 1;
      tr->stop = env->hg_dim;
      break;
    case GFNX_ENV_BITSEQ: /* build_bitseq train.cpp:381-427; vocab cap 256 (k <= 8) */
      if (env->bs_k < 1 || env->bs_k > 8 || env->bs_n_bits % env->bs_k != 0) {
        rc = fail(tr, "bitseq: k must divide n_bits (1 <= k <= 8)");
        break;
      }
      tr->bs_slots = env->bs_n_bits / env->bs_k;
      tr->bs_vocab = 1 << env->bs_k;
      if (tr->bs_slots > ORC_MAX_SLOTS) rc = fail(tr, "bitseq: too many slots");
      if (env->bs_scheme != 0 && env->bs_scheme != 1) {
        rc = fail(tr, "bitseq: scheme must be 0 (non-autoregressive) or 1 (autoregressive fixed)");
        break;
      }
      tr->A = env->bs_scheme ? tr->bs_vocab : tr->bs_slots * tr->bs_vocab;
      tr->Ab = env->bs_scheme ? 1 : tr->bs_slots;
      tr->O = tr->bs_slots * (tr->bs_vocab + 1) + 1;
      tr->T = tr->bs_slots;
      tr->stop = -1;
      if (!rc) rc = generate_modes(tr);
      break;
    case GFNX_ENV_ISING:
      if (env->is_side < 2 || env->is_side * env->is_side > ORC_MAX_SLOTS) {
        rc = fail(tr, "ising: lattice side must be >= 2");
        break;
      }
      tr->is_D = env->is_side * env->is_side;
      tr->A = 2 * tr->is_D;
      tr->Ab = tr->is_D;
      tr->O = 3 * tr->is_D;
      tr->T = tr->is_D;
      tr->stop = -1;
      toroidal_coupling(tr);
      break;
    case GFNX_ENV_DAG:
      tr->dag_d = env->dag_d;
      rc = dag_build(tr);
      tr->A = env->dag_d * (env->dag_d - 1) + 1;
      tr->Ab = tr->A;
      tr->O = env->dag_d * env->dag_d;
      tr->T = env->dag_d * (env->dag_d - 1) / 2 + 1;
      tr->stop = env->dag_d * (env->dag_d - 1);
      break;
    default:
      rc = fail(tr, "unknown env kind %d", env->kind);
  }
  if (!rc) {
    if (train->objective == GFNX_OBJ_FLDB) rc = fail(tr, "fldb objective is out of scope");
    else if (train->objective < 0 || train->objective > 4) rc = fail(tr, "unknown objective");
    else if (train->learned_backward) rc = fail(tr, "learned backward policy not supported");
    else if (train->objective == GFNX_OBJ_MDB && tr->stop < 0)
      rc = fail(tr, "mdb objective needs the stop action index");
    else if (train->objective == GFNX_OBJ_SUBTB &&
             (train->subtb_lambda <= 0.0 || train->subtb_lambda > 1.0))
      rc = fail(tr, "subtb lambda must lie in (0, 1]");
    else if (train->num_hidden < 1 || train->num_hidden > 8)
      rc = fail(tr, "mlp_init: need at least one hidden layer");
    else if (train->batch_size < 1) rc = fail(tr, "forward_rollout: num_envs must be >= 1");
  }
  if (rc) {
    if (err) snprintf(err, errlen, "%s", tr->err);
    orc_destroy(tr);
    return NULL;
  }
  tr->state_words = env_state_words(tr);
  tr->n_trunk = train->num_hidden;
  tr->dims[0] = tr->O;
  for (int l = 0; l < tr->n_trunk; ++l) tr->dims[l + 1] = train->hidden[l];
  mlp_layout(tr);
  tr->params = (double*)calloc(tr->n_params, sizeof(double));
  tr->grads = (double*)calloc(tr->n_params, sizeof(double));
  tr->adam_m = (double*)calloc(tr->n_params, sizeof(double));
  tr->adam_v = (double*)calloc(tr->n_params, sizeof(double));
  mlp_init(tr);
  tr->B = train->batch_size;
  tr->b0 = nb > 0 ? b0 : 0;
  tr->nb = nb > 0 ? nb : train->batch_size;
  const size_t nbt = (size_t)tr->nb * tr->T;
  tr->lengths = (int32_t*)calloc(tr->nb, sizeof(int32_t));
  tr->fwd_actions = (int32_t*)malloc(nbt * sizeof(int32_t));
  tr->bwd_actions = (int32_t*)malloc(nbt * sizeof(int32_t));
  tr->log_rewards = (double*)calloc(tr->nb, sizeof(double));
  tr->log_pb = (double*)calloc(nbt, sizeof(double));
  tr->delta = (double*)calloc(nbt, sizeof(double));
  tr->terminal_state = (uint32_t*)calloc((size_t)tr->nb * tr->state_words, sizeof(uint32_t));
  tr->states = (orc_state*)malloc(sizeof(orc_state) * (size_t)tr->nb * (tr->T + 1));
  return tr;
}

void orc_destroy(orc_trainer* tr) {
  if (!tr) return;
  free(tr->modes);
  free(tr->J);
  free(tr->dag_cache);
  free(tr->params);
  free(tr->grads);
  free(tr->adam_m);
  free(tr->adam_v);
  free(tr->lengths);
  free(tr->fwd_actions);
  free(tr->bwd_actions);
  free(tr->log_rewards);
  free(tr->log_pb);
  free(tr->delta);
  free(tr->terminal_state);
  free(tr->states);
  free(tr);
}

const char* orc_last_error(const orc_trainer* tr) { return tr->err; }

int32_t orc_shape(const orc_trainer* tr, gfnx_env_shape* out) {
  out->num_actions = tr->A;
  out->num_backward_actions = tr->Ab;
  out->obs_dim = tr->O;
  out->max_traj_len = tr->T;
  out->stop_action = tr->stop;
  out->state_words = tr->state_words;
  return 0;
}

int64_t orc_num_params(const orc_trainer* tr) { return tr->n_params; }
void orc_get_params(const orc_trainer* tr, double* flat, double* log_z) {
  if (flat) memcpy(flat, tr->params, sizeof(double) * tr->n_params);
  if (log_z) *log_z = tr->log_z;
}
void orc_set_params(orc_trainer* tr, const double* flat, double log_z) {
  if (flat) memcpy(tr->params, flat, sizeof(double) * tr->n_params);
  tr->log_z = log_z;
}
void orc_get_adam(const orc_trainer* tr, double* m, double* v, int64_t* t, double* zm, double* zv,
                  int64_t* zt) {
  if (m) memcpy(m, tr->adam_m, sizeof(double) * tr->n_params);
  if (v) memcpy(v, tr->adam_v, sizeof(double) * tr->n_params);
  if (t) *t = tr->adam_t;
  if (zm) *zm = tr->z_m;
  if (zv) *zv = tr->z_v;
  if (zt) *zt = tr->z_t;
}
void orc_set_adam(orc_trainer* tr, const double* m, const double* v, int64_t t, double zm,
                  double zv, int64_t zt) {
  if (m) memcpy(tr->adam_m, m, sizeof(double) * tr->n_params);
  if (v) memcpy(tr->adam_v, v, sizeof(double) * tr->n_params);
  tr->adam_t = t;
  tr->z_m = zm;
  tr->z_v = zv;
  tr->z_t = zt;
}

/* ====================================================================== */
/* Rollouts — proj/include/gfn/env_core.hpp                                */
/* ====================================================================== */

/* rollout_from_actions (env_core.hpp:166-229): re-simulates and records. */
static int record_from_actions(orc_trainer* tr, const int32_t* actions) {
  const int T = tr->T;
  const int mdb = tr->tr.objective == GFNX_OBJ_MDB;
  uint8_t* mask = (uint8_t*)malloc(tr->A);
  for (int b = 0; b < tr->nb; ++b) {
    orc_state* st = tr->states + (size_t)b * (T + 1);
    env_reset(tr, &st[0]);
    tr->lengths[b] = 0;
    tr->log_rewards[b] = 0.0;
    for (int t = 0; t < T; ++t) {
      tr->fwd_actions[(size_t)b * T + t] = -1;
      tr->bwd_actions[(size_t)b * T + t] = -1;
      tr->log_pb[(size_t)b * T + t] = 0.0;
      tr->delta[(size_t)b * T + t] = 0.0;
    }
    int t = 0;
    for (; t < T; ++t) {
      const int a = actions[(size_t)b * T + t];
      if (st[t].is_terminal || a < 0) break;
      env_action_mask(tr, &st[t], mask);
      if (a >= tr->A || !mask[a]) {
        free(mask);
        return fail(tr, "rollout: illegal action in replay");
      }
      st[t + 1] = st[t];
      double prev_log_r = 0.0;
      if (mdb) prev_log_r = state_log_reward(tr, &st[t]);
      const double log_r = env_step(tr, &st[t + 1], a);
      tr->fwd_actions[(size_t)b * T + t] = a;
      tr->bwd_actions[(size_t)b * T + t] = env_backward_action(tr, a);
      const int legal_bwd = env_num_parents(tr, &st[t + 1]);
      if (legal_bwd < 1) {
        free(mask);
        return fail(tr, "rollout: reached state with no parent");
      }
      tr->log_pb[(size_t)b * T + t] = -log((double)legal_bwd);
      if (mdb && !st[t + 1].is_terminal)
        tr->delta[(size_t)b * T + t] = state_log_reward(tr, &st[t + 1]) - prev_log_r;
      if (st[t + 1].is_terminal) {
        tr->log_rewards[b] = log_r;
        tr->lengths[b] = t + 1;
        env_pack(tr, &st[t + 1], tr->terminal_state + (size_t)b * tr->state_words);
      }
    }
    if (!st[t].is_terminal) {
      free(mask);
      return fail(tr, "rollout: trajectory did not reach a terminal state");
    }
  }
  free(mask);
  tr->has_batch = 1;
  return 0;
}

int32_t orc_replay(orc_trainer* tr, const int32_t* actions) { return record_from_actions(tr, actions); }

/* forward_rollout (env_core.hpp:232-274). use_policy == 0 is the eps = 1 rollout without
 * the policy forward: eps_uniform (objectives.cpp:242-264) then gives (1 - 1) * p_i / z +
 * 1 / legal = 1 / legal exactly for every finite logit row, so the draws do not depend on
 * the MLP (the reference still evaluates it, only to reject non-finite logits). Used by the
 * parity tests at the benchmarked batch sizes, where the fp64 MLP per state would dominate. */
static int32_t rollout_impl(orc_trainer* tr, int64_t it, double eps, int use_policy) {
  if (eps < 0.0 || eps > 1.0) return fail(tr, "exploration eps must lie in [0,1]");
  const int T = tr->T, A = tr->A, nb = tr->nb;
  uint64_t root[2], key[2];
  orc_make_key(tr->tr.seed, root);
  orc_fold_in(root, 1000 + (uint64_t)it, key); /* train.cpp:228 */
  orc_state* cur = (orc_state*)malloc(sizeof(orc_state) * nb);
  int32_t* actions = (int32_t*)malloc(sizeof(int32_t) * (size_t)nb * T);
  for (int b = 0; b < nb; ++b) env_reset(tr, &cur[b]);
  for (size_t i = 0; i < (size_t)nb * T; ++i) actions[i] = -1;
  double* obs = (double*)malloc(sizeof(double) * tr->O);
  double* logits = (double*)malloc(sizeof(double) * A);
  double* probs = (double*)malloc(sizeof(double) * A);
  uint8_t* mask = (uint8_t*)malloc(A);
  int rc = 0;
  for (int t = 0; t < T && !rc; ++t) {
    int any_live = 0;
    for (int b = 0; b < nb; ++b) any_live |= !cur[b].is_terminal;
    if (!any_live) break;
    uint64_t step_key[2];
    orc_fold_in(key, (uint64_t)t, step_key); /* env_core.hpp:259 */
    for (int b = 0; b < nb; ++b) {
      if (cur[b].is_terminal) continue;
      env_action_mask(tr, &cur[b], mask);
      if (use_policy) {
        env_encode_obs(tr, &cur[b], obs);
        orc_mlp_forward(tr, obs, 1, logits, NULL); /* row-independent mlp_forward (nn.cpp:60-89) */
      } else {
        for (int i = 0; i < A; ++i) logits[i] = 0.0;
      }
      for (int i = 0; i < A; ++i)
        if (!isfinite(logits[i])) rc = fail(tr, "forward_rollout: non-finite policy logits");
      if (rc) break;
      const int legal = orc_eps_uniform(logits, mask, A, eps, probs);
      if (legal == 0) { rc = fail(tr, "eps_uniform: no legal action"); break; }
      if (legal < 0) { rc = fail(tr, "eps_uniform: non-finite logits"); break; }
      uint64_t dk[2];
      orc_fold_in(step_key, (uint64_t)(tr->b0 + b), dk); /* global trajectory index */
      const int a = orc_categorical(dk, probs, A);
      if (a < 0) { rc = fail(tr, "categorical: no positive weight"); break; }
      actions[(size_t)b * T + t] = a;
      env_step(tr, &cur[b], a);
    }
  }
  if (!rc) rc = record_from_actions(tr, actions);
  free(cur);
  free(actions);
  free(obs);
  free(logits);
  free(probs);
  free(mask);
  return rc;
}

int32_t orc_rollout(orc_trainer* tr, int64_t it, double eps) { return rollout_impl(tr, it, eps, 1); }
int32_t orc_rollout_uniform(orc_trainer* tr, int64_t it) { return rollout_impl(tr, it, 1.0, 0); }

void orc_batch(const orc_trainer* tr, orc_batch_view* out) {
  out->nb = tr->nb;
  out->T = tr->T;
  out->state_words = tr->state_words;
  out->lengths = tr->lengths;
  out->fwd_actions = tr->fwd_actions;
  out->bwd_actions = tr->bwd_actions;
  out->log_rewards = tr->log_rewards;
  out->log_pb = tr->log_pb;
  out->delta = tr->delta;
  out->terminal_state = tr->terminal_state;
}

void orc_local_counts(const orc_trainer* tr, int64_t* n_steps, int64_t* n_mdb) {
  int64_t s = 0, m = 0;
  for (int b = 0; b < tr->nb; ++b) {
    s += tr->lengths[b];
    m += tr->lengths[b] > 1 ? tr->lengths[b] - 1 : 0;
  }
  if (n_steps) *n_steps = s;
  if (n_mdb) *n_mdb = m;
}

/* ====================================================================== */
/* Loss + analytic gradient (objectives.cpp:42-240 + tape.cpp:321-485)      */
/* ====================================================================== */

/* ---- bf16 operand model (TEST INFRASTRUCTURE: the numerics of the device's bf16 fast
 * path, stated on top of this restatement so device-vs-model differences isolate
 * implementation error from the bf16 operand rounding the design accepts) ---- */
static double bf16r(double x) { /* fp32 then round-to-nearest-even to bf16 (cvt.rn.bf16.f32) */
  float f = (float)x;
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return (double)f;
  u += 0x7fffu + ((u >> 16) & 1u);
  u &= 0xffff0000u;
  memcpy(&f, &u, 4);
  return (double)f;
}

/* Trunk of one row under the model flags: weights from Pm; ORC_BFM_ACT rounds every post-ReLU
 * activation to bf16; ORC_BFM_ISING_L1 forms layer 1 like the persistent Ising rollout
 * (lockstep.cu k_ls_ising_l1img / k_ls_h1init): the all-unassigned pre-activation
 * b1 + sum_s bf16(W1[3s+2]) plus, per assigned site, bf16(bf16(W1[3s+u]) - bf16(W1[3s+2])). */
static void model_trunk_row(const orc_trainer* tr, const double* Pm, int flags, const orc_state* s,
                            const double* obs, double** acts) {
  const double* h = obs;
  for (int l = 0; l < tr->n_trunk; ++l) {
    const int out = tr->dims[l + 1];
    if (l == 0 && (flags & ORC_BFM_ISING_L1) && tr->env.kind == GFNX_ENV_ISING) {
      const double* W1 = tr->params + tr->off_w[0];
      const double* b1 = tr->params + tr->off_b[0];
      for (int j = 0; j < out; ++j) {
        double z = b1[j];
        for (int site = 0; site < tr->is_D; ++site) z += bf16r(W1[(size_t)(3 * site + 2) * out + j]);
        for (int site = 0; site < tr->is_D; ++site) {
          if (s->v[site] == 0) continue;
          const int u = s->v[site] > 0 ? 1 : 0;
          z += bf16r(bf16r(W1[(size_t)(3 * site + u) * out + j]) - bf16r(W1[(size_t)(3 * site + 2) * out + j]));
        }
        acts[0][j] = z < 0.0 ? 0.0 : z;
      }
    } else {
      dense_row(h, tr->dims[l], Pm + tr->off_w[l], Pm + tr->off_b[l], out, acts[l], 1);
    }
    if (flags & ORC_BFM_ACT)
      for (int j = 0; j < out; ++j) acts[l][j] = bf16r(acts[l][j]);
    h = acts[l];
  }
}

static int32_t compute_grads_impl(orc_trainer* tr, double norm, int flags, double* loss_out,
                                  double* g, double* dlogz_out, double* row_logpf) {
  if (!tr->has_batch) return fail(tr, "train_step: no batch");
  const int T = tr->T, A = tr->A, nt = tr->n_trunk;
  const int H = tr->dims[nt];
  const int obj = tr->tr.objective;
  const int need_flow = obj == GFNX_OBJ_DB || obj == GFNX_OBJ_SUBTB;
  int64_t n_steps, n_mdb;
  orc_local_counts(tr, &n_steps, &n_mdb);
  if (norm <= 0.0)
    norm = obj == GFNX_OBJ_DB ? (double)n_steps
         : obj == GFNX_OBJ_MDB ? (double)n_mdb : (double)tr->B;
  /* rows = real states t < L_b in (b, t) order */
  int64_t R = n_steps;
  int64_t* row0 = (int64_t*)malloc(sizeof(int64_t) * (tr->nb + 1));
  row0[0] = 0;
  for (int b = 0; b < tr->nb; ++b) row0[b + 1] = row0[b] + tr->lengths[b];
  int64_t act_sz = 0;
  for (int l = 0; l < nt; ++l) act_sz += tr->dims[l + 1];
  double* obs = (double*)malloc(sizeof(double) * (size_t)R * tr->O);
  double* act = (double*)malloc(sizeof(double) * (size_t)R * act_sz);  /* post-ReLU per layer */
  double* logp = (double*)malloc(sizeof(double) * (size_t)R * A);
  uint8_t* mask = (uint8_t*)malloc((size_t)R * A);
  double* flow = (double*)calloc((size_t)R, sizeof(double));
  double* glogp = (double*)calloc((size_t)R * A, sizeof(double));
  double* gflow = (double*)calloc((size_t)R, sizeof(double));
  double* acts[10];
  /* parameters the matmuls read: the fp64 master, or (ORC_BFM_W) its weight matrices rounded
   * to bf16 like the device's operand images; biases stay unrounded */
  double* wq = NULL;
  const double* Pm = tr->params;
  if (flags & ORC_BFM_W) {
    wq = (double*)malloc(sizeof(double) * tr->n_params);
    memcpy(wq, tr->params, sizeof(double) * tr->n_params);
    for (int l = 0; l < nt; ++l)
      for (int64_t i = 0; i < (int64_t)tr->dims[l] * tr->dims[l + 1]; ++i)
        wq[tr->off_w[l] + i] = bf16r(wq[tr->off_w[l] + i]);
    for (int64_t i = 0; i < (int64_t)H * A; ++i) wq[tr->off_fw + i] = bf16r(wq[tr->off_fw + i]);
    for (int64_t i = 0; i < (int64_t)H * tr->Ab; ++i) wq[tr->off_bw + i] = bf16r(wq[tr->off_bw + i]);
    for (int64_t i = 0; i < H; ++i) wq[tr->off_flw + i] = bf16r(wq[tr->off_flw + i]);
    Pm = wq;
  }
  /* ---- forward: mlp_forward_tape (nn.cpp:91-126) + masked_log_softmax (tape.cpp:177-213) */
  for (int b = 0; b < tr->nb; ++b)
    for (int t = 0; t < tr->lengths[b]; ++t) {
      const int64_t r = row0[b] + t;
      const orc_state* s = tr->states + (size_t)b * (T + 1) + t;
      env_encode_obs(tr, s, obs + (size_t)r * tr->O);
      env_action_mask(tr, s, mask + (size_t)r * A);
      int64_t o = 0;
      for (int l = 0; l < nt; ++l) {
        acts[l] = act + (size_t)r * act_sz + o;
        o += tr->dims[l + 1];
      }
      model_trunk_row(tr, Pm, flags, s, obs + (size_t)r * tr->O, acts);
      double* x = logp + (size_t)r * A;
      dense_row(acts[nt - 1], H, Pm + tr->off_fw, Pm + tr->off_fb, A, x, 0);
      if (flags & ORC_BFM_LOGIT)
        for (int c = 0; c < A; ++c) x[c] = bf16r(x[c]);
      if (need_flow)
        dense_row(acts[nt - 1], H, Pm + tr->off_flw, Pm + tr->off_flb, 1, flow + r, 0);
      const uint8_t* mr = mask + (size_t)r * A;
      double hi = -INFINITY;
      int legal = 0;
      for (int c = 0; c < A; ++c)
        if (mr[c]) {
          ++legal;
          if (x[c] > hi) hi = x[c];
        }
      if (!isfinite(hi)) {
        free(row0); free(obs); free(act); free(logp); free(mask); free(flow); free(glogp); free(gflow); free(wq);
        return fail(tr, "masked_log_softmax: non-finite logits");
      }
      double ssum = 0.0;
      for (int c = 0; c < A; ++c)
        if (mr[c]) ssum += exp(x[c] - hi);
      const double lse = hi + log(ssum);
      for (int c = 0; c < A; ++c) x[c] = mr[c] ? x[c] - lse : -1e30;
    }
  /* ---- objective ---- */
  double loss = 0.0, dlogz = 0.0;
  const double log_z = tr->log_z;
  if (obj == GFNX_OBJ_TB) { /* tb_loss objectives.cpp:120-142 */
    const double w = 1.0 / norm;
    for (int b = 0; b < tr->nb; ++b) {
      double cum = 0.0;
      for (int t = 0; t < tr->lengths[b]; ++t) {
        const int64_t r = row0[b] + t;
        const double pf = logp[(size_t)r * A + tr->fwd_actions[(size_t)b * T + t]];
        const double d = pf + -tr->log_pb[(size_t)b * T + t];
        cum += d;
      }
      const double res = (cum + log_z) + -tr->log_rewards[b];
      loss += res * res * w;
      const double g = 2.0 * res * w;
      dlogz += g;
      for (int t = 0; t < tr->lengths[b]; ++t) {
        const int64_t r = row0[b] + t;
        glogp[(size_t)r * A + tr->fwd_actions[(size_t)b * T + t]] += g;
      }
    }
  } else if (obj == GFNX_OBJ_DB) { /* transition_loss objectives.cpp:94-118 */
    for (int b = 0; b < tr->nb; ++b) {
      const int L = tr->lengths[b];
      for (int t = 0; t < L; ++t) {
        const int64_t r = row0[b] + t;
        const double pf = logp[(size_t)r * A + tr->fwd_actions[(size_t)b * T + t]];
        const double d = pf + -tr->log_pb[(size_t)b * T + t];
        const double f0 = flow[r];
        const double f1 = (t + 1 < L) ? flow[r + 1] : tr->log_rewards[b];
        const double res = (f0 - f1) + d;
        const double w = (t == L - 1 ? tr->tr.terminal_penalty : 1.0) / norm;
        loss += res * res * w;
        const double g = 2.0 * res * w;
        gflow[r] += g;
        if (t + 1 < L) gflow[r + 1] += -g;
        glogp[(size_t)r * A + tr->fwd_actions[(size_t)b * T + t]] += g;
      }
    }
  } else if (obj == GFNX_OBJ_SUBTB) { /* subtb_loss objectives.cpp:144-180 */
    const double lam = tr->tr.subtb_lambda;
    double* cum = (double*)malloc(sizeof(double) * (T + 1));
    double* F = (double*)malloc(sizeof(double) * (T + 1));
    double* gcum = (double*)malloc(sizeof(double) * (T + 1));
    double* gpair = (double*)malloc(sizeof(double) * (size_t)(T + 1) * (T + 1));
    for (int b = 0; b < tr->nb; ++b) {
      const int L = tr->lengths[b];
      cum[0] = 0.0;
      for (int t = 0; t < L; ++t) {
        const int64_t r = row0[b] + t;
        const double pf = logp[(size_t)r * A + tr->fwd_actions[(size_t)b * T + t]];
        cum[t + 1] = cum[t] + (pf + -tr->log_pb[(size_t)b * T + t]);
        F[t] = flow[r];
      }
      F[L] = tr->log_rewards[b];
      double nrm = 0.0;
      for (int j = 0; j < L; ++j)
        for (int k = j + 1; k <= L; ++k) nrm += pow(lam, k - j);
      if (nrm <= 0.0) continue;
      for (int k = 0; k <= L; ++k) gcum[k] = 0.0;
      int np = 0;
      for (int j = 0; j < L; ++j)
        for (int k = j + 1; k <= L; ++k) {
          const double w = pow(lam, k - j) / nrm / norm;
          const double res = (F[j] - F[k]) + (cum[k] - cum[j]);
          loss += res * res * w;
          gpair[np++] = 2.0 * res * w;
        }
      /* Tape reverse order. GCC evaluates the operands of
       * add(sub(take(flows,fj), take(flows,fk)), sub(take(cum,ck), take(cum,cj)))
       * right to left (objectives.cpp:177-178), so backward visits take(flows,fj),
       * take(flows,fk), take(cum,ck), take(cum,cj) in that order. */
      np = 0;
      for (int j = 0; j < L; ++j)
        for (int k = j + 1; k <= L; ++k) gflow[row0[b] + j] += gpair[np++];
      np = 0;
      for (int j = 0; j < L; ++j)
        for (int k = j + 1; k <= L; ++k) {
          if (k < L) gflow[row0[b] + k] += -gpair[np];
          ++np;
        }
      np = 0;
      for (int j = 0; j < L; ++j)
        for (int k = j + 1; k <= L; ++k) gcum[k] += gpair[np++];
      np = 0;
      for (int j = 0; j < L; ++j)
        for (int k = j + 1; k <= L; ++k) gcum[j] += -gpair[np++];
      /* exclusive_row_cumsum backward (tape.cpp:448-461): d grid[t] = sum_{c > t} dcum[c] */
      double acc = 0.0;
      for (int c = L; c >= 0; --c) {
        if (c < L) {
          const int64_t r = row0[b] + c;
          glogp[(size_t)r * A + tr->fwd_actions[(size_t)b * T + c]] += acc;
        }
        acc += gcum[c];
      }
    }
    free(cum);
    free(F);
    free(gcum);
    free(gpair);
  } else if (obj == GFNX_OBJ_MDB) { /* mdb_loss objectives.cpp:186-226 */
    const double w = 1.0 / norm;
    const int stop = tr->stop;
    for (int b = 0; b < tr->nb; ++b) {
      const int L = tr->lengths[b];
      for (int t = 0; t + 1 < L; ++t) {
        const int64_t r = row0[b] + t;
        const int a = tr->fwd_actions[(size_t)b * T + t];
        if (a == stop) {
          free(row0); free(obs); free(act); free(logp); free(mask); free(flow); free(glogp); free(gflow); free(wq);
          return fail(tr, "stop action before trajectory end");
        }
        double res = logp[(size_t)r * A + a] +
                     (logp[(size_t)(r + 1) * A + stop] - logp[(size_t)r * A + stop]);
        res = res + -tr->log_pb[(size_t)b * T + t];
        res = res + -tr->delta[(size_t)b * T + t];
        loss += res * res * w;
        const double g = 2.0 * res * w;
        glogp[(size_t)r * A + a] += g;
        glogp[(size_t)(r + 1) * A + stop] += g;
        glogp[(size_t)r * A + stop] += -g;
      }
    }
  }
  if (!isfinite(loss)) {
    free(row0); free(obs); free(act); free(logp); free(mask); free(flow); free(glogp); free(gflow); free(wq);
    return fail(tr, "training loss is not finite");
  }
  /* ---- backward through masked log-softmax (tape.cpp:413-434) and the MLP ---- */
  memset(g, 0, sizeof(double) * tr->n_params);
  int maxw = 0;
  for (int l = 0; l <= nt; ++l) maxw = tr->dims[l] > maxw ? tr->dims[l] : maxw;
  double* gx = (double*)malloc(sizeof(double) * A);
  double* gh = (double*)malloc(sizeof(double) * maxw);
  double* gz = (double*)malloc(sizeof(double) * maxw);
  for (int64_t r = 0; r < R; ++r) {
    const uint8_t* mr = mask + (size_t)r * A;
    const double* lp = logp + (size_t)r * A;
    const double* gr = glogp + (size_t)r * A;
    double gsum = 0.0;
    for (int c = 0; c < A; ++c)
      if (mr[c]) gsum += gr[c];
    for (int c = 0; c < A; ++c) gx[c] = mr[c] ? gr[c] - exp(lp[c]) * gsum : 0.0;
    double gfl = need_flow ? gflow[r] : 0.0;
    if (flags & ORC_BFM_GRAD) { /* bf16 dlogits / dflow operand images */
      for (int c = 0; c < A; ++c) gx[c] = bf16r(gx[c]);
      gfl = bf16r(gfl);
    }
    int64_t o = 0;
    for (int l = 0; l < nt; ++l) {
      acts[l] = act + (size_t)r * act_sz + o;
      o += tr->dims[l + 1];
    }
    const double* h = acts[nt - 1];
    /* head weight/bias grads (matmul_tn_acc + add_rowvec backward) */
    for (int p = 0; p < H; ++p) {
      double* gw = g + tr->off_fw + (size_t)p * A;
      for (int j = 0; j < A; ++j) gw[j] += h[p] * gx[j];
    }
    for (int j = 0; j < A; ++j) g[tr->off_fb + j] += gx[j];
    if (need_flow) {
      for (int p = 0; p < H; ++p) g[tr->off_flw + p] += h[p] * gfl;
      g[tr->off_flb] += gfl;
    }
    /* dh = flow contribution then fwd contribution (reverse node order) */
    for (int p = 0; p < H; ++p) {
      double v = 0.0;
      if (need_flow) v += gfl * Pm[tr->off_flw + p];
      double acc = 0.0;
      const double* wr = Pm + tr->off_fw + (size_t)p * A;
      for (int j = 0; j < A; ++j) acc += gx[j] * wr[j];
      gh[p] = v + acc;
    }
    for (int l = nt - 1; l >= 0; --l) {
      const int out = tr->dims[l + 1], in = tr->dims[l];
      for (int j = 0; j < out; ++j) gz[j] = acts[l][j] > 0.0 ? gh[j] : 0.0;
      if (flags & ORC_BFM_GRAD)
        for (int j = 0; j < out; ++j) gz[j] = bf16r(gz[j]);
      const double* hin = l > 0 ? acts[l - 1] : obs + (size_t)r * tr->O;
      for (int p = 0; p < in; ++p) {
        const double av = hin[p];
        double* gw = g + tr->off_w[l] + (size_t)p * out;
        for (int j = 0; j < out; ++j) gw[j] += av * gz[j];
      }
      for (int j = 0; j < out; ++j) g[tr->off_b[l] + j] += gz[j];
      if (l > 0) {
        const double* W = Pm + tr->off_w[l];
        for (int p = 0; p < in; ++p) {
          double acc = 0.0;
          const double* wr = W + (size_t)p * out;
          for (int j = 0; j < out; ++j) acc += gz[j] * wr[j];
          gh[p] = acc;
        }
      }
    }
  }
  if (dlogz_out) *dlogz_out = obj == GFNX_OBJ_TB ? dlogz : 0.0;
  if (row_logpf) {
    memset(row_logpf, 0, sizeof(double) * (size_t)tr->nb * T);
    for (int b = 0; b < tr->nb; ++b)
      for (int t = 0; t < tr->lengths[b]; ++t)
        row_logpf[(size_t)b * T + t] =
            logp[(size_t)(row0[b] + t) * A + tr->fwd_actions[(size_t)b * T + t]];
  }
  free(gx); free(gh); free(gz);
  free(row0); free(obs); free(act); free(logp); free(mask); free(flow); free(glogp); free(gflow); free(wq);
  if (loss_out) *loss_out = loss;
  return 0;
}

int32_t orc_compute_grads(orc_trainer* tr, double norm, double* loss_out) {
  return compute_grads_impl(tr, norm, 0, loss_out, tr->grads, &tr->dlogz, NULL);
}

int32_t orc_model_grads(orc_trainer* tr, double norm, int32_t flags, double* loss, double* grads,
                        double* dlogz, double* row_logpf) {
  double* g = (double*)malloc(sizeof(double) * tr->n_params);
  const int32_t rc = compute_grads_impl(tr, norm, flags, loss, g, dlogz, row_logpf);
  if (!rc && grads) memcpy(grads, g, sizeof(double) * tr->n_params);
  free(g);
  return rc;
}

/* The action the reference sampler (fp64 policy, eps_uniform + categorical with the
 * reference key fold_in(fold_in(fold_in(root, 1000 + it), t), b0 + b), env_core.hpp:259-268)
 * would draw at every real state of the RESIDENT batch (teacher forcing on its states);
 * -1 past each trajectory's end. The device/oracle action-agreement rate at eps < 1. */
int32_t orc_teacher_actions(orc_trainer* tr, int64_t it, double eps, int32_t* out) {
  if (!tr->has_batch) return fail(tr, "teacher_actions: no batch");
  const int T = tr->T, A = tr->A;
  uint64_t root[2], key[2], step_key[2], dk[2];
  orc_make_key(tr->tr.seed, root);
  orc_fold_in(root, 1000 + (uint64_t)it, key);
  double* obs = (double*)malloc(sizeof(double) * tr->O);
  double* logits = (double*)malloc(sizeof(double) * A);
  double* probs = (double*)malloc(sizeof(double) * A);
  uint8_t* mask = (uint8_t*)malloc(A);
  for (size_t i = 0; i < (size_t)tr->nb * T; ++i) out[i] = -1;
  for (int t = 0; t < T; ++t) {
    orc_fold_in(key, (uint64_t)t, step_key);
    for (int b = 0; b < tr->nb; ++b) {
      if (t >= tr->lengths[b]) continue;
      const orc_state* s = tr->states + (size_t)b * (T + 1) + t;
      env_encode_obs(tr, s, obs);
      env_action_mask(tr, s, mask);
      orc_mlp_forward(tr, obs, 1, logits, NULL);
      if (orc_eps_uniform(logits, mask, A, eps, probs) <= 0) continue;
      orc_fold_in(step_key, (uint64_t)(tr->b0 + b), dk);
      out[(size_t)b * T + t] = orc_categorical(dk, probs, A);
    }
  }
  free(obs); free(logits); free(probs); free(mask);
  return 0;
}

void orc_get_grads(const orc_trainer* tr, double* flat, double* dlogz) {
  if (flat) memcpy(flat, tr->grads, sizeof(double) * tr->n_params);
  if (dlogz) *dlogz = tr->dlogz;
}
void orc_set_grads(orc_trainer* tr, const double* flat, double dlogz) {
  if (flat) memcpy(tr->grads, flat, sizeof(double) * tr->n_params);
  tr->dlogz = dlogz;
}

static void adam_update(double* p, const double* g, double* m, double* v, int64_t n, int64_t* t,
                        double lr, double b1, double b2, double eps, double wd) {
  /* adam_step optim.cpp:19-43 */
  *t += 1;
  const double bc1 = 1.0 - pow(b1, (double)*t);
  const double bc2 = 1.0 - pow(b2, (double)*t);
  for (int64_t j = 0; j < n; ++j) {
    const double gj = g[j];
    m[j] = b1 * m[j] + (1.0 - b1) * gj;
    v[j] = b2 * v[j] + (1.0 - b2) * gj * gj;
    const double mhat = m[j] / bc1;
    const double vhat = v[j] / bc2;
    p[j] -= lr * (mhat / (sqrt(vhat) + eps) + wd * p[j]);
  }
}

void orc_apply_adam(orc_trainer* tr, double lr) { /* train.cpp:184-190 */
  const gfnx_train_desc* s = &tr->tr;
  adam_update(tr->params, tr->grads, tr->adam_m, tr->adam_v, tr->n_params, &tr->adam_t, lr,
              s->beta1, s->beta2, s->adam_eps, s->weight_decay);
  if (s->objective == GFNX_OBJ_TB) {
    double g = tr->dlogz;
    adam_update(&tr->log_z, &g, &tr->z_m, &tr->z_v, 1, &tr->z_t, s->z_lr, s->beta1, s->beta2,
                s->adam_eps, 0.0);
  }
}

int32_t orc_iteration(orc_trainer* tr, int64_t it, double* loss) { /* train.cpp:224-229 */
  const double lr = orc_schedule_value(&tr->tr.lr, it);
  const double eps = orc_schedule_value(&tr->tr.explore, it);
  if (orc_rollout(tr, it, eps)) return -1;
  double l = 0.0;
  if (orc_compute_grads(tr, 0.0, &l)) return -1;
  orc_apply_adam(tr, lr);
  if (loss) *loss = l;
  return 0;
}

/* ---- test helpers ---- */

int32_t orc_obs_after(const orc_trainer* tr, const int32_t* actions, int32_t n, double* obs,
                      uint8_t* mask) {
  orc_state s;
  env_reset(tr, &s);
  for (int i = 0; i < n; ++i) env_step(tr, &s, actions[i]);
  if (obs) env_encode_obs(tr, &s, obs);
  if (mask) env_action_mask(tr, &s, mask);
  return 0;
}

int32_t orc_bitseq_modes(const orc_trainer* tr, uint8_t* out, int32_t cap) {
  const int n = tr->env.bs_n_bits;
  for (int m = 0; m < tr->n_modes && m < cap; ++m) memcpy(out + (size_t)m * n, tr->modes + (size_t)m * n, n);
  return tr->n_modes;
}

int32_t orc_dag_cache(const orc_trainer* tr, double* out, int32_t cap) {
  const int n = tr->dag_d * (1 << tr->dag_d);
  if (out && cap >= n) memcpy(out, tr->dag_cache, sizeof(double) * n);
  return n;
}

int32_t orc_dag_true_adj(const orc_trainer* tr, uint32_t* out) {
  for (int u = 0; u < tr->dag_d; ++u) out[u] = tr->dag_true_adj[u];
  return tr->dag_d;
}
