// host.cpp — host-side setup for libgfnx: environment tables (rewards tabulated with
// the reference's own fp64 expressions so the device reproduces them bit for bit),
// the DAG score cache, mode sets, parameter init, schedules and per-env defaults.
// Compiled with -ffp-contract=off (no FMA contraction), like the reference build
// the parity tests compare against.
#include "host.h"

#include <math.h>
#include <string.h>

#include <algorithm>
#include <numeric>
#include <set>

#include "engine.h"

namespace gfnx {

namespace {

void random_uniform(Key key, size_t n, double* out) {  // rng.cpp:52-62
  for (size_t i = 0; i < n; i += 2) {
    uint64_t a, b;
    threefry2x64(key, i / 2, 0, a, b);
    out[i] = to_unit(a);
    if (i + 1 < n) out[i + 1] = to_unit(b);
  }
}

void random_normal(Key key, size_t n, double* out) {  // rng.cpp:68-80
  for (size_t i = 0; i < n; i += 2) {
    uint64_t a, b;
    threefry2x64(key, i / 2, 1, a, b);
    double u1 = to_unit(a);
    const double u2 = to_unit(b);
    if (u1 <= 0.0) u1 = 0x1.0p-53;
    const double r = sqrt(-2.0 * log(u1));
    out[i] = r * cos(2.0 * M_PI * u2);
    if (i + 1 < n) out[i + 1] = r * sin(2.0 * M_PI * u2);
  }
}

int random_range(Key key, int n) { return (int)(uniform_scalar(key) * n) % n; }  // rng.cpp:82-85

double cholesky_logdet(std::vector<double>& a, int n, bool* ok) {  // dag.cpp:20-38
  double logdet = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = a[(size_t)i * n + j];
      for (int k = 0; k < j; ++k) s -= a[(size_t)i * n + k] * a[(size_t)j * n + k];
      if (i == j) {
        if (!(s > 0.0)) *ok = false;
        a[(size_t)i * n + j] = sqrt(s);
        logdet += 2.0 * log(a[(size_t)i * n + j]);
      } else {
        a[(size_t)i * n + j] = s / a[(size_t)j * n + j];
      }
    }
  return logdet;
}

void cholesky_solve(const std::vector<double>& l, int n, std::vector<double>& b) {  // :41-54
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

double log_multivariate_gamma(int ell, double a) {  // dag.cpp:56-60
  double v = 0.25 * ell * (ell - 1) * log(M_PI);
  for (int i = 1; i <= ell; ++i) v += lgamma(a + 0.5 * (1.0 - i));
  return v;
}

// generate_er_dataset (dag.cpp:70-119) + LocalScoreCache::{lingauss,bge} (:163-298)
std::string build_dag(const gfnx_env_desc& e, HostEnv* out) {
  const int d = e.dag_d, n = e.dag_data_n;
  if (d < 2 || d > kMaxDagD) return "dag env: d must lie in [2, 8] on the device path";
  if (n < 1) return "er dataset: n must be >= 1";
  if (e.dag_expected_in_degree < 0.0) return "er dataset: negative in-degree";
  const Key key = fold_in(make_key(e.dag_data_seed), 0xDA7A);  // train.cpp:563-566
  std::vector<int> order(d);
  std::iota(order.begin(), order.end(), 0);
  for (int i = d - 1; i > 0; --i) {
    const int j = random_range(fold_in(key, 1000 + (uint64_t)i), i + 1);
    std::swap(order[i], order[j]);
  }
  const double p = std::min(1.0, 2.0 * e.dag_expected_in_degree / (d - 1));
  const Key edge_key = fold_in(key, 1), weight_key = fold_in(key, 2);
  std::vector<double> weights((size_t)d * d), tw((size_t)d * d, 0.0);
  random_normal(weight_key, weights.size(), weights.data());
  std::vector<uint32_t> adj(d, 0);
  uint64_t draw = 0;
  for (int i = 0; i < d; ++i)
    for (int j = i + 1; j < d; ++j) {
      const int u = order[i], v = order[j];
      if (uniform_scalar(fold_in(edge_key, draw++)) < p) {
        adj[u] |= 1u << v;
        tw[(size_t)u * d + v] = weights[(size_t)u * d + v];
      }
    }
  const double noise_sd = sqrt(0.1);
  std::vector<double> eps((size_t)n * d), x((size_t)n * d, 0.0);
  random_normal(fold_in(key, 3), eps.size(), eps.data());
  for (int row = 0; row < n; ++row)
    for (int pos = 0; pos < d; ++pos) {
      const int j = order[pos];
      double mean = 0.0;
      for (int u = 0; u < d; ++u)
        if (adj[u] & (1u << j)) mean += tw[(size_t)u * d + j] * x[(size_t)row * d + u];
      x[(size_t)row * d + j] = mean + noise_sd * eps[(size_t)row * d + j];
    }
  out->dag_true_adj = adj;
  const uint32_t nmask = 1u << d;
  out->dag_cache.assign((size_t)d * nmask, 0.0);
  const double nn = (double)n;
  bool ok = true;
  if (e.dag_score == GFNX_DAG_LINGAUSS) {
    const double s2 = e.dag_noise_var, w2 = e.dag_weight_var;
    if (!(s2 > 0.0) || !(w2 > 0.0)) return "score cache: variances must be positive";
    std::vector<double> gram((size_t)d * d, 0.0);
    for (int i = 0; i < n; ++i)
      for (int a = 0; a < d; ++a)
        for (int b = 0; b <= a; ++b) {
          const double v = x[(size_t)i * d + a] * x[(size_t)i * d + b];
          gram[(size_t)a * d + b] += v;
          if (a != b) gram[(size_t)b * d + a] += v;
        }
    for (int j = 0; j < d; ++j) {
      const double yy = gram[(size_t)j * d + j];
      for (uint32_t mask = 0; mask < nmask; ++mask) {
        if (mask & (1u << j)) continue;
        std::vector<int> pa;
        for (int i = 0; i < d; ++i)
          if (mask & (1u << i)) pa.push_back(i);
        const int np = (int)pa.size();
        double quad = yy / s2;
        double logdet = nn * log(s2);
        if (np > 0) {
          std::vector<double> bm((size_t)np * np), v(np);
          for (int a = 0; a < np; ++a) {
            v[a] = gram[(size_t)pa[a] * d + j];
            for (int c = 0; c < np; ++c)
              bm[(size_t)a * np + c] = gram[(size_t)pa[a] * d + pa[c]] / s2 + (a == c ? 1.0 / w2 : 0.0);
          }
          const double logdet_b = cholesky_logdet(bm, np, &ok);
          std::vector<double> xs = v;
          cholesky_solve(bm, np, xs);
          double vx = 0.0;
          for (int a = 0; a < np; ++a) vx += v[a] * xs[a];
          quad -= vx / (s2 * s2);
          logdet += np * log(w2) + logdet_b;
        }
        out->dag_cache[(size_t)j * nmask + mask] = -0.5 * (nn * log(2.0 * M_PI) + logdet + quad);
      }
    }
  } else {
    const double alpha_mu = e.dag_alpha_mu;
    const double alpha_w = e.dag_alpha_w > 0.0 ? e.dag_alpha_w : d + 2.0;
    if (!(alpha_mu > 0.0)) return "bge: alpha_mu must be positive";
    if (!(alpha_w > d - 1)) return "bge: alpha_w must exceed d - 1";
    std::vector<double> xbar(d, 0.0), r((size_t)d * d, 0.0);
    for (int i = 0; i < n; ++i)
      for (int a = 0; a < d; ++a) xbar[a] += x[(size_t)i * d + a];
    for (int a = 0; a < d; ++a) xbar[a] /= nn;
    for (int i = 0; i < n; ++i)
      for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b)
          r[(size_t)a * d + b] += (x[(size_t)i * d + a] - xbar[a]) * (x[(size_t)i * d + b] - xbar[b]);
    const double shrink = nn * alpha_mu / (nn + alpha_mu);
    for (int a = 0; a < d; ++a) {
      for (int b = 0; b < d; ++b) r[(size_t)a * d + b] += shrink * xbar[a] * xbar[b];
      r[(size_t)a * d + a] += 1.0;
    }
    std::vector<double> logdet_r(nmask, 0.0), subset_ml(nmask, 0.0);
    for (uint32_t mask = 1; mask < nmask; ++mask) {
      std::vector<int> mem;
      for (int i = 0; i < d; ++i)
        if (mask & (1u << i)) mem.push_back(i);
      const int ell = (int)mem.size();
      std::vector<double> sub((size_t)ell * ell);
      for (int a = 0; a < ell; ++a)
        for (int b = 0; b < ell; ++b) sub[(size_t)a * ell + b] = r[(size_t)mem[a] * d + mem[b]];
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
        out->dag_cache[(size_t)j * nmask + mask] = subset_ml[mask | (1u << j)] - subset_ml[mask];
      }
  }
  if (!ok) return "cholesky: matrix not positive definite";
  return "";
}

// generate_modes (sequences.cpp:72-98) with key fold_in(make_key(modes_seed), 0x30DE)
std::string build_modes(const gfnx_env_desc& e, HostEnv* out) {
  static const char* words[5] = {"00000000", "11111111", "11110000", "00001111", "00111100"};
  const int n = e.bs_n_bits;
  if (n <= 0 || n % 8 != 0) return "generate_modes: need 8 | n";
  if (e.bs_num_modes < 1) return "generate_modes: target_count must be positive";
  if (n > 64 * kMaxModeWords) return "bitseq: n_bits exceeds device cap (512)";
  const int blocks = n / 8;
  double distinct = 1.0;
  for (int i = 0; i < blocks; ++i) distinct *= 5.0;
  const int cap = distinct < (double)e.bs_num_modes ? (int)distinct : e.bs_num_modes;
  const Key key = fold_in(make_key(e.bs_modes_seed), 0x30DE);
  std::set<std::string> seen;
  uint64_t draw = 0;
  while ((int)seen.size() < cap) {
    std::string mode;
    for (int b = 0; b < blocks; ++b) mode += words[random_range(fold_in(key, draw++), 5)];
    seen.insert(mode);
  }
  out->n_modes = (int)seen.size();
  out->mode_words = (n + 63) / 64;
  out->modes.assign((size_t)out->n_modes * out->mode_words, 0);
  int m = 0;
  for (const auto& s : seen) {
    for (int i = 0; i < n; ++i)
      if (s[i] == '1') out->modes[(size_t)m * out->mode_words + i / 64] |= 1ull << (63 - i % 64);
    ++m;
  }
  out->bs_logr.resize(n + 1);
  for (int dd = 0; dd <= n; ++dd)  // ModeSet::log_reward :54
    out->bs_logr[dd] = -e.bs_beta * (double)dd / (double)n;
  return "";
}

}  // namespace

std::string build_host_env(const gfnx_env_desc& e, HostEnv* out) {
  gfnx_env_shape& s = out->shape;
  int max_parents = 1;
  switch (e.kind) {
    case GFNX_ENV_HYPERGRID: {  // HypergridEnv::validate + shape (hypergrid.hpp:32-36)
      if (e.hg_dim < 1 || e.hg_dim > kMaxHgDim) return "hypergrid: dim must lie in [1, 8]";
      if (e.hg_side < 2 || e.hg_side > 256) return "hypergrid: side must lie in [2, 256]";
      if (e.hg_r0 < 0.0 || e.hg_r1 < 0.0 || e.hg_r2 < 0.0)
        return "hypergrid: reward terms must be nonnegative";
      if (e.hg_r0 <= 0.0) return "hypergrid: r0 must be positive for log rewards";
      s.num_actions = s.num_backward_actions = e.hg_dim + 1;
      s.obs_dim = e.hg_dim * e.hg_side;
      s.max_traj_len = e.hg_dim * (e.hg_side - 1) + 1;
      s.stop_action = e.hg_dim;
      s.state_words = (e.hg_dim + 3) / 4;
      for (int c = 0; c < e.hg_side; ++c) {  // grid_log_reward per-coordinate tests (:111-119)
        const double x = fabs((double)c / (e.hg_side - 1) - 0.5);
        if (0.25 < x) out->hg_f1[c >> 5] |= 1u << (c & 31);
        if (0.3 < x && x < 0.4) out->hg_f2[c >> 5] |= 1u << (c & 31);
      }
      for (int p1 = 0; p1 < 2; ++p1)
        for (int p2 = 0; p2 < 2; ++p2)
          out->hg_logr[p1 | (p2 << 1)] = log(e.hg_r0 + e.hg_r1 * (double)p1 + e.hg_r2 * (double)p2);
      max_parents = e.hg_dim;
      break;
    }
    case GFNX_ENV_BITSEQ: {  // build_bitseq (train.cpp:381-427): NAR, or the AR-fixed scheme
      if (e.bs_k < 1 || e.bs_k > 8 || e.bs_n_bits % e.bs_k != 0)
        return "bitseq: k must divide n_bits (1 <= k <= 8)";
      if (e.bs_scheme != 0 && e.bs_scheme != 1)
        return "bitseq: scheme must be 0 (non-autoregressive) or 1 (autoregressive fixed)";
      out->bs_slots = e.bs_n_bits / e.bs_k;
      out->bs_vocab = 1 << e.bs_k;
      if (out->bs_slots > kMaxSlots) return "bitseq: n_bits / k exceeds device cap (64 slots)";
      // num_actions / num_backward_actions (sequences.cpp:200-218): NAR pos * vocab + word over
      // every slot, one remove-per-slot backward action; AR fixed: the next token, remove-last
      s.num_actions = e.bs_scheme ? out->bs_vocab : out->bs_slots * out->bs_vocab;
      s.num_backward_actions = e.bs_scheme ? 1 : out->bs_slots;
      s.obs_dim = out->bs_slots * (out->bs_vocab + 1) + 1;
      s.max_traj_len = out->bs_slots;
      s.stop_action = -1;
      s.state_words = (out->bs_slots + 3) / 4 + (out->bs_slots + 31) / 32;
      const std::string err = build_modes(e, out);
      if (!err.empty()) return err;
      max_parents = out->bs_slots;
      break;
    }
    case GFNX_ENV_ISING: {  // toroidal_coupling (ising.cpp:15-31)
      const int side = e.is_side;
      if (side < 2) return "ising: lattice side must be >= 2";
      const int D = side * side;
      if (D > kMaxIsingD) return "ising: side^2 exceeds device cap (256)";
      out->is_D = D;
      std::vector<double> J((size_t)D * D, 0.0);
      auto site = [side](int r, int c) { return ((r + side) % side) * side + (c + side) % side; };
      const int dr[4] = {1, -1, 0, 0}, dc[4] = {0, 0, 1, -1};
      for (int r = 0; r < side; ++r)
        for (int c = 0; c < side; ++c) {
          const int a = site(r, c);
          for (int q = 0; q < 4; ++q) {
            const int b = site(r + dr[q], c + dc[q]);
            if (a != b) J[(size_t)a * D + b] = e.is_sigma;
          }
        }
      out->is_nbr.assign((size_t)D * 4, -1);
      out->is_J.assign((size_t)D * 4, 0.0);
      for (int a = 0; a < D; ++a) {
        int q = 0;
        for (int b = 0; b < D; ++b)
          if (J[(size_t)a * D + b] != 0.0) {
            if (q >= 4) return "ising: coupling row has more than 4 nonzeros";
            out->is_nbr[(size_t)a * 4 + q] = (int16_t)b;
            out->is_J[(size_t)a * 4 + q] = J[(size_t)a * D + b];
            ++q;
          }
      }
      s.num_actions = 2 * D;
      s.num_backward_actions = D;
      s.obs_dim = 3 * D;
      s.max_traj_len = D;
      s.stop_action = -1;
      s.state_words = 2 * ((D + 31) / 32);
      max_parents = D;
      break;
    }
    case GFNX_ENV_DAG: {
      const std::string err = build_dag(e, out);
      if (!err.empty()) return err;
      const int d = e.dag_d;
      s.num_actions = s.num_backward_actions = d * (d - 1) + 1;
      s.obs_dim = d * d;
      s.max_traj_len = d * (d - 1) / 2 + 1;
      s.stop_action = d * (d - 1);
      s.state_words = (d + 1) / 2;
      max_parents = d * (d - 1) / 2 + 1;
      break;
    }
    default:
      return "unknown env kind";
  }
  out->neglog.assign(max_parents + 1, 0.0);
  for (int k = 1; k <= max_parents; ++k) out->neglog[k] = -log((double)k);  // env_core.hpp:207
  return "";
}

std::string validate_train(const gfnx_train_desc& t, const gfnx_env_shape& s) {
  if (t.objective == GFNX_OBJ_FLDB) return "fldb objective is out of scope (phylo only)";
  if (t.objective < 0 || t.objective > 4) return "unknown objective";
  if (t.learned_backward != 0 && t.learned_backward != 1) return "learned_backward must be 0 or 1";
  if (t.learned_backward && t.precision != GFNX_PREC_FP64_CHECK)
    return "learned backward policy: fp64 check mode only (the bf16 paths use the uniform P_B)";
  if (t.objective == GFNX_OBJ_MDB && s.stop_action < 0)
    return "mdb objective needs the stop action index";
  if (t.objective == GFNX_OBJ_SUBTB && (t.subtb_lambda <= 0.0 || t.subtb_lambda > 1.0))
    return "subtb lambda must lie in (0, 1]";
  if (t.num_hidden < 1 || t.num_hidden > 8) return "mlp_init: need 1..8 hidden layers";
  for (int l = 0; l < t.num_hidden; ++l)
    if (t.hidden[l] < 1 || t.hidden[l] > 512) return "mlp_init: hidden width must lie in [1, 512]";
  if (t.batch_size < 1) return "forward_rollout: num_envs must be >= 1";
  if (t.deterministic != 0 && t.deterministic != 1) return "deterministic must be 0 or 1";
  if (t.precision != GFNX_PREC_BF16 && t.precision != GFNX_PREC_FP64_CHECK)
    return "unknown precision";
  return "";
}

void make_layout(const gfnx_train_desc& t, const gfnx_env_shape& s, MlpLayout* L) {
  L->n_trunk = t.num_hidden;
  L->dims[0] = s.obs_dim;
  for (int l = 0; l < t.num_hidden; ++l) L->dims[l + 1] = t.hidden[l];
  int64_t off = 0;
  for (int l = 0; l < L->n_trunk; ++l) {
    L->off_w[l] = off;
    off += (int64_t)L->dims[l] * L->dims[l + 1];
    L->off_b[l] = off;
    off += L->dims[l + 1];
  }
  const int H = L->H();
  L->off_fw = off; off += (int64_t)H * s.num_actions;
  L->off_fb = off; off += s.num_actions;
  L->off_bw = off; off += (int64_t)H * s.num_backward_actions;
  L->off_bb = off; off += s.num_backward_actions;
  L->off_flw = off; off += H;
  L->off_flb = off; off += 1;
  L->n_params = off;
}

void init_params(const gfnx_train_desc& t, const MlpLayout& L, int A, int Ab,
                 std::vector<double>* params) {
  params->assign(L.n_params, 0.0);
  const Key key = fold_in(make_key(t.seed), 0);
  int k = 0;
  auto dense = [&](int64_t off, int in, int out) {  // dense_init nn.cpp:28-39
    const double bound = 1.0 / sqrt((double)in);
    const size_t n = (size_t)in * out;
    std::vector<double> u(n);
    random_uniform(fold_in(key, k++), n, u.data());
    for (size_t i = 0; i < n; ++i) (*params)[off + i] = (2.0 * u[i] - 1.0) * bound;
  };
  for (int l = 0; l < L.n_trunk; ++l) dense(L.off_w[l], L.dims[l], L.dims[l + 1]);
  dense(L.off_fw, L.H(), A);
  dense(L.off_bw, L.H(), Ab);
  dense(L.off_flw, L.H(), 1);
}

std::vector<double> ising_dense_coupling(int side, double sigma) {  // toroidal_coupling ising.cpp:15-31
  const int D = side * side;
  std::vector<double> J((size_t)D * D, 0.0);
  auto site = [side](int r, int c) { return ((r + side) % side) * side + (c + side) % side; };
  const int dr[4] = {1, -1, 0, 0}, dc[4] = {0, 0, 1, -1};
  for (int r = 0; r < side; ++r)
    for (int c = 0; c < side; ++c) {
      const int a = site(r, c);
      for (int q = 0; q < 4; ++q) {
        const int b = site(r + dr[q], c + dc[q]);
        if (a != b) J[(size_t)a * D + b] = sigma;
      }
    }
  return J;
}

namespace {
double dense_energy(const std::vector<int8_t>& s, const std::vector<double>& J, int D) {  // ising.cpp:40-51
  double quad = 0.0;
  for (int a = 0; a < D; ++a) {
    double row = 0.0;
    for (int b = 0; b < D; ++b) row += J[(size_t)a * D + b] * s[b];
    quad += s[a] * row;
  }
  return -quad;
}
}  // namespace

// gibbs_data_sampler (ising.cpp:185-220) with gibbs_sweep / heat_bath_prob_up (:162-183):
// heat-bath sweeps of chain 0 (+ parallel tempering when chains > 1), burn-in, thinning.
// One-time synthetic data generation for EB-GFN (train.cpp:899-907), like build_dag's data.
std::vector<int8_t> ising_gibbs_data(const std::vector<double>& J, int D, Key key, int64_t n_samples,
                                     int64_t burn_in, int64_t thinning, int chains, double hottest_beta) {
  std::vector<double> betas(chains, 1.0);
  for (int c = 1; c < chains; ++c) {
    const double frac = (double)c / (chains - 1);
    betas[c] = exp(log(1.0) + frac * (log(hottest_beta)));
  }
  std::vector<std::vector<int8_t>> state(chains, std::vector<int8_t>(D));
  std::vector<double> u(D);
  for (int c = 0; c < chains; ++c) {
    random_uniform(fold_in(fold_in(key, 7777), (uint64_t)c), (size_t)D, u.data());
    for (int a = 0; a < D; ++a) state[c][a] = u[a] < 0.5 ? -1 : 1;
  }
  std::vector<int8_t> out;
  out.reserve((size_t)n_samples * D);
  int64_t sweep = 0, got = 0;
  while (got < n_samples) {
    const Key sweep_key = fold_in(key, (uint64_t)sweep);
    for (int c = 0; c < chains; ++c) {
      const Key ck = fold_in(sweep_key, (uint64_t)c);
      std::vector<int8_t>& sp = state[c];
      for (int site = 0; site < D; ++site) {
        double h = 0.0;
        for (int b = 0; b < D; ++b)
          if (b != site) h += J[(size_t)site * D + b] * sp[b];
        const double p_up = 1.0 / (1.0 + exp(-4.0 * betas[c] * h));
        sp[site] = uniform_scalar(fold_in(ck, (uint64_t)site)) < p_up ? 1 : -1;
      }
    }
    if (chains > 1) {
      for (int c = (int)(sweep % 2); c + 1 < chains; c += 2) {
        const double e_lo = dense_energy(state[c], J, D);
        const double e_hi = dense_energy(state[c + 1], J, D);
        const double log_a = (betas[c] - betas[c + 1]) * (e_lo - e_hi);
        if (log(uniform_scalar(fold_in(fold_in(sweep_key, 999), (uint64_t)c))) < log_a) std::swap(state[c], state[c + 1]);
      }
    }
    ++sweep;
    if (sweep > burn_in && (sweep - burn_in) % thinning == 0) {
      out.insert(out.end(), state[0].begin(), state[0].end());
      ++got;
    }
  }
  return out;
}

double schedule_value(const gfnx_schedule& s, int64_t step) {
  if (s.warmup > 0 && step < s.warmup) return s.start_value * (double)step / (double)s.warmup;
  const double prog = s.horizon > 0 ? std::min(1.0, (double)(step - s.warmup) / (double)s.horizon) : 1.0;
  switch (s.kind) {
    case 0: return s.start_value;
    case 1:
      if (s.horizon <= 0) return s.end_value;
      return s.start_value + (s.end_value - s.start_value) * prog;
    case 2:
      if (s.horizon <= 0) return s.end_value;
      return s.end_value + 0.5 * (s.start_value - s.end_value) * (1.0 + cos(M_PI * prog));
  }
  return s.start_value;
}

void resolve_schedule(gfnx_schedule* s, int64_t iterations) {
  if (s->horizon < 0) s->horizon = std::max<int64_t>(1, iterations / 2);
  if (s->horizon == 0) s->horizon = std::max<int64_t>(1, iterations - s->warmup);
}

void default_env(int kind, gfnx_env_desc* e) {  // builder defaults train.cpp:361-366,388-396,531-583,637-640
  memset(e, 0, sizeof *e);
  e->kind = kind;
  e->hg_dim = 2; e->hg_side = 8; e->hg_r0 = 1e-3; e->hg_r1 = 0.5; e->hg_r2 = 2.0;
  e->bs_n_bits = 8; e->bs_k = 2; e->bs_beta = 3.0; e->bs_num_modes = 60; e->bs_modes_seed = 0;
  e->is_side = 3; e->is_sigma = 0.2;
  e->dag_d = 5; e->dag_score = GFNX_DAG_LINGAUSS; e->dag_alpha_mu = 1.0; e->dag_alpha_w = 0.0;
  e->dag_noise_var = 0.1; e->dag_weight_var = 1.0; e->dag_expected_in_degree = 1.0;
  e->dag_data_n = 100; e->dag_data_seed = 0;
}

void default_train(int kind, gfnx_train_desc* t) {  // EnvDefaults + read_settings
  memset(t, 0, sizeof *t);
  int64_t iterations = 1000;
  int batch = 16;
  double lr = 1e-3, z_lr = 0.1, wd = 0.0, eps0 = 0.0, eps1 = 0.0;
  int64_t eps_h = 0;
  int hidden[4] = {256, 256, 0, 0}, nh = 2;
  int objective = GFNX_OBJ_TB;
  switch (kind) {
    case GFNX_ENV_HYPERGRID: iterations = 62500; break;
    case GFNX_ENV_BITSEQ: iterations = 50000; z_lr = 0.05; wd = 1e-5; eps0 = eps1 = 1e-3; break;
    case GFNX_ENV_DAG:
      iterations = 100000; batch = 128; lr = 1e-4; hidden[0] = hidden[1] = 128;
      objective = GFNX_OBJ_MDB; eps0 = 1.0; eps1 = 0.1; eps_h = -1;
      break;
    case GFNX_ENV_ISING:
      iterations = 20000; batch = 256; nh = 4; hidden[2] = hidden[3] = 256;
      break;
  }
  t->objective = objective;
  t->subtb_lambda = 0.9;
  t->terminal_penalty = 1.0;
  t->batch_size = batch;
  t->num_hidden = nh;
  for (int i = 0; i < nh; ++i) t->hidden[i] = hidden[i];
  t->beta1 = 0.9; t->beta2 = 0.999; t->adam_eps = 1e-8; t->weight_decay = wd; t->z_lr = z_lr;
  t->lr.kind = 0; t->lr.start_value = lr; t->lr.end_value = lr;
  t->explore.kind = eps0 == eps1 ? 0 : 1;
  t->explore.start_value = eps0; t->explore.end_value = eps1; t->explore.horizon = eps_h;
  t->iterations = iterations;
  t->precision = GFNX_PREC_BF16;
}

}  // namespace gfnx
