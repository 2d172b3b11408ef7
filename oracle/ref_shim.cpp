// ref_shim.cpp — C ABI over the UNMODIFIED reference library (gfnkit) built from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libgfnref.so.
//
// TEST INFRASTRUCTURE ONLY: used to pin the oracle restatement (oracle/gfn_oracle.c)
// and to generate golden fixtures (tests/golden/make_golden.py), and as the
// "reference" CPU baseline in bench.py. Everything on the numeric path goes
// through the reference's public API: forward_rollout (env_core.hpp:232-274),
// mlp_forward_tape (nn.cpp:91-126), build_loss (objectives.cpp:230-240),
// Tape::backward (tape.cpp:321-333), adam_step (optim.cpp:19-43) and, for the
// stock benchmark, run_bench (train.cpp:801-809). The ~20 lines of train_step
// glue mirror train.cpp:164-192, which sits in an anonymous namespace.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <type_traits>
#include <vector>

#include "gfn/checkpoint.hpp"
#include "gfn/config.hpp"
#include "gfn/env_core.hpp"
#include "gfn/envs/dag.hpp"
#include "gfn/envs/hypergrid.hpp"
#include "gfn/envs/ising.hpp"
#include "gfn/envs/sequences.hpp"
#include "gfn/errors.hpp"
#include "gfn/exact.hpp"
#include "gfn/metrics.hpp"
#include "gfn/nn.hpp"
#include "gfn/objectives.hpp"
#include "gfn/optim.hpp"
#include "gfn/rng.hpp"
#include "gfn/train.hpp"

#include "../include/gfnx.h"

namespace {

using namespace gfn;

thread_local std::string g_err;

Schedule to_sched(const gfnx_schedule& s, int64_t iterations) {
  Schedule o;
  o.kind = s.kind == 1 ? Schedule::Kind::kLinear
         : s.kind == 2 ? Schedule::Kind::kCosine : Schedule::Kind::kConstant;
  o.start_value = s.start_value;
  o.end_value = s.end_value;
  o.warmup = s.warmup;
  int64_t h = s.horizon;
  if (h < 0) h = std::max<int64_t>(1, iterations / 2);
  if (h == 0) h = std::max<int64_t>(1, iterations - s.warmup);
  o.horizon = h;
  return o;
}

struct SessionBase {
  virtual ~SessionBase() = default;
  virtual void rollout(int64_t it, double eps) = 0;
  virtual double compute_grads() = 0;
  virtual void apply_adam(double lr) = 0;
  virtual const TrajectoryBatch& batch() const = 0;
  virtual MlpParams& policy() = 0;
  // distance of the policy's exact terminal marginal (exact_policy_marginal, exact.hpp:76)
  // to the target: TV for hypergrid (grid_exact_distribution) and Ising
  // (ising_exact_distribution), JSD for DAG (dag_exact_posterior) - acceptance criteria 1, 3, 5
  virtual double exact_divergence() { throw config_error("exact divergence: hypergrid, DAG and Ising only"); }
  // the bitseq `pearson` metric (train.cpp:440-454): Pearson correlation of the Monte-Carlo
  // terminal log-probabilities (mc_terminal_logprob, exact.hpp:229-241, `mc` backward samples)
  // and the log-rewards over the builder's test set (generate_test_set, train.cpp:431-433)
  virtual double pearson_metric(int64_t, int, uint64_t) { throw config_error("pearson: bitseq only"); }
  // mc_terminal_logprob (exact.hpp:229-241) of one packed terminal state
  virtual double mc_logprob(const uint32_t*, int, const RngKey&) = 0;
  // backward_rollout (env_core.hpp:314-370) of n packed terminal states -> the session batch
  virtual void backward_batch(const uint32_t*, int, const RngKey&) = 0;
  virtual void set_packing(int state_words) = 0;
  virtual std::vector<double>& grads() = 0;
  virtual double& dlogz() = 0;
  virtual AdamState& opt_main() = 0;
  virtual AdamState& opt_z() = 0;
};

template <VectorEnv E>
struct Session : SessionBase {
  E env;
  typename E::Params params;
  gfnx_train_desc td;
  LossConfig loss;
  AdamConfig adam, adam_z;
  RngKey root;
  MlpParams pol;
  AdamState om, oz;
  TrajectoryBatch tb;
  std::vector<double> g;
  double dz = 0.0;

  Session(typename E::Params p, const gfnx_train_desc& t, int stop) : params(std::move(p)), td(t) {
    loss.objective = static_cast<Objective>(t.objective);
    loss.subtb_lambda = t.subtb_lambda;
    loss.learned_backward = t.learned_backward != 0;
    loss.terminal_penalty = t.terminal_penalty;
    loss.stop_action = stop;
    adam.beta1 = t.beta1;
    adam.beta2 = t.beta2;
    adam.eps = t.adam_eps;
    adam.weight_decay = t.weight_decay;
    adam.lr = t.lr.start_value;
    adam_z = adam;
    adam_z.lr = t.z_lr;
    adam_z.weight_decay = 0.0;
    root = make_key(t.seed);
    std::vector<int> hidden(t.hidden, t.hidden + t.num_hidden);
    pol = mlp_init(env.obs_dim(params), hidden, env.num_actions(params),
                   env.num_backward_actions(params), fold_in(root, 0), t.logz_init);
    om = adam_init(pol.tensors());
    std::vector<Tensor*> zp = {&pol.log_z};
    oz = adam_init(zp);
  }
  void rollout(int64_t it, double eps) override {
    RolloutOptions ropt;
    ropt.record_delta_log_reward = loss.objective == Objective::kMDB;
    tb = forward_rollout(env, params, pol, td.batch_size, fold_in(root, 1000 + it), eps, ropt);
  }
  // train.cpp:164-183 (forward, loss, finite check, backward)
  double compute_grads() override {
    const bool need_flow = loss.objective == Objective::kDB ||
                           loss.objective == Objective::kSubTB ||
                           loss.objective == Objective::kFLDB;
    Tape tape;
    MlpTapeBind bind = mlp_forward_tape(tape, pol, tb.obs_tensor(), loss.learned_backward, need_flow);
    HeadVars heads;
    heads.fwd_logits = bind.fwd_logits;
    heads.bwd_logits = bind.bwd_logits;
    heads.log_flow = bind.log_flow;
    heads.log_z = bind.log_z;
    const Tape::Var l = build_loss(tape, tb, heads, loss);
    const double lv = tape.value(l).data[0];
    if (!std::isfinite(lv)) throw numeric_error("training loss is not finite");
    tape.backward(l);
    g.clear();
    for (Tape::Var v : bind.leaves) {
      const Tensor& gt = tape.grad(v);
      g.insert(g.end(), gt.data.begin(), gt.data.end());
    }
    dz = tape.grad(bind.log_z_leaf).data[0];
    return lv;
  }
  // train.cpp:184-190
  void apply_adam(double lr) override {
    auto tensors = pol.tensors();
    std::vector<Tensor> gts;
    size_t off = 0;
    for (Tensor* t : tensors) {
      Tensor gt(t->shape);
      std::copy(g.begin() + off, g.begin() + off + gt.data.size(), gt.data.begin());
      off += gt.data.size();
      gts.push_back(std::move(gt));
    }
    std::vector<const Tensor*> gp;
    for (auto& x : gts) gp.push_back(&x);
    adam_step(om, tensors, gp, adam, lr);
    if (loss.objective == Objective::kTB) {
      std::vector<Tensor*> zp = {&pol.log_z};
      Tensor zg = Tensor::scalar(dz);
      std::vector<const Tensor*> zgp = {&zg};
      adam_step(oz, zp, zgp, adam_z);
    }
  }
  const TrajectoryBatch& batch() const override { return tb; }
  MlpParams& policy() override { return pol; }
  double exact_divergence() override {
    if constexpr (std::is_same_v<E, HypergridEnv>) {
      auto graph = enumerate_state_graph(env, params);
      return tv_distance(exact_policy_marginal(env, params, graph, pol), grid_exact_distribution(params));
    } else if constexpr (std::is_same_v<E, DagEnv>) {
      auto graph = enumerate_state_graph(env, params);
      return jsd(exact_policy_marginal(env, params, graph, pol), dag_exact_posterior(*params.score));
    } else if constexpr (std::is_same_v<E, IsingEnv>) {  // criterion 5 (acceptance.cpp:342-360)
      auto graph = enumerate_state_graph(env, params);
      return tv_distance(exact_policy_marginal(env, params, graph, pol), ising_exact_distribution(*params.coupling));
    } else {
      return SessionBase::exact_divergence();
    }
  }
  // the env's terminal instance of packed device state words (DESIGN.md §4 layouts)
  typename E::Instance terminal_of(const uint32_t* w) const {
    typename E::Instance inst = env.reset_instance(params);
    if constexpr (std::is_same_v<E, HypergridEnv>) {
      int sum = 0;
      for (int i = 0; i < params.dim; ++i) {  // packed: byte i = coordinate i
        inst.coords[i] = static_cast<int>((w[i >> 2] >> (8 * (i & 3))) & 0xffu);
        sum += inst.coords[i];
      }
      inst.is_terminal = true;
      inst.step_count = sum + 1;
    } else if constexpr (std::is_same_v<E, DagEnv>) {  // packed: row u in half (u & 1) of word u >> 1
      const int d = params.d;
      for (int u = 0; u < d; ++u) {
        inst.adj[u] = (w[u >> 1] >> (16 * (u & 1))) & 0xffffu;
        inst.num_edges += __builtin_popcount(inst.adj[u]);
      }
      inst.closure_t = closure_from_adjacency(inst.adj);
      inst.is_terminal = true;
      inst.step_count = inst.num_edges + 1;
    } else if constexpr (std::is_same_v<E, SequenceEnv>) {  // token bytes, then the filled mask
      const int slots = params.max_len, tw = (slots + 3) / 4;
      std::string key;
      for (int i = 0; i < slots; ++i) {
        if (!((w[tw + (i >> 5)] >> (i & 31)) & 1u)) throw contract_violation("packed bitseq: empty slot");
        const int tok = static_cast<int>((w[i >> 2] >> (8 * (i & 3))) & 0xffu);
        for (int b = params.bit_block - 1; b >= 0; --b) key += ((tok >> b) & 1) ? '1' : '0';
      }
      inst = env.terminal_from_key(key, params);
    } else {  // Ising: assigned mask words, then the up mask words
      const int dim = params.coupling->dim();
      std::vector<int8_t> spins(dim);
      for (int i = 0; i < dim; ++i) {
        const bool as = (w[i >> 5] >> (i & 31)) & 1u;
        const bool up = (w[pk_half + (i >> 5)] >> (i & 31)) & 1u;
        spins[i] = as ? (up ? 1 : -1) : 0;
      }
      inst = env.terminal_from_spins(spins, params);
    }
    return inst;
  }
  int pk_half = 0;  // Ising: word offset of the up mask in the packed state (state_words / 2)
  double mc_logprob(const uint32_t* w, int K, const RngKey& key) override {
    return mc_terminal_logprob(env, params, pol, loss.learned_backward, terminal_of(w), K, key);
  }
  void backward_batch(const uint32_t* w, int n, const RngKey& key) override {
    EnvState<E> terms;
    for (int i = 0; i < n; ++i) terms.push_back(terminal_of(w + (size_t)i * sw));
    RolloutOptions ropt;
    ropt.record_delta_log_reward = loss.objective == Objective::kMDB;
    tb = backward_rollout(env, params, &pol, loss.learned_backward, terms, key, ropt);
  }
  int sw = 1;  // packed state words per state
  double pearson_metric(int64_t step, int mc, uint64_t test_seed) override {
    if constexpr (std::is_same_v<E, SequenceEnv>) {
      const auto* modes = dynamic_cast<const ModeSet*>(params.reward.get());
      if (!modes) throw config_error("pearson: mode-set reward only");
      const auto test_set = generate_test_set(*modes, fold_in(make_key(test_seed), 0x7E57));
      const RngKey mkey = fold_in(fold_in(make_key(td.seed), 0x3E7A), step);
      std::vector<double> log_p, log_r;
      for (size_t i = 0; i < test_set.size(); ++i) {
        auto inst = env.terminal_from_key(test_set[i], params);
        log_p.push_back(mc_terminal_logprob(env, params, pol, loss.learned_backward, inst, mc, fold_in(mkey, i)));
        log_r.push_back(modes->log_reward(test_set[i]));
      }
      return pearson(log_p, log_r);
    } else {
      return SessionBase::pearson_metric(step, mc, test_seed);
    }
  }
  void set_packing(int state_words) override {
    sw = state_words;
    pk_half = state_words / 2;
  }
  std::vector<double>& grads() override { return g; }
  double& dlogz() override { return dz; }
  AdamState& opt_main() override { return om; }
  AdamState& opt_z() override { return oz; }
};

std::unique_ptr<SessionBase> make_session_raw(const gfnx_env_desc& e, const gfnx_train_desc& t) {
  switch (e.kind) {
    case GFNX_ENV_HYPERGRID: {
      HypergridEnv::Params p;
      p.dim = e.hg_dim;
      p.side = e.hg_side;
      p.r0 = e.hg_r0;
      p.r1 = e.hg_r1;
      p.r2 = e.hg_r2;
      HypergridEnv::validate(p);
      return std::make_unique<Session<HypergridEnv>>(p, t, p.dim);
    }
    case GFNX_ENV_BITSEQ: {  // build_bitseq train.cpp:381-427
      auto modes = std::make_shared<ModeSet>(generate_modes(
          e.bs_n_bits, e.bs_beta, e.bs_num_modes, fold_in(make_key(e.bs_modes_seed), 0x30DE)));
      modes->beta = e.bs_beta;
      SequenceEnv::Params p;
      p.scheme = e.bs_scheme == 1 ? SeqScheme::kAutoregressiveFixed : SeqScheme::kNonAutoregressive;
      p.max_len = e.bs_n_bits / e.bs_k;
      p.vocab = 1 << e.bs_k;
      p.bit_block = e.bs_k;
      p.reward = modes;
      SequenceEnv::validate(p);
      return std::make_unique<Session<SequenceEnv>>(p, t, -1);
    }
    case GFNX_ENV_ISING: {  // build_ising train.cpp:637-657
      IsingEnv::Params p;
      p.coupling = std::make_shared<IsingCoupling>(toroidal_coupling(e.is_side, e.is_sigma));
      IsingEnv::validate(p);
      return std::make_unique<Session<IsingEnv>>(p, t, -1);
    }
    case GFNX_ENV_DAG: {  // build_dag train.cpp:523-586
      DagDataset data = generate_er_dataset(e.dag_d, e.dag_expected_in_degree, e.dag_data_n,
                                            fold_in(make_key(e.dag_data_seed), 0xDA7A));
      std::shared_ptr<LocalScoreCache> cache;
      if (e.dag_score == GFNX_DAG_LINGAUSS) {
        LocalScoreCache::LinGaussConfig lc;
        lc.noise_var = e.dag_noise_var;
        lc.weight_var = e.dag_weight_var;
        cache = std::make_shared<LocalScoreCache>(LocalScoreCache::lingauss(data, lc));
      } else {
        LocalScoreCache::BgeConfig bc;
        bc.alpha_mu = e.dag_alpha_mu;
        bc.alpha_w = e.dag_alpha_w;
        cache = std::make_shared<LocalScoreCache>(LocalScoreCache::bge(data, bc));
      }
      DagEnv::Params p;
      p.d = e.dag_d;
      p.score = cache;
      DagEnv::validate(p);
      return std::make_unique<Session<DagEnv>>(p, t, p.d * (p.d - 1));
    }
  }
  throw config_error("unknown env kind");
}

std::unique_ptr<SessionBase> make_session(const gfnx_env_desc& e, const gfnx_train_desc& t) {
  auto s = make_session_raw(e, t);
  // packed device state words: hypergrid a byte per coordinate; bitseq token
  // bytes + filled mask; Ising assigned + up masks; DAG 16-bit adjacency rows
  int sw = 1;
  switch (e.kind) {
    case GFNX_ENV_HYPERGRID: sw = (e.hg_dim + 3) / 4; break;
    case GFNX_ENV_BITSEQ: {
      const int slots = e.bs_n_bits / e.bs_k;
      sw = (slots + 3) / 4 + (slots + 31) / 32;
      break;
    }
    case GFNX_ENV_ISING: sw = 2 * ((e.is_side * e.is_side + 31) / 32); break;
    case GFNX_ENV_DAG: sw = (e.dag_d + 1) / 2; break;
  }
  s->set_packing(sw);
  return s;
}

struct RefSession {
  gfnx_env_desc env;
  gfnx_train_desc train;
  std::unique_ptr<SessionBase> s;
  std::string err;
};

template <class F>
int guard(RefSession* rs, F&& f) {
  try {
    f();
    return 0;
  } catch (const config_error& e) {
    (rs ? rs->err : g_err) = std::string("config_error: ") + e.what();
    return 1;
  } catch (const contract_violation& e) {
    (rs ? rs->err : g_err) = std::string("contract_violation: ") + e.what();
    return 2;
  } catch (const numeric_error& e) {
    (rs ? rs->err : g_err) = std::string("numeric_error: ") + e.what();
    return 3;
  } catch (const std::exception& e) {
    (rs ? rs->err : g_err) = std::string("error: ") + e.what();
    return 9;
  }
}

}  // namespace

extern "C" {

void* ref_create(const gfnx_env_desc* env, const gfnx_train_desc* train) {
  auto* rs = new RefSession{*env, *train, nullptr, ""};
  if (guard(nullptr, [&] { rs->s = make_session(*env, *train); })) {
    delete rs;
    return nullptr;
  }
  return rs;
}
void ref_destroy(void* h) { delete static_cast<RefSession*>(h); }
const char* ref_last_error(void* h) { return h ? static_cast<RefSession*>(h)->err.c_str() : g_err.c_str(); }

int ref_rollout(void* h, int64_t it, double eps) {
  auto* rs = static_cast<RefSession*>(h);
  return guard(rs, [&] { rs->s->rollout(it, eps); });
}

// Padded TrajectoryBatch fields; T = batch max_steps.
int ref_batch(void* h, int32_t* lengths, int32_t* fwd_actions, int32_t* bwd_actions,
              double* log_rewards, double* log_pb, double* delta) {
  auto* rs = static_cast<RefSession*>(h);
  const TrajectoryBatch& tb = rs->s->batch();
  const size_t bt = static_cast<size_t>(tb.num_traj) * tb.max_steps;
  if (lengths) std::copy(tb.lengths.begin(), tb.lengths.end(), lengths);
  if (fwd_actions) std::copy(tb.fwd_actions.begin(), tb.fwd_actions.begin() + bt, fwd_actions);
  if (bwd_actions) std::copy(tb.bwd_actions.begin(), tb.bwd_actions.begin() + bt, bwd_actions);
  if (log_rewards) std::copy(tb.log_rewards.begin(), tb.log_rewards.end(), log_rewards);
  if (log_pb) std::copy(tb.log_pb_uniform.begin(), tb.log_pb_uniform.begin() + bt, log_pb);
  if (delta) std::copy(tb.delta_log_reward.begin(), tb.delta_log_reward.begin() + bt, delta);
  return 0;
}

// Terminal keys (encode_terminal) joined with '\n' into buf.
int ref_terminal_keys(void* h, char* buf, int64_t cap) {
  auto* rs = static_cast<RefSession*>(h);
  std::string all;
  for (const auto& k : rs->s->batch().terminal_keys) all += k + "\n";
  if (static_cast<int64_t>(all.size()) + 1 > cap) return -1;
  std::memcpy(buf, all.c_str(), all.size() + 1);
  return static_cast<int>(all.size());
}

int ref_compute_grads(void* h, double* loss) {
  auto* rs = static_cast<RefSession*>(h);
  return guard(rs, [&] { *loss = rs->s->compute_grads(); });
}

int64_t ref_num_params(void* h) {
  auto* rs = static_cast<RefSession*>(h);
  int64_t n = 0;
  for (const Tensor* t : rs->s->policy().tensors()) n += t->size();
  return n;
}

void ref_get_grads(void* h, double* flat, double* dlogz) {
  auto* rs = static_cast<RefSession*>(h);
  std::copy(rs->s->grads().begin(), rs->s->grads().end(), flat);
  *dlogz = rs->s->dlogz();
}

void ref_apply_adam(void* h, double lr) { static_cast<RefSession*>(h)->s->apply_adam(lr); }

void ref_get_params(void* h, double* flat, double* log_z) {
  auto* rs = static_cast<RefSession*>(h);
  size_t off = 0;
  for (const Tensor* t : rs->s->policy().tensors()) {
    std::copy(t->data.begin(), t->data.end(), flat + off);
    off += t->data.size();
  }
  *log_z = rs->s->policy().log_z.data[0];
}

void ref_set_params(void* h, const double* flat, double log_z) {
  auto* rs = static_cast<RefSession*>(h);
  size_t off = 0;
  for (Tensor* t : rs->s->policy().tensors()) {
    std::copy(flat + off, flat + off + t->data.size(), t->data.begin());
    off += t->data.size();
  }
  rs->s->policy().log_z.data[0] = log_z;
}

// One train_scenario iteration (train.cpp:224-229).
int ref_iteration(void* h, int64_t it, double* loss) {
  auto* rs = static_cast<RefSession*>(h);
  return guard(rs, [&] {
    const double lr = schedule_value(to_sched(rs->train.lr, rs->train.iterations), it);
    const double eps = schedule_value(to_sched(rs->train.explore, rs->train.iterations), it);
    rs->s->rollout(it, eps);
    *loss = rs->s->compute_grads();
    rs->s->apply_adam(lr);
  });
}

// the reference's own GFNCKPT1 writer / reader on the session's policy and Adam states
int ref_save_checkpoint(void* h, const char* path, int64_t step) {
  auto* rs = static_cast<RefSession*>(h);
  return guard(rs, [&] {
    Checkpoint c;
    c.params = rs->s->policy();
    c.opt_main = rs->s->opt_main();
    c.opt_z = rs->s->opt_z();
    c.step = step;
    save_checkpoint(c, path);
  });
}

int ref_load_checkpoint(void* h, const char* path, int64_t* step) {
  auto* rs = static_cast<RefSession*>(h);
  return guard(rs, [&] {
    Checkpoint c = load_checkpoint(path);
    rs->s->policy() = c.params;
    rs->s->opt_main() = c.opt_main;
    rs->s->opt_z() = c.opt_z;
    *step = c.step;
  });
}

int ref_mc_logprob(void* h, const uint32_t* term, int K, uint64_t key_hi, uint64_t key_lo, double* out) {
  RefSession* rs = static_cast<RefSession*>(h);
  return guard(rs, [&] {
    RngKey k;
    k.hi = key_hi;
    k.lo = key_lo;
    *out = rs->s->mc_logprob(term, K, k);
  });
}

int ref_backward_rollout(void* h, const uint32_t* terms, int n, uint64_t key_hi, uint64_t key_lo) {
  RefSession* rs = static_cast<RefSession*>(h);
  return guard(rs, [&] {
    RngKey k;
    k.hi = key_hi;
    k.lo = key_lo;
    rs->s->backward_batch(terms, n, k);
  });
}

int ref_pearson(void* h, int64_t step, int mc, uint64_t test_seed, double* out) {
  RefSession* rs = static_cast<RefSession*>(h);
  return guard(rs, [&] { *out = rs->s->pearson_metric(step, mc, test_seed); });
}

int ref_exact_divergence(void* h, double* out) {
  auto* rs = static_cast<RefSession*>(h);
  return guard(rs, [&] { *out = rs->s->exact_divergence(); });
}

double ref_uniform_fold(uint64_t hi, uint64_t lo, uint64_t idx) {
  return uniform_scalar(fold_in(RngKey{hi, lo}, idx));
}
void ref_threefry(uint64_t hi, uint64_t lo, uint64_t c0, uint64_t c1, uint64_t* out) {
  auto w = threefry2x64(RngKey{hi, lo}, c0, c1);
  out[0] = w[0];
  out[1] = w[1];
}

// gibbs_data_sampler (ising.cpp:185-220) on toroidal_coupling(side, sigma): n x D spins
int ref_gibbs_data(int side, double sigma, uint64_t seed, int64_t n, int64_t burn_in, int64_t thinning,
                   int chains, double hottest_beta, int8_t* out) {
  return guard(nullptr, [&] {
    GibbsConfig gc;
    gc.burn_in = burn_in;
    gc.thinning = thinning;
    gc.num_chains = chains;
    gc.hottest_beta = hottest_beta;
    auto d = gibbs_data_sampler(toroidal_coupling(side, sigma), fold_in(make_key(seed), 0x919B), n, gc);
    size_t o = 0;
    for (const auto& v : d)
      for (int8_t x : v) out[o++] = x;
  });
}

// The reference's own benchmark harness (run_bench -> bench_scenario, train.cpp:294-334,
// 801-809) through its Config front door. Returns mean it/s (and 3-sigma stderr).
int ref_run_bench(const char* env_name, const char* const* keys, const char* const* values,
                  int n_kv, double* mean_its, double* stderr3) {
  return guard(nullptr, [&] {
    Config cfg;
    cfg.set("env.name", env_name);
    for (int i = 0; i < n_kv; ++i) cfg.set(keys[i], values[i]);
    BenchReport r = run_bench(cfg);
    *mean_its = r.mean_iters_per_second;
    *stderr3 = r.stderr3;
  });
}

}  // extern "C"
