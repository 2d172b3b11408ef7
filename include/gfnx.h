/*
 * gfnx.h — C ABI of the B200-native GFlowNet training engine (libgfnx.so).
 *
 * This is the drop-in boundary for the reference's training hot path
 *   forward_rollout -> build_loss -> Tape::backward -> adam_step
 * (reference: proj/include/gfn/env_core.hpp:232-274, proj/src/objectives.cpp:230-240,
 *  proj/src/tape.cpp:321-485, proj/src/optim.cpp:19-43, glued by train_step
 *  proj/src/train.cpp:164-192 and the loop body proj/src/train.cpp:224-243).
 *
 * Plain C types only: no torch, no STL. One gfnx_ctx owns one CUDA device's
 * memory, stream and (optionally) an NCCL communicator; calls on a ctx are
 * serialised on its stream. Every entry point returns a gfnx_status; the
 * message of the last failure is available from gfnx_last_error().
 *
 * The same descriptor structs are consumed by the CPU oracle (oracle/gfn_oracle.h)
 * so parity tests drive both sides from one description.
 */
#ifndef GFNX_H_
#define GFNX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GFNX_ABI_VERSION 1

/* Error classes mirror proj/include/gfn/errors.hpp:6-16 plus device/NCCL failures. */
typedef enum gfnx_status {
  GFNX_OK = 0,
  GFNX_ERR_CONFIG = 1,   /* gfn::config_error */
  GFNX_ERR_CONTRACT = 2, /* gfn::contract_violation (illegal action, bad batch, ...) */
  GFNX_ERR_NUMERIC = 3,  /* gfn::numeric_error (non-finite logits / loss) */
  GFNX_ERR_CUDA = 4,
  GFNX_ERR_NCCL = 5
} gfnx_status;

/* Environment kinds on the device hot path. */
typedef enum gfnx_env_kind {
  GFNX_ENV_HYPERGRID = 0, /* proj/include/gfn/envs/hypergrid.hpp:12-55 */
  GFNX_ENV_BITSEQ = 1,    /* SequenceEnv, non-autoregressive scheme + ModeSet, sequences.hpp:74-124 */
  GFNX_ENV_ISING = 2,     /* proj/include/gfn/envs/ising.hpp:33-71 */
  GFNX_ENV_DAG = 3        /* proj/include/gfn/envs/dag.hpp:70-115 */
} gfnx_env_kind;

/* Same numbering as gfn::Objective (proj/include/gfn/objectives.hpp:11). */
typedef enum gfnx_objective {
  GFNX_OBJ_DB = 0,
  GFNX_OBJ_TB = 1,
  GFNX_OBJ_SUBTB = 2,
  GFNX_OBJ_FLDB = 3, /* phylo-only in the reference; rejected (out of scope) */
  GFNX_OBJ_MDB = 4
} gfnx_objective;

typedef enum gfnx_precision {
  GFNX_PREC_BF16 = 0,       /* fast path: bf16 tcgen05 GEMMs, fp32 accumulate, fp32 master */
  GFNX_PREC_FP64_CHECK = 1  /* check mode: fp64 SIMT, reference operation order */
} gfnx_precision;

typedef enum gfnx_dag_score { GFNX_DAG_LINGAUSS = 0, GFNX_DAG_BGE = 1 } gfnx_dag_score;

/* gfn::Schedule (proj/include/gfn/optim.hpp:30-37). kind: 0 constant, 1 linear, 2 cosine.
 * horizon < 0 means "half of train.iterations", 0 means "iterations - warmup"
 * (read_schedule, proj/src/train.cpp:83-103); resolved at gfnx_create. */
typedef struct gfnx_schedule {
  int32_t kind;
  int32_t pad_;
  double start_value;
  double end_value;
  int64_t warmup;
  int64_t horizon;
} gfnx_schedule;

typedef struct gfnx_env_desc {
  int32_t kind; /* gfnx_env_kind */
  /* hypergrid: HypergridEnv::Params (hypergrid.hpp:17-23) */
  int32_t hg_dim;
  int32_t hg_side;
  int32_t pad0_;
  double hg_r0, hg_r1, hg_r2;
  /* bitseq (build_bitseq, train.cpp:381-427): n_bits, k (vocab 2^k), beta, modes */
  int32_t bs_n_bits;
  int32_t bs_k;
  double bs_beta;
  int32_t bs_num_modes;
  int32_t bs_scheme;   /* SeqScheme: 0 non-autoregressive (build_bitseq), 1 autoregressive fixed */
  uint64_t bs_modes_seed;
  /* ising (build_ising, train.cpp:637-657): toroidal coupling sigma * A_N */
  int32_t is_side;
  int32_t pad2_;
  double is_sigma;
  /* dag (build_dag, train.cpp:523-586) */
  int32_t dag_d;
  int32_t dag_score; /* gfnx_dag_score */
  double dag_alpha_mu, dag_alpha_w;        /* BGe; alpha_w <= 0 means d + 2 */
  double dag_noise_var, dag_weight_var;    /* lingauss */
  double dag_expected_in_degree;
  int32_t dag_data_n;
  int32_t pad3_;
  uint64_t dag_data_seed;
} gfnx_env_desc;

typedef struct gfnx_train_desc {
  int32_t objective; /* gfnx_objective */
  int32_t learned_backward; /* must be 0 (uniform P_B) on the device path */
  double subtb_lambda;
  double terminal_penalty;
  int32_t batch_size; /* GLOBAL trajectories per iteration (B); ranks take slices */
  int32_t num_hidden;
  int32_t hidden[8];
  double logz_init;
  double beta1, beta2, adam_eps, weight_decay; /* main optimizer (AdamConfig) */
  double z_lr;                                 /* logZ optimizer lr (TB only) */
  gfnx_schedule lr;                            /* optimizer.lr_anneal.* */
  gfnx_schedule explore;                       /* explore.* (epsilon-uniform mix) */
  int64_t iterations;                          /* only used to resolve schedule horizons */
  uint64_t seed;
  int32_t precision; /* gfnx_precision */
  /* bf16 hypergrid / DAG path: 1 = run-to-run bit-identical results (static per-CTA
   * trajectory ranges and row regions instead of work stealing, as the reference's
   * byte-identical runs require, test_config_train.cpp:80-122); 0 = dynamic (faster).
   * fp64 check mode and the lockstep paths are always deterministic. */
  int32_t deterministic;
} gfnx_train_desc;

/* Per-environment defaults of the reference drivers (train.cpp:43-62, 105-137, 353-657). */
gfnx_status gfnx_default_env_desc(int32_t kind, gfnx_env_desc* out);
gfnx_status gfnx_default_train_desc(int32_t kind, gfnx_train_desc* out);

/* Static shape of an environment: A, Ab, obs_dim, T (max_traj_len), stop action (-1 if none). */
typedef struct gfnx_env_shape {
  int32_t num_actions;
  int32_t num_backward_actions;
  int32_t obs_dim;
  int32_t max_traj_len;
  int32_t stop_action;
  int32_t state_words; /* 32-bit words of the packed device state per trajectory */
} gfnx_env_shape;
gfnx_status gfnx_env_shape_of(const gfnx_env_desc* env, gfnx_env_shape* out);

typedef struct gfnx_ctx gfnx_ctx;

/* nccl_id: 128-byte ncclUniqueId from gfnx_nccl_unique_id on rank 0 (NULL when world == 1). */
gfnx_status gfnx_create(const gfnx_env_desc* env, const gfnx_train_desc* train, int32_t device,
                        int32_t rank, int32_t world, const void* nccl_id, gfnx_ctx** out);
void gfnx_destroy(gfnx_ctx* ctx);
gfnx_status gfnx_nccl_unique_id(void* out128);
/* In-process communicator: the ranks of one job as threads of ONE process (one ctx per rank,
 * one thread per ctx; the ranks may share a GPU or sit on peer-accessible GPUs of a node).
 * The job's all-reduce is then a libgfnx kernel that reads every rank's buffer over peer
 * memory and sums in rank order (deterministic, identical on every rank) instead of NCCL.
 * Destroy the member ctxs before the group. Replaces nothing in the reference, which is
 * single-process and single-threaded; it is the data-parallel plumbing of
 * SURVEY §8(e) for single-process drivers and for testing world > 1 on one GPU. */
typedef struct gfnx_group gfnx_group;
gfnx_status gfnx_group_create(int32_t world, gfnx_group** out);
gfnx_status gfnx_group_destroy(gfnx_group* group);
gfnx_status gfnx_create_in_group(const gfnx_env_desc* env, const gfnx_train_desc* train, int32_t device,
                                 int32_t rank, gfnx_group* group, gfnx_ctx** out);
/* Last error message for ctx (or of the last failed gfnx_create when ctx == NULL). */
const char* gfnx_last_error(const gfnx_ctx* ctx);
int32_t gfnx_abi_version(void);

/* Parameters in MlpParams::tensors() order (nn.cpp:8-19): trunk (W[in x out], b)...,
 * fwd head, bwd head, flow head; log_z separate. fp64 on the host side. */
gfnx_status gfnx_num_params(const gfnx_ctx* ctx, int64_t* n);
gfnx_status gfnx_set_params(gfnx_ctx* ctx, const double* flat, int64_t n, double log_z);
gfnx_status gfnx_get_params(gfnx_ctx* ctx, double* flat, int64_t n, double* log_z);
/* Adam state: main m, v (n each) + step t; logZ m, v, t. NULL pointers skip a field. */
gfnx_status gfnx_set_adam_state(gfnx_ctx* ctx, const double* m, const double* v, int64_t t,
                                double z_m, double z_v, int64_t z_t);
gfnx_status gfnx_get_adam_state(gfnx_ctx* ctx, double* m, double* v, int64_t* t, double* z_m,
                                double* z_v, int64_t* z_t);

/* One forward rollout of this rank's trajectory slice for iteration `it`
 * (key fold_in(make_key(seed), 1000 + it), env_core.hpp:232-274) at exploration eps.
 * The batch stays resident on the device. */
/* GFNCKPT1 checkpoint files, byte-compatible with the reference's save_checkpoint /
 * load_checkpoint (checkpoint.cpp:11-107): policy (fp64), both Adam states, step counter. */
gfnx_status gfnx_save_checkpoint(gfnx_ctx* ctx, const char* path, int64_t step);
gfnx_status gfnx_load_checkpoint(gfnx_ctx* ctx, const char* path, int64_t* step);

/* Exact terminal marginal of the current policy on the hypergrid (exact_policy_marginal,
 * exact.hpp:76-113): one batched policy forward over every cell + a level-by-level DP on the
 * device. marginal: n = side^dim doubles in row-major cell order (coordinate 0 fastest), or
 * NULL; tv: total variation to R / Z (the `tv_exact` metric), or NULL. bf16 fast path. */
gfnx_status gfnx_exact_terminal_marginal(gfnx_ctx* ctx, double* marginal, int64_t n, double* tv);

/* Monte-Carlo terminal log-probability (mc_terminal_logprob, exact.hpp:229-241) of n packed
 * terminal states under the current policy, every env and precision: num_samples backward
 * trajectories each from the uniform backward policy, walked on the device exactly as
 * backward_rollout draws them with key {keys[2i], keys[2i+1]} (RngKey words,
 * env_core.hpp:314-370), scored by the device policy forward (score_trajectories,
 * objectives.cpp:294-316); out[i] = logsumexp_k(log_pf - log_pb) - log(num_samples).
 * Hypergrid / DAG bf16: one batched forward over all transitions on eval buffers. Bitseq /
 * Ising and fp64 check mode: teacher-forced batches of local_batch walks through the resident
 * batch, which is consumed (call gfnx_rollout again before training). */
gfnx_status gfnx_mc_terminal_logprob(gfnx_ctx* ctx, const uint32_t* terminals, int64_t n, int32_t num_samples,
                                     const uint64_t* keys, double* out);

/* The bitseq `pearson` metric (train.cpp:440-454) of the current policy, on the device: the
 * builder's test set (generate_test_set, sequences.cpp:100-119, key
 * fold_in(make_key(test_seed), 0x7E57); n_modes * n_bits strings), mc_samples-walk
 * gfnx_mc_terminal_logprob of each with key fold_in(fold_in(fold_in(make_key(seed), 0x3E7A),
 * step), i), Pearson correlation with the log-rewards (metrics.cpp:96-116). Consumes the
 * resident batch like gfnx_mc_terminal_logprob does. NUMERIC on zero variance. */
gfnx_status gfnx_pearson(gfnx_ctx* ctx, int64_t step, int32_t mc_samples, uint64_t test_seed, double* out);

/* ---- EB-GFN (run_eb_gfn, train.cpp:875-1018) on an Ising ctx -----------------------------
 * The ctx's env (is_side, is_sigma) is the TRUE coupling J* that generates the data; the
 * sampler is trained with TB (train desc: batch_size = the sampler batch) on the energy of
 * the learned coupling J (zero at start), which is fitted by contrastive divergence with
 * MH-corrected back-and-forth proposals (ising.cpp:222-373). Everything per iteration runs
 * on the device: mixture selection, data-backed backward walks, the mixed rollout (sampled
 * + teacher-forced rows), train_step, the k-step back-and-forth proposals, MH acceptance,
 * cd_gradient, the J update and neg_log_rmse. Data: ctx-generated with the reference's Gibbs
 * sampler (gibbs_data_sampler, key fold_in(make_key(seed), 0x919B)) or caller supplied. */
typedef struct gfnx_eb_desc {
  int32_t data_samples;      /* env.data_samples (2000) */
  int32_t k;                 /* eb.k: back-and-forth steps; <= 0 means D */
  int64_t gibbs_burn_in;     /* gibbs.burn_in (2000) */
  int64_t gibbs_thinning;    /* gibbs.thinning (10) */
  int32_t gibbs_chains;      /* gibbs.chains (1) */
  int32_t data_batch;        /* eb.data_batch; <= 0 means the sampler batch */
  double gibbs_hottest_beta; /* gibbs.hottest_beta (0.2) */
  double alpha;              /* eb.alpha: on-policy fraction of the sampler batch (0.5) */
  double coupling_lr;        /* eb.coupling_lr (0.05) */
  double coupling_lr_end;    /* eb.coupling_lr_end (= coupling_lr) */
} gfnx_eb_desc;

gfnx_status gfnx_eb_default_desc(gfnx_eb_desc* out);
/* gibbs_data_sampler (ising.cpp:185-220) on toroidal_coupling(side, sigma) with key
 * fold_in(make_key(seed), 0x919B) (train.cpp:905-906): n x side^2 spins (host, no ctx) */
gfnx_status gfnx_ising_gibbs_data(int32_t side, double sigma, uint64_t seed, const gfnx_eb_desc* desc,
                                  int8_t* out, int64_t n);
/* data: NULL (Gibbs-sample data_samples states from J*) or n x D spins in {-1, +1} */
gfnx_status gfnx_eb_init(gfnx_ctx* ctx, const gfnx_eb_desc* desc, const int8_t* data, int64_t n);
/* iterations it0 .. it0 + n - 1; out (or NULL): per iteration {loss, logZ, neg_log_rmse,
 * accepted proposals} (the metrics.csv columns of train.cpp:938-1003 before interval
 * averaging) */
gfnx_status gfnx_eb_run(gfnx_ctx* ctx, int64_t it0, int64_t n, double* out);
/* j_model / j_true: D x D row-major (either may be NULL); init_nlr: neg_log_rmse at start */
gfnx_status gfnx_eb_coupling(gfnx_ctx* ctx, double* j_model, double* j_true, int64_t n, double* init_nlr);
/* the data set: n_samples x D spins (n_samples from gfnx_eb_init) */
gfnx_status gfnx_eb_dataset(gfnx_ctx* ctx, int8_t* out, int64_t n);

/* backward_rollout (env_core.hpp:314-370) under the uniform backward policy: n = local_batch
 * packed terminal states (this rank's slice, gfnx_batch_dims) walked back to s0 on the device
 * (draw b = first_traj + i of `key`), then replayed forward (rollout_from_actions) into the
 * resident batch — gfnx_compute_grads / gfnx_train_step / gfnx_export_batch act on it.
 * CONTRACT on a non-terminal state. */
gfnx_status gfnx_backward_rollout(gfnx_ctx* ctx, const uint32_t* terminals, int64_t n, uint64_t key_hi,
                                  uint64_t key_lo);

/* rollout_from_actions (env_core.hpp:166-229): n = local_batch * max_traj_len forward actions
 * (row b = trajectory b, -1 after its end) replayed into the resident batch. CONTRACT on an
 * illegal action or a trajectory that does not terminate. */
gfnx_status gfnx_rollout_from_actions(gfnx_ctx* ctx, const int32_t* actions, int64_t n);

/* Terminal-state FIFO of the `tv_buffer` metric, hypergrid (FifoBuffer, buffer.hpp:13-55,
 * fed by buffer.push_batch(batch.terminal_keys), train.cpp:231). reset: new empty buffer of
 * `capacity` >= 1 (the reference default is 200000); push: appends the resident batch's
 * terminal states in trajectory order, oldest evicted first (stream-ordered, no host sync);
 * tv_buffer: tv_distance(buffer.empirical(), grid_exact_distribution) (metrics.cpp:35-48)
 * and the buffer size. Each rank's buffer holds its own trajectory slice. */
gfnx_status gfnx_buffer_reset(gfnx_ctx* ctx, int64_t capacity);
gfnx_status gfnx_buffer_push(gfnx_ctx* ctx);
gfnx_status gfnx_tv_buffer(gfnx_ctx* ctx, int64_t* size, double* tv);

gfnx_status gfnx_rollout(gfnx_ctx* ctx, int64_t it, double eps);
/* Loss + gradient over the resident batch, NCCL all-reduce (world > 1), Adam on
 * the main params with learning rate lr and (TB) on logZ with z_lr (train.cpp:164-192).
 * *loss receives the global loss value (NULL: no device->host read). */
gfnx_status gfnx_train_step(gfnx_ctx* ctx, double lr, double* loss);
/* Same as gfnx_train_step without the Adam update (gradients kept for gfnx_get_grads). */
gfnx_status gfnx_compute_grads(gfnx_ctx* ctx, double* loss);
gfnx_status gfnx_get_grads(gfnx_ctx* ctx, double* flat, int64_t n, double* d_log_z);
/* Per-row log pi_F(a_t | s_t) [local_batch * max_len], (b, t) order, 0 past each trajectory's
 * end, of the policy the last training pass scored the resident batch with — the
 * `masked_log_softmax` + `take` values of the reference tape (tape.cpp:177-245,
 * objectives.cpp:67-69), for per-row parity checks. */
gfnx_status gfnx_export_row_logpf(gfnx_ctx* ctx, double* out, int64_t n);
/* Terminal log-rewards of packed states (the packed layout of gfnx_export_batch's
 * terminal_state): log_reward_of of every env — hypergrid.cpp:111-119,
 * ModeSet::log_reward sequences.cpp:50-55, ising_energy ising.cpp:40-51 (log R = -E),
 * graph_log_reward dag.cpp:313-322 — bit-identical to the reference. Host buffers
 * states[n][state_words], out[n]; raises GFNX_ERR_CONTRACT for a non-terminal state where the
 * reference throws (incomplete Ising configuration / bit string). */
gfnx_status gfnx_log_rewards(gfnx_ctx* ctx, const uint32_t* states, int64_t n, double* out);
/* Same over DEVICE buffers, word-major states_soa[state_words][n] (coalesced), out[n];
 * stream-ordered on the ctx stream, no synchronisation (errors at the next sync point). */
gfnx_status gfnx_log_rewards_device(gfnx_ctx* ctx, const uint32_t* states_soa, int64_t n, double* out);
/* Diagnostics (read-only): copy an internal device buffer of the lockstep fast path by name
 * ("h<l>", "dz<l>", "mask<l>", "dlog", "rowbuf", "coef"); out == NULL returns the size. */
gfnx_status gfnx_debug_buffer(gfnx_ctx* ctx, const char* name, void* out, int64_t cap, int64_t* bytes);
/* Full iteration `it`: schedules, rollout, train step (train.cpp:224-229). */
gfnx_status gfnx_iteration(gfnx_ctx* ctx, int64_t it, double* loss);
/* n iterations it0..it0+n-1 enqueued back to back on the ctx stream with no host
 * synchronisation in between (stream-ordered launches, no CUDA graph); losses[n] may be NULL. */
gfnx_status gfnx_run(gfnx_ctx* ctx, int64_t it0, int64_t n, double* losses);
gfnx_status gfnx_synchronize(gfnx_ctx* ctx);

/* Pipelined end-to-end iteration with pinned host staging owned by the ctx.
 * gfnx_iteration_async enqueues iteration `it` (as gfnx_iteration) followed by
 * device->host copies of its loss, lengths, log-rewards and packed terminal states into
 * pinned slot `slot` (0 or 1) and returns without waiting; gfnx_slot_wait blocks until
 * that slot's copies have landed and returns pointers into the pinned slot (valid until
 * the slot is reused). A host loop alternates slots so the device never waits for the
 * host (what train_scenario does with the batch: buffer.push_batch, train.cpp:231). */
typedef struct gfnx_slot_view {
  int64_t it;
  double loss;
  int32_t n; /* local trajectories */
  int32_t state_words;
  const int32_t* lengths;
  const double* log_rewards;
  const uint32_t* terminal_state;
} gfnx_slot_view;
gfnx_status gfnx_iteration_async(gfnx_ctx* ctx, int64_t it, int32_t slot);
gfnx_status gfnx_slot_wait(gfnx_ctx* ctx, int32_t slot, gfnx_slot_view* out);

/* Host view of this rank's resident batch (TrajectoryBatch fields, trajectory.hpp:15-33).
 * Caller-owned buffers sized by gfnx_batch_dims; NULL pointers are skipped. */
typedef struct gfnx_host_batch {
  int32_t* lengths;        /* [Bl] */
  int32_t* fwd_actions;    /* [Bl * T], -1 on padding */
  int32_t* bwd_actions;    /* [Bl * T], -1 on padding */
  double* log_rewards;     /* [Bl] */
  double* log_pb;          /* [Bl * T] log_pb_uniform, 0 on padding */
  double* delta_log_reward;/* [Bl * T] (MDB only, 0 elsewhere) */
  uint32_t* terminal_state;/* [Bl * state_words] packed terminal state */
} gfnx_host_batch;
gfnx_status gfnx_batch_dims(const gfnx_ctx* ctx, int32_t* local_batch, int32_t* first_traj,
                            int32_t* max_len, int32_t* state_words);
gfnx_status gfnx_export_batch(gfnx_ctx* ctx, gfnx_host_batch* out);

/* Kernel launches issued by this ctx since creation (evidence for bench.py). */
int64_t gfnx_kernel_launches(const gfnx_ctx* ctx);
/* Device time (ms) of the last gfnx_rollout / train-step phases, measured with CUDA events. */
gfnx_status gfnx_last_phase_ms(const gfnx_ctx* ctx, double* rollout_ms, double* train_ms);

/* CUDA events on the ctx stream (bench.py device timing): slots 0..15. */
gfnx_status gfnx_event_record(gfnx_ctx* ctx, int32_t slot);
gfnx_status gfnx_event_elapsed(gfnx_ctx* ctx, int32_t slot_a, int32_t slot_b, double* ms);
/* Per-kernel CUDA-event brackets while enabled (enable = 1: every launch, 2: the rollout
 * kernel only, so the brackets do not perturb the rest of the iteration); profile_read
 * returns the number of distinct kernels, their '\n'-separated names, summed ms and launch
 * counts, and clears the record. */
gfnx_status gfnx_profile(gfnx_ctx* ctx, int32_t enable);
/* out[0] rows (states) processed since creation, out[1] rollouts, out[2] rows and out[3]
 * MDB transitions of the resident batch. */
gfnx_status gfnx_counters(gfnx_ctx* ctx, int64_t* out, int32_t n);
int32_t gfnx_profile_read(gfnx_ctx* ctx, char* names, int32_t names_cap, double* total_ms,
                          int32_t* counts, int32_t cap);
/* Diagnostic clock64 totals of the persistent rollout's phases (fast path, hypergrid/DAG):
 * mode 1 enables, 0 disables, 2 copies up to n totals into out and clears them.
 * out: [layer1, hidden mma, hidden epilogue, head mma, sample+step, loop barrier,
 *       tile steps, active slot-steps] summed over CTAs. */
gfnx_status gfnx_phase_timers(gfnx_ctx* ctx, int32_t mode, int64_t* out, int32_t n);

/* Stand-alone device kernels exposed for unit tests (threefry KAT, GEMM). */
/* tcgen05.mma 128 x n x 256 (bf16, SW128 smem operands) issue-to-completion clocks per CTA
 * for `reps` back-to-back MMAs (mode 0: wait after each, 1: K-split issue, 2: one wait). */
gfnx_status gfnx_test_mma_rate(int32_t n, int32_t reps, int32_t mode, int32_t grid, int64_t* cycles);
/* D[128x256] = A[128x256] B[256x256]^T (bf16 bits, row-major; A staged in tensor memory). */
gfnx_status gfnx_test_ts_mma(const uint16_t* a, const uint16_t* b, float* d);
gfnx_status gfnx_test_threefry(const uint64_t* keys_hi_lo, const uint64_t* ctr, int64_t n,
                               uint64_t* out);
gfnx_status gfnx_test_uniform_fold(uint64_t key_hi, uint64_t key_lo, const uint64_t* idx,
                                   int64_t n, double* out);

#ifdef __cplusplus
}
#endif
#endif /* GFNX_H_ */
