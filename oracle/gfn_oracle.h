/*
 * gfn_oracle.h — CPU oracle for the GFlowNet training hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This is a plain-C, fp64, single-threaded
 * restatement of the reference (gfnkit, /root/reference/proj) hot path:
 * Threefry RNG, the hypergrid / bitseq-NAR / Ising / DAG environments,
 * the MLP policy, epsilon-uniform masked categorical sampling, forward
 * rollouts, TB / DB / SubTB / MDB losses with analytic gradients, and Adam.
 * Every function cites the reference file:line it follows.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it; the product (libgfnx.so) never links it. It is pinned against the
 * compiled reference (oracle/_ref, built by oracle/Makefile) and the golden
 * fixtures in tests/golden/ (see tests/test_oracle.py).
 *
 * Descriptors are the product's own (include/gfnx.h) so a parity test drives
 * both sides from one description.
 */
#ifndef GFN_ORACLE_H_
#define GFN_ORACLE_H_

#include <stdint.h>

#include "../include/gfnx.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- RNG (proj/src/rng.cpp:10-100) ---- */
void orc_make_key(uint64_t seed, uint64_t out[2]);
void orc_threefry2x64(const uint64_t key[2], uint64_t c0, uint64_t c1, uint64_t out[2]);
void orc_fold_in(const uint64_t key[2], uint64_t index, uint64_t out[2]);
double orc_uniform_scalar(const uint64_t key[2]);
/* returns the sampled index, or -1 when no weight is positive (reference throws) */
int32_t orc_categorical(const uint64_t key[2], const double* w, int32_t n);
/* returns number of legal entries (0 -> reference throws contract_violation) */
int32_t orc_eps_uniform(const double* logits, const uint8_t* mask, int32_t n, double eps,
                        double* probs);
double orc_schedule_value(const gfnx_schedule* s, int64_t step);

/* ---- trainer ---- */
typedef struct orc_trainer orc_trainer;

/* b0/nb: this rank's slice [b0, b0+nb) of the global batch (nb == 0: whole batch) */
orc_trainer* orc_create(const gfnx_env_desc* env, const gfnx_train_desc* train, int32_t b0,
                        int32_t nb, char* err, int32_t errlen);
void orc_destroy(orc_trainer* tr);
const char* orc_last_error(const orc_trainer* tr);
int32_t orc_shape(const orc_trainer* tr, gfnx_env_shape* out);

int64_t orc_num_params(const orc_trainer* tr);
void orc_get_params(const orc_trainer* tr, double* flat, double* log_z);
void orc_set_params(orc_trainer* tr, const double* flat, double log_z);
void orc_get_adam(const orc_trainer* tr, double* m, double* v, int64_t* t, double* zm, double* zv,
                  int64_t* zt);
void orc_set_adam(orc_trainer* tr, const double* m, const double* v, int64_t t, double zm,
                  double zv, int64_t zt);

/* forward_rollout + rollout_from_actions (env_core.hpp:166-274) for iteration it */
int32_t orc_rollout(orc_trainer* tr, int64_t it, double eps);
/* The eps = 1 rollout without evaluating the policy (the draws are exactly 1/#legal). */
int32_t orc_rollout_uniform(orc_trainer* tr, int64_t it);
/* Replace the resident batch by replaying explicit actions [nb * T] (-1 padded). */
int32_t orc_replay(orc_trainer* tr, const int32_t* actions);
/* Local normaliser counts: real transitions (DB) and MDB transitions. */
void orc_local_counts(const orc_trainer* tr, int64_t* n_steps, int64_t* n_mdb);
/* Loss partial + gradients of the resident batch with GLOBAL normaliser `norm`
 * (B for TB/SubTB, n_steps for DB, n_mdb for MDB; <= 0: use local counts). */
int32_t orc_compute_grads(orc_trainer* tr, double norm, double* loss);
void orc_get_grads(const orc_trainer* tr, double* flat, double* dlogz);
/* bf16 operand model of the device fast path (test infrastructure): the same loss/gradient
 * with the rounding points of the bf16 kernels switched on by `flags`; flags == 0 is
 * bit-identical to orc_compute_grads. Outputs: loss, grads [n_params], dlogz, and the
 * per-row log pi_F(a_t | s_t) [nb * T] (0 past each end); any may be NULL. */
#define ORC_BFM_W 1        /* weight matrices rounded to bf16 (operand images) */
#define ORC_BFM_ACT 2      /* post-ReLU activations rounded to bf16 (activation images) */
#define ORC_BFM_GRAD 4     /* dlogits, dflow and masked dz rounded to bf16 (gradient images) */
#define ORC_BFM_LOGIT 8    /* logits rounded to bf16 (lockstep path's logits image) */
#define ORC_BFM_ISING_L1 16 /* persistent Ising rollout's layer-1 delta image */
int32_t orc_model_grads(orc_trainer* tr, double norm, int32_t flags, double* loss, double* grads,
                        double* dlogz, double* row_logpf);
/* Actions the fp64 reference sampler draws at every state of the resident batch [nb * T]. */
int32_t orc_teacher_actions(orc_trainer* tr, int64_t it, double eps, int32_t* out);
void orc_set_grads(orc_trainer* tr, const double* flat, double dlogz);
/* Adam on main params (lr) and, for TB, on logZ (adam_z) — train.cpp:184-190 */
void orc_apply_adam(orc_trainer* tr, double lr);
/* One full reference iteration (train.cpp:224-229). */
int32_t orc_iteration(orc_trainer* tr, int64_t it, double* loss);

typedef struct orc_batch_view {
  int32_t nb, T, state_words;
  const int32_t* lengths;
  const int32_t* fwd_actions;
  const int32_t* bwd_actions;
  const double* log_rewards;
  const double* log_pb;
  const double* delta;
  const uint32_t* terminal_state;
} orc_batch_view;
void orc_batch(const orc_trainer* tr, orc_batch_view* out);

/* Environment helpers used by tests (host restatements of env methods). */
double orc_log_reward_of_state(const orc_trainer* tr, const uint32_t* packed_state);
/* mlp_forward on explicit obs rows [n x obs_dim] -> fwd logits [n x A], flow [n] */
int32_t orc_mlp_forward(const orc_trainer* tr, const double* obs, int32_t n, double* fwd_logits,
                        double* flow);
/* encode_obs of the state reached after replaying `actions` (length n) from s0 */
int32_t orc_obs_after(const orc_trainer* tr, const int32_t* actions, int32_t n, double* obs,
                      uint8_t* mask);
/* Bitseq modes (ModeSet::modes as 0/1 bytes, [num_modes x n_bits]); returns count. */
int32_t orc_bitseq_modes(const orc_trainer* tr, uint8_t* out, int32_t cap);
/* DAG local score cache [d x 2^d] and dataset summary. */
int32_t orc_dag_cache(const orc_trainer* tr, double* out, int32_t cap);
int32_t orc_dag_true_adj(const orc_trainer* tr, uint32_t* out);

#ifdef __cplusplus
}
#endif
#endif
