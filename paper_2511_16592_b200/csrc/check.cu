// check.cu — fp64 "check mode": SIMT kernels that reproduce the reference's
// operation order (compiled with --fmad=false so no FMA contraction happens, like the
// -ffp-contract=off reference build in oracle/_ref). Used for teacher-forced parity:
// sampled actions, terminal states, masks and log-rewards come out bit-exact; losses,
// gradients and updated parameters agree to the last few ulps (device exp/log vs glibc).
//
//   k_check_rollout  forward_rollout + rollout_from_actions  env_core.hpp:166-274
//   k_check_fwd      mlp_forward_tape + masked_log_softmax    nn.cpp:91-126, tape.cpp:177-213
//   k_check_loss     tb/db/subtb/mdb losses + their backward  objectives.cpp:94-226
//   k_check_bwd      masked log-softmax / MLP backward rows   tape.cpp:344-434
//   k_check_wgrad    matmul_tn_acc / add_rowvec weight grads  tensor.cpp:92-102, tape.cpp:380-389
//   k_check_adam     adam_step                                optim.cpp:19-43
#include <math.h>

#include "engine.h"
#include "check_common.cuh"
#include "walk.cuh"

namespace gfnx {

namespace {

template <class Env>
__global__ void k_check_rollout(EnvParams P, DevLayout D, const double* __restrict__ params,
                                Key key, double eps, int b0, int Bl, DeviceBatch batch,
                                double* obs_scratch, double* logit_scratch, int32_t* err,
                                const int16_t* __restrict__ forced) {
  const int b = blockIdx.x;
  if (b >= Bl) return;
  __shared__ typename Env::State s;
  __shared__ double hbuf[2][512];
  __shared__ int s_done;
  const int T = P.T, A = P.A;
  double* obs = obs_scratch + (size_t)b * P.O;
  double* w = logit_scratch + (size_t)b * A;
  if (threadIdx.x == 0) {
    Env::reset(P, s);
    batch.lengths[b] = 0;
    batch.log_rewards[b] = 0.0;
  }
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    batch.actions[(size_t)b * T + t] = -1;
    batch.nparents[(size_t)b * T + t] = 0;
    batch.delta[(size_t)b * T + t] = 0.0;
  }
  __syncthreads();
  // teacher-forced trajectory (rollout_from_actions, env_core.hpp:166-229) unless its row
  // starts with -1 (sampled: the EB-GFN mixed batches, train.cpp:949-971)
  const bool fb = forced && forced[(size_t)b * T] >= 0;
  for (int t = 0; t < T; ++t) {
    if (fb) {  // the action is given
      if (threadIdx.x == 0) {
        const int a = forced[(size_t)b * T + t];
        s_done = 1;
        if (a < 0 || a >= A || !Env::legal(P, s, a)) {
          atomicExch(err, GFNX_ERR_CONTRACT);
        } else {
          const double prev_r = P.mdb ? Env::log_reward(P, s) : 0.0;
          const bool term = Env::step(P, s, a);
          batch.actions[(size_t)b * T + t] = (int16_t)a;
          batch.nparents[(size_t)b * T + t] = (uint16_t)Env::num_parents(P, s);
          if (P.mdb && !term) batch.delta[(size_t)b * T + t] = Env::log_reward(P, s) - prev_r;
          if (term) {
            batch.lengths[b] = t + 1;
            batch.log_rewards[b] = Env::log_reward(P, s);
            Env::pack(P, s, batch.term_state + (size_t)b * P.SW);
          } else {
            s_done = 0;
          }
        }
      }
      __syncthreads();
      if (s_done) break;
      continue;
    }
    for (int i = threadIdx.x; i < P.O; i += blockDim.x) obs[i] = 0.0;
    __syncthreads();
    if (threadIdx.x == 0) Env::features(P, s, [&](int f, double v) { obs[f] = v; });
    __syncthreads();
    const double* h = obs;
    int in = P.O;
    for (int l = 0; l < D.n_trunk; ++l) {
      double* z = hbuf[l & 1];
      dense_block(h, in, params + D.off_w[l], params + D.off_b[l], D.dims[l + 1], z, true);
      __syncthreads();
      h = z;
      in = D.dims[l + 1];
    }
    dense_block(h, in, params + D.off_fw, params + D.off_fb, A, w, false);
    __syncthreads();
    if (threadIdx.x == 0) {
      // eps_uniform (objectives.cpp:242-264) then categorical (rng.cpp:87-100)
      int legal = 0;
      double hi = -INFINITY;
      bool finite = true;
      for (int i = 0; i < A; ++i) {
        finite &= isfinite(w[i]);
        if (Env::legal(P, s, i)) {
          ++legal;
          if (w[i] > hi) hi = w[i];
        }
      }
      int a = -1;
      if (!finite) {
        atomicExch(err, GFNX_ERR_NUMERIC);
      } else if (legal == 0) {
        atomicExch(err, GFNX_ERR_CONTRACT);
      } else {
        double z = 0.0;
        for (int i = 0; i < A; ++i) {
          if (Env::legal(P, s, i)) {
            const double p = exp(w[i] - hi);
            w[i] = p;
            z += p;
          } else {
            w[i] = 0.0;
          }
        }
        const double u = eps / legal;
        double total = 0.0;
        for (int i = 0; i < A; ++i) {
          if (Env::legal(P, s, i)) w[i] = (1.0 - eps) * w[i] / z + u;
          total += w[i];
        }
        const double uu =
            uniform_scalar(fold_in(fold_in(key, (uint64_t)t), (uint64_t)(b0 + b))) * total;
        double acc = 0.0;
        for (int i = 0; i < A; ++i) {
          acc += w[i];
          if (uu < acc) {
            a = i;
            break;
          }
        }
        if (a < 0)
          for (int i = A - 1; i >= 0; --i)
            if (w[i] > 0.0) {
              a = i;
              break;
            }
      }
      s_done = 1;
      if (a >= 0) {
        // rollout_from_actions bookkeeping (env_core.hpp:190-217)
        const double prev_r = P.mdb ? Env::log_reward(P, s) : 0.0;
        const bool term = Env::step(P, s, a);
        batch.actions[(size_t)b * T + t] = (int16_t)a;
        batch.nparents[(size_t)b * T + t] = (uint16_t)Env::num_parents(P, s);
        if (P.mdb && !term) batch.delta[(size_t)b * T + t] = Env::log_reward(P, s) - prev_r;
        if (term) {
          batch.lengths[b] = t + 1;
          batch.log_rewards[b] = Env::log_reward(P, s);
          Env::pack(P, s, batch.term_state + (size_t)b * P.SW);
        } else {
          s_done = 0;
        }
      }
    }
    __syncthreads();
    if (s_done) break;
  }
  if (threadIdx.x == 0 && batch.lengths[b] == 0) atomicExch(err, GFNX_ERR_CONTRACT);
}

// Row r -> trajectory through the exclusive prefix of lengths.
__device__ int find_traj(const int32_t* row0, int Bl, int r) {
  int lo = 0, hi = Bl;  // row0[lo] <= r < row0[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (row0[mid] <= r) lo = mid; else hi = mid;
  }
  return lo;
}

// bwd = 1: the learned backward policy's pass (mlp_forward_tape's bwd head at s_{t+1},
// nn.cpp:111-121, masked by backward_action_mask): row r = step t of its trajectory holds
// s_{t+1}, D carries the bwd head's offsets with A = Ab, bidx[r] = the step's backward action
template <class Env>
__global__ void k_check_fwd(EnvParams P, DevLayout D, const double* __restrict__ params,
                            DeviceBatch batch, int Bl, int R, int need_flow, double* obs_out,
                            double* act_out, double* logp_out, uint8_t* mask_out,
                            double* flow_out, int32_t* err, int bwd, int32_t* bidx) {
  const int r = blockIdx.x;
  if (r >= R) return;
  __shared__ typename Env::State s;
  __shared__ double red;
  const int T = P.T, A = bwd ? P.Ab : P.A;
  double* obs = obs_out + (size_t)r * P.O;
  double* act = act_out + (size_t)r * D.act_sz;
  double* x = logp_out + (size_t)r * A;
  uint8_t* mask = mask_out + (size_t)r * A;
  if (threadIdx.x == 0) {
    const int b = find_traj(batch.row0, Bl, r);
    const int t = r - batch.row0[b];
    Env::reset(P, s);
    for (int q = 0; q < t + bwd; ++q) Env::step(P, s, batch.actions[(size_t)b * T + q]);
    if (bwd) bidx[r] = Env::backward_action(P, batch.actions[(size_t)b * T + t]);
  }
  for (int i = threadIdx.x; i < P.O; i += blockDim.x) obs[i] = 0.0;
  __syncthreads();
  if (threadIdx.x == 0) Env::features(P, s, [&](int f, double v) { obs[f] = v; });
  for (int i = threadIdx.x; i < A; i += blockDim.x)
    mask[i] = (bwd ? bwd_legal<Env>(P, s, i) : Env::legal(P, s, i)) ? 1 : 0;
  __syncthreads();
  const double* h = obs;
  int in = P.O;
  for (int l = 0; l < D.n_trunk; ++l) {
    double* z = act + D.act_off[l];
    dense_block(h, in, params + D.off_w[l], params + D.off_b[l], D.dims[l + 1], z, true);
    __syncthreads();
    h = z;
    in = D.dims[l + 1];
  }
  dense_block(h, in, params + D.off_fw, params + D.off_fb, A, x, false);
  if (need_flow && threadIdx.x == 0) {
    double acc = 0.0;
    for (int p = 0; p < in; ++p) acc += h[p] * params[D.off_flw + p];
    acc += params[D.off_flb];
    flow_out[r] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // masked_log_softmax (tape.cpp:177-213)
    double hi = -INFINITY;
    for (int c = 0; c < A; ++c)
      if (mask[c] && x[c] > hi) hi = x[c];
    if (!isfinite(hi)) {
      atomicExch(err, GFNX_ERR_NUMERIC);
      hi = 0.0;
    }
    double ssum = 0.0;
    for (int c = 0; c < A; ++c)
      if (mask[c]) ssum += exp(x[c] - hi);
    red = hi + log(ssum);
  }
  __syncthreads();
  const double lse = red;
  for (int c = threadIdx.x; c < A; c += blockDim.x) x[c] = mask[c] ? x[c] - lse : -1e30;
}

// Objectives, one thread, the reference's accumulation order (gfn_oracle.c mirrors it):
// tb_loss :120-142, transition_loss :94-118, subtb_loss :144-180, mdb_loss :186-226.
__global__ void k_check_loss(int obj, int A, int T, int B_global, double terminal_penalty,
                             int stop, const double* lampow, const double* neglog,
                             DeviceBatch batch, int Bl, const int32_t* gcounts,
                             const double* logp, const double* flow, double* glogp,
                             double* gflow, double* gpair, double* scalars, int32_t* err,
                             int Ab, const double* blogp, const int32_t* bidx, double* bglogp) {
  // learned backward policy (blogp != null): log P_B = the bwd head's masked log-softmax at
  // s_{t+1} (step_log_ratio objectives.cpp:57-70: pf - pb), gradient -g into bglogp
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  auto pb_idx = [&](int64_t r) { return r * Ab + bidx[r]; };
  const double log_z = scalars[0];
  double norm = (double)B_global;
  if (obj == GFNX_OBJ_DB) norm = (double)gcounts[0];
  if (obj == GFNX_OBJ_MDB) norm = (double)gcounts[1];
  double loss = 0.0, dlogz = 0.0;
  for (int b = 0; b < Bl; ++b) {
    const int L = batch.lengths[b];
    const int64_t r0 = batch.row0[b];
    const int16_t* acts = batch.actions + (size_t)b * T;
    const uint16_t* np = batch.nparents + (size_t)b * T;
    const double logr = batch.log_rewards[b];
    if (obj == GFNX_OBJ_TB) {
      const double w = 1.0 / norm;
      double cum = 0.0;
      for (int t = 0; t < L; ++t)
        cum += blogp ? logp[(r0 + t) * A + acts[t]] - blogp[pb_idx(r0 + t)]
                     : logp[(r0 + t) * A + acts[t]] + -neglog[np[t]];
      const double res = (cum + log_z) + -logr;
      loss += res * res * w;
      const double g = 2.0 * res * w;
      dlogz += g;
      for (int t = 0; t < L; ++t) {
        glogp[(r0 + t) * A + acts[t]] += g;
        if (blogp) bglogp[pb_idx(r0 + t)] += -g;
      }
    } else if (obj == GFNX_OBJ_DB) {
      for (int t = 0; t < L; ++t) {
        const int64_t r = r0 + t;
        const double d = blogp ? logp[r * A + acts[t]] - blogp[pb_idx(r)] : logp[r * A + acts[t]] + -neglog[np[t]];
        const double f1 = (t + 1 < L) ? flow[r + 1] : logr;
        const double res = (flow[r] - f1) + d;
        const double w = (t == L - 1 ? terminal_penalty : 1.0) / norm;
        loss += res * res * w;
        const double g = 2.0 * res * w;
        gflow[r] += g;
        if (t + 1 < L) gflow[r + 1] += -g;
        glogp[r * A + acts[t]] += g;
        if (blogp) bglogp[pb_idx(r)] += -g;
      }
    } else if (obj == GFNX_OBJ_SUBTB) {
      double* cum = gpair;                       // [T+1]
      double* F = gpair + (T + 1);               // [T+1]
      double* gcum = gpair + 2 * (T + 1);        // [T+1]
      double* gp = gpair + 3 * (T + 1);          // [(T+1)^2]
      cum[0] = 0.0;
      for (int t = 0; t < L; ++t) {
        cum[t + 1] = cum[t] + (blogp ? logp[(r0 + t) * A + acts[t]] - blogp[pb_idx(r0 + t)]
                                     : logp[(r0 + t) * A + acts[t]] + -neglog[np[t]]);
        F[t] = flow[r0 + t];
      }
      F[L] = logr;
      double nrm = 0.0;
      for (int j = 0; j < L; ++j)
        for (int k = j + 1; k <= L; ++k) nrm += lampow[k - j];
      if (nrm <= 0.0) continue;
      for (int k = 0; k <= L; ++k) gcum[k] = 0.0;
      int n = 0;
      for (int j = 0; j < L; ++j)
        for (int k = j + 1; k <= L; ++k) {
          const double w = lampow[k - j] / nrm / norm;
          const double res = (F[j] - F[k]) + (cum[k] - cum[j]);
          loss += res * res * w;
          gp[n++] = 2.0 * res * w;
        }
      // backward visit order of the right-to-left-built tape (see gfn_oracle.c)
      n = 0;
      for (int j = 0; j < L; ++j)
        for (int k = j + 1; k <= L; ++k) gflow[r0 + j] += gp[n++];
      n = 0;
      for (int j = 0; j < L; ++j)
        for (int k = j + 1; k <= L; ++k) {
          if (k < L) gflow[r0 + k] += -gp[n];
          ++n;
        }
      n = 0;
      for (int j = 0; j < L; ++j)
        for (int k = j + 1; k <= L; ++k) gcum[k] += gp[n++];
      n = 0;
      for (int j = 0; j < L; ++j)
        for (int k = j + 1; k <= L; ++k) gcum[j] += -gp[n++];
      double acc = 0.0;  // exclusive_row_cumsum backward (tape.cpp:448-461)
      for (int c = L; c >= 0; --c) {
        if (c < L) {
          glogp[(r0 + c) * A + acts[c]] += acc;
          if (blogp) bglogp[pb_idx(r0 + c)] += -acc;
        }
        acc += gcum[c];
      }
    } else if (obj == GFNX_OBJ_MDB) {
      const double w = 1.0 / norm;
      for (int t = 0; t + 1 < L; ++t) {
        const int64_t r = r0 + t;
        const int a = acts[t];
        if (a == stop) atomicExch(err, GFNX_ERR_CONTRACT);
        double res = logp[r * A + a] + (logp[(r + 1) * A + stop] - logp[r * A + stop]);
        res = blogp ? res - blogp[pb_idx(r)] : res + -neglog[np[t]];
        res = res + -batch.delta[(size_t)b * T + t];
        loss += res * res * w;
        const double g = 2.0 * res * w;
        glogp[r * A + a] += g;
        glogp[(r + 1) * A + stop] += g;
        glogp[r * A + stop] += -g;
        if (blogp) bglogp[pb_idx(r)] += -g;
      }
    }
  }
  if (!isfinite(loss)) atomicExch(err, GFNX_ERR_NUMERIC);
  scalars[4] = loss;
  scalars[3] = obj == GFNX_OBJ_TB ? dlogz : 0.0;
}

// Per row: masked log-softmax backward (tape.cpp:413-434), head dgrad, trunk dgrads.
// Stores gx [R x A] and gz [R x act_sz] (gradient w.r.t. each trunk layer's pre-activation).
__global__ void k_check_bwd(DevLayout D, const double* __restrict__ params, int R, int need_flow,
                            const double* act, const double* logp, const uint8_t* mask,
                            const double* glogp, const double* gflow, double* gx_out,
                            double* gz_out) {
  const int r = blockIdx.x;
  if (r >= R) return;
  __shared__ double gsum_s;
  __shared__ double gh[512];
  const int A = D.A;
  const double* lp = logp + (size_t)r * A;
  const double* gr = glogp + (size_t)r * A;
  const uint8_t* mr = mask + (size_t)r * A;
  double* gx = gx_out + (size_t)r * A;
  double* gz = gz_out + (size_t)r * D.act_sz;
  const double* a_r = act + (size_t)r * D.act_sz;
  if (threadIdx.x == 0) {
    double gsum = 0.0;
    for (int c = 0; c < A; ++c)
      if (mr[c]) gsum += gr[c];
    gsum_s = gsum;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < A; c += blockDim.x)
    gx[c] = mr[c] ? gr[c] - exp(lp[c]) * gsum_s : 0.0;
  __syncthreads();
  const int H = D.H;
  const double gf = need_flow ? gflow[r] : 0.0;
  for (int p = threadIdx.x; p < H; p += blockDim.x) {  // flow node first, then fwd head
    double v = 0.0;
    if (need_flow) v += gf * params[D.off_flw + p];
    double acc = 0.0;
    const double* wr = params + D.off_fw + (size_t)p * A;
    for (int j = 0; j < A; ++j) acc += gx[j] * wr[j];
    gh[p] = v + acc;
  }
  __syncthreads();
  for (int l = D.n_trunk - 1; l >= 0; --l) {
    const int out = D.dims[l + 1], in = D.dims[l];
    double* gzl = gz + D.act_off[l];
    const double* al = a_r + D.act_off[l];
    for (int j = threadIdx.x; j < out; j += blockDim.x) gzl[j] = al[j] > 0.0 ? gh[j] : 0.0;
    __syncthreads();
    if (l > 0) {
      const double* W = params + D.off_w[l];
      for (int p = threadIdx.x; p < in; p += blockDim.x) {
        double acc = 0.0;
        const double* wr = W + (size_t)p * out;
        for (int j = 0; j < out; ++j) acc += gzl[j] * wr[j];
        gh[p] = acc;
      }
    }
    __syncthreads();
  }
}

// One thread per parameter element, rows accumulated sequentially in (b, t) order:
// matmul_tn_acc (tensor.cpp:92-102) and the add_rowvec bias backward (tape.cpp:380-389).
// (learned backward: a second row set — the s_{t+1} rows of the bwd head — adds to the trunk
// and owns the bwd head; R2 = 0 otherwise)
__global__ void k_check_wgrad(DevLayout D, int R, int need_flow, const double* obs,
                              const double* act, const double* gx, const double* gz,
                              const double* gflow, double* grads, int R2, const double* obs2,
                              const double* act2, const double* gx2, const double* gz2, int64_t off_bw,
                              int64_t off_bb, int Ab) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int A = D.A;
  // trunk weights / biases
  for (int l = 0; l < D.n_trunk; ++l) {
    const int in = D.dims[l], out = D.dims[l + 1];
    const int64_t nw = (int64_t)in * out;
    if (e >= D.off_w[l] && e < D.off_w[l] + nw) {
      const int64_t q = e - D.off_w[l];
      const int p = (int)(q / out), j = (int)(q % out);
      double acc = 0.0;
      for (int r = 0; r < R; ++r) {
        const double av = l == 0 ? obs[(size_t)r * D.O + p] : act[(size_t)r * D.act_sz + D.act_off[l - 1] + p];
        acc += av * gz[(size_t)r * D.act_sz + D.act_off[l] + j];
      }
      for (int r = 0; r < R2; ++r) {
        const double av = l == 0 ? obs2[(size_t)r * D.O + p] : act2[(size_t)r * D.act_sz + D.act_off[l - 1] + p];
        acc += av * gz2[(size_t)r * D.act_sz + D.act_off[l] + j];
      }
      grads[e] = acc;
      return;
    }
    if (e >= D.off_b[l] && e < D.off_b[l] + out) {
      const int j = (int)(e - D.off_b[l]);
      double acc = 0.0;
      for (int r = 0; r < R; ++r) acc += gz[(size_t)r * D.act_sz + D.act_off[l] + j];
      for (int r = 0; r < R2; ++r) acc += gz2[(size_t)r * D.act_sz + D.act_off[l] + j];
      grads[e] = acc;
      return;
    }
  }
  const int H = D.H;
  const int last = D.act_off[D.n_trunk - 1];
  if (e >= D.off_fw && e < D.off_fw + (int64_t)H * A) {
    const int64_t q = e - D.off_fw;
    const int p = (int)(q / A), j = (int)(q % A);
    double acc = 0.0;
    for (int r = 0; r < R; ++r) acc += act[(size_t)r * D.act_sz + last + p] * gx[(size_t)r * A + j];
    grads[e] = acc;
    return;
  }
  if (e >= D.off_fb && e < D.off_fb + A) {
    const int j = (int)(e - D.off_fb);
    double acc = 0.0;
    for (int r = 0; r < R; ++r) acc += gx[(size_t)r * A + j];
    grads[e] = acc;
    return;
  }
  if (need_flow && e >= D.off_flw && e < D.off_flw + H) {
    const int p = (int)(e - D.off_flw);
    double acc = 0.0;
    for (int r = 0; r < R; ++r) acc += act[(size_t)r * D.act_sz + last + p] * gflow[r];
    grads[e] = acc;
    return;
  }
  if (need_flow && e == D.off_flb) {
    double acc = 0.0;
    for (int r = 0; r < R; ++r) acc += gflow[r];
    grads[e] = acc;
  }
  if (R2 > 0 && e >= off_bw && e < off_bw + (int64_t)H * Ab) {  // bwd head [H][Ab]
    const int64_t q = e - off_bw;
    const int p = (int)(q / Ab), j = (int)(q % Ab);
    double acc = 0.0;
    for (int r = 0; r < R2; ++r) acc += act2[(size_t)r * D.act_sz + last + p] * gx2[(size_t)r * Ab + j];
    grads[e] = acc;
    return;
  }
  if (R2 > 0 && e >= off_bb && e < off_bb + Ab) {
    const int j = (int)(e - off_bb);
    double acc = 0.0;
    for (int r = 0; r < R2; ++r) acc += gx2[(size_t)r * Ab + j];
    grads[e] = acc;
  }
}

// adam_step (optim.cpp:19-43). Bias corrections 1 - beta^t from the device-owned step
// counters; a step whose iteration raised the device error word is skipped and not counted
// (the reference throws before adam_step, train.cpp:174-183).
__global__ void k_check_adam(double* p, const double* g, double* m, double* v, int64_t n,
                             double lr, double b1, double b2, double eps, double wd, double* scalars,
                             int do_z, double z_lr, int64_t* steps, const int32_t* err) {
  __shared__ int skip;
  __shared__ double bc[4];
  if (threadIdx.x == 0) {
    skip = *err != 0;
    const double t = (double)(steps[0] + 1), zt = (double)(steps[1] + 1);
    bc[0] = 1.0 - pow(b1, t);
    bc[1] = 1.0 - pow(b2, t);
    bc[2] = 1.0 - pow(b1, zt);
    bc[3] = 1.0 - pow(b2, zt);
  }
  __syncthreads();
  if (skip) return;
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) {
    const double gj = g[j];
    m[j] = b1 * m[j] + (1.0 - b1) * gj;
    v[j] = b2 * v[j] + (1.0 - b2) * gj * gj;
    const double mhat = m[j] / bc[0];
    const double vhat = v[j] / bc[1];
    p[j] -= lr * (mhat / (sqrt(vhat) + eps) + wd * p[j]);
  }
  if (do_z && j == 0) {  // logZ: separate AdamState, weight decay 0 (train.cpp:125-128,186-190)
    const double gj = scalars[3];
    scalars[1] = b1 * scalars[1] + (1.0 - b1) * gj;
    scalars[2] = b2 * scalars[2] + (1.0 - b2) * gj * gj;
    const double mhat = scalars[1] / bc[2];
    const double vhat = scalars[2] / bc[3];
    scalars[0] -= z_lr * (mhat / (sqrt(vhat) + eps) + 0.0 * scalars[0]);
  }
  adam_commit(steps, do_z);
}

template <class Env>
void rollout_impl(Ctx& c, Key key, double eps, const int16_t* forced) {
  const DevLayout D = make_dev_layout(c);
  k_check_rollout<Env><<<c.Bl, 256, 0, c.stream>>>(c.P, D, c.p64, key, eps, c.b0, c.Bl, c.batch,
                                                    c.ck_obs, c.ck_logp, c.batch.counters + 3, forced);
  c.launches++;
}

// the learned backward head as the "head" of DevLayout (A = Ab, nn.cpp:111-121 bwd leaves)
DevLayout bwd_layout(const Ctx& c) {
  DevLayout d = make_dev_layout(c);
  d.off_fw = c.L.off_bw;
  d.off_fb = c.L.off_bb;
  d.A = c.shape.num_backward_actions;
  return d;
}

template <class Env>
void fwd_impl(Ctx& c, int R, int need_flow) {
  const DevLayout D = make_dev_layout(c);
  k_check_fwd<Env><<<R, 256, 0, c.stream>>>(c.P, D, c.p64, c.batch, c.Bl, R, need_flow, c.ck_obs,
                                            c.ck_act, c.ck_logp, c.ck_mask, c.ck_flow,
                                            c.batch.counters + 3, 0, nullptr);
  c.launches++;
  if (c.train.learned_backward) {  // the bwd head over the s_{t+1} rows
    const DevLayout Db = bwd_layout(c);
    k_check_fwd<Env><<<R, 256, 0, c.stream>>>(c.P, Db, c.p64, c.batch, c.Bl, R, 0, c.ck_bobs, c.ck_bact,
                                              c.ck_blogp, c.ck_bmask, nullptr, c.batch.counters + 3, 1,
                                              c.ck_bidx);
    c.launches++;
  }
}

void ensure_scratch(Ctx& c, int64_t rows) {
  if (rows <= c.ck_rows_cap) return;
  const DevLayout D = make_dev_layout(c);
  cudaFree(c.ck_obs);
  cudaFree(c.ck_act);
  cudaFree(c.ck_logp);
  cudaFree(c.ck_mask);
  cudaFree(c.ck_flow);
  cudaFree(c.ck_glogp);
  cudaFree(c.ck_gflow);
  cudaFree(c.ck_gz);
  cudaFree(c.ck_gx);
  const int64_t n = rows > c.Bl ? rows : c.Bl;
  cuda_check(cudaMalloc(&c.ck_obs, sizeof(double) * n * D.O), "check scratch");
  cuda_check(cudaMalloc(&c.ck_act, sizeof(double) * n * D.act_sz), "check scratch");
  cuda_check(cudaMalloc(&c.ck_logp, sizeof(double) * n * D.A), "check scratch");
  cuda_check(cudaMalloc(&c.ck_mask, n * D.A), "check scratch");
  cuda_check(cudaMalloc(&c.ck_flow, sizeof(double) * n), "check scratch");
  cuda_check(cudaMalloc(&c.ck_glogp, sizeof(double) * n * D.A), "check scratch");
  cuda_check(cudaMalloc(&c.ck_gflow, sizeof(double) * n), "check scratch");
  cuda_check(cudaMalloc(&c.ck_gz, sizeof(double) * n * D.act_sz), "check scratch");
  cuda_check(cudaMalloc(&c.ck_gx, sizeof(double) * n * D.A), "check scratch");
  if (c.train.learned_backward) {
    const int Ab = c.shape.num_backward_actions;
    void* old[] = {c.ck_bobs, c.ck_bact, c.ck_blogp, c.ck_bmask, c.ck_bglogp, c.ck_bgx, c.ck_bgz, c.ck_bidx};
    for (void* p : old) cudaFree(p);
    cuda_check(cudaMalloc(&c.ck_bobs, sizeof(double) * n * D.O), "check scratch");
    cuda_check(cudaMalloc(&c.ck_bact, sizeof(double) * n * D.act_sz), "check scratch");
    cuda_check(cudaMalloc(&c.ck_blogp, sizeof(double) * n * Ab), "check scratch");
    cuda_check(cudaMalloc(&c.ck_bmask, n * Ab), "check scratch");
    cuda_check(cudaMalloc(&c.ck_bglogp, sizeof(double) * n * Ab), "check scratch");
    cuda_check(cudaMalloc(&c.ck_bgx, sizeof(double) * n * Ab), "check scratch");
    cuda_check(cudaMalloc(&c.ck_bgz, sizeof(double) * n * D.act_sz), "check scratch");
    cuda_check(cudaMalloc(&c.ck_bidx, sizeof(int32_t) * n), "check scratch");
  }
  c.ck_rows_cap = n;
}

}  // namespace

void check_rollout(Ctx& c, Key key, double eps, const int16_t* forced) {
  ensure_scratch(c, c.Bl);
  switch (c.env.kind) {
    case GFNX_ENV_HYPERGRID: rollout_impl<HypergridEnv>(c, key, eps, forced); break;
    case GFNX_ENV_BITSEQ: rollout_impl<BitseqEnv>(c, key, eps, forced); break;
    case GFNX_ENV_ISING: rollout_impl<IsingEnv>(c, key, eps, forced); break;
    case GFNX_ENV_DAG: rollout_impl<DagEnv>(c, key, eps, forced); break;
  }
}

// the policy forward + masked log-softmax over the resident batch's rows (no loss): the
// per-row log pi of a teacher-forced batch (score_trajectories, objectives.cpp:294-316)
void check_forward(Ctx& c) {
  const int R = (int)total_rows(c);
  ensure_scratch(c, R);
  switch (c.env.kind) {
    case GFNX_ENV_HYPERGRID: fwd_impl<HypergridEnv>(c, R, 0); break;
    case GFNX_ENV_BITSEQ: fwd_impl<BitseqEnv>(c, R, 0); break;
    case GFNX_ENV_ISING: fwd_impl<IsingEnv>(c, R, 0); break;
    case GFNX_ENV_DAG: fwd_impl<DagEnv>(c, R, 0); break;
  }
}

// Computes loss + gradients into c.g64 / scalars[3]; the caller handles allreduce + Adam.
void check_train(Ctx& c, bool /*apply*/, double /*lr*/, double* /*loss*/) {
  const int obj = c.train.objective;
  const int need_flow = obj == GFNX_OBJ_DB || obj == GFNX_OBJ_SUBTB;
  const int R = (int)total_rows(c);
  ensure_scratch(c, R);
  const DevLayout D = make_dev_layout(c);
  switch (c.env.kind) {
    case GFNX_ENV_HYPERGRID: fwd_impl<HypergridEnv>(c, R, need_flow); break;
    case GFNX_ENV_BITSEQ: fwd_impl<BitseqEnv>(c, R, need_flow); break;
    case GFNX_ENV_ISING: fwd_impl<IsingEnv>(c, R, need_flow); break;
    case GFNX_ENV_DAG: fwd_impl<DagEnv>(c, R, need_flow); break;
  }
  cudaMemsetAsync(c.ck_glogp, 0, sizeof(double) * (size_t)R * D.A, c.stream);
  cudaMemsetAsync(c.ck_gflow, 0, sizeof(double) * (size_t)R, c.stream);
  const bool lb = c.train.learned_backward != 0;
  const int Ab = c.shape.num_backward_actions;
  if (lb) cudaMemsetAsync(c.ck_bglogp, 0, sizeof(double) * (size_t)R * Ab, c.stream);
  const int T = c.shape.max_traj_len;
  if (!c.ck_lampow) {  // pow(lambda, k), k = 0..T (glibc pow), and the SubTB pair scratch
    cuda_check(cudaMalloc(&c.ck_lampow, sizeof(double) * (T + 1)), "lampow");
    cuda_check(cudaMalloc(&c.ck_gpair, sizeof(double) * ((size_t)(T + 1) * (T + 1) + 3 * (T + 1))), "gpair");
    std::vector<double> lp(T + 1);
    for (int k = 0; k <= T; ++k) lp[k] = pow(c.train.subtb_lambda, (double)k);
    cuda_check(cudaMemcpy(c.ck_lampow, lp.data(), sizeof(double) * (T + 1), cudaMemcpyHostToDevice), "lampow");
  }
  double* lampow = c.ck_lampow;
  double* gpair = c.ck_gpair;
  // global normaliser counts live in counters[4..5] (all-reduced by the caller when world > 1)
  k_check_loss<<<1, 1, 0, c.stream>>>(obj, D.A, T, c.B, c.train.terminal_penalty,
                                      c.shape.stop_action, lampow, c.d_neglog, c.batch, c.Bl,
                                      c.batch.counters + 4, c.ck_logp, c.ck_flow, c.ck_glogp,
                                      c.ck_gflow, gpair, c.d_scalars, c.batch.counters + 3, Ab,
                                      lb ? c.ck_blogp : nullptr, c.ck_bidx, c.ck_bglogp);
  k_check_bwd<<<R, 256, 0, c.stream>>>(D, c.p64, R, need_flow, c.ck_act, c.ck_logp, c.ck_mask,
                                       c.ck_glogp, c.ck_gflow, c.ck_gx, c.ck_gz);
  if (lb) {  // bwd head + trunk over the s_{t+1} rows
    k_check_bwd<<<R, 256, 0, c.stream>>>(bwd_layout(c), c.p64, R, 0, c.ck_bact, c.ck_blogp, c.ck_bmask,
                                         c.ck_bglogp, nullptr, c.ck_bgx, c.ck_bgz);
    c.launches++;
  }
  cudaMemsetAsync(c.g64, 0, sizeof(double) * c.L.n_params, c.stream);
  const int64_t n = c.L.n_params;
  k_check_wgrad<<<(unsigned)((n + 127) / 128), 128, 0, c.stream>>>(
      D, R, need_flow, c.ck_obs, c.ck_act, c.ck_gx, c.ck_gz, c.ck_gflow, c.g64, lb ? R : 0, c.ck_bobs,
      c.ck_bact, c.ck_bgx, c.ck_bgz, c.L.off_bw, c.L.off_bb, Ab);
  c.launches += 3;
}

void check_adam(Ctx& c, double lr) {
  const gfnx_train_desc& s = c.train;
  const int do_z = s.objective == GFNX_OBJ_TB;
  const int64_t n = c.L.n_params;
  k_check_adam<<<(unsigned)((n + 255) / 256), 256, 0, c.stream>>>(
      c.p64, c.g64, c.m64, c.v64, n, lr, s.beta1, s.beta2, s.adam_eps, s.weight_decay, c.d_scalars, do_z, s.z_lr,
      c.d_steps, c.batch.counters + 3);
  c.launches++;
}

namespace {
// backward_rollout with the learned backward policy (env_core.hpp:331-359, learned branch):
// one block per walk, the bwd head's logits at the current state (fp64, reference order),
// eps_uniform(bwd_logits, backward mask, Ab, 0.0) then categorical(fold_in(step_key, b));
// walk j <-> global walk g = min(j0 + j, N - 1), terminal g / K, draw as k_bwd_walk's
template <class Env>
__global__ void k_check_bwd_walk(EnvParams P, DevLayout Db, const double* __restrict__ params,
                                 const uint32_t* __restrict__ terms, int n_walks, int64_t j0, int64_t N, int K,
                                 const uint64_t* __restrict__ keys, Key key, int64_t draw_base, int T,
                                 int16_t* __restrict__ act, uint16_t* __restrict__ np, int32_t* __restrict__ len,
                                 double* obs_scratch, double* logit_scratch, int32_t* err) {
  const int j = blockIdx.x;
  if (j >= n_walks) return;
  __shared__ typename Env::State s;
  __shared__ double hbuf[2][512];
  __shared__ int s_L, s_bad;
  const int Ab = P.Ab;
  double* obs = obs_scratch + (size_t)j * P.O;
  double* w = logit_scratch + (size_t)j * Ab;
  const int64_t g = j0 + j < N ? j0 + j : N - 1;
  const int64_t i = g / K;
  const Key base = keys ? Key{keys[2 * (size_t)i], keys[2 * (size_t)i + 1]} : key;
  const uint64_t draw = keys ? (uint64_t)(g % K) : (uint64_t)(draw_base + g);
  int16_t* a_out = act + (size_t)j * T;
  uint16_t* n_out = np + (size_t)j * T;
  if (threadIdx.x == 0) {
    unpack_terminal<Env>(P, terms + (size_t)i * P.SW, s);
    s_bad = terminal_ok<Env>(P, s) ? 0 : GFNX_ERR_CONTRACT;
    s_L = s_bad ? 0 : walk_length<Env>(P, s);
    len[j] = s_L;
    for (int t = s_L; t < T; ++t) {
      a_out[t] = -1;
      n_out[t] = 0;
    }
  }
  __syncthreads();
  const int L = s_L;
  for (int t = 0; t < L; ++t) {
    for (int q = threadIdx.x; q < P.O; q += blockDim.x) obs[q] = 0.0;
    __syncthreads();
    if (threadIdx.x == 0) Env::features(P, s, [&](int f, double v) { obs[f] = v; });
    __syncthreads();
    const double* h = obs;
    int in = P.O;
    for (int l = 0; l < Db.n_trunk; ++l) {
      double* z = hbuf[l & 1];
      dense_block(h, in, params + Db.off_w[l], params + Db.off_b[l], Db.dims[l + 1], z, true);
      __syncthreads();
      h = z;
      in = Db.dims[l + 1];
    }
    dense_block(h, in, params + Db.off_fw, params + Db.off_fb, Ab, w, false);
    __syncthreads();
    if (threadIdx.x == 0) {
      int legal = 0;  // eps_uniform(bwd_logits, mask, ab, 0.0) (objectives.cpp:242-264)
      double hi = -INFINITY;
      for (int c = 0; c < Ab; ++c)
        if (bwd_legal<Env>(P, s, c)) {
          ++legal;
          if (w[c] > hi) hi = w[c];
        }
      if (legal == 0 || !isfinite(hi)) {
        s_bad = legal == 0 ? GFNX_ERR_CONTRACT : GFNX_ERR_NUMERIC;
      } else {
        double z = 0.0;
        for (int c = 0; c < Ab; ++c) {
          if (bwd_legal<Env>(P, s, c)) {
            const double p = exp(w[c] - hi);
            w[c] = p;
            z += p;
          } else {
            w[c] = 0.0;
          }
        }
        const double u = 0.0 / legal;
        double total = 0.0;
        for (int c = 0; c < Ab; ++c) {
          if (bwd_legal<Env>(P, s, c)) w[c] = (1.0 - 0.0) * w[c] / z + u;
          total += w[c];
        }
        const double uu = uniform_scalar(fold_in(fold_in(base, (uint64_t)t), draw)) * total;
        int ab = -1;
        double acc = 0.0;
        for (int c = 0; c < Ab; ++c) {
          acc += w[c];
          if (uu < acc) {
            ab = c;
            break;
          }
        }
        if (ab < 0)
          for (int c = Ab - 1; c >= 0; --c)
            if (w[c] > 0.0) {
              ab = c;
              break;
            }
        const int f = L - 1 - t;
        n_out[f] = (uint16_t)legal;
        a_out[f] = (int16_t)bwd_apply<Env>(P, s, ab);
      }
    }
    __syncthreads();
    if (s_bad) break;
  }
  if (threadIdx.x == 0 && s_bad) atomicExch(err, s_bad);
}

__global__ void k_check_row_logpf(DeviceBatch batch, const double* __restrict__ logp, int A, int Bl, int T,
                                  double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= Bl * T) return;
  const int b = i / T, t = i % T;
  out[i] = t < batch.lengths[b] ? logp[(size_t)(batch.row0[b] + t) * A + batch.actions[i]] : 0.0;
}
}  // namespace

void check_bwd_walk(Ctx& c, const uint32_t* d_terms, int n_walks, int64_t j0, int64_t N, int K,
                    const uint64_t* d_keys, Key key, int64_t draw_base, int16_t* d_act, uint16_t* d_np,
                    int32_t* d_len) {
  if (n_walks <= 0) return;
  double *obs = nullptr, *logit = nullptr;
  cuda_check(cudaMallocAsync(&obs, sizeof(double) * (size_t)n_walks * c.P.O, c.stream), "bwd walk");
  cuda_check(cudaMallocAsync(&logit, sizeof(double) * (size_t)n_walks * c.P.Ab, c.stream), "bwd walk");
  const DevLayout Db = bwd_layout(c);
  auto go = [&](auto e) {
    using Env = decltype(e);
    k_check_bwd_walk<Env><<<n_walks, 256, 0, c.stream>>>(c.P, Db, c.p64, d_terms, n_walks, j0, N, K, d_keys, key,
                                                          draw_base, c.P.T, d_act, d_np, d_len, obs, logit,
                                                          c.batch.counters + 3);
  };
  switch (c.env.kind) {
    case GFNX_ENV_HYPERGRID: go(HypergridEnv{}); break;
    case GFNX_ENV_BITSEQ: go(BitseqEnv{}); break;
    case GFNX_ENV_ISING: go(IsingEnv{}); break;
    case GFNX_ENV_DAG: go(DagEnv{}); break;
  }
  c.launches++;
  cudaFreeAsync(obs, c.stream);
  cudaFreeAsync(logit, c.stream);
}

namespace {
// per-row learned log P_B of the last check_forward, (b, t) order (0 past each end)
__global__ void k_check_row_logpb(DeviceBatch batch, const double* __restrict__ blogp,
                                  const int32_t* __restrict__ bidx, int Ab, int Bl, int T, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= Bl * T) return;
  const int b = i / T, t = i % T;
  if (t >= batch.lengths[b]) {
    out[i] = 0.0;
    return;
  }
  const int64_t r = batch.row0[b] + t;
  out[i] = blogp[r * Ab + bidx[r]];
}
}  // namespace

void check_row_logpb(Ctx& c, double* out) {
  const int n = c.Bl * c.P.T;
  k_check_row_logpb<<<(n + 255) / 256, 256, 0, c.stream>>>(c.batch, c.ck_blogp, c.ck_bidx, c.P.Ab, c.Bl, c.P.T, out);
  c.launches++;
}

void check_row_logpf(Ctx& c, double* out) {
  const int n = c.Bl * c.P.T;
  k_check_row_logpf<<<(n + 255) / 256, 256, 0, c.stream>>>(c.batch, c.ck_logp, c.P.A, c.Bl, c.P.T, out);
  c.launches++;
}

}  // namespace gfnx
