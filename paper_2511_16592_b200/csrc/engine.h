// engine.h — host-side engine context shared by the kernel translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/gfnx.h"
#include "envs.cuh"

namespace gfnx {

// Layout of the flat parameter vector in MlpParams::tensors() order (nn.cpp:8-19).
struct MlpLayout {
  int n_trunk = 0;
  int dims[10] = {0};  // dims[0] = obs_dim, dims[l+1] = hidden width of trunk layer l
  int64_t off_w[10] = {0}, off_b[10] = {0};
  int64_t off_fw = 0, off_fb = 0, off_bw = 0, off_bb = 0, off_flw = 0, off_flb = 0;
  int64_t n_params = 0;
  int H() const { return dims[n_trunk]; }
};

// Device-resident trajectory batch of this rank's slice (compact SoA, not the padded
// B*(T+1)*obs_dim fp64 TrajectoryBatch of trajectory.hpp:15-33).
struct DeviceBatch {
  int32_t* lengths = nullptr;     // [Bl]
  int16_t* actions = nullptr;     // [Bl * T], -1 pad
  double* log_rewards = nullptr;  // [Bl]
  double* delta = nullptr;        // [Bl * T] (MDB)
  uint16_t* nparents = nullptr;   // [Bl * T] #legal backward actions at s_{t+1} (log_pb = -log n)
  uint32_t* term_state = nullptr; // [Bl * SW]
  int32_t* row0 = nullptr;        // [Bl + 1] exclusive prefix of lengths
  int32_t* row_bt = nullptr;      // [sum L] row -> b * T + t (state row of the training pass)
  int32_t* scan_part = nullptr;   // scan scratch
  int32_t* counters = nullptr;    // [4]: total rows, mdb rows, work counter, error word
};

struct Ctx;
struct Group;  // in-process communicator (group.cu)

// element types of the job's all-reduces
constexpr int kDtypeF32 = 0, kDtypeF64 = 1, kDtypeI32 = 2;
Group* group_new(int world);
int group_world(const Group* g);
void group_delete(Group* g);
void group_join(Ctx& c, Group* g, int rank);
void group_leave(Ctx& c, Group* g, int rank);
void group_allreduce(Ctx& c, void* buf, size_t n, int dtype, cudaStream_t s);
// world > 1: all-reduce the gradient bucket g[0, n) on the comm stream once the compute
// stream's work so far is done (SURVEY §8(e) bucketed all-reduce behind the backward); the
// rest of the gradient follows in do_train after the compute stream joins — api.cu
void grad_bucket_async(Ctx& c, float* g, int64_t n);

// check-mode (fp64 SIMT, reference operation order) — check.cu
// forced: [Bl * T] actions of a teacher-forced batch (rollout_from_actions), or null to sample
void check_rollout(Ctx& c, Key key, double eps, const int16_t* forced = nullptr);
void check_forward(Ctx& c);  // per-row log-softmax of the resident batch (check_row_logpf reads it)
// learned backward policy (check mode): walks sampled from the bwd head, per-row log P_B
void check_bwd_walk(Ctx& c, const uint32_t* d_terms, int n_walks, int64_t j0, int64_t N, int K,
                    const uint64_t* d_keys, Key key, int64_t draw_base, int16_t* d_act, uint16_t* d_np,
                    int32_t* d_len);
void check_row_logpb(Ctx& c, double* out);
void check_train(Ctx& c, bool apply, double lr, double* loss);
void check_adam(Ctx& c, double lr);

// fast mode (bf16 tcgen05) — fast.cu
void fast_init(Ctx& c);
void fast_free(Ctx& c);
void fast_rollout(Ctx& c, Key key, double eps);
void fast_train(Ctx& c, bool apply, double lr, double* loss);  // gradients -> g32, scalars
void fast_adam(Ctx& c, double lr);
void fast_sync_weights(Ctx& c);  // fp32 master -> bf16 operand images
void fast_row_logpf(Ctx& c, double* out);   // per-row log pi_F of the training record [Bl*T] (device)
void check_row_logpf(Ctx& c, double* out);

// fixed-length (lockstep) fast path for bitseq / Ising — lockstep.cu
bool ls_supported(const Ctx& c, std::string* why);
void ls_init(Ctx& c);
void ls_free(Ctx& c);
void ls_sync_weights(Ctx& c);
void ls_rollout(Ctx& c, Key key, double eps, const int16_t* forced = nullptr);
void ls_train(Ctx& c);
void ls_row_logpf(Ctx& c, double* out);
bool ls_debug_buffer(Ctx& c, const std::string& name, const void** ptr, size_t* bytes);

// diagnostics — fast.cu
void test_mma_rate(int n, int reps, int mode, int grid, long long* host_out);
void test_ts_mma(const uint16_t* a, const uint16_t* b, float* d);

// shared small kernels — batch.cu
void launch_row_scan(Ctx& c, bool counts = true);
// batched terminal log-rewards over word-major packed states [SW][n] (device) — reward.cu
void reward_soa(Ctx& c, const uint32_t* st, int64_t n, double* out);
void reward_free(Ctx& c);
void ensure_row0(Ctx& c);              // row0 / row_bt of the resident batch (lazy after a fused rollout)
bool fast_rollout_counts(const Ctx& c);  // the fast rollout publishes the row counts itself
void fast_hg_marginal(Ctx& c, std::vector<double>* pt);  // exact terminal marginal (hypergrid)
// tv_buffer metric (hypergrid): terminal-state FIFO + histogram on the device — fast.cu
// mc_terminal_logprob (exact.hpp:229-241), hypergrid fast path — fast.cu
// (device buffers: terminals [n][SW], keys [n][2], out [n])
void fast_mc_terminal_logprob(Ctx& c, const uint32_t* d_terms, int64_t n, int K, const uint64_t* d_keys,
                              double* d_out);
void fast_forced_rollout(Ctx& c, const int16_t* d_forced);  // rollout_from_actions, bf16 paths
// backward walks, teacher-forced batches, MC terminal log-probabilities — walk.cu
void launch_bwd_walk(Ctx& c, const uint32_t* d_terms, int n_walks, int64_t j0, int64_t N, int K,
                     const uint64_t* d_keys, Key key, int64_t draw_base, int16_t* d_act, uint16_t* d_np,
                     int32_t* d_len, uint32_t* d_stst);
void launch_replay(Ctx& c, const int16_t* d_forced, uint32_t* d_stst);
void exclusive_scan_i32(Ctx& c, const int32_t* d_in, int32_t* d_out, int n);
void launch_walk_rows(Ctx& c, const int32_t* d_len, const int32_t* d_row0, int n, int32_t* d_rows,
                      int32_t* d_tiles, int tile_rows);
void launch_mc_terms_rows(Ctx& c, const float* rowbuf, int rs, const int32_t* d_row0, const uint16_t* d_np,
                          const int32_t* d_len, int n, double* d_terms);
void launch_mc_lse(Ctx& c, const double* d_terms, int n, int K, double* d_out);
void forced_rollout(Ctx& c, const int16_t* d_forced);
void backward_rollout(Ctx& c, const uint32_t* d_terms, Key key);
// EB-GFN (run_eb_gfn, train.cpp:875-1018) — eb.cu
void eb_default_desc(gfnx_eb_desc* d);
void eb_init(Ctx& c, const gfnx_eb_desc& d, const int8_t* data, int64_t n);
void eb_free(Ctx& c);
void eb_ensure_metrics(Ctx& c, int64_t n);
const int16_t* eb_pre(Ctx& c, Key it_key);
void eb_post(Ctx& c, Key it_key, double j_lr, int64_t i);
const double* eb_metrics(Ctx& c);
double eb_coupling_lr(Ctx& c, int64_t it);
void eb_coupling(Ctx& c, double* jm, double* jt, double* init_nlr);
int64_t eb_dataset(Ctx& c, int8_t* out, int64_t n);
void bitseq_pearson(Ctx& c, int64_t step, int mc, uint64_t test_seed, double* d_out);
void mc_terminal_logprob_chunked(Ctx& c, const uint32_t* d_terms, int64_t n, int K, const uint64_t* d_keys,
                                 double* d_out);
void hg_buffer_reset(Ctx& c, int64_t capacity);
void hg_buffer_push(Ctx& c);
double hg_buffer_tv(Ctx& c);
void hg_buffer_free(Ctx& c);

struct Ctx {
  gfnx_env_desc env{};
  gfnx_train_desc train{};
  gfnx_env_shape shape{};
  EnvParams P{};
  MlpLayout L{};   // device layout (bf16 fast paths: hidden widths zero-padded to the kernel's)
  MlpLayout Lx{};  // the user's layout (MlpParams::tensors() of the requested widths): the ABI
  std::vector<int64_t> xmap;  // user parameter index -> device index (empty: same layout)
  int device = 0, rank = 0, world = 1;
  int B = 0, Bl = 0, b0 = 0;  // global batch, local slice [b0, b0+Bl)
  int Bcap = 0;               // trajectory capacity of the batch arrays (>= Bl: lockstep pads to 128)
  cudaStream_t stream = nullptr;
  void* nccl = nullptr;  // ncclComm_t (one process per GPU)
  Group* group = nullptr;  // or an in-process group (one thread per rank)
  std::string err;
  int64_t launches = 0;

  // environment tables (device)
  uint64_t* d_modes = nullptr;
  double* d_bs_logr = nullptr;
  int16_t* d_is_nbr = nullptr;
  double* d_is_J = nullptr;
  double* d_dag_cache = nullptr;
  double* d_neglog = nullptr;
  std::vector<double> h_dag_cache;
  std::vector<int16_t> h_is_nbr;  // [D][4] ascending neighbours (host copy, reward tables)
  std::vector<double> h_is_J;
  double* d_is_rowtab = nullptr;  // [D][16] Ising row sums per neighbour pattern (reward.cu)

  // parameters: fp64 master (check mode) or fp32 master (fast mode)
  double* p64 = nullptr;
  double* g64 = nullptr;
  double* m64 = nullptr;
  double* v64 = nullptr;
  float* p32 = nullptr;
  float* g32 = nullptr;
  float* m32 = nullptr;
  float* v32 = nullptr;
  double* d_scalars = nullptr;  // [8]: log_z, z_m, z_v, dlogz, loss, norm, ...
  int64_t* d_steps = nullptr;   // [4]: adam_t, z_t, commit ticket (device-owned, see adam_commit)

  DeviceBatch batch;
  bool has_batch = false;
  bool has_grads = false;

  // check-mode scratch
  double* ck_obs = nullptr;
  double* ck_act = nullptr;
  double* ck_logp = nullptr;
  uint8_t* ck_mask = nullptr;
  double* ck_flow = nullptr;
  double* ck_glogp = nullptr;
  double* ck_gflow = nullptr;
  double* ck_gz = nullptr;
  double* ck_gx = nullptr;
  double* ck_pair = nullptr;
  double* ck_lampow = nullptr;  // [T + 1] pow(lambda, k)
  double* ck_gpair = nullptr;   // SubTB pair scratch
  // learned backward policy (check mode): the bwd head's rows (s_{t+1} of every step)
  double *ck_bobs = nullptr, *ck_bact = nullptr, *ck_blogp = nullptr, *ck_bglogp = nullptr, *ck_bgx = nullptr,
         *ck_bgz = nullptr;
  uint8_t* ck_bmask = nullptr;
  int32_t* ck_bidx = nullptr;
  int64_t ck_rows_cap = 0;

  // optional rollout phase clocks (env GFNX_PHASE_TIMERS=1 at create): [8] int64
  long long* phase = nullptr;
  bool rows_stale = false;  // row0 / row_bt not derived for the resident batch yet

  // fast-mode state (opaque, fast.cu)
  void* fast = nullptr;
  // EB-GFN state (opaque, eb.cu)
  void* eb = nullptr;

  // terminal-state FIFO of the tv_buffer metric (FifoBuffer, buffer.hpp:13-55): ring of
  // cell indices + per-cell counts on the device; head / size tracked on the host (every
  // push appends exactly Bl items, stream-ordered)
  struct TermBuffer {
    int32_t* fifo = nullptr;  // [cap] cell index (coordinate 0 fastest)
    int32_t* hist = nullptr;  // [cells] occurrences in the ring
    double* p = nullptr;      // [cells] grid_exact_distribution probabilities
    double* out = nullptr;    // [1] last tv
    int64_t cap = 0, head = 0, size = 0, cells = 0;
  } tbuf;

  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t user_ev[16] = {};
  // pinned staging slots for gfnx_iteration_async
  struct Slot {
    uint8_t* host = nullptr;  // [loss f64 | err i32 pad | lengths | log_rewards | term_state]
    uint8_t* dev = nullptr;   // the same bytes staged on the device (one gather kernel)
    cudaEvent_t staged = nullptr, done = nullptr;
    int64_t it = -1;
  };
  Slot slots[2];
  cudaStream_t copy_stream = nullptr;  // slot device->host copies, off the compute stream
  cudaStream_t comm_stream = nullptr;  // world > 1: the early gradient bucket's all-reduce
  cudaEvent_t comm_ev[2] = {nullptr, nullptr};
  int64_t grad_bucket0 = 0;            // gradient entries [0, grad_bucket0) already in flight
  // per-kernel CUDA-event profiling (bench.py roofline): records (name, start, stop)
  struct ProfRec {
    const char* name;
    cudaEvent_t a, b;
  };
  bool profiling = false;
  bool profile_rollout_only = false;  // gfnx_profile(ctx, 2): bracket the rollout kernel only
  std::vector<ProfRec> prof;
  std::vector<cudaEvent_t> ev_pool;
  double last_rollout_ms = 0.0, last_train_ms = 0.0;

  bool check_mode() const { return train.precision == GFNX_PREC_FP64_CHECK; }
};

// RAII bracket of one kernel launch with CUDA events on the ctx stream (when profiling)
struct ProfScope {
  Ctx& c;
  int idx = -1;
  ProfScope(Ctx& ctx, const char* name);
  ~ProfScope();
};

#ifdef __CUDACC__
// Adam step commit: the last block of an Adam kernel to finish advances the device step
// counters (every block read them at its start, before any block took a ticket).
__device__ __forceinline__ void adam_commit(int64_t* steps, int do_z) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned long long k = atomicAdd(reinterpret_cast<unsigned long long*>(steps + 2), 1ull);
    if (k == gridDim.x - 1) {
      steps[0] += 1;
      if (do_z) steps[1] += 1;
      steps[2] = 0;
      __threadfence();
    }
  }
}
#endif

// error reporting from kernel TUs
void cuda_check(cudaError_t e, const char* what);
[[noreturn]] void raise_error(int code, const std::string& msg);
int64_t total_rows(Ctx& c);  // reads counters[0] (sync)

}  // namespace gfnx
