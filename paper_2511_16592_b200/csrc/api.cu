// api.cu — the C ABI of libgfnx (include/gfnx.h): context lifetime, parameter/optimizer
// state import/export, the per-iteration pipeline (rollout -> loss/grad -> NCCL all-reduce
// -> Adam) and batch export. The pipeline mirrors train_scenario's loop body
// (proj/src/train.cpp:224-229) and train_step (:164-192).
#include <dlfcn.h>
#include <math.h>
#include <nccl.h>
#include <string.h>

#include <algorithm>
#include <cstdio>
#include <string>
#include <vector>

#include "engine.h"
#include "host.h"

namespace gfnx {

namespace {
thread_local std::string g_create_err;

struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl_api() {  // loaded lazily: single-GPU runs never touch NCCL
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
      api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
      api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
      api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
      api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
      api.ok = api.GetUniqueId && api.CommInitRank && api.AllReduce && api.CommDestroy;
    }
  }
  return api;
}

struct Failure {
  gfnx_status code;
  std::string msg;
};

}  // namespace

void raise_error(int code, const std::string& msg) { throw Failure{(gfnx_status)code, msg}; }

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Failure{GFNX_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}

// ---------------------------------------------------------------------------
// small kernels shared by both precisions

ProfScope::ProfScope(Ctx& ctx, const char* name) : c(ctx) {
  if (!c.profiling) return;
  if (c.profile_rollout_only && strcmp(name, "k_fast_rollout") != 0 && strcmp(name, "k_ls_persist") != 0) return;
  auto take = [&]() {
    if (c.ev_pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = c.ev_pool.back();
    c.ev_pool.pop_back();
    return e;
  };
  Ctx::ProfRec r{name, take(), take()};
  cudaEventRecord(r.a, c.stream);
  c.prof.push_back(r);
  idx = (int)c.prof.size() - 1;
}

ProfScope::~ProfScope() {
  if (idx >= 0) cudaEventRecord(c.prof[idx].b, c.stream);
}

// lengths -> row0 (exclusive prefix of lengths), row_bt (row -> b*T + t), counters:
// counters[0] = sum L, [1] = sum max(L-1, 0), [4..5] = the same (global when world == 1,
// all-reduced otherwise), [8..11] = int64 running totals (rows, rollouts) for bench.py.
// Three coalesced passes over 1024-trajectory blocks (the partial sums are tiny).
constexpr int kScanBlock = 1024;

__device__ __forceinline__ int block_excl_scan(int v, int* warp_sums, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    warp_sums[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  const int base = warp > 0 ? warp_sums[warp - 1] : 0;
  if (total) *total = warp_sums[(blockDim.x >> 5) - 1];
  return base + x - v;
}

__global__ void k_len_partials(const int32_t* __restrict__ lengths, int Bl, int2* part) {
  __shared__ int ws[32], ws2[32];
  const int b = blockIdx.x * kScanBlock + threadIdx.x;
  const int L = b < Bl ? lengths[b] : 0;
  int v = L, v2 = L > 1 ? L - 1 : 0;
  for (int o = 16; o > 0; o >>= 1) {
    v += __shfl_xor_sync(0xffffffffu, v, o);
    v2 += __shfl_xor_sync(0xffffffffu, v2, o);
  }
  if ((threadIdx.x & 31) == 0) {
    ws[threadIdx.x >> 5] = v;
    ws2[threadIdx.x >> 5] = v2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0, s2 = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      s += ws[w];
      s2 += ws2[w];
    }
    part[blockIdx.x] = make_int2(s, s2);
  }
}

__global__ void k_len_scan_partials(int2* part, int nparts, int32_t* counters, int counts) {
  if (threadIdx.x != 0) return;
  int run = 0, run2 = 0;
  for (int i = 0; i < nparts; ++i) {  // <= 64 entries at B = 65536
    const int2 p = part[i];
    part[i] = make_int2(run, 0);
    run += p.x;
    run2 += p.y;
  }
  if (!counts) return;
  long long* acc = reinterpret_cast<long long*>(counters + 8);
  acc[0] += run;
  acc[1] += 1;
  counters[0] = run;
  counters[1] = run2;
  counters[4] = run;
  counters[5] = run2;
}

__global__ void k_len_finish(const int32_t* __restrict__ lengths, int Bl, int T,
                             const int2* part, int32_t* row0, int32_t* row_bt, const int32_t* counters) {
  __shared__ int ws[32];
  const int b = blockIdx.x * kScanBlock + threadIdx.x;
  const int L = b < Bl ? lengths[b] : 0;
  const int r0 = part[blockIdx.x].x + block_excl_scan(L, ws, nullptr);
  if (b < Bl) {
    row0[b] = r0;
    for (int t = 0; t < L; ++t) row_bt[r0 + t] = b * T + t;
  }
  if (b == Bl) row0[Bl] = counters[0];
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0 && Bl % kScanBlock == 0) row0[Bl] = counters[0];
}

void ensure_row0(Ctx& c) {
  if (!c.rows_stale) return;
  launch_row_scan(c, false);
  c.rows_stale = false;
}

void launch_row_scan(Ctx& c, bool counts) {
  ProfScope ps(c, "k_row_scan");
  const int nb = (c.Bl + kScanBlock - 1) / kScanBlock;
  int2* part = reinterpret_cast<int2*>(c.batch.scan_part);
  k_len_partials<<<nb, kScanBlock, 0, c.stream>>>(c.batch.lengths, c.Bl, part);
  k_len_scan_partials<<<1, 32, 0, c.stream>>>(part, nb, c.batch.counters, counts ? 1 : 0);
  k_len_finish<<<nb, kScanBlock, 0, c.stream>>>(c.batch.lengths, c.Bl, c.P.T, part, c.batch.row0,
                                                c.batch.row_bt, c.batch.counters);
  c.launches += 3;
}

int64_t total_rows(Ctx& c) {
  int32_t v = 0;
  cuda_check(cudaMemcpyAsync(&v, c.batch.counters, sizeof v, cudaMemcpyDeviceToHost, c.stream),
             "read rows");
  cuda_check(cudaStreamSynchronize(c.stream), "sync");
  return v;
}

__global__ void k_threefry(const uint64_t* keys, const uint64_t* ctr, int64_t n, uint64_t* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t a, b;
  threefry2x64(Key{keys[2 * i], keys[2 * i + 1]}, ctr[2 * i], ctr[2 * i + 1], a, b);
  out[2 * i] = a;
  out[2 * i + 1] = b;
}

__global__ void k_uniform_fold(Key k, const uint64_t* idx, int64_t n, double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = uniform_scalar(fold_in(k, idx[i]));
}

__global__ void k_copy_f64_to_f32(const double* a, float* b, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = (float)a[i];
}
__global__ void k_copy_f32_to_f64(const float* a, double* b, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = (double)a[i];
}

}  // namespace gfnx

using namespace gfnx;

struct gfnx_ctx {
  Ctx c;
};

namespace {

template <class F>
gfnx_status guard(gfnx_ctx* ctx, F&& f) {
  try {
    if (ctx && ctx->c.stream) cuda_check(cudaSetDevice(ctx->c.device), "cudaSetDevice");  // per calling thread
    f();
    return GFNX_OK;
  } catch (const Failure& e) {
    if (ctx) ctx->c.err = e.msg; else g_create_err = e.msg;
    return e.code;
  }
}

[[noreturn]] void fail(gfnx_status code, const std::string& msg) { throw Failure{code, msg}; }

void check_device_error(Ctx& c) {
  int32_t e = 0;
  cuda_check(cudaMemcpyAsync(&e, c.batch.counters + 3, sizeof e, cudaMemcpyDeviceToHost, c.stream),
             "error word");
  cuda_check(cudaStreamSynchronize(c.stream), "sync");
  if (e != 0) {
    cudaMemsetAsync(c.batch.counters + 3, 0, sizeof(int32_t), c.stream);
    if (e == GFNX_ERR_NUMERIC) fail(GFNX_ERR_NUMERIC, "non-finite policy logits or loss");
    fail((gfnx_status)e, "contract violation detected on device (illegal action / no legal action)");
  }
}

// the job's all-reduce (sum, in place, stream-ordered on `st`, default the compute stream):
// in-process group or NCCL
void nccl_sum(Ctx& c, void* buf, size_t n, ncclDataType_t t, cudaStream_t st = nullptr) {
  if (c.world <= 1) return;
  if (!st) st = c.stream;
  if (c.group) {
    group_allreduce(c, buf, n, t == ncclFloat64 ? kDtypeF64 : t == ncclFloat32 ? kDtypeF32 : kDtypeI32, st);
    return;
  }
  NcclApi& api = nccl_api();
  const ncclResult_t r = api.AllReduce(buf, buf, n, t, ncclSum, (ncclComm_t)c.nccl, st);
  if (r != ncclSuccess) fail(GFNX_ERR_NCCL, std::string("ncclAllReduce: ") + api.GetErrorString(r));
}

}  // namespace

void gfnx::grad_bucket_async(Ctx& c, float* g, int64_t n) {
  if (c.world <= 1 || n <= 0) return;
  if (!c.comm_stream) {
    cuda_check(cudaStreamCreateWithFlags(&c.comm_stream, cudaStreamNonBlocking), "comm stream");
    for (auto& e : c.comm_ev) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "comm event");
  }
  cuda_check(cudaEventRecord(c.comm_ev[0], c.stream), "bucket ready");
  cuda_check(cudaStreamWaitEvent(c.comm_stream, c.comm_ev[0], 0), "bucket wait");
  nccl_sum(c, g, (size_t)n, ncclFloat32, c.comm_stream);
  cuda_check(cudaEventRecord(c.comm_ev[1], c.comm_stream), "bucket done");
  c.grad_bucket0 = n;
}

namespace {

void do_rollout(Ctx& c, int64_t it, double eps) {
  if (eps < 0.0 || eps > 1.0) fail(GFNX_ERR_CONFIG, "exploration eps must lie in [0,1]");
  const Key key = fold_in(make_key(c.train.seed), 1000 + (uint64_t)it);  // train.cpp:228
  cudaEventRecord(c.ev[0], c.stream);
  if (c.check_mode()) check_rollout(c, key, eps);
  else fast_rollout(c, key, eps);
  if (c.check_mode() || !fast_rollout_counts(c)) {
    launch_row_scan(c);
    c.rows_stale = false;
  } else {
    c.rows_stale = true;  // counts published by the rollout; row0 derived on demand
  }
  if (c.world > 1) nccl_sum(c, c.batch.counters + 4, 2, ncclInt32);
  cudaEventRecord(c.ev[1], c.stream);
  cuda_check(cudaGetLastError(), "rollout launch");
  c.has_batch = true;
  c.has_grads = false;
}

// a teacher-forced batch just landed in the resident batch (rollout_from_actions): row
// counts, the global normalisers, batch flags
void finish_forced(Ctx& c) {
  launch_row_scan(c);
  c.rows_stale = false;
  if (c.world > 1) nccl_sum(c, c.batch.counters + 4, 2, ncclInt32);
  cuda_check(cudaGetLastError(), "forced rollout launch");
  c.has_batch = true;
  c.has_grads = false;
}

// gradient + (optionally) Adam; loss read back when loss != nullptr
void do_train(Ctx& c, bool apply, double lr, double* loss) {
  if (!c.has_batch) fail(GFNX_ERR_CONTRACT, "train_step: no resident batch (call gfnx_rollout)");
  const int64_t n = c.L.n_params;
  if (c.check_mode()) {
    check_train(c, apply, lr, loss);
    if (c.world > 1) {
      cudaMemcpyAsync(c.g64 + n, c.d_scalars + 3, 2 * sizeof(double), cudaMemcpyDeviceToDevice, c.stream);
      nccl_sum(c, c.g64, (size_t)n + 2, ncclFloat64);
      cudaMemcpyAsync(c.d_scalars + 3, c.g64 + n, 2 * sizeof(double), cudaMemcpyDeviceToDevice, c.stream);
    }
    if (apply) check_adam(c, lr);
  } else {
    fast_train(c, apply, lr, loss);
    if (c.world > 1) {  // the early bucket (fast_train: dW1 | db1 behind wgrad), then the rest
      const int64_t n0 = c.grad_bucket0;
      if (n0 > 0) cuda_check(cudaStreamWaitEvent(c.stream, c.comm_ev[1], 0), "bucket join");
      c.grad_bucket0 = 0;
      nccl_sum(c, c.g32 + n0, (size_t)(n - n0), ncclFloat32);
      nccl_sum(c, c.d_scalars + 3, 2, ncclFloat64);
    }
    if (apply) fast_adam(c, lr);
  }
  cudaEventRecord(c.ev[2], c.stream);
  cuda_check(cudaGetLastError(), "train launch");
  c.has_grads = true;
  if (loss) {
    double v = 0.0;
    cuda_check(cudaMemcpyAsync(&v, c.d_scalars + 4, sizeof v, cudaMemcpyDeviceToHost, c.stream), "loss");
    check_device_error(c);
    *loss = v;
  }
}

}  // namespace

namespace {
// The bf16 fast paths run fixed hidden widths: lockstep (bitseq / Ising) 256 per layer,
// hypergrid two equal layers of 128 or 256, DAG two of 128. A narrower network runs there
// zero-padded: the extra units have zero weights in and out and zero bias, so they stay
// exactly 0 through ReLU (their products add exact zeros to the real units' tensor-core
// sums), their ReLU masks are 0, every gradient into them is exactly 0 and Adam (with or
// without weight decay) keeps them at 0 — the real units compute what the requested widths
// compute. The ABI (params, grads, Adam state, checkpoints) keeps the user's layout.
void pad_layout(Ctx& c) {
  const int kind = c.env.kind, nh = c.train.num_hidden;
  int maxw = 0;
  for (int l = 0; l < nh; ++l) maxw = std::max(maxw, (int)c.train.hidden[l]);
  int target = 0;
  if (kind == GFNX_ENV_BITSEQ || kind == GFNX_ENV_ISING) {
    if (maxw <= 256 && nh >= 2) target = 256;
  } else if (nh == 2) {
    if (kind == GFNX_ENV_DAG) target = maxw <= 128 ? 128 : 0;
    else target = maxw <= 128 ? 128 : maxw <= 256 ? 256 : 0;
  }
  if (!target) return;  // unsupported widths: the fast path's own check reports them
  bool same = true;
  for (int l = 0; l < nh; ++l) same = same && c.train.hidden[l] == target;
  if (same) return;
  gfnx_train_desc tp = c.train;
  for (int l = 0; l < nh; ++l) tp.hidden[l] = target;
  make_layout(tp, c.shape, &c.L);
  const MlpLayout &X = c.Lx, &D = c.L;
  c.xmap.assign(X.n_params, -1);
  auto block = [&](int64_t xo, int64_t dof, int rows, int cols, int dcols) {  // [rows][cols]
    for (int i = 0; i < rows; ++i)
      for (int j = 0; j < cols; ++j) c.xmap[xo + (int64_t)i * cols + j] = dof + (int64_t)i * dcols + j;
  };
  for (int l = 0; l < nh; ++l) {
    block(X.off_w[l], D.off_w[l], X.dims[l], X.dims[l + 1], D.dims[l + 1]);
    block(X.off_b[l], D.off_b[l], 1, X.dims[l + 1], D.dims[l + 1]);
  }
  const int A = c.shape.num_actions, Ab = c.shape.num_backward_actions, H = X.H();
  block(X.off_fw, D.off_fw, H, A, A);
  block(X.off_fb, D.off_fb, 1, A, A);
  block(X.off_bw, D.off_bw, H, Ab, Ab);
  block(X.off_bb, D.off_bb, 1, Ab, Ab);
  block(X.off_flw, D.off_flw, H, 1, 1);
  block(X.off_flb, D.off_flb, 1, 1, 1);
}
}  // namespace

// user-layout vector -> device-layout vector (padding zero), and back
std::vector<double> to_device_layout(const Ctx& c, const double* x) {
  if (c.xmap.empty()) return std::vector<double>(x, x + c.L.n_params);
  std::vector<double> d(c.L.n_params, 0.0);
  for (int64_t i = 0; i < c.Lx.n_params; ++i) d[c.xmap[i]] = x[i];
  return d;
}
template <class T>
void to_user_layout(const Ctx& c, const T* d, double* x) {
  if (c.xmap.empty()) {
    for (int64_t i = 0; i < c.L.n_params; ++i) x[i] = d[i];
  } else {
    for (int64_t i = 0; i < c.Lx.n_params; ++i) x[i] = d[c.xmap[i]];
  }
}

extern "C" {

int32_t gfnx_abi_version(void) { return GFNX_ABI_VERSION; }

gfnx_status gfnx_default_env_desc(int32_t kind, gfnx_env_desc* out) {
  if (kind < 0 || kind > 3 || !out) return GFNX_ERR_CONFIG;
  default_env(kind, out);
  return GFNX_OK;
}

gfnx_status gfnx_default_train_desc(int32_t kind, gfnx_train_desc* out) {
  if (kind < 0 || kind > 3 || !out) return GFNX_ERR_CONFIG;
  default_train(kind, out);
  return GFNX_OK;
}

gfnx_status gfnx_env_shape_of(const gfnx_env_desc* env, gfnx_env_shape* out) {
  return guard(nullptr, [&] {
    HostEnv he;
    const std::string err = build_host_env(*env, &he);
    if (!err.empty()) fail(GFNX_ERR_CONFIG, err);
    *out = he.shape;
  });
}

const char* gfnx_last_error(const gfnx_ctx* ctx) {
  return ctx ? ctx->c.err.c_str() : g_create_err.c_str();
}

gfnx_status gfnx_nccl_unique_id(void* out128) {
  return guard(nullptr, [&] {
    NcclApi& api = nccl_api();
    if (!api.ok) fail(GFNX_ERR_NCCL, "libnccl.so.2 not found");
    ncclUniqueId id;
    const ncclResult_t r = api.GetUniqueId(&id);
    if (r != ncclSuccess) fail(GFNX_ERR_NCCL, api.GetErrorString(r));
    memcpy(out128, &id, sizeof id);
  });
}


namespace {
gfnx_status create_impl(const gfnx_env_desc* env, const gfnx_train_desc* train, int32_t device, int32_t rank,
                        int32_t world, const void* nccl_id, Group* group, gfnx_ctx** out) {
  *out = nullptr;
  auto* h = new gfnx_ctx();
  Ctx& c = h->c;
  const gfnx_status st = guard(nullptr, [&] {
    c.env = *env;
    c.train = *train;
    if (world < 1 || rank < 0 || rank >= world) fail(GFNX_ERR_CONFIG, "bad rank/world");
    HostEnv he;
    std::string err = build_host_env(*env, &he);
    if (!err.empty()) fail(GFNX_ERR_CONFIG, err);
    c.shape = he.shape;
    err = validate_train(*train, c.shape);
    if (!err.empty()) fail(GFNX_ERR_CONFIG, err);
    resolve_schedule(&c.train.lr, c.train.iterations);
    resolve_schedule(&c.train.explore, c.train.iterations);
    make_layout(c.train, c.shape, &c.Lx);
    c.L = c.Lx;
    if (train->precision != GFNX_PREC_FP64_CHECK) pad_layout(c);
    c.device = device;
    c.rank = rank;
    c.world = world;
    c.B = train->batch_size;
    // contiguous slices; rank r takes [r*B/W, (r+1)*B/W) — global indices keep the RNG stream
    c.b0 = (int)((int64_t)c.B * rank / world);
    c.Bl = (int)((int64_t)c.B * (rank + 1) / world) - c.b0;
    if (c.Bl < 1) fail(GFNX_ERR_CONFIG, "batch_size smaller than world size");
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    cuda_check(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking), "stream");
    for (auto& e : c.ev) cuda_check(cudaEventCreate(&e), "event");
    // env tables
    EnvParams& P = c.P;
    P.kind = env->kind;
    P.A = c.shape.num_actions;
    P.Ab = c.shape.num_backward_actions;
    P.O = c.shape.obs_dim;
    P.T = c.shape.max_traj_len;
    P.stop = c.shape.stop_action;
    P.SW = c.shape.state_words;
    P.mdb = train->objective == GFNX_OBJ_MDB;
    P.hg_dim = env->hg_dim;
    P.hg_side = env->hg_side;
    memcpy(P.hg_f1, he.hg_f1, sizeof P.hg_f1);
    memcpy(P.hg_f2, he.hg_f2, sizeof P.hg_f2);
    memcpy(P.hg_logr, he.hg_logr, sizeof P.hg_logr);
    P.bs_slots = he.bs_slots;
    P.bs_vocab = he.bs_vocab;
    P.bs_k = env->bs_k;
    P.bs_nbits = env->bs_n_bits;
    P.bs_words = he.mode_words;
    P.n_modes = he.n_modes;
    P.bs_ar = env->kind == GFNX_ENV_BITSEQ && env->bs_scheme == 1;
    P.is_D = he.is_D;
    P.dag_d = env->dag_d;
    auto up = [&](auto** dst, const auto& vec) {
      using T = typename std::decay_t<decltype(vec)>::value_type;
      if (vec.empty()) return;
      cuda_check(cudaMalloc((void**)dst, sizeof(T) * vec.size()), "table alloc");
      cuda_check(cudaMemcpy(*dst, vec.data(), sizeof(T) * vec.size(), cudaMemcpyHostToDevice), "table");
    };
    up(&c.d_modes, he.modes);
    up(&c.d_bs_logr, he.bs_logr);
    up(&c.d_is_nbr, he.is_nbr);
    up(&c.d_is_J, he.is_J);
    up(&c.d_dag_cache, he.dag_cache);
    up(&c.d_neglog, he.neglog);
    c.h_dag_cache = he.dag_cache;
    c.h_is_nbr = he.is_nbr;
    c.h_is_J = he.is_J;
    P.modes = c.d_modes;
    P.bs_logr = c.d_bs_logr;
    P.is_nbr = c.d_is_nbr;
    P.is_J = c.d_is_J;
    P.dag_cache = c.d_dag_cache;
    P.neglog = c.d_neglog;
    // batch (the lockstep paths lay out whole 128-trajectory tiles: pad rows past Bl)
    const bool lockstep_env = env->kind == GFNX_ENV_BITSEQ || env->kind == GFNX_ENV_ISING;
    c.Bcap = (lockstep_env && train->precision != GFNX_PREC_FP64_CHECK) ? (c.Bl + 127) / 128 * 128 : c.Bl;
    const int T = P.T, Bl = c.Bcap;
    DeviceBatch& bt = c.batch;
    cuda_check(cudaMalloc(&bt.lengths, sizeof(int32_t) * Bl), "batch");
    cuda_check(cudaMalloc(&bt.actions, sizeof(int16_t) * (size_t)Bl * T), "batch");
    cuda_check(cudaMalloc(&bt.log_rewards, sizeof(double) * Bl), "batch");
    cuda_check(cudaMalloc(&bt.delta, sizeof(double) * (size_t)Bl * T), "batch");
    cuda_check(cudaMemset(bt.delta, 0, sizeof(double) * (size_t)Bl * T), "batch");
    cuda_check(cudaMalloc(&bt.nparents, sizeof(uint16_t) * (size_t)Bl * T), "batch");
    cuda_check(cudaMalloc(&bt.term_state, sizeof(uint32_t) * (size_t)Bl * P.SW), "batch");
    cuda_check(cudaMalloc(&bt.row0, sizeof(int32_t) * (Bl + 1)), "batch");
    cuda_check(cudaMalloc(&bt.row_bt, sizeof(int32_t) * ((size_t)Bl * T + 1)), "batch");
    cuda_check(cudaMalloc(&bt.scan_part, sizeof(int32_t) * 2 * ((Bl + 1023) / 1024 + 1)), "batch");
    cuda_check(cudaMalloc(&bt.counters, sizeof(int32_t) * 16), "batch");
    cuda_check(cudaMemset(bt.counters, 0, sizeof(int32_t) * 16), "batch");
    // parameters
    std::vector<double> p0;
    init_params(c.train, c.Lx, P.A, P.Ab, &p0);  // the reference's mlp_init at the user's widths
    p0 = to_device_layout(c, p0.data());
    const int64_t n = c.L.n_params;
    cuda_check(cudaMalloc(&c.d_scalars, sizeof(double) * 8), "scalars");
    std::vector<double> sc(8, 0.0);
    sc[0] = train->logz_init;
    cuda_check(cudaMemcpy(c.d_scalars, sc.data(), sizeof(double) * 8, cudaMemcpyHostToDevice), "scalars");
    cuda_check(cudaMalloc(&c.d_steps, sizeof(int64_t) * 4), "steps");
    cuda_check(cudaMemset(c.d_steps, 0, sizeof(int64_t) * 4), "steps");
    if (c.check_mode()) {
      cuda_check(cudaMalloc(&c.p64, sizeof(double) * n), "params");
      cuda_check(cudaMalloc(&c.g64, sizeof(double) * (n + 2)), "grads");
      cuda_check(cudaMalloc(&c.m64, sizeof(double) * n), "adam");
      cuda_check(cudaMalloc(&c.v64, sizeof(double) * n), "adam");
      cuda_check(cudaMemcpy(c.p64, p0.data(), sizeof(double) * n, cudaMemcpyHostToDevice), "params");
      cuda_check(cudaMemset(c.g64, 0, sizeof(double) * (n + 2)), "grads");
      cuda_check(cudaMemset(c.m64, 0, sizeof(double) * n), "adam");
      cuda_check(cudaMemset(c.v64, 0, sizeof(double) * n), "adam");
    } else {
      std::vector<float> pf(p0.begin(), p0.end());
      cuda_check(cudaMalloc(&c.p32, sizeof(float) * n), "params");
      cuda_check(cudaMalloc(&c.g32, sizeof(float) * (n + 2)), "grads");
      cuda_check(cudaMalloc(&c.m32, sizeof(float) * n), "adam");
      cuda_check(cudaMalloc(&c.v32, sizeof(float) * n), "adam");
      cuda_check(cudaMemcpy(c.p32, pf.data(), sizeof(float) * n, cudaMemcpyHostToDevice), "params");
      cuda_check(cudaMemset(c.g32, 0, sizeof(float) * (n + 2)), "grads");
      cuda_check(cudaMemset(c.m32, 0, sizeof(float) * n), "adam");
      cuda_check(cudaMemset(c.v32, 0, sizeof(float) * n), "adam");
      fast_init(c);
    }
    if (group) {
      if (group_world(group) != world) fail(GFNX_ERR_CONFIG, "group world differs from the ctx world");
      group_join(c, group, rank);
      c.group = group;
    } else if (world > 1) {
      NcclApi& api = nccl_api();
      if (!api.ok) fail(GFNX_ERR_NCCL, "libnccl.so.2 not found");
      if (!nccl_id) fail(GFNX_ERR_CONFIG, "world > 1 needs an NCCL unique id");
      ncclUniqueId id;
      memcpy(&id, nccl_id, sizeof id);
      ncclComm_t comm;
      const ncclResult_t r = api.CommInitRank(&comm, world, id, rank);
      if (r != ncclSuccess) fail(GFNX_ERR_NCCL, std::string("ncclCommInitRank: ") + api.GetErrorString(r));
      c.nccl = comm;
    }
    cuda_check(cudaDeviceSynchronize(), "create");
  });
  if (st != GFNX_OK) {
    gfnx_destroy(h);
    return st;
  }
  *out = h;
  return GFNX_OK;
}
}  // namespace

gfnx_status gfnx_create(const gfnx_env_desc* env, const gfnx_train_desc* train, int32_t device,
                        int32_t rank, int32_t world, const void* nccl_id, gfnx_ctx** out) {
  return create_impl(env, train, device, rank, world, nccl_id, nullptr, out);
}

gfnx_status gfnx_group_create(int32_t world, gfnx_group** out) {
  *out = nullptr;
  return guard(nullptr, [&] { *out = reinterpret_cast<gfnx_group*>(group_new(world)); });
}

gfnx_status gfnx_group_destroy(gfnx_group* g) {
  return guard(nullptr, [&] { group_delete(reinterpret_cast<Group*>(g)); });
}

gfnx_status gfnx_create_in_group(const gfnx_env_desc* env, const gfnx_train_desc* train, int32_t device,
                                 int32_t rank, gfnx_group* group, gfnx_ctx** out) {
  if (!group) return GFNX_ERR_CONFIG;
  Group* g = reinterpret_cast<Group*>(group);
  return create_impl(env, train, device, rank, group_world(g), nullptr, g, out);
}

void gfnx_destroy(gfnx_ctx* h) {
  if (!h) return;
  Ctx& c = h->c;
  if (c.stream) cudaStreamSynchronize(c.stream);
  if (c.nccl) nccl_api().CommDestroy((ncclComm_t)c.nccl);
  if (c.group) group_leave(c, c.group, c.rank);
  reward_free(c);
  eb_free(c);
  if (c.fast) fast_free(c);
  hg_buffer_free(c);
  if (c.phase) cudaFree(c.phase);
  void* ptrs[] = {c.d_modes, c.d_bs_logr, c.d_is_nbr, c.d_is_J, c.d_dag_cache, c.d_neglog,
                  c.p64, c.g64, c.m64, c.v64, c.p32, c.g32, c.m32, c.v32, c.d_scalars, c.d_steps,
                  c.batch.lengths, c.batch.actions, c.batch.log_rewards, c.batch.delta,
                  c.batch.nparents, c.batch.term_state, c.batch.row0, c.batch.counters,
                  c.batch.row_bt, c.batch.scan_part,
                  c.ck_obs, c.ck_act, c.ck_logp, c.ck_mask, c.ck_flow, c.ck_glogp, c.ck_gflow,
                  c.ck_bobs, c.ck_bact, c.ck_blogp, c.ck_bglogp, c.ck_bgx, c.ck_bgz, c.ck_bmask, c.ck_bidx,
                  c.ck_gz, c.ck_gx, c.ck_lampow, c.ck_gpair};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (auto& e : c.ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c.user_ev)
    if (e) cudaEventDestroy(e);
  for (auto& r : c.prof) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : c.ev_pool) cudaEventDestroy(e);
  if (c.copy_stream) cudaStreamSynchronize(c.copy_stream);
  for (auto& s : c.slots) {
    if (s.host) cudaFreeHost(s.host);
    if (s.dev) cudaFree(s.dev);
    if (s.done) cudaEventDestroy(s.done);
    if (s.staged) cudaEventDestroy(s.staged);
  }
  if (c.copy_stream) cudaStreamDestroy(c.copy_stream);
  if (c.comm_stream) {
    cudaStreamSynchronize(c.comm_stream);
    cudaStreamDestroy(c.comm_stream);
  }
  for (auto e : c.comm_ev)
    if (e) cudaEventDestroy(e);
  if (c.stream) cudaStreamDestroy(c.stream);
  delete h;
}

gfnx_status gfnx_num_params(const gfnx_ctx* h, int64_t* n) {
  *n = h->c.Lx.n_params;
  return GFNX_OK;
}

gfnx_status gfnx_set_params(gfnx_ctx* h, const double* flat, int64_t n, double log_z) {
  return guard(h, [&] {
    Ctx& c = h->c;
    if (n != c.Lx.n_params) fail(GFNX_ERR_CONFIG, "set_params: size mismatch");
    if (c.check_mode()) {
      cuda_check(cudaMemcpyAsync(c.p64, flat, sizeof(double) * n, cudaMemcpyHostToDevice, c.stream), "params");
    } else {
      const std::vector<double> d = to_device_layout(c, flat);
      std::vector<float> f(d.begin(), d.end());
      cuda_check(cudaMemcpyAsync(c.p32, f.data(), sizeof(float) * f.size(), cudaMemcpyHostToDevice, c.stream), "params");
      cuda_check(cudaStreamSynchronize(c.stream), "sync");
      fast_sync_weights(c);
    }
    cuda_check(cudaMemcpyAsync(c.d_scalars, &log_z, sizeof(double), cudaMemcpyHostToDevice, c.stream), "logz");
    cuda_check(cudaStreamSynchronize(c.stream), "sync");
  });
}

gfnx_status gfnx_get_params(gfnx_ctx* h, double* flat, int64_t n, double* log_z) {
  return guard(h, [&] {
    Ctx& c = h->c;
    if (n != c.Lx.n_params) fail(GFNX_ERR_CONFIG, "get_params: size mismatch");
    if (flat) {
      if (c.check_mode()) {
        cuda_check(cudaMemcpyAsync(flat, c.p64, sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream), "params");
      } else {
        std::vector<float> f(c.L.n_params);
        cuda_check(cudaMemcpyAsync(f.data(), c.p32, sizeof(float) * f.size(), cudaMemcpyDeviceToHost, c.stream), "params");
        cuda_check(cudaStreamSynchronize(c.stream), "sync");
        to_user_layout(c, f.data(), flat);
      }
    }
    if (log_z) cuda_check(cudaMemcpyAsync(log_z, c.d_scalars, sizeof(double), cudaMemcpyDeviceToHost, c.stream), "logz");
    cuda_check(cudaStreamSynchronize(c.stream), "sync");
  });
}

gfnx_status gfnx_set_adam_state(gfnx_ctx* h, const double* m, const double* v, int64_t t,
                                double z_m, double z_v, int64_t z_t) {
  return guard(h, [&] {
    Ctx& c = h->c;
    const int64_t n = c.L.n_params;
    // queued Adam kernels must not overwrite the restored state (the ctx stream is non-blocking)
    cuda_check(cudaStreamSynchronize(c.stream), "sync");
    if (c.check_mode()) {
      if (m) cuda_check(cudaMemcpy(c.m64, m, sizeof(double) * n, cudaMemcpyHostToDevice), "adam");
      if (v) cuda_check(cudaMemcpy(c.v64, v, sizeof(double) * n, cudaMemcpyHostToDevice), "adam");
    } else {
      auto put = [&](const double* x, float* dst) {
        if (!x) return;
        const std::vector<double> d = to_device_layout(c, x);
        std::vector<float> f(d.begin(), d.end());
        cuda_check(cudaMemcpy(dst, f.data(), sizeof(float) * n, cudaMemcpyHostToDevice), "adam");
      };
      put(m, c.m32);
      put(v, c.v32);
    }
    double zs[2] = {z_m, z_v};
    cuda_check(cudaMemcpy(c.d_scalars + 1, zs, sizeof zs, cudaMemcpyHostToDevice), "adam z");
    const int64_t steps[4] = {t, z_t, 0, 0};
    cuda_check(cudaMemcpy(c.d_steps, steps, sizeof steps, cudaMemcpyHostToDevice), "adam steps");
  });
}

gfnx_status gfnx_get_adam_state(gfnx_ctx* h, double* m, double* v, int64_t* t, double* z_m,
                                double* z_v, int64_t* z_t) {
  return guard(h, [&] {
    Ctx& c = h->c;
    cuda_check(cudaStreamSynchronize(c.stream), "sync");
    const int64_t n = c.L.n_params;
    auto get = [&](double* dst, const double* s64, const float* s32) {
      if (!dst) return;
      if (c.check_mode()) {
        cuda_check(cudaMemcpy(dst, s64, sizeof(double) * n, cudaMemcpyDeviceToHost), "adam");
      } else {
        std::vector<float> f(n);
        cuda_check(cudaMemcpy(f.data(), s32, sizeof(float) * n, cudaMemcpyDeviceToHost), "adam");
        to_user_layout(c, f.data(), dst);
      }
    };
    get(m, c.m64, c.m32);
    get(v, c.v64, c.v32);
    double zs[2];
    cuda_check(cudaMemcpy(zs, c.d_scalars + 1, sizeof zs, cudaMemcpyDeviceToHost), "adam z");
    if (z_m) *z_m = zs[0];
    if (z_v) *z_v = zs[1];
    int64_t steps[4];
    cuda_check(cudaMemcpy(steps, c.d_steps, sizeof steps, cudaMemcpyDeviceToHost), "adam steps");
    if (t) *t = steps[0];
    if (z_t) *z_t = steps[1];
  });
}

// ---------------------------------------------------------------------------
// GFNCKPT1 checkpoints (checkpoint.cpp:11-107): magic, trunk depth, every Dense as
// (rank, dims, fp64 values) for weight [in x out] and bias [out], fwd / bwd / flow heads,
// log_z [1], then the main Adam state (t, tensor count, m tensors, v tensors), the log_z
// Adam state and the step counter. Byte-compatible with the reference's save / load.
namespace {
constexpr char kCkptMagic[8] = {'G', 'F', 'N', 'C', 'K', 'P', 'T', '1'};

struct CkptTensor {
  std::vector<int64_t> shape;
  int64_t off, n;
};

std::vector<CkptTensor> ckpt_tensors(const Ctx& c) {  // MlpParams::tensors() order (nn.cpp:8-19)
  const MlpLayout& L = c.Lx;
  std::vector<CkptTensor> v;
  for (int l = 0; l < L.n_trunk; ++l) {
    v.push_back({{L.dims[l], L.dims[l + 1]}, L.off_w[l], (int64_t)L.dims[l] * L.dims[l + 1]});
    v.push_back({{L.dims[l + 1]}, L.off_b[l], L.dims[l + 1]});
  }
  const int64_t H = L.H(), A = c.shape.num_actions, Ab = c.shape.num_backward_actions;
  v.push_back({{H, A}, L.off_fw, H * A});
  v.push_back({{A}, L.off_fb, A});
  v.push_back({{H, Ab}, L.off_bw, H * Ab});
  v.push_back({{Ab}, L.off_bb, Ab});
  v.push_back({{H, 1}, L.off_flw, H});
  v.push_back({{1}, L.off_flb, 1});
  return v;
}

void put_i64(std::FILE* f, int64_t x) { std::fwrite(&x, 8, 1, f); }
int64_t get_i64(std::FILE* f) {
  int64_t x = 0;
  if (std::fread(&x, 8, 1, f) != 1) fail(GFNX_ERR_CONFIG, "checkpoint: truncated file");
  return x;
}
void put_tensor(std::FILE* f, const std::vector<int64_t>& shape, const double* x, int64_t n) {
  put_i64(f, (int64_t)shape.size());
  for (int64_t d : shape) put_i64(f, d);
  std::fwrite(x, sizeof(double), (size_t)n, f);
}
void get_tensor(std::FILE* f, const std::vector<int64_t>& shape, double* x, int64_t n) {
  const int64_t rank = get_i64(f);
  if (rank != (int64_t)shape.size()) fail(GFNX_ERR_CONFIG, "checkpoint: tensor rank does not match the model");
  for (int64_t d : shape)
    if (get_i64(f) != d) fail(GFNX_ERR_CONFIG, "checkpoint: tensor shape does not match the model");
  if (std::fread(x, sizeof(double), (size_t)n, f) != (size_t)n) fail(GFNX_ERR_CONFIG, "checkpoint: truncated tensor data");
}
}  // namespace

gfnx_status gfnx_save_checkpoint(gfnx_ctx* h, const char* path, int64_t step) {
  return guard(h, [&] {
    Ctx& c = h->c;
    const int64_t n = c.Lx.n_params;
    std::vector<double> p(n), m(n), v(n);
    double z = 0, zm = 0, zv = 0;
    int64_t t = 0, zt = 0;
    if (gfnx_get_params(h, p.data(), n, &z) != GFNX_OK) fail(GFNX_ERR_CUDA, c.err);
    if (gfnx_get_adam_state(h, m.data(), v.data(), &t, &zm, &zv, &zt) != GFNX_OK) fail(GFNX_ERR_CUDA, c.err);
    std::FILE* f = std::fopen(path, "wb");
    if (!f) fail(GFNX_ERR_CONFIG, std::string("checkpoint: cannot open for write: ") + path);
    const auto ts = ckpt_tensors(c);
    std::fwrite(kCkptMagic, 1, 8, f);
    put_i64(f, c.Lx.n_trunk);
    for (const auto& x : ts) put_tensor(f, x.shape, p.data() + x.off, x.n);
    put_tensor(f, {1}, &z, 1);
    put_i64(f, t);
    put_i64(f, (int64_t)ts.size());
    for (const auto& x : ts) put_tensor(f, x.shape, m.data() + x.off, x.n);
    for (const auto& x : ts) put_tensor(f, x.shape, v.data() + x.off, x.n);
    put_i64(f, zt);
    put_i64(f, 1);
    put_tensor(f, {1}, &zm, 1);
    put_tensor(f, {1}, &zv, 1);
    put_i64(f, step);
    const bool ok = std::ferror(f) == 0;
    std::fclose(f);
    if (!ok) fail(GFNX_ERR_CONFIG, std::string("checkpoint: write failed: ") + path);
  });
}

gfnx_status gfnx_load_checkpoint(gfnx_ctx* h, const char* path, int64_t* step) {
  return guard(h, [&] {
    Ctx& c = h->c;
    const int64_t n = c.Lx.n_params;
    std::vector<double> p(n), m(n), v(n);
    double z = 0, zm = 0, zv = 0;
    std::FILE* f = std::fopen(path, "rb");
    if (!f) fail(GFNX_ERR_CONFIG, std::string("checkpoint: cannot open: ") + path);
    struct Closer {
      std::FILE* f;
      ~Closer() { std::fclose(f); }
    } closer{f};
    char magic[8];
    if (std::fread(magic, 1, 8, f) != 8 || memcmp(magic, kCkptMagic, 8) != 0)
      fail(GFNX_ERR_CONFIG, std::string("checkpoint: bad magic in ") + path);
    if (get_i64(f) != c.Lx.n_trunk) fail(GFNX_ERR_CONFIG, "checkpoint: trunk depth does not match the model");
    const auto ts = ckpt_tensors(c);
    for (const auto& x : ts) get_tensor(f, x.shape, p.data() + x.off, x.n);
    get_tensor(f, {1}, &z, 1);
    const int64_t t = get_i64(f);
    if (get_i64(f) != (int64_t)ts.size()) fail(GFNX_ERR_CONFIG, "checkpoint: optimizer state does not match the model");
    for (const auto& x : ts) get_tensor(f, x.shape, m.data() + x.off, x.n);
    for (const auto& x : ts) get_tensor(f, x.shape, v.data() + x.off, x.n);
    const int64_t zt = get_i64(f);
    if (get_i64(f) != 1) fail(GFNX_ERR_CONFIG, "checkpoint: log_z optimizer state malformed");
    get_tensor(f, {1}, &zm, 1);
    get_tensor(f, {1}, &zv, 1);
    const int64_t st = get_i64(f);
    if (gfnx_set_params(h, p.data(), n, z) != GFNX_OK) fail(GFNX_ERR_CUDA, c.err);
    if (gfnx_set_adam_state(h, m.data(), v.data(), t, zm, zv, zt) != GFNX_OK) fail(GFNX_ERR_CUDA, c.err);
    if (step) *step = st;
  });
}

gfnx_status gfnx_exact_terminal_marginal(gfnx_ctx* h, double* marginal, int64_t n, double* tv) {
  return guard(h, [&] {
    Ctx& c = h->c;
    if (c.check_mode()) fail(GFNX_ERR_CONFIG, "exact terminal marginal: bf16 fast path only");
    std::vector<double> pt;
    fast_hg_marginal(c, &pt);
    if (marginal) {
      if (n != (int64_t)pt.size()) fail(GFNX_ERR_CONFIG, "exact terminal marginal: wrong buffer size");
      memcpy(marginal, pt.data(), sizeof(double) * pt.size());
    }
    if (tv) {  // against R / Z over all cells (grid_exact_distribution, hypergrid.cpp:111-119)
      const int d = c.env.hg_dim, side = c.env.hg_side;
      std::vector<double> r(pt.size());
      double zsum = 0.0;
      for (size_t x = 0; x < pt.size(); ++x) {
        int64_t y = (int64_t)x;
        bool p1 = true, p2 = true;
        for (int i = 0; i < d; ++i) {
          const double a = fabs((double)(y % side) / (double)(side - 1) - 0.5);
          y /= side;
          p1 = p1 && 0.25 < a;
          p2 = p2 && 0.3 < a && a < 0.4;
        }
        r[x] = c.env.hg_r0 + (p1 ? c.env.hg_r1 : 0.0) + (p2 ? c.env.hg_r2 : 0.0);
        zsum += r[x];
      }
      double s = 0.0;
      for (size_t x = 0; x < pt.size(); ++x) s += fabs(pt[x] - r[x] / zsum);
      *tv = 0.5 * s;
    }
  });
}

gfnx_status gfnx_mc_terminal_logprob(gfnx_ctx* h, const uint32_t* terminals, int64_t n, int32_t num_samples,
                                     const uint64_t* keys, double* out) {
  return guard(h, [&] {
    Ctx& c = h->c;
    if (!terminals || !keys || !out) fail(GFNX_ERR_CONFIG, "mc terminal log-prob: null buffer");
    if (n < 1 || num_samples < 1) fail(GFNX_ERR_CONFIG, "mc terminal log-prob: empty batch");
    uint32_t* d_t = nullptr;
    uint64_t* d_k = nullptr;
    double* d_o = nullptr;
    cuda_check(cudaMallocAsync(&d_t, sizeof(uint32_t) * n * c.P.SW, c.stream), "mc");
    cuda_check(cudaMallocAsync(&d_k, sizeof(uint64_t) * 2 * n, c.stream), "mc");
    cuda_check(cudaMallocAsync(&d_o, sizeof(double) * n, c.stream), "mc");
    cuda_check(cudaMemcpyAsync(d_t, terminals, sizeof(uint32_t) * n * c.P.SW, cudaMemcpyHostToDevice, c.stream), "mc");
    cuda_check(cudaMemcpyAsync(d_k, keys, sizeof(uint64_t) * 2 * n, cudaMemcpyHostToDevice, c.stream), "mc");
    const bool rows_path = !c.check_mode() && (c.env.kind == GFNX_ENV_HYPERGRID || c.env.kind == GFNX_ENV_DAG);
    if (rows_path) fast_mc_terminal_logprob(c, d_t, n, num_samples, d_k, d_o);
    else mc_terminal_logprob_chunked(c, d_t, n, num_samples, d_k, d_o);
    cuda_check(cudaMemcpyAsync(out, d_o, sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream), "mc");
    for (void* p : {(void*)d_t, (void*)d_k, (void*)d_o}) cudaFreeAsync(p, c.stream);
    check_device_error(c);
  });
}

gfnx_status gfnx_pearson(gfnx_ctx* h, int64_t step, int32_t mc_samples, uint64_t test_seed, double* out) {
  return guard(h, [&] {
    Ctx& c = h->c;
    if (!out) fail(GFNX_ERR_CONFIG, "pearson: null buffer");
    if (mc_samples < 1) fail(GFNX_ERR_CONFIG, "pearson: mc_samples must be >= 1");
    double* d = nullptr;
    cuda_check(cudaMallocAsync(&d, sizeof(double), c.stream), "pearson");
    bitseq_pearson(c, step, mc_samples, test_seed, d);
    cuda_check(cudaMemcpyAsync(out, d, sizeof(double), cudaMemcpyDeviceToHost, c.stream), "pearson");
    cudaFreeAsync(d, c.stream);
    check_device_error(c);
  });
}

gfnx_status gfnx_eb_default_desc(gfnx_eb_desc* out) {
  if (!out) return GFNX_ERR_CONFIG;
  eb_default_desc(out);
  return GFNX_OK;
}

gfnx_status gfnx_ising_gibbs_data(int32_t side, double sigma, uint64_t seed, const gfnx_eb_desc* desc,
                                  int8_t* out, int64_t n) {
  return guard(nullptr, [&] {
    if (!desc || !out) fail(GFNX_ERR_CONFIG, "gibbs: null buffer");
    if (side < 2) fail(GFNX_ERR_CONFIG, "ising: lattice side must be >= 2");
    if (desc->gibbs_chains < 1) fail(GFNX_ERR_CONFIG, "gibbs: need at least one chain");
    if (desc->gibbs_thinning < 1 || n < 0) fail(GFNX_ERR_CONFIG, "gibbs: bad sample counts");
    const int D = side * side;
    const auto d = ising_gibbs_data(ising_dense_coupling(side, sigma), D, fold_in(make_key(seed), 0x919B), n,
                                    desc->gibbs_burn_in, desc->gibbs_thinning, desc->gibbs_chains,
                                    desc->gibbs_hottest_beta);
    std::copy(d.begin(), d.end(), out);
  });
}

gfnx_status gfnx_eb_init(gfnx_ctx* h, const gfnx_eb_desc* desc, const int8_t* data, int64_t n) {
  return guard(h, [&] {
    if (!desc) fail(GFNX_ERR_CONFIG, "eb-gfn: null desc");
    cuda_check(cudaStreamSynchronize(h->c.stream), "sync");
    eb_init(h->c, *desc, data, n);
    h->c.has_batch = false;
    h->c.has_grads = false;
  });
}

// run_eb_gfn's loop body (train.cpp:940-1003): the sampler update on the mixed batch
// (forward rollout of the on-policy rows + backward_rollout of the data rows, one device
// rollout with teacher-forced rows), then the energy-model update
gfnx_status gfnx_eb_run(gfnx_ctx* h, int64_t it0, int64_t n, double* out) {
  return guard(h, [&] {
    Ctx& c = h->c;
    if (n < 0) fail(GFNX_ERR_CONFIG, "eb-gfn: negative iteration count");
    eb_ensure_metrics(c, std::max<int64_t>(n, 1));
    const Key root = make_key(c.train.seed);
    for (int64_t i = 0; i < n; ++i) {
      const int64_t it = it0 + i;
      const Key it_key = fold_in(root, 1000 + (uint64_t)it);
      const double eps = schedule_value(c.train.explore, it);
      const double lr = schedule_value(c.train.lr, it);
      const int16_t* forced = eb_pre(c, it_key);
      if (c.check_mode()) check_rollout(c, fold_in(it_key, 3), eps, forced);
      else ls_rollout(c, fold_in(it_key, 3), eps, forced);
      finish_forced(c);
      do_train(c, true, lr, nullptr);
      eb_post(c, it_key, eb_coupling_lr(c, it), i);
    }
    if (out && n > 0)
      cuda_check(cudaMemcpyAsync(out, eb_metrics(c), sizeof(double) * 4 * n, cudaMemcpyDeviceToHost, c.stream),
                 "eb metrics");
    check_device_error(c);
  });
}

gfnx_status gfnx_eb_coupling(gfnx_ctx* h, double* j_model, double* j_true, int64_t n, double* init_nlr) {
  return guard(h, [&] {
    Ctx& c = h->c;
    if ((j_model || j_true) && n != (int64_t)c.P.is_D * c.P.is_D) fail(GFNX_ERR_CONFIG, "eb coupling: n must be D*D");
    eb_coupling(c, j_model, j_true, init_nlr);
  });
}

gfnx_status gfnx_eb_dataset(gfnx_ctx* h, int8_t* out, int64_t n) {
  return guard(h, [&] { eb_dataset(h->c, out, n); });
}

gfnx_status gfnx_backward_rollout(gfnx_ctx* h, const uint32_t* terminals, int64_t n, uint64_t key_hi,
                                  uint64_t key_lo) {
  return guard(h, [&] {
    Ctx& c = h->c;
    if (!terminals) fail(GFNX_ERR_CONFIG, "backward_rollout: null buffer");
    if (n != c.Bl) fail(GFNX_ERR_CONFIG, "backward_rollout: n must equal the local batch (gfnx_batch_dims)");
    uint32_t* d_t = nullptr;
    cuda_check(cudaMallocAsync(&d_t, sizeof(uint32_t) * n * c.P.SW, c.stream), "backward rollout");
    cuda_check(cudaMemcpyAsync(d_t, terminals, sizeof(uint32_t) * n * c.P.SW, cudaMemcpyHostToDevice, c.stream),
               "backward rollout");
    backward_rollout(c, d_t, Key{key_hi, key_lo});
    cudaFreeAsync(d_t, c.stream);
    finish_forced(c);
    check_device_error(c);
  });
}

gfnx_status gfnx_rollout_from_actions(gfnx_ctx* h, const int32_t* actions, int64_t n) {
  return guard(h, [&] {
    Ctx& c = h->c;
    const int64_t nt = (int64_t)c.Bl * c.P.T;
    if (!actions) fail(GFNX_ERR_CONFIG, "rollout_from_actions: null buffer");
    if (n != nt) fail(GFNX_ERR_CONFIG, "rollout_from_actions: size must be local_batch * max_traj_len");
    std::vector<int16_t> a16(nt);
    for (int64_t i = 0; i < nt; ++i) {
      if (actions[i] < -1 || actions[i] >= c.P.A) fail(GFNX_ERR_CONTRACT, "rollout_from_actions: action out of range");
      if (i % c.P.T == 0 && actions[i] < 0) fail(GFNX_ERR_CONTRACT, "rollout_from_actions: empty trajectory");
      a16[i] = (int16_t)actions[i];
    }
    int16_t* d_a = nullptr;
    cuda_check(cudaMallocAsync(&d_a, sizeof(int16_t) * nt, c.stream), "rollout_from_actions");
    cuda_check(cudaMemcpyAsync(d_a, a16.data(), sizeof(int16_t) * nt, cudaMemcpyHostToDevice, c.stream),
               "rollout_from_actions");
    forced_rollout(c, d_a);
    cudaFreeAsync(d_a, c.stream);
    finish_forced(c);
    check_device_error(c);
  });
}

gfnx_status gfnx_buffer_reset(gfnx_ctx* h, int64_t capacity) {
  return guard(h, [&] { hg_buffer_reset(h->c, capacity); });
}

gfnx_status gfnx_buffer_push(gfnx_ctx* h) {
  return guard(h, [&] { hg_buffer_push(h->c); });
}

gfnx_status gfnx_tv_buffer(gfnx_ctx* h, int64_t* size, double* tv) {
  return guard(h, [&] {
    const double v = hg_buffer_tv(h->c);
    if (size) *size = h->c.tbuf.size;
    if (tv) *tv = v;
  });
}

gfnx_status gfnx_rollout(gfnx_ctx* h, int64_t it, double eps) {
  return guard(h, [&] {
    do_rollout(h->c, it, eps);
    check_device_error(h->c);
  });
}

gfnx_status gfnx_train_step(gfnx_ctx* h, double lr, double* loss) {
  return guard(h, [&] { do_train(h->c, true, lr, loss); });
}

gfnx_status gfnx_compute_grads(gfnx_ctx* h, double* loss) {
  return guard(h, [&] {
    double l = 0.0;
    do_train(h->c, false, 0.0, &l);
    if (loss) *loss = l;
  });
}

gfnx_status gfnx_get_grads(gfnx_ctx* h, double* flat, int64_t n, double* d_log_z) {
  return guard(h, [&] {
    Ctx& c = h->c;
    if (n != c.Lx.n_params) fail(GFNX_ERR_CONFIG, "get_grads: size mismatch");
    if (!c.has_grads) fail(GFNX_ERR_CONTRACT, "get_grads: no gradients computed");
    cuda_check(cudaStreamSynchronize(c.stream), "sync");
    if (flat) {
      if (c.check_mode()) {
        cuda_check(cudaMemcpy(flat, c.g64, sizeof(double) * n, cudaMemcpyDeviceToHost), "grads");
      } else {
        std::vector<float> f(c.L.n_params);
        cuda_check(cudaMemcpy(f.data(), c.g32, sizeof(float) * f.size(), cudaMemcpyDeviceToHost), "grads");
        to_user_layout(c, f.data(), flat);
      }
    }
    if (d_log_z) cuda_check(cudaMemcpy(d_log_z, c.d_scalars + 3, sizeof(double), cudaMemcpyDeviceToHost), "dlogz");
  });
}

gfnx_status gfnx_export_row_logpf(gfnx_ctx* h, double* out, int64_t n) {
  return guard(h, [&] {
    Ctx& c = h->c;
    if (n != (int64_t)c.Bl * c.P.T) fail(GFNX_ERR_CONFIG, "export_row_logpf: size mismatch (local_batch * max_len)");
    if (!c.has_batch || !c.has_grads) fail(GFNX_ERR_CONTRACT, "export_row_logpf: no training pass on the resident batch");
    double* d = nullptr;
    cuda_check(cudaMallocAsync(&d, sizeof(double) * n, c.stream), "row logpf");
    if (c.check_mode()) {
      ensure_row0(c);
      check_row_logpf(c, d);
    } else {
      fast_row_logpf(c, d);
    }
    cuda_check(cudaMemcpyAsync(out, d, sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream), "row logpf");
    cuda_check(cudaFreeAsync(d, c.stream), "row logpf");
    cuda_check(cudaStreamSynchronize(c.stream), "row logpf");
  });
}

gfnx_status gfnx_debug_buffer(gfnx_ctx* h, const char* name, void* out, int64_t cap, int64_t* bytes) {
  return guard(h, [&] {
    Ctx& c = h->c;
    const void* p = nullptr;
    size_t n = 0;
    const bool lock = !c.check_mode() && (c.env.kind == GFNX_ENV_BITSEQ || c.env.kind == GFNX_ENV_ISING);
    if (!lock || !ls_debug_buffer(c, name, &p, &n)) fail(GFNX_ERR_CONFIG, std::string("debug_buffer: unknown buffer ") + name);
    if (bytes) *bytes = (int64_t)n;
    if (out) {
      if (cap < (int64_t)n) fail(GFNX_ERR_CONFIG, "debug_buffer: buffer too small");
      cuda_check(cudaStreamSynchronize(c.stream), "sync");
      cuda_check(cudaMemcpy(out, p, n, cudaMemcpyDeviceToHost), "debug_buffer");
    }
  });
}

gfnx_status gfnx_log_rewards_device(gfnx_ctx* h, const uint32_t* states_soa, int64_t n, double* out) {
  return guard(h, [&] {
    if (n < 0) fail(GFNX_ERR_CONFIG, "log_rewards: negative count");
    reward_soa(h->c, states_soa, n, out);
  });
}

gfnx_status gfnx_log_rewards(gfnx_ctx* h, const uint32_t* states, int64_t n, double* out) {
  return guard(h, [&] {
    Ctx& c = h->c;
    if (n < 0) fail(GFNX_ERR_CONFIG, "log_rewards: negative count");
    if (n == 0) return;
    const int SW = c.P.SW;
    std::vector<uint32_t> soa((size_t)SW * n);
    for (int64_t i = 0; i < n; ++i)
      for (int k = 0; k < SW; ++k) soa[(size_t)k * n + i] = states[(size_t)i * SW + k];
    uint32_t* d_st = nullptr;
    double* d_out = nullptr;
    cuda_check(cudaMallocAsync(&d_st, sizeof(uint32_t) * soa.size(), c.stream), "log_rewards");
    cuda_check(cudaMallocAsync(&d_out, sizeof(double) * n, c.stream), "log_rewards");
    cuda_check(cudaMemcpyAsync(d_st, soa.data(), sizeof(uint32_t) * soa.size(), cudaMemcpyHostToDevice, c.stream),
               "log_rewards");
    reward_soa(c, d_st, n, d_out);
    cuda_check(cudaMemcpyAsync(out, d_out, sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream), "log_rewards");
    cudaFreeAsync(d_st, c.stream);
    cudaFreeAsync(d_out, c.stream);
    check_device_error(c);
  });
}

gfnx_status gfnx_iteration(gfnx_ctx* h, int64_t it, double* loss) {
  return guard(h, [&] {
    Ctx& c = h->c;
    const double lr = schedule_value(c.train.lr, it);       // train.cpp:225
    const double eps = schedule_value(c.train.explore, it); // train.cpp:226
    do_rollout(c, it, eps);
    do_train(c, true, lr, loss);
    if (!loss) check_device_error(c);  // a failed batch is reported by this call, not a later one
  });
}

gfnx_status gfnx_run(gfnx_ctx* h, int64_t it0, int64_t n, double* losses) {
  return guard(h, [&] {
    Ctx& c = h->c;
    for (int64_t i = 0; i < n; ++i) {
      const int64_t it = it0 + i;
      do_rollout(c, it, schedule_value(c.train.explore, it));
      do_train(c, true, schedule_value(c.train.lr, it), losses ? losses + i : nullptr);
    }
    check_device_error(c);
  });
}

namespace {
size_t slot_bytes(const Ctx& c) {
  return 16 + sizeof(int32_t) * c.Bl + sizeof(double) * c.Bl + sizeof(uint32_t) * (size_t)c.Bl * c.P.SW;
}

}  // namespace

namespace gfnx {
// one launch gathers an iteration's results into the slot's device staging buffer (the
// layout of the pinned host slot), so the next iteration may overwrite the batch while the
// device->host copy runs on the copy stream
__global__ void k_slot_stage(uint32_t* __restrict__ dst, const double* __restrict__ loss,
                             const int32_t* __restrict__ err, const int32_t* __restrict__ len,
                             const double* __restrict__ logr, const uint32_t* __restrict__ term, int Bl, int SW) {
  const size_t n1 = (size_t)Bl, n2 = 2 * (size_t)Bl, n3 = (size_t)Bl * SW, total = 4 + n1 + n2 + n3;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t v;
    if (i < 2) v = reinterpret_cast<const uint32_t*>(loss)[i];
    else if (i == 2) v = (uint32_t)*err;
    else if (i == 3) v = 0u;
    else if (i < 4 + n1) v = (uint32_t)len[i - 4];
    else if (i < 4 + n1 + n2) v = reinterpret_cast<const uint32_t*>(logr)[i - 4 - n1];
    else v = term[i - 4 - n1 - n2];
    dst[i] = v;
  }
}
}  // namespace gfnx

gfnx_status gfnx_iteration_async(gfnx_ctx* h, int64_t it, int32_t slot) {
  return guard(h, [&] {
    Ctx& c = h->c;
    if (slot < 0 || slot > 1) fail(GFNX_ERR_CONFIG, "slot must be 0 or 1");
    Ctx::Slot& s = c.slots[slot];
    const size_t nb = slot_bytes(c);
    if (!s.host) {
      cuda_check(cudaHostAlloc((void**)&s.host, nb, cudaHostAllocDefault), "pinned slot");
      cuda_check(cudaMalloc(&s.dev, nb), "slot staging");
      cuda_check(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming), "slot event");
      cuda_check(cudaEventCreateWithFlags(&s.staged, cudaEventDisableTiming), "slot event");
    }
    if (!c.copy_stream) cuda_check(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking), "copy stream");
    do_rollout(c, it, schedule_value(c.train.explore, it));
    do_train(c, true, schedule_value(c.train.lr, it), nullptr);
    // the staging buffer of this slot is free once its previous device->host copy is done
    if (s.it >= 0) cuda_check(cudaStreamWaitEvent(c.stream, s.done, 0), "slot reuse");
    const size_t words = nb / 4;
    k_slot_stage<<<(unsigned)std::min<size_t>((words + 255) / 256, 4 * 148), 256, 0, c.stream>>>(
        reinterpret_cast<uint32_t*>(s.dev), c.d_scalars + 4, c.batch.counters + 3, c.batch.lengths,
        c.batch.log_rewards, c.batch.term_state, c.Bl, c.P.SW);
    c.launches++;
    cuda_check(cudaEventRecord(s.staged, c.stream), "slot record");
    cuda_check(cudaStreamWaitEvent(c.copy_stream, s.staged, 0), "slot copy");
    cuda_check(cudaMemcpyAsync(s.host, s.dev, nb, cudaMemcpyDeviceToHost, c.copy_stream), "slot copy");
    cuda_check(cudaEventRecord(s.done, c.copy_stream), "slot record");
    s.it = it;
  });
}

gfnx_status gfnx_slot_wait(gfnx_ctx* h, int32_t slot, gfnx_slot_view* out) {
  return guard(h, [&] {
    Ctx& c = h->c;
    if (slot < 0 || slot > 1 || !c.slots[slot].host) fail(GFNX_ERR_CONFIG, "slot not in use");
    Ctx::Slot& s = c.slots[slot];
    cuda_check(cudaEventSynchronize(s.done), "slot wait");
    int32_t err = 0;
    memcpy(&err, s.host + 8, sizeof err);
    if (err != 0) {
      cudaMemsetAsync(c.batch.counters + 3, 0, sizeof(int32_t), c.stream);
      fail((gfnx_status)err, "device error in iteration " + std::to_string(s.it));
    }
    uint8_t* p = s.host;
    out->it = s.it;
    memcpy(&out->loss, p, sizeof(double));
    out->n = c.Bl;
    out->state_words = c.P.SW;
    p += 16;
    out->lengths = reinterpret_cast<const int32_t*>(p);
    p += sizeof(int32_t) * c.Bl;
    out->log_rewards = reinterpret_cast<const double*>(p);
    p += sizeof(double) * c.Bl;
    out->terminal_state = reinterpret_cast<const uint32_t*>(p);
  });
}

gfnx_status gfnx_synchronize(gfnx_ctx* h) {
  return guard(h, [&] {
    cuda_check(cudaStreamSynchronize(h->c.stream), "sync");
    check_device_error(h->c);
  });
}

gfnx_status gfnx_batch_dims(const gfnx_ctx* h, int32_t* local_batch, int32_t* first_traj,
                            int32_t* max_len, int32_t* state_words) {
  if (local_batch) *local_batch = h->c.Bl;
  if (first_traj) *first_traj = h->c.b0;
  if (max_len) *max_len = h->c.P.T;
  if (state_words) *state_words = h->c.P.SW;
  return GFNX_OK;
}

gfnx_status gfnx_export_batch(gfnx_ctx* h, gfnx_host_batch* out) {
  return guard(h, [&] {
    Ctx& c = h->c;
    if (!c.has_batch) fail(GFNX_ERR_CONTRACT, "export_batch: no resident batch");
    cuda_check(cudaStreamSynchronize(c.stream), "sync");
    const int Bl = c.Bl, T = c.P.T;
    const size_t bt = (size_t)Bl * T;
    // steps t >= L_b are padding (actions -1, log P_B and delta 0): the device does not keep
    // them, the export derives them from the lengths
    std::vector<int32_t> len(Bl);
    cuda_check(cudaMemcpy(len.data(), c.batch.lengths, sizeof(int32_t) * Bl, cudaMemcpyDeviceToHost), "export");
    if (out->lengths) memcpy(out->lengths, len.data(), sizeof(int32_t) * Bl);
    if (out->log_rewards) cuda_check(cudaMemcpy(out->log_rewards, c.batch.log_rewards, sizeof(double) * Bl, cudaMemcpyDeviceToHost), "export");
    if (out->delta_log_reward) {
      cuda_check(cudaMemcpy(out->delta_log_reward, c.batch.delta, sizeof(double) * bt, cudaMemcpyDeviceToHost), "export");
      for (int b = 0; b < Bl; ++b)  // delta is defined for non-terminal steps t < L - 1
        for (int t = std::max(len[b] - 1, 0); t < T; ++t) out->delta_log_reward[(size_t)b * T + t] = 0.0;
    }
    if (out->terminal_state) cuda_check(cudaMemcpy(out->terminal_state, c.batch.term_state, sizeof(uint32_t) * Bl * c.P.SW, cudaMemcpyDeviceToHost), "export");
    if (!out->fwd_actions && !out->bwd_actions && !out->log_pb) return;
    std::vector<int16_t> a(bt);
    std::vector<uint16_t> np(bt);
    cuda_check(cudaMemcpy(a.data(), c.batch.actions, sizeof(int16_t) * bt, cudaMemcpyDeviceToHost), "export");
    cuda_check(cudaMemcpy(np.data(), c.batch.nparents, sizeof(uint16_t) * bt, cudaMemcpyDeviceToHost), "export");
    HostEnv he;
    build_host_env(c.env, &he);
    for (size_t i = 0; i < bt; ++i) {
      const int act = (int)(i % T) < len[i / T] ? a[i] : -1;
      if (out->fwd_actions) out->fwd_actions[i] = act;
      if (out->bwd_actions) {
        int ba = -1;
        if (act >= 0) {
          switch (c.env.kind) {  // get_backward_action of each env
            case GFNX_ENV_BITSEQ: ba = act / c.P.bs_vocab; break;
            case GFNX_ENV_ISING: ba = act / 2; break;
            default: ba = act;
          }
        }
        out->bwd_actions[i] = ba;
      }
      if (out->log_pb) out->log_pb[i] = act >= 0 ? he.neglog[np[i]] : 0.0;
    }
  });
}

int64_t gfnx_kernel_launches(const gfnx_ctx* h) { return h->c.launches; }

gfnx_status gfnx_last_phase_ms(const gfnx_ctx* h, double* rollout_ms, double* train_ms) {
  return guard(const_cast<gfnx_ctx*>(h), [&] {
    const Ctx& c = h->c;
    cuda_check(cudaEventSynchronize(c.ev[2]), "event");
    float a = 0.f, b = 0.f;
    cuda_check(cudaEventElapsedTime(&a, c.ev[0], c.ev[1]), "event");
    cuda_check(cudaEventElapsedTime(&b, c.ev[1], c.ev[2]), "event");
    if (rollout_ms) *rollout_ms = a;
    if (train_ms) *train_ms = b;
  });
}

gfnx_status gfnx_event_record(gfnx_ctx* h, int32_t slot) {
  return guard(h, [&] {
    Ctx& c = h->c;
    if (slot < 0 || slot >= 16) fail(GFNX_ERR_CONFIG, "event slot out of range");
    if (!c.user_ev[slot]) cuda_check(cudaEventCreate(&c.user_ev[slot]), "event");
    cuda_check(cudaEventRecord(c.user_ev[slot], c.stream), "event record");
  });
}

gfnx_status gfnx_event_elapsed(gfnx_ctx* h, int32_t a, int32_t b, double* ms) {
  return guard(h, [&] {
    Ctx& c = h->c;
    if (a < 0 || a >= 16 || b < 0 || b >= 16 || !c.user_ev[a] || !c.user_ev[b])
      fail(GFNX_ERR_CONFIG, "event slot not recorded");
    cuda_check(cudaEventSynchronize(c.user_ev[b]), "event sync");
    float f = 0.f;
    cuda_check(cudaEventElapsedTime(&f, c.user_ev[a], c.user_ev[b]), "elapsed");
    *ms = f;
  });
}

gfnx_status gfnx_counters(gfnx_ctx* h, int64_t* out, int32_t n) {
  return guard(h, [&] {
    Ctx& c = h->c;
    int32_t raw[16];
    cuda_check(cudaMemcpyAsync(raw, c.batch.counters, sizeof raw, cudaMemcpyDeviceToHost, c.stream), "counters");
    cuda_check(cudaStreamSynchronize(c.stream), "sync");
    int64_t acc[2];
    memcpy(acc, raw + 8, sizeof acc);
    const int64_t vals[4] = {acc[0], acc[1], raw[0], raw[1]};
    for (int i = 0; i < n && i < 4; ++i) out[i] = vals[i];
  });
}

// diagnostic clock slots: rollout [0..8], wgrad passes [9..11], sampler sub-phases [12..14],
// bwd phases [15..20]
constexpr int kPhaseSlots = 32;

gfnx_status gfnx_phase_timers(gfnx_ctx* h, int32_t mode, int64_t* out, int32_t n) {
  return guard(h, [&] {
    Ctx& c = h->c;
    if (mode == 1) {
      if (!c.phase) cuda_check(cudaMalloc(&c.phase, sizeof(long long) * kPhaseSlots), "phase timers");
      cuda_check(cudaMemsetAsync(c.phase, 0, sizeof(long long) * kPhaseSlots, c.stream), "phase timers");
    } else if (mode == 0) {
      if (c.phase) {
        cudaStreamSynchronize(c.stream);
        cudaFree(c.phase);
      }
      c.phase = nullptr;
    } else if (c.phase) {
      long long v[kPhaseSlots];
      cuda_check(cudaMemcpyAsync(v, c.phase, sizeof v, cudaMemcpyDeviceToHost, c.stream), "phase timers");
      cuda_check(cudaStreamSynchronize(c.stream), "sync");
      for (int i = 0; i < n && i < kPhaseSlots; ++i) out[i] = v[i];
      cuda_check(cudaMemsetAsync(c.phase, 0, sizeof v, c.stream), "phase timers");
    }
  });
}

gfnx_status gfnx_profile(gfnx_ctx* h, int32_t enable) {
  h->c.profiling = enable != 0;
  h->c.profile_rollout_only = enable == 2;
  return GFNX_OK;
}

int32_t gfnx_profile_read(gfnx_ctx* h, char* names, int32_t names_cap, double* total_ms,
                          int32_t* counts, int32_t cap) {
  Ctx& c = h->c;
  cudaStreamSynchronize(c.stream);
  std::vector<std::string> keys;
  std::vector<double> tot;
  std::vector<int> cnt;
  for (auto& r : c.prof) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    size_t k = 0;
    while (k < keys.size() && keys[k] != r.name) ++k;
    if (k == keys.size()) {
      keys.push_back(r.name);
      tot.push_back(0.0);
      cnt.push_back(0);
    }
    tot[k] += ms;
    cnt[k] += 1;
    c.ev_pool.push_back(r.a);
    c.ev_pool.push_back(r.b);
  }
  c.prof.clear();
  std::string joined;
  int n = 0;
  for (size_t k = 0; k < keys.size() && (int)k < cap; ++k, ++n) {
    joined += keys[k] + "\n";
    total_ms[k] = tot[k];
    counts[k] = cnt[k];
  }
  if (names && names_cap > 0) {
    const size_t m = std::min<size_t>(joined.size(), (size_t)names_cap - 1);
    memcpy(names, joined.data(), m);
    names[m] = 0;
  }
  return n;
}

gfnx_status gfnx_test_threefry(const uint64_t* keys, const uint64_t* ctr, int64_t n, uint64_t* out) {
  return guard(nullptr, [&] {
    uint64_t *dk, *dc, *dout;
    cuda_check(cudaMalloc(&dk, 16 * n), "alloc");
    cuda_check(cudaMalloc(&dc, 16 * n), "alloc");
    cuda_check(cudaMalloc(&dout, 16 * n), "alloc");
    cudaMemcpy(dk, keys, 16 * n, cudaMemcpyHostToDevice);
    cudaMemcpy(dc, ctr, 16 * n, cudaMemcpyHostToDevice);
    k_threefry<<<(unsigned)((n + 255) / 256), 256>>>(dk, dc, n, dout);
    cuda_check(cudaMemcpy(out, dout, 16 * n, cudaMemcpyDeviceToHost), "threefry");
    cudaFree(dk);
    cudaFree(dc);
    cudaFree(dout);
  });
}

gfnx_status gfnx_test_mma_rate(int32_t n, int32_t reps, int32_t mode, int32_t grid, int64_t* cycles) {
  return guard(nullptr, [&] {
    test_mma_rate(n, reps, mode, grid, reinterpret_cast<long long*>(cycles));
    cuda_check(cudaGetLastError(), "mma rate");
  });
}

gfnx_status gfnx_test_ts_mma(const uint16_t* a, const uint16_t* b, float* d) {
  return guard(nullptr, [&] {
    test_ts_mma(a, b, d);
    cuda_check(cudaGetLastError(), "ts mma");
  });
}

gfnx_status gfnx_test_uniform_fold(uint64_t key_hi, uint64_t key_lo, const uint64_t* idx, int64_t n,
                                   double* out) {
  return guard(nullptr, [&] {
    uint64_t* di;
    double* dout;
    cuda_check(cudaMalloc(&di, 8 * n), "alloc");
    cuda_check(cudaMalloc(&dout, 8 * n), "alloc");
    cudaMemcpy(di, idx, 8 * n, cudaMemcpyHostToDevice);
    k_uniform_fold<<<(unsigned)((n + 255) / 256), 256>>>(Key{key_hi, key_lo}, di, n, dout);
    cuda_check(cudaMemcpy(out, dout, 8 * n, cudaMemcpyDeviceToHost), "uniform");
    cudaFree(di);
    cudaFree(dout);
  });
}

}  // extern "C"
