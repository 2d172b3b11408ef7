// group.cu — in-process communicator: the ranks of one data-parallel job driven by the
// threads of ONE process (one gfnx_ctx per rank, on one or several GPUs of a node).
//
// The job's single exchange step — the sum of the gradient / loss partials and of the DB/MDB
// normaliser counts (objectives.cpp:112-113,224) — is a hand-written kernel
// that reads every rank's buffer directly (peer memory over NVLink when the ranks sit on
// different GPUs, plain device memory when they share one) and adds them in rank order, so
// every rank obtains the identical, deterministic sum. Ordering across the ranks' streams uses
// CUDA events published through a host barrier at enqueue time; no stream is ever synchronised
// on the host:
//   1. rank r records ready[r] after the producers of its buffer        -> barrier
//   2. rank r's stream waits for ready[q] (all q), sums all buffers into its scratch,
//      records done[r]                                                   -> barrier
//   3. rank r's stream waits for done[q] (every peer finished reading buf[r]), then copies
//      scratch -> buf[r].
// The NCCL path (one process per GPU) is the other transport; both are selected at create.
#include <algorithm>
#include <condition_variable>
#include <mutex>
#include <vector>

#include "engine.h"

namespace gfnx {

struct Group {
  int world = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t gen = 0;
  struct Member {
    int device = -1;
    cudaStream_t stream = nullptr;
    cudaEvent_t ready = nullptr, done = nullptr;
    void* buf = nullptr;
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    bool joined = false;
  };
  std::vector<Member> m;

  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const int64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

namespace {

constexpr int kMaxWorld = 16;
struct Srcs {
  const void* p[kMaxWorld];
};

template <class T>
__global__ void k_group_sum(Srcs s, int world, size_t n, T* __restrict__ out) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    T acc = static_cast<const T*>(s.p[0])[i];
    for (int q = 1; q < world; ++q) acc += static_cast<const T*>(s.p[q])[i];  // rank order
    out[i] = acc;
  }
}

size_t dtype_size(int dtype) { return dtype == kDtypeF64 ? 8 : 4; }

}  // namespace

Group* group_new(int world) {
  if (world < 1 || world > kMaxWorld) raise_error(GFNX_ERR_CONFIG, "group world must lie in [1, 16]");
  auto* g = new Group();
  g->world = world;
  g->m.resize(world);
  return g;
}

int group_world(const Group* g) { return g->world; }

void group_delete(Group* g) {
  if (!g) return;
  for (auto& mb : g->m) {
    if (mb.joined) raise_error(GFNX_ERR_CONTRACT, "group destroyed while a member context is alive");
  }
  delete g;
}

void group_join(Ctx& c, Group* g, int rank) {
  std::lock_guard<std::mutex> lk(g->mu);
  Group::Member& mb = g->m[rank];
  if (mb.joined) raise_error(GFNX_ERR_CONFIG, "group rank already taken");
  mb.device = c.device;
  mb.stream = c.stream;
  cuda_check(cudaEventCreateWithFlags(&mb.ready, cudaEventDisableTiming), "group event");
  cuda_check(cudaEventCreateWithFlags(&mb.done, cudaEventDisableTiming), "group event");
  mb.joined = true;
  // peer access to the members already on other devices (NVLink P2P), both directions
  for (int q = 0; q < g->world; ++q) {
    const Group::Member& o = g->m[q];
    if (q == rank || !o.joined || o.device == c.device) continue;
    int ok = 0;
    cudaDeviceCanAccessPeer(&ok, c.device, o.device);
    if (!ok) raise_error(GFNX_ERR_CONFIG, "group: no peer access between the member GPUs");
    cudaSetDevice(c.device);
    cudaError_t e = cudaDeviceEnablePeerAccess(o.device, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) cuda_check(e, "peer access");
    cudaSetDevice(o.device);
    e = cudaDeviceEnablePeerAccess(c.device, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) cuda_check(e, "peer access");
    cudaSetDevice(c.device);
  }
  cudaGetLastError();
}

void group_leave(Ctx& c, Group* g, int rank) {
  std::lock_guard<std::mutex> lk(g->mu);
  Group::Member& mb = g->m[rank];
  if (mb.ready) cudaEventDestroy(mb.ready);
  if (mb.done) cudaEventDestroy(mb.done);
  if (mb.scratch) cudaFree(mb.scratch);
  mb = Group::Member{};
  (void)c;
}

// Sum of `buf` over the group, in place on every rank (stream-ordered on `st`). Every
// member must call it with the same n / dtype in the same order (a collective).
void group_allreduce(Ctx& c, void* buf, size_t n, int dtype, cudaStream_t st) {
  Group* g = c.group;
  Group::Member& me = g->m[c.rank];
  const size_t bytes = n * dtype_size(dtype);
  if (me.scratch_bytes < bytes) {
    if (me.scratch) cudaFree(me.scratch);
    cuda_check(cudaMalloc(&me.scratch, bytes), "group scratch");
    me.scratch_bytes = bytes;
  }
  me.buf = buf;
  cuda_check(cudaEventRecord(me.ready, st), "group ready");
  g->barrier();
  Srcs s{};
  for (int q = 0; q < g->world; ++q) {
    s.p[q] = g->m[q].buf;
    if (q != c.rank) cuda_check(cudaStreamWaitEvent(st, g->m[q].ready, 0), "group wait");
  }
  const int threads = 256;
  const int blocks = (int)std::min<size_t>((n + threads - 1) / threads, 4 * 148);
  if (dtype == kDtypeF64)
    k_group_sum<double><<<blocks, threads, 0, st>>>(s, g->world, n, static_cast<double*>(me.scratch));
  else if (dtype == kDtypeF32)
    k_group_sum<float><<<blocks, threads, 0, st>>>(s, g->world, n, static_cast<float*>(me.scratch));
  else
    k_group_sum<int32_t><<<blocks, threads, 0, st>>>(s, g->world, n, static_cast<int32_t*>(me.scratch));
  c.launches++;
  cuda_check(cudaEventRecord(me.done, st), "group done");
  g->barrier();
  for (int q = 0; q < g->world; ++q)
    if (q != c.rank) cuda_check(cudaStreamWaitEvent(st, g->m[q].done, 0), "group wait");
  cuda_check(cudaMemcpyAsync(buf, me.scratch, bytes, cudaMemcpyDeviceToDevice, st), "group copy");
}

}  // namespace gfnx
