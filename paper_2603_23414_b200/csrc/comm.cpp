// comm.cpp — NCCL and in-process transports of the replica exchange (comm.hpp).
#include "comm.hpp"
#include "srl.h"

#include <dlfcn.h>

#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>

#include <nccl.h>

namespace srl {

// ------------------------------------------------------------------ NCCL (dlopen)
// The NCCL C API types come from nccl.h (the copy shipped with the torch NCCL
// wheel: NCCL 2.28, ncclConfig_t with the non-blocking flag); the entry points
// are resolved with dlsym from the libnccl already mapped into the process.
namespace nccl {
typedef int (*GetUniqueId_t)(ncclUniqueId*);
typedef int (*CommInitRankConfig_t)(ncclComm_t*, int, ncclUniqueId, int, ncclConfig_t*);
typedef int (*CommDestroy_t)(ncclComm_t);
typedef int (*CommAbort_t)(ncclComm_t);
typedef int (*CommGetAsyncError_t)(ncclComm_t, ncclResult_t*);
typedef int (*AllGather_t)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
typedef int (*Broadcast_t)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
typedef int (*Group_t)();
typedef const char* (*GetErrorString_t)(ncclResult_t);

struct Api {
  GetUniqueId_t GetUniqueId = nullptr;
  CommInitRankConfig_t CommInitRankConfig = nullptr;
  CommDestroy_t CommDestroy = nullptr;
  CommAbort_t CommAbort = nullptr;
  CommGetAsyncError_t CommGetAsyncError = nullptr;
  AllGather_t AllGather = nullptr;
  Broadcast_t Broadcast = nullptr;
  Group_t GroupStart = nullptr, GroupEnd = nullptr;
  GetErrorString_t GetErrorString = nullptr;
  bool ok = false;
  std::string why;
};

const Api& api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    // prefer the libnccl already mapped into the process (torch's), then the
    // loader's search path
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
      return;
    }
#define SRL_SYM(f, name)                                        \
  a.f = reinterpret_cast<decltype(a.f)>(dlsym(h, name));        \
  if (!a.f) {                                                   \
    a.why = std::string("libnccl.so.2 lacks ") + name;          \
    return;                                                     \
  }
    SRL_SYM(GetUniqueId, "ncclGetUniqueId");
    SRL_SYM(CommInitRankConfig, "ncclCommInitRankConfig");
    SRL_SYM(CommDestroy, "ncclCommDestroy");
    SRL_SYM(CommAbort, "ncclCommAbort");
    SRL_SYM(CommGetAsyncError, "ncclCommGetAsyncError");
    SRL_SYM(AllGather, "ncclAllGather");
    SRL_SYM(Broadcast, "ncclBroadcast");
    SRL_SYM(GroupStart, "ncclGroupStart");
    SRL_SYM(GroupEnd, "ncclGroupEnd");
    SRL_SYM(GetErrorString, "ncclGetErrorString");
#undef SRL_SYM
    a.ok = true;
  });
  return a;
}

int check(int rc, const char* what, std::string& err) {
  if (rc == ncclSuccess || rc == ncclInProgress) return 0;
  err = std::string(what) + ": " + (api().GetErrorString ? api().GetErrorString((ncclResult_t)rc) : "nccl error");
  return -1;
}
}  // namespace nccl

class NcclComm : public Comm {
 public:
  ncclComm_t comm = nullptr;
  bool aborted = false;
  ~NcclComm() override {
    if (comm && !aborted) nccl::api().CommDestroy(comm);
  }
  // a non-blocking communicator may return ncclInProgress from an enqueue: wait
  // (bounded) until the operation is enqueued before the stream is used further
  int settle(int rc, const char* what, std::string& err) {
    if (nccl::check(rc, what, err)) return -1;
    if (rc != ncclInProgress) return 0;
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
      ncclResult_t st = ncclSuccess;
      nccl::api().CommGetAsyncError(comm, &st);
      if (st == ncclSuccess) return 0;
      if (st != ncclInProgress) return nccl::check(st, what, err);
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(300)) return err = std::string(what) + ": enqueue timed out", -1;
      std::this_thread::yield();
    }
  }
  int allgather_inplace(void* buf, size_t seg, cudaStream_t st, std::string& err) override {
    const nccl::Api& a = nccl::api();
    uint8_t* b = (uint8_t*)buf;
    return settle(a.AllGather(b + (size_t)rank * seg, b, seg, ncclUint8, comm, st), "ncclAllGather", err);
  }
  int broadcast_inplace(const std::vector<Range>& ranges, cudaStream_t st, std::string& err) override {
    const nccl::Api& a = nccl::api();
    if (nccl::check(a.GroupStart(), "ncclGroupStart", err)) return -1;
    int rc = 0;
    for (const Range& r : ranges)
      if (r.bytes && !rc) rc = nccl::check(a.Broadcast(r.p, r.p, r.bytes, ncclUint8, 0, comm, st), "ncclBroadcast", err);
    std::string e2;
    if (settle(a.GroupEnd(), "ncclGroupEnd", e2) && !rc) {
      err = e2;
      rc = -1;
    }
    return rc;
  }
  int poll_error(std::string& err) override {
    if (aborted) return err = "communicator aborted", -1;
    ncclResult_t st = ncclSuccess;
    if (nccl::api().CommGetAsyncError(comm, &st) != ncclSuccess) return err = "ncclCommGetAsyncError failed", -1;
    if (st == ncclSuccess || st == ncclInProgress) return 0;
    return nccl::check(st, "NCCL asynchronous error", err);
  }
  void abort() override {
    if (comm && !aborted) nccl::api().CommAbort(comm);
    aborted = true;
  }
};

int nccl_unique_id(uint8_t* out, std::string& err) {
  const nccl::Api& a = nccl::api();
  if (!a.ok) return err = a.why, -1;
  ncclUniqueId id;
  if (nccl::check(a.GetUniqueId(&id), "ncclGetUniqueId", err)) return -1;
  memcpy(out, id.internal, 128);
  return 0;
}

Comm* comm_create_nccl(const uint8_t* uid, int rank, int world, int timeout_ms, std::string& err) {
  const nccl::Api& a = nccl::api();
  if (!a.ok) return err = a.why, nullptr;
  ncclUniqueId id;
  memcpy(id.internal, uid, 128);
  NcclComm* c = new NcclComm();
  c->rank = rank;
  c->world = world;
  // non-blocking initialisation, polled with a deadline: a rank that never joins
  // fails every other rank's srl_create instead of hanging it
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
  cfg.blocking = 0;
  if (nccl::check(a.CommInitRankConfig(&c->comm, world, id, rank, &cfg), "ncclCommInitRankConfig", err)) {
    c->comm = nullptr;
    delete c;
    return nullptr;
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    ncclResult_t st = ncclInProgress;
    a.CommGetAsyncError(c->comm, &st);
    if (st == ncclSuccess) break;
    const bool late = std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(timeout_ms);
    if (st != ncclInProgress || late) {
      if (st != ncclInProgress) nccl::check(st, "ncclCommInitRankConfig", err);
      else err = "ncclCommInitRankConfig: timed out waiting for the other ranks";
      a.CommAbort(c->comm);
      c->aborted = true;
      delete c;
      return nullptr;
    }
    std::this_thread::sleep_for(std::chrono::milliseconds(1));
  }
  return c;
}

// ------------------------------------------------------------------ in-process group
struct LocalGroup {
  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  bool broken = false;
  std::vector<std::vector<void*>> ptrs;      // [rank] published addresses of the current call
  std::vector<cudaEvent_t> ev_ready, ev_done;  // [rank], created by the owning rank on its device
  explicit LocalGroup(int w) : world(w), ptrs(w), ev_ready(w, nullptr), ev_done(w, nullptr) {}

  // returns false on timeout (another rank died): the group is then broken for good
  bool barrier(long long timeout_ms) {
    std::unique_lock<std::mutex> lk(mu);
    if (broken) return false;
    const long long my = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    const bool ok = cv.wait_for(lk, std::chrono::milliseconds(timeout_ms), [&] { return gen != my || broken; });
    if (!ok || broken) {
      broken = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
};

void* local_group_create(int world) { return world >= 1 ? new LocalGroup(world) : nullptr; }
void local_group_destroy(void* g) { delete (LocalGroup*)g; }

class LocalComm : public Comm {
 public:
  LocalGroup* g = nullptr;
  long long timeout_ms = 300000;
  ~LocalComm() override {
    if (g) {
      if (g->ev_ready[rank]) cudaEventDestroy(g->ev_ready[rank]);
      if (g->ev_done[rank]) cudaEventDestroy(g->ev_done[rank]);
      g->ev_ready[rank] = g->ev_done[rank] = nullptr;
    }
  }
  // publish addresses + "inputs ready", copy peers' data after their ready event,
  // then make every rank's stream wait until all peers finished reading from it
  template <class F>
  int exchange(const std::vector<void*>& mine, cudaStream_t st, F copies, std::string& err) {
    g->ptrs[rank] = mine;
    if (cudaEventRecord(g->ev_ready[rank], st) != cudaSuccess) return err = "cudaEventRecord", -1;
    if (!g->barrier(timeout_ms)) return err = "local group barrier timed out (a peer rank failed)", -1;
    if (copies()) return err = "cudaMemcpyAsync (local peer copy) failed", -1;
    if (cudaEventRecord(g->ev_done[rank], st) != cudaSuccess) return err = "cudaEventRecord", -1;
    if (!g->barrier(timeout_ms)) return err = "local group barrier timed out (a peer rank failed)", -1;
    for (int p = 0; p < world; ++p)
      if (p != rank) cudaStreamWaitEvent(st, g->ev_done[p], 0);
    return 0;
  }
  int allgather_inplace(void* buf, size_t seg, cudaStream_t st, std::string& err) override {
    uint8_t* b = (uint8_t*)buf;
    return exchange({buf}, st, [&]() -> int {
      for (int p = 0; p < world; ++p) {
        if (p == rank) continue;
        cudaStreamWaitEvent(st, g->ev_ready[p], 0);
        const uint8_t* src = (const uint8_t*)g->ptrs[p][0] + (size_t)p * seg;
        if (cudaMemcpyAsync(b + (size_t)p * seg, src, seg, cudaMemcpyDefault, st) != cudaSuccess) return -1;
      }
      return 0;
    }, err);
  }
  int poll_error(std::string& err) override {
    std::lock_guard<std::mutex> lk(g->mu);
    return g->broken ? (err = "local group broken (a peer rank failed or timed out)", -1) : 0;
  }
  void abort() override {
    std::lock_guard<std::mutex> lk(g->mu);
    g->broken = true;
    g->cv.notify_all();
  }
  int broadcast_inplace(const std::vector<Range>& ranges, cudaStream_t st, std::string& err) override {
    std::vector<void*> mine;
    for (const Range& r : ranges) mine.push_back(r.p);
    return exchange(mine, st, [&]() -> int {
      if (rank == 0) return 0;
      if (g->ptrs[0].size() != ranges.size()) return -1;
      cudaStreamWaitEvent(st, g->ev_ready[0], 0);
      for (size_t i = 0; i < ranges.size(); ++i)
        if (ranges[i].bytes &&
            cudaMemcpyAsync(ranges[i].p, g->ptrs[0][i], ranges[i].bytes, cudaMemcpyDefault, st) != cudaSuccess)
          return -1;
      return 0;
    }, err);
  }
};

Comm* comm_create_local(void* group, int rank, int world, int timeout_ms, std::string& err) {
  LocalGroup* g = (LocalGroup*)group;
  if (!g) return err = "null local group", nullptr;
  if (g->world != world) return err = "local group size differs from comm->world", nullptr;
  if (g->ev_ready[rank]) return err = "rank already joined this local group", nullptr;
  LocalComm* c = new LocalComm();
  c->g = g;
  c->timeout_ms = timeout_ms;
  c->rank = rank;
  c->world = world;
  if (cudaEventCreateWithFlags(&g->ev_ready[rank], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&g->ev_done[rank], cudaEventDisableTiming) != cudaSuccess) {
    delete c;
    return err = "cudaEventCreate", nullptr;
  }
  return c;
}

// ------------------------------------------------------------------ host callbacks
class HostComm : public Comm {
 public:
  srl_host_transport t{};
  uint8_t* h = nullptr;
  size_t cap = 0;
  bool failed = false;
  ~HostComm() override {
    if (h) cudaFreeHost(h);
  }
  int grow(size_t bytes, std::string& err) {
    if (bytes <= cap) return 0;
    if (h) cudaFreeHost(h);
    h = nullptr;
    cap = 0;
    if (cudaHostAlloc((void**)&h, bytes, cudaHostAllocDefault) != cudaSuccess) return err = "cudaHostAlloc", -1;
    cap = bytes;
    return 0;
  }
  int allgather_inplace(void* buf, size_t seg, cudaStream_t st, std::string& err) override {
    if (failed) return err = "host transport failed earlier", -1;
    if (grow(seg * world, err)) return -1;
    uint8_t* b = (uint8_t*)buf;
    if (cudaMemcpyAsync(h + (size_t)rank * seg, b + (size_t)rank * seg, seg, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return err = "device -> host staging of the all-gather", -1;
    if (t.allgather(t.ctx, h, (uint64_t)seg) != 0) return failed = true, err = "host all-gather callback failed", -1;
    if (cudaMemcpyAsync(b, h, seg * world, cudaMemcpyHostToDevice, st) != cudaSuccess)
      return err = "host -> device of the all-gather", -1;
    return cudaStreamSynchronize(st) == cudaSuccess ? 0 : (err = "all-gather upload", -1);
  }
  int broadcast_inplace(const std::vector<Range>& ranges, cudaStream_t st, std::string& err) override {
    if (failed) return err = "host transport failed earlier", -1;
    for (const Range& r : ranges) {
      if (!r.bytes) continue;
      if (grow(r.bytes, err)) return -1;
      if (rank == 0 && (cudaMemcpyAsync(h, r.p, r.bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
                        cudaStreamSynchronize(st) != cudaSuccess))
        return err = "device -> host staging of the broadcast", -1;
      if (t.broadcast(t.ctx, h, (uint64_t)r.bytes) != 0) return failed = true, err = "host broadcast callback failed", -1;
      if (rank != 0 && (cudaMemcpyAsync(r.p, h, r.bytes, cudaMemcpyHostToDevice, st) != cudaSuccess ||
                        cudaStreamSynchronize(st) != cudaSuccess))
        return err = "host -> device of the broadcast", -1;
    }
    return 0;
  }
  int poll_error(std::string& err) override { return failed ? (err = "host transport failed", -1) : 0; }
  void abort() override { failed = true; }
};

Comm* comm_create_host(const void* transport, int rank, int world, std::string& err) {
  const srl_host_transport* t = (const srl_host_transport*)transport;
  if (!t || !t->allgather || !t->broadcast) return err = "srl_comm.host: null transport / callback", nullptr;
  HostComm* c = new HostComm();
  c->t = *t;
  c->rank = rank;
  c->world = world;
  return c;
}

}  // namespace srl
