// comm.cpp — NCCL and in-process transports of the replica exchange (comm.hpp).
#include "comm.hpp"

#include <dlfcn.h>

#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>

namespace srl {

// ------------------------------------------------------------------ NCCL (dlopen)
// The handful of NCCL entry points used here, declared from the NCCL C API
// (nccl.h): opaque communicator, 128-byte unique id, int result codes.
namespace nccl {
typedef struct ncclComm* comm_t;
typedef struct {
  char internal[128];
} uid_t;
constexpr int kSuccess = 0;
constexpr int kInProgress = 7;
constexpr int kUint8 = 1;

struct Api {
  int (*GetUniqueId)(uid_t*) = nullptr;
  int (*CommInitRank)(comm_t*, int, uid_t, int) = nullptr;
  int (*CommDestroy)(comm_t) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, comm_t, cudaStream_t) = nullptr;
  int (*Broadcast)(const void*, void*, size_t, int, int, comm_t, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
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
    SRL_SYM(CommInitRank, "ncclCommInitRank");
    SRL_SYM(CommDestroy, "ncclCommDestroy");
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
  if (rc == kSuccess || rc == kInProgress) return 0;
  err = std::string(what) + ": " + (api().GetErrorString ? api().GetErrorString(rc) : "nccl error");
  return -1;
}
}  // namespace nccl

class NcclComm : public Comm {
 public:
  nccl::comm_t comm = nullptr;
  ~NcclComm() override {
    if (comm) nccl::api().CommDestroy(comm);
  }
  int allgather_inplace(void* buf, size_t seg, cudaStream_t st, std::string& err) override {
    const nccl::Api& a = nccl::api();
    uint8_t* b = (uint8_t*)buf;
    return nccl::check(a.AllGather(b + (size_t)rank * seg, b, seg, nccl::kUint8, comm, st), "ncclAllGather", err);
  }
  int broadcast_inplace(const std::vector<Range>& ranges, cudaStream_t st, std::string& err) override {
    const nccl::Api& a = nccl::api();
    if (nccl::check(a.GroupStart(), "ncclGroupStart", err)) return -1;
    int rc = 0;
    for (const Range& r : ranges)
      if (r.bytes && !rc) rc = nccl::check(a.Broadcast(r.p, r.p, r.bytes, nccl::kUint8, 0, comm, st), "ncclBroadcast", err);
    std::string e2;
    if (nccl::check(a.GroupEnd(), "ncclGroupEnd", e2) && !rc) {
      err = e2;
      rc = -1;
    }
    return rc;
  }
};

int nccl_unique_id(uint8_t* out, std::string& err) {
  const nccl::Api& a = nccl::api();
  if (!a.ok) return err = a.why, -1;
  nccl::uid_t id;
  if (nccl::check(a.GetUniqueId(&id), "ncclGetUniqueId", err)) return -1;
  memcpy(out, id.internal, 128);
  return 0;
}

Comm* comm_create_nccl(const uint8_t* uid, int rank, int world, std::string& err) {
  const nccl::Api& a = nccl::api();
  if (!a.ok) return err = a.why, nullptr;
  nccl::uid_t id;
  memcpy(id.internal, uid, 128);
  NcclComm* c = new NcclComm();
  c->rank = rank;
  c->world = world;
  if (nccl::check(a.CommInitRank(&c->comm, world, id, rank), "ncclCommInitRank", err)) {
    c->comm = nullptr;
    delete c;
    return nullptr;
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
  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (broken) return false;
    const long long my = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    const bool ok = cv.wait_for(lk, std::chrono::seconds(300), [&] { return gen != my || broken; });
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
    if (!g->barrier()) return err = "local group barrier timed out (a peer rank failed)", -1;
    if (copies()) return err = "cudaMemcpyAsync (local peer copy) failed", -1;
    if (cudaEventRecord(g->ev_done[rank], st) != cudaSuccess) return err = "cudaEventRecord", -1;
    if (!g->barrier()) return err = "local group barrier timed out (a peer rank failed)", -1;
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

Comm* comm_create_local(void* group, int rank, int world, std::string& err) {
  LocalGroup* g = (LocalGroup*)group;
  if (!g) return err = "null local group", nullptr;
  if (g->world != world) return err = "local group size differs from comm->world", nullptr;
  if (g->ev_ready[rank]) return err = "rank already joined this local group", nullptr;
  LocalComm* c = new LocalComm();
  c->g = g;
  c->rank = rank;
  c->world = world;
  if (cudaEventCreateWithFlags(&g->ev_ready[rank], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&g->ev_done[rank], cudaEventDisableTiming) != cudaSuccess) {
    delete c;
    return err = "cudaEventCreate", nullptr;
  }
  return c;
}

}  // namespace srl
