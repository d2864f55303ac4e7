// comm.hpp — the replica exchange of the data-parallel rollout (SURVEY §8(e),
// rows a14 and a17): an in-place all-gather of every replica's sampled
// (token, logprob) rows after each decode step, and an in-place broadcast of
// the refreshed policy from rank 0 after each early update.
//
// Three transports behind one interface:
//   NCCL   one process per GPU (torch.distributed launch); libnccl is resolved
//          at run time with dlopen -- the copy torch already loaded -- so the
//          library does not pin an NCCL version at link time;
//   LOCAL  several engines in ONE process (one host thread each, any devices,
//          including several on the same GPU): peer copies with
//          cudaMemcpyAsync ordered by CUDA events and a host barrier.  This is
//          what lets one B200 run the R > 1 lockstep path bit-exactly against
//          the oracle;
//   HOST   caller-supplied host callbacks (srl_host_transport): the rows are
//          staged through pinned host memory and exchanged by the caller (e.g.
//          a torch.distributed gloo group) -- several processes on one GPU, or
//          any host network.  Slow, but it runs the engine's replica protocol
//          across processes where NCCL cannot (one GPU per rank).
// Every call is collective: all ranks issue the same calls in the same order.
// Failure handling: the engine never blocks on a stream that holds a
// collective; it polls completion with a deadline and poll_error(), and calls
// abort() (ncclCommAbort) on an asynchronous error or a timeout, after which
// the engine reports SRL_E_NCCL for good.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <string>
#include <vector>

namespace srl {

struct Range {
  void* p;
  size_t bytes;
};

class Comm {
 public:
  int rank = 0, world = 1;
  virtual ~Comm() = default;
  // buf holds `world` segments of seg_bytes; this rank's segment (rank * seg_bytes)
  // is the input, every other segment is overwritten with the owner's.
  virtual int allgather_inplace(void* buf, size_t seg_bytes, cudaStream_t st, std::string& err) = 0;
  // every rank passes the same list (its own addresses); rank 0's bytes are copied
  // into every other rank's ranges.
  virtual int broadcast_inplace(const std::vector<Range>& ranges, cudaStream_t st, std::string& err) = 0;
  // non-zero (with a message) once the transport has failed asynchronously
  virtual int poll_error(std::string& err) { (void)err; return 0; }
  // tear down after a failure or timeout: pending collectives are abandoned
  virtual void abort() {}
};

// timeout_ms bounds the communicator's initialisation (non-blocking NCCL init polled)
Comm* comm_create_nccl(const uint8_t* unique_id, int rank, int world, int timeout_ms, std::string& err);
Comm* comm_create_local(void* group, int rank, int world, int timeout_ms, std::string& err);
Comm* comm_create_host(const void* transport /* srl_host_transport */, int rank, int world, std::string& err);
int nccl_unique_id(uint8_t* out128, std::string& err);
void* local_group_create(int world);
void local_group_destroy(void* g);

}  // namespace srl
