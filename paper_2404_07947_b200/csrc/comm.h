// Point-to-point transport between the ranks of a multi-GPU layout.
//
// The multi-stage executor (multi.cu) runs the same host loop on every rank;
// each exchange step of the method -- a pipeline hop of hidden states
// (PAPER.md:109, 196), the TP exchange of fp32 partial sums,
// the WAA KV handoff and the token return -- is a send /
// recv pair between the two ranks owning the GPUs involved, issued at the same
// point of the loop on both.  Sends and recvs between a pair of ranks match in
// issue order (NCCL's p2p rule); ops between group_start / group_end are
// posted together so symmetric exchanges cannot deadlock.
//
//   NcclComm  -- one process per GPU, ncclSend / ncclRecv over NVLink.
//   LocalComm -- `world` ranks as threads of one process on one device; a
//                transfer is a device copy on the receiver's stream ordered by
//                events against the sender's stream.  It exists so the
//                multi-rank executor can be tested on a single GPU.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <vector>

namespace exg {

struct Comm {
  virtual ~Comm() = default;
  virtual int rank() const = 0;
  virtual int world() const = 0;
  virtual void group_start() = 0;
  virtual void group_end() = 0;
  virtual void send(const void* buf, size_t bytes, int peer, cudaStream_t st) = 0;
  virtual void recv(void* buf, size_t bytes, int peer, cudaStream_t st) = 0;
  // Collective over ALL ranks, identical arguments on every rank: set up the
  // sub-communicators of these rank groups (each ascending, >= 2 ranks) --
  // the TP groups of a layout.  NCCL: ncclCommSplit.
  virtual void prepare_groups(const std::vector<std::vector<int>>& groups) { (void)groups; }
  // Native in-place fp32 sum over a prepared group (called by every member,
  // on its stream).  Transports without one (has_allreduce() false) leave
  // the caller to exchange the partials with send / recv.
  virtual bool has_allreduce() const { return false; }
  virtual void allreduce_sum(float* buf, size_t n, const std::vector<int>& group, cudaStream_t st) {
    (void)buf, (void)n, (void)group, (void)st;
    throw std::logic_error("transport has no native all-reduce");
  }
  // Surface asynchronous transport errors (NCCL: ncclCommGetAsyncError of the
  // communicator and its sub-communicators); throws on error.
  virtual void check_async() {}
};

// NCCL communicator over `world` processes (uid from nccl_unique_id on rank 0)
std::unique_ptr<Comm> make_nccl_comm(const uint8_t uid[128], int rank, int world);
void nccl_unique_id(uint8_t uid[128]);

// `world` thread-ranks sharing one hub; make_local_comms returns one Comm per rank
struct LocalHub;
std::shared_ptr<LocalHub> make_local_hub(int world);
std::unique_ptr<Comm> make_local_comm(std::shared_ptr<LocalHub> hub, int rank);

}  // namespace exg
