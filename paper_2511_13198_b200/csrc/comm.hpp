// Collective backends of the strategy library: NCCL (one process per GPU over
// NVLink / NVSwitch) and an in-process loopback group (P virtual ranks on one
// device, host threads + CUDA events) that lets a single B200 run every
// strategy at P = 2, 4, 8 with the same strategy code.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <condition_variable>
#include <mutex>
#include <vector>

#include "../../include/paradyse.h"

namespace pds {

enum DType { DT_BF16 = 0, DT_F32 = 1 };

struct Comm {
  int P = 1, rank = 0;
  virtual ~Comm() {}
  // recv [P][count] <- send [count] of every rank (rank order).  send may alias
  // recv + rank*count (in place).
  virtual pds_status all_gather(const void* send, void* recv, int64_t count, DType dt, cudaStream_t st) = 0;
  // recv [count] <- sum over ranks of send[rank*count ...].  recv may alias
  // send + rank*count (in place).
  virtual pds_status reduce_scatter(const void* send, void* recv, int64_t count, DType dt, cudaStream_t st) = 0;
  // in-place sum (fp32)
  virtual pds_status all_reduce(void* buf, int64_t count, DType dt, cudaStream_t st) = 0;
  // recv[j][count] <- send_j[rank][count]  (chunk `rank` of every source j)
  virtual pds_status all_to_all(const void* send, void* recv, int64_t count, DType dt, cudaStream_t st) = 0;
  // A communicator for collectives issued on a second stream concurrently with this
  // one's (NCCL: a split of the same ranks, so two in-flight collectives never share
  // one communicator; loopback / self: the same object).  Collective: every rank
  // calls it at the same point of the program.
  virtual Comm* side(pds_status* st) { return this; }
  // true when every collective is an identity (one rank, no library)
  virtual bool trivial() const { return false; }
};

Comm* make_nccl_comm(int P, int rank, const void* uid, pds_status* st);
Comm* make_self_comm();

struct LoopGroup {
  int P;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<const void*> ptr;
  std::vector<cudaEvent_t> ready, done;
  void barrier();
};
Comm* make_loop_comm(LoopGroup* g, int rank, pds_status* st);

int64_t dt_size(DType dt);

}  // namespace pds
