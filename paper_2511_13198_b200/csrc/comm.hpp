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

// one point-to-point transfer of a p2p() call: `bytes` from / to device memory `ptr`;
// a send to `peer` is matched with that peer's receive from this rank of the same tag
struct P2P {
  int peer;
  int tag;
  void* ptr;
  int64_t bytes;
};

struct Comm {
  int P = 1, rank = 0;
  virtual ~Comm() {}
  // grouped point-to-point sends and receives (ring passes, the zigzag exchange of the
  // context-parallel attention); a send to this rank itself is a device copy into the
  // matching receive.  Every rank calls it at the same point of the program.
  virtual pds_status p2p(const P2P* sends, int ns, const P2P* recvs, int nr, cudaStream_t st) = 0;
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
  // ---- tile-overlapped collectives (MegatronTS over P ranks) ----
  // Both are issued on the side stream `st`, which the caller has ordered after the
  // compute stream `main`'s producers; the GEMM they overlap runs on `main`.
  // all_gather_flagged: recv [P][count] holds this rank's chunk at slot `rank`; the
  // chunks of ranks rank+1, rank+2, ... (mod P) land in that order and after chunk j
  // has landed flags[j] := epoch (a stream memory write: no SM involved), which the
  // consuming GEMM polls per tile (GemmArgs::wait_flags).
  virtual pds_status all_gather_flagged(void* recv, int64_t count, DType dt, cudaStream_t main, cudaStream_t st,
                                        uint32_t* flags, uint32_t epoch) {
    return PDS_ENOTIMPL;
  }
  // reduce_scatter_gated: send [P][count] partials from the producing GEMM; chunk j of
  // ranks rank+1, rank+2, ... is sent to rank j once ctr[j] has reached `target`
  // (a stream wait on the GEMM's store counter, GemmArgs::done_ctr), and the partial of
  // rank i for this rank's chunk lands in recv + i*count (recv slot `rank` untouched).
  // After joining `st` the caller sums recv[i != rank] and send[rank] in rank order.
  virtual pds_status reduce_scatter_gated(const void* send, void* recv, int64_t count, DType dt, cudaStream_t main,
                                          cudaStream_t st, const uint32_t* ctr, uint32_t target) {
    return PDS_ENOTIMPL;
  }
  // all_to_all_gated: send [P][count] blocks from the producing GEMM (column-blocked
  // epilogue); block j is sent to rank j once ctr[j] has reached `target` (own block:
  // copied into recv + rank*count), and rank i's block for this rank lands in
  // recv + i*count.
  virtual pds_status all_to_all_gated(const void* send, void* recv, int64_t count, DType dt, cudaStream_t main,
                                      cudaStream_t st, const uint32_t* ctr, uint32_t target) {
    return PDS_ENOTIMPL;
  }
  // SMs a GEMM must leave free while one of the above is in flight (the collective's
  // own kernels must be able to run beside a persistent GEMM that polls for them)
  virtual int overlap_sm_reserve() const { return 0; }
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

// 32-bit stream memory operations (driver API, no SM involved): `*addr := v` after the
// stream's prior work; block the stream until (int32)(*addr - v) >= 0
pds_status stream_write32(cudaStream_t st, uint32_t* addr, uint32_t v);
pds_status stream_wait32_geq(cudaStream_t st, const uint32_t* addr, uint32_t v);

}  // namespace pds
