#include "comm.hpp"

#include <nccl.h>

#include <cstring>
#include <string>

#include "internal.hpp"

namespace pds {

// defined in kernels/norm.cu
int sum_bf16_p(const void* const* srcs, int P, void* dst, int64_t n, cudaStream_t st);
int sum_f32_p(const void* const* srcs, int P, void* dst, int64_t n, cudaStream_t st);

int64_t dt_size(DType dt) { return dt == DT_BF16 ? 2 : 4; }

// ------------------------------------------------------------------ P = 1
struct SelfComm : Comm {
  bool trivial() const override { return true; }
  pds_status all_gather(const void* send, void* recv, int64_t count, DType dt, cudaStream_t st) override {
    if (send != recv) PDS_CUDA(cudaMemcpyAsync(recv, send, count * dt_size(dt), cudaMemcpyDeviceToDevice, st));
    return PDS_OK;
  }
  pds_status reduce_scatter(const void* send, void* recv, int64_t count, DType dt, cudaStream_t st) override {
    return all_gather(send, recv, count, dt, st);
  }
  pds_status all_reduce(void*, int64_t, DType, cudaStream_t) override { return PDS_OK; }
  pds_status all_to_all(const void* send, void* recv, int64_t count, DType dt, cudaStream_t st) override {
    return all_gather(send, recv, count, dt, st);
  }
};
Comm* make_self_comm() { return new SelfComm(); }

// ------------------------------------------------------------------ NCCL
#define PDS_NCCL(expr)                                                          \
  do {                                                                          \
    ncclResult_t r__ = (expr);                                                  \
    if (r__ != ncclSuccess) {                                                   \
      set_error(std::string(#expr) + ": " + ncclGetErrorString(r__));          \
      return PDS_ENCCL;                                                         \
    }                                                                           \
  } while (0)

static ncclDataType_t nt(DType dt) { return dt == DT_BF16 ? ncclBfloat16 : ncclFloat32; }

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  NcclComm* side_ = nullptr;
  ~NcclComm() override {
    delete side_;
    if (comm) ncclCommDestroy(comm);
  }
  Comm* side(pds_status* st) override {
    if (!side_) {
      ncclComm_t c2 = nullptr;
      ncclResult_t r = ncclCommSplit(comm, 0, rank, &c2, nullptr);
      if (r != ncclSuccess) {
        set_error(std::string("ncclCommSplit: ") + ncclGetErrorString(r));
        *st = PDS_ENCCL;
        return nullptr;
      }
      side_ = new NcclComm();
      side_->P = P;
      side_->rank = rank;
      side_->comm = c2;
    }
    return side_;
  }
  pds_status all_gather(const void* send, void* recv, int64_t count, DType dt, cudaStream_t st) override {
    PDS_NCCL(ncclAllGather(send, recv, (size_t)count, nt(dt), comm, st));
    return PDS_OK;
  }
  pds_status reduce_scatter(const void* send, void* recv, int64_t count, DType dt, cudaStream_t st) override {
    PDS_NCCL(ncclReduceScatter(send, recv, (size_t)count, nt(dt), ncclSum, comm, st));
    return PDS_OK;
  }
  pds_status all_reduce(void* buf, int64_t count, DType dt, cudaStream_t st) override {
    PDS_NCCL(ncclAllReduce(buf, buf, (size_t)count, nt(dt), ncclSum, comm, st));
    return PDS_OK;
  }
  pds_status all_to_all(const void* send, void* recv, int64_t count, DType dt, cudaStream_t st) override {
    const int64_t b = count * dt_size(dt);
    PDS_NCCL(ncclGroupStart());
    for (int j = 0; j < P; ++j) {
      PDS_NCCL(ncclSend(static_cast<const char*>(send) + j * b, (size_t)count, nt(dt), j, comm, st));
      PDS_NCCL(ncclRecv(static_cast<char*>(recv) + j * b, (size_t)count, nt(dt), j, comm, st));
    }
    PDS_NCCL(ncclGroupEnd());
    return PDS_OK;
  }
};

Comm* make_nccl_comm(int P, int rank, const void* uid, pds_status* st) {
  NcclComm* c = new NcclComm();
  c->P = P;
  c->rank = rank;
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof(id));
  ncclResult_t r = ncclCommInitRank(&c->comm, P, id, rank);
  if (r != ncclSuccess) {
    set_error(std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    *st = PDS_ENCCL;
    delete c;
    return nullptr;
  }
  *st = PDS_OK;
  return c;
}

// ------------------------------------------------------------------ loopback
void LoopGroup::barrier() {
  std::unique_lock<std::mutex> lk(mu);
  const uint64_t g = gen;
  if (++arrived == P) {
    arrived = 0;
    ++gen;
    cv.notify_all();
  } else {
    cv.wait(lk, [&] { return gen != g; });
  }
}

struct LoopComm : Comm {
  LoopGroup* g;
  void* scratch = nullptr;
  int64_t scratch_bytes = 0;
  ~LoopComm() override {
    if (scratch) cudaFree(scratch);
  }
  pds_status ensure(int64_t bytes, cudaStream_t st) {
    if (bytes <= scratch_bytes) return PDS_OK;
    PDS_CUDA(cudaStreamSynchronize(st));
    if (scratch) PDS_CUDA(cudaFree(scratch));
    scratch = nullptr;
    PDS_CUDA(cudaMalloc(&scratch, bytes));
    scratch_bytes = bytes;
    return PDS_OK;
  }
  // publish `p` (device pointer) + an event recorded on st; wait until all ranks published
  void publish(const void* p, cudaStream_t st) {
    g->ptr[rank] = p;
    cudaEventRecord(g->ready[rank], st);
    g->barrier();
  }
  // after this rank's reads: record done, wait for everyone, then order st after all reads
  void finish(cudaStream_t st) {
    cudaEventRecord(g->done[rank], st);
    g->barrier();
    for (int j = 0; j < P; ++j)
      if (j != rank) cudaStreamWaitEvent(st, g->done[j], 0);
  }
  void wait_ready(cudaStream_t st) {
    for (int j = 0; j < P; ++j)
      if (j != rank) cudaStreamWaitEvent(st, g->ready[j], 0);
  }
  pds_status all_gather(const void* send, void* recv, int64_t count, DType dt, cudaStream_t st) override {
    const int64_t b = count * dt_size(dt);
    publish(send, st);
    wait_ready(st);
    for (int j = 0; j < P; ++j) {
      char* dst = static_cast<char*>(recv) + j * b;
      if (dst != g->ptr[j]) PDS_CUDA(cudaMemcpyAsync(dst, g->ptr[j], b, cudaMemcpyDeviceToDevice, st));
    }
    finish(st);
    return PDS_OK;
  }
  pds_status reduce_scatter(const void* send, void* recv, int64_t count, DType dt, cudaStream_t st) override {
    const int64_t b = count * dt_size(dt);
    PDS_TRY(ensure(b, st));
    publish(send, st);
    wait_ready(st);
    const void* srcs[8];
    for (int j = 0; j < P; ++j) srcs[j] = static_cast<const char*>(g->ptr[j]) + rank * b;
    // the sum reads every source's chunk `rank`; write into a scratch first when in place
    void* tmp = scratch;
    int rc = dt == DT_BF16 ? sum_bf16_p(srcs, P, tmp, count, st) : sum_f32_p(srcs, P, tmp, count, st);
    if (rc) PDS_FAIL(PDS_ECUDA, std::string("loopback reduce_scatter: ") + cudaGetErrorString((cudaError_t)rc));
    finish(st);
    PDS_CUDA(cudaMemcpyAsync(recv, tmp, b, cudaMemcpyDeviceToDevice, st));
    return PDS_OK;
  }
  pds_status all_reduce(void* buf, int64_t count, DType dt, cudaStream_t st) override {
    const int64_t b = count * dt_size(dt);
    PDS_TRY(ensure(b, st));
    publish(buf, st);
    wait_ready(st);
    const void* srcs[8];
    for (int j = 0; j < P; ++j) srcs[j] = g->ptr[j];
    void* tmp = scratch;
    int rc = dt == DT_BF16 ? sum_bf16_p(srcs, P, tmp, count, st) : sum_f32_p(srcs, P, tmp, count, st);
    if (rc) PDS_FAIL(PDS_ECUDA, "loopback all_reduce");
    finish(st);
    PDS_CUDA(cudaMemcpyAsync(buf, tmp, b, cudaMemcpyDeviceToDevice, st));
    return PDS_OK;
  }
  pds_status all_to_all(const void* send, void* recv, int64_t count, DType dt, cudaStream_t st) override {
    const int64_t b = count * dt_size(dt);
    publish(send, st);
    wait_ready(st);
    for (int j = 0; j < P; ++j)
      PDS_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + j * b,
                               static_cast<const char*>(g->ptr[j]) + rank * b, b,
                               cudaMemcpyDeviceToDevice, st));
    finish(st);
    return PDS_OK;
  }
};

Comm* make_loop_comm(LoopGroup* g, int rank, pds_status* st) {
  LoopComm* c = new LoopComm();
  c->g = g;
  c->P = g->P;
  c->rank = rank;
  *st = PDS_OK;
  return c;
}

}  // namespace pds
