#include "comm.hpp"

#include <cuda.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <vector>
#include <cstring>
#include <string>

#include "internal.hpp"

namespace pds {

// defined in kernels/norm.cu
int sum_bf16_p(const void* const* srcs, int P, void* dst, int64_t n, cudaStream_t st);
int sum_f32_p(const void* const* srcs, int P, void* dst, int64_t n, cudaStream_t st);

int64_t dt_size(DType dt) { return dt == DT_BF16 ? 2 : 4; }

// ------------------------------------------------------------------ stream memops
namespace {
typedef CUresult (*PfnWrite32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PfnWait32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
template <class F>
F driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(p);
}
}  // namespace

pds_status stream_write32(cudaStream_t st, uint32_t* addr, uint32_t v) {
  static PfnWrite32 fn = driver_fn<PfnWrite32>("cuStreamWriteValue32");
  if (!fn) PDS_FAIL(PDS_ECUDA, "cuStreamWriteValue32 unavailable");
  // default flags: the write is ordered after (and fenced behind) the stream's prior work
  if (fn((CUstream)st, (CUdeviceptr)addr, v, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
    PDS_FAIL(PDS_ECUDA, "cuStreamWriteValue32 failed");
  return PDS_OK;
}

pds_status stream_wait32_geq(cudaStream_t st, const uint32_t* addr, uint32_t v) {
  static PfnWait32 fn = driver_fn<PfnWait32>("cuStreamWaitValue32");
  if (!fn) PDS_FAIL(PDS_ECUDA, "cuStreamWaitValue32 unavailable");
  if (fn((CUstream)st, (CUdeviceptr)addr, v, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
    PDS_FAIL(PDS_ECUDA, "cuStreamWaitValue32 failed");
  return PDS_OK;
}

// sends to this rank itself: device copies into the matching receives (same tag)
static pds_status self_p2p(int rank, const P2P* sends, int ns, const P2P* recvs, int nr, cudaStream_t st) {
  for (int i = 0; i < ns; ++i) {
    if (sends[i].peer != rank) continue;
    int j = 0;
    while (j < nr && !(recvs[j].peer == rank && recvs[j].tag == sends[i].tag)) ++j;
    if (j == nr || recvs[j].bytes != sends[i].bytes) PDS_FAIL(PDS_EINVAL, "p2p: unmatched self transfer");
    if (recvs[j].ptr != sends[i].ptr)
      PDS_CUDA(cudaMemcpyAsync(recvs[j].ptr, sends[i].ptr, sends[i].bytes, cudaMemcpyDeviceToDevice, st));
  }
  return PDS_OK;
}

// ------------------------------------------------------------------ P = 1
struct SelfComm : Comm {
  pds_status p2p(const P2P* sends, int ns, const P2P* recvs, int nr, cudaStream_t st) override {
    return self_p2p(0, sends, ns, recvs, nr, st);
  }
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

static int side_ctas() {
  static int v = [] {
    const char* e = getenv("PDS_OVERLAP_CTAS");
    const int n = e ? atoi(e) : 8;
    return n < 2 ? 2 : (n > 32 ? 32 : n & ~1);
  }();
  return v;
}

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  NcclComm* side_ = nullptr;
  ~NcclComm() override {
    delete side_;
    if (comm) ncclCommDestroy(comm);
  }
  Comm* side(pds_status* st) override {
    if (!side_) {
      // the side communicator runs beside persistent GEMMs: cap its CTAs, and the
      // GEMMs that poll for it leave that many SMs free (overlap_sm_reserve)
      ncclComm_t c2 = nullptr;
      ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
      cfg.minCTAs = 1;
      cfg.maxCTAs = side_ctas();
      ncclResult_t r = ncclCommSplit(comm, 0, rank, &c2, &cfg);
      if (r != ncclSuccess) {
        set_error(std::string("ncclCommSplit: ") + ncclGetErrorString(r));
        *st = PDS_ENCCL;
        return nullptr;
      }
      side_ = new NcclComm();
      side_->P = P;
      side_->rank = rank;
      side_->comm = c2;
      side_->max_ctas = cfg.maxCTAs;
      // NCCL connects point-to-point peers lazily, which can take a while; connect them
      // now so no tile-polling GEMM ever waits on connection setup
      if (side_->warm_p2p() != PDS_OK) {
        *st = PDS_ENCCL;
        return nullptr;
      }
    }
    return side_;
  }
  pds_status all_gather(const void* send, void* recv, int64_t count, DType dt, cudaStream_t st) override {
    PDS_NCCL(ncclAllGather(send, recv, (size_t)count, nt(dt), comm, st));
    return PDS_OK;
  }
  // one NCCL group; between two ranks, sends and receives match in issue order, so
  // both sides issue their transfers to / from each peer sorted by tag
  pds_status p2p(const P2P* sends, int ns, const P2P* recvs, int nr, cudaStream_t st) override {
    PDS_TRY(self_p2p(rank, sends, ns, recvs, nr, st));
    std::vector<int> si, ri;
    for (int i = 0; i < ns; ++i)
      if (sends[i].peer != rank) si.push_back(i);
    for (int i = 0; i < nr; ++i)
      if (recvs[i].peer != rank) ri.push_back(i);
    std::sort(si.begin(), si.end(), [&](int a, int b) { return sends[a].tag < sends[b].tag; });
    std::sort(ri.begin(), ri.end(), [&](int a, int b) { return recvs[a].tag < recvs[b].tag; });
    PDS_NCCL(ncclGroupStart());
    for (int i : si) PDS_NCCL(ncclSend(sends[i].ptr, (size_t)sends[i].bytes, ncclUint8, sends[i].peer, comm, st));
    for (int i : ri) PDS_NCCL(ncclRecv(recvs[i].ptr, (size_t)recvs[i].bytes, ncclUint8, recvs[i].peer, comm, st));
    PDS_NCCL(ncclGroupEnd());
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
  // P - 1 pairwise steps on the (CTA-limited) side communicator; step k exchanges with
  // ranks rank +- k, so every GPU sends and receives one chunk per step over NVSwitch
  pds_status all_gather_flagged(void* recv, int64_t count, DType dt, cudaStream_t, cudaStream_t st,
                                uint32_t* flags, uint32_t epoch) override {
    const int64_t b = count * dt_size(dt);
    char* base = static_cast<char*>(recv);
    PDS_TRY(stream_write32(st, flags + rank, epoch));     // own chunk: in place already
    for (int k = 1; k < P; ++k) {
      const int from = (rank + k) % P, to = (rank - k + P) % P;
      PDS_NCCL(ncclGroupStart());
      PDS_NCCL(ncclSend(base + rank * b, (size_t)count, nt(dt), to, comm, st));
      PDS_NCCL(ncclRecv(base + from * b, (size_t)count, nt(dt), from, comm, st));
      PDS_NCCL(ncclGroupEnd());
      PDS_TRY(stream_write32(st, flags + from, epoch));
    }
    return PDS_OK;
  }
  pds_status reduce_scatter_gated(const void* send, void* recv, int64_t count, DType dt, cudaStream_t,
                                  cudaStream_t st, const uint32_t* ctr, uint32_t target) override {
    const int64_t b = count * dt_size(dt);
    for (int k = 1; k < P; ++k) {
      const int to = (rank + k) % P, from = (rank - k + P) % P;
      PDS_TRY(stream_wait32_geq(st, ctr + to, target));
      PDS_NCCL(ncclGroupStart());
      PDS_NCCL(ncclSend(static_cast<const char*>(send) + to * b, (size_t)count, nt(dt), to, comm, st));
      PDS_NCCL(ncclRecv(static_cast<char*>(recv) + from * b, (size_t)count, nt(dt), from, comm, st));
      PDS_NCCL(ncclGroupEnd());
    }
    return PDS_OK;
  }
  pds_status all_to_all_gated(const void* send, void* recv, int64_t count, DType dt, cudaStream_t,
                              cudaStream_t st, const uint32_t* ctr, uint32_t target) override {
    const int64_t b = count * dt_size(dt);
    const char* sb = static_cast<const char*>(send);
    char* rb = static_cast<char*>(recv);
    PDS_TRY(stream_wait32_geq(st, ctr + rank, target));
    PDS_CUDA(cudaMemcpyAsync(rb + rank * b, sb + rank * b, b, cudaMemcpyDeviceToDevice, st));
    for (int k = 1; k < P; ++k) {
      const int to = (rank + k) % P, from = (rank - k + P) % P;
      PDS_TRY(stream_wait32_geq(st, ctr + to, target));
      PDS_NCCL(ncclGroupStart());
      PDS_NCCL(ncclSend(sb + to * b, (size_t)count, nt(dt), to, comm, st));
      PDS_NCCL(ncclRecv(rb + from * b, (size_t)count, nt(dt), from, comm, st));
      PDS_NCCL(ncclGroupEnd());
    }
    return PDS_OK;
  }
  int overlap_sm_reserve() const override { return max_ctas; }
  pds_status warm_p2p() {
    void* buf = nullptr;
    cudaStream_t s = nullptr;
    PDS_CUDA(cudaMalloc(&buf, 2 * 256));
    PDS_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    pds_status rc = PDS_OK;
    for (int k = 1; k < P && rc == PDS_OK; ++k) {
      const int to = (rank + k) % P, from = (rank - k + P) % P;
      if (ncclGroupStart() != ncclSuccess ||
          ncclSend(buf, 64, ncclFloat32, to, comm, s) != ncclSuccess ||
          ncclRecv(static_cast<char*>(buf) + 256, 64, ncclFloat32, from, comm, s) != ncclSuccess ||
          ncclGroupEnd() != ncclSuccess) {
        set_error("NCCL point-to-point warm-up failed");
        rc = PDS_ENCCL;
      }
    }
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    cudaFree(buf);
    return rc;
  }
  int max_ctas = 0;
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
    if (ag_done) cudaEventDestroy(ag_done);
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
  // every rank publishes its receive list (a host array); each rank then copies its
  // sends into the matching peer receives once that peer's stream reached the call
  pds_status p2p(const P2P* sends, int ns, const P2P* recvs, int nr, cudaStream_t st) override {
    std::vector<P2P> mine(recvs, recvs + nr);
    mine.push_back(P2P{-1, 0, nullptr, 0});            // terminator
    publish(mine.data(), st);
    for (int i = 0; i < ns; ++i) {
      const P2P* theirs = static_cast<const P2P*>(g->ptr[sends[i].peer]);
      const P2P* m = theirs;
      while (m->peer >= 0 && !(m->peer == rank && m->tag == sends[i].tag)) ++m;
      if (m->peer < 0 || m->bytes != sends[i].bytes) {
        g->barrier();                                   // keep the peers' barrier count
        PDS_FAIL(PDS_EINVAL, "p2p: unmatched loopback transfer");
      }
      if (sends[i].peer != rank) PDS_CUDA(cudaStreamWaitEvent(st, g->ready[sends[i].peer], 0));
      if (m->ptr != sends[i].ptr)
        PDS_CUDA(cudaMemcpyAsync(m->ptr, sends[i].ptr, sends[i].bytes, cudaMemcpyDeviceToDevice, st));
    }
    finish(st);                                         // every peer's copy into our receives is done
    return PDS_OK;
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
  // One GPU hosts every virtual rank, so a persistent GEMM polling for chunks could hold
  // the SMs that a peer's producer kernel (or a copy) needs: here the compute stream
  // waits for the whole gather before the GEMM starts, which still runs the GEMM's
  // flag protocol (epochs, chunk order) but never makes it spin on SM-bound work.
  cudaEvent_t ag_done = nullptr;
  pds_status all_gather_flagged(void* recv, int64_t count, DType dt, cudaStream_t main, cudaStream_t st,
                                uint32_t* flags, uint32_t epoch) override {
    const int64_t b = count * dt_size(dt);
    char* base = static_cast<char*>(recv);
    if (!ag_done) PDS_CUDA(cudaEventCreateWithFlags(&ag_done, cudaEventDisableTiming));
    publish(base + rank * b, st);
    PDS_TRY(stream_write32(st, flags + rank, epoch));     // own chunk: in place already
    for (int k = 1; k < P; ++k) {
      const int j = (rank + k) % P;
      PDS_CUDA(cudaStreamWaitEvent(st, g->ready[j], 0));
      PDS_CUDA(cudaMemcpyAsync(base + j * b, g->ptr[j], b, cudaMemcpyDeviceToDevice, st));
      PDS_TRY(stream_write32(st, flags + j, epoch));
    }
    finish(st);
    PDS_CUDA(cudaEventRecord(ag_done, st));
    PDS_CUDA(cudaStreamWaitEvent(main, ag_done, 0));
    return PDS_OK;
  }
  pds_status reduce_scatter_gated(const void* send, void* recv, int64_t count, DType dt, cudaStream_t,
                                  cudaStream_t st, const uint32_t* ctr, uint32_t target) override {
    const int64_t b = count * dt_size(dt);
    publish(recv, st);                          // this rank's receive buffer is free
    for (int k = 1; k < P; ++k) {
      const int j = (rank + k) % P;
      PDS_TRY(stream_wait32_geq(st, ctr + j, target));
      PDS_CUDA(cudaStreamWaitEvent(st, g->ready[j], 0));
      PDS_CUDA(cudaMemcpyAsync(static_cast<char*>(const_cast<void*>(g->ptr[j])) + rank * b,
                               static_cast<const char*>(send) + j * b, b, cudaMemcpyDeviceToDevice, st));
    }
    finish(st);                                 // every peer's copy into recv is done
    return PDS_OK;
  }
  pds_status all_to_all_gated(const void* send, void* recv, int64_t count, DType dt, cudaStream_t,
                              cudaStream_t st, const uint32_t* ctr, uint32_t target) override {
    const int64_t b = count * dt_size(dt);
    const char* sb = static_cast<const char*>(send);
    publish(recv, st);                          // this rank's receive buffer is free
    PDS_TRY(stream_wait32_geq(st, ctr + rank, target));
    PDS_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + rank * b, sb + rank * b, b, cudaMemcpyDeviceToDevice, st));
    for (int k = 1; k < P; ++k) {
      const int j = (rank + k) % P;
      PDS_TRY(stream_wait32_geq(st, ctr + j, target));
      PDS_CUDA(cudaStreamWaitEvent(st, g->ready[j], 0));
      PDS_CUDA(cudaMemcpyAsync(static_cast<char*>(const_cast<void*>(g->ptr[j])) + rank * b, sb + j * b, b,
                               cudaMemcpyDeviceToDevice, st));
    }
    finish(st);                                 // every peer's block has landed in recv
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
