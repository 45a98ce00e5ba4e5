// The switchable functional parallelism library:
// one Transformer layer f_{pi,FFN} o f_{pi,MHA} per strategy pi, forward and
// backward, over the unified boundary layout [s/P, b, h] (Table 2 spec row,
// PAPER.md:139).  Every strategy consumes and produces the same layout, so a
// layer-wise switch is a different function pointer, never a redistribution
// (PAPER.md:45, 224, 294).
//
//   MegatronTS  AG(s) -> column-parallel QKV(+RoPE) / FC1(+GELU) -> row-parallel
//               proj / FC2 -> RS(s)
//   UlyssesZ    AG(weights, ZeRO3) -> local QKV packed per head group -> A2A
//               seq->heads -> attention -> A2A heads->seq
//   METP        the TS dataflow in c waves of s/(Pc) rows per rank, per-wave AG/RS,
//               GEMMs reading / writing position-ordered buffers through TMA row
//               remaps (no gather copies), FFN recomputed in bwd  (R-11)
//
// Readings R-1..R-36 of DESIGN.md; buffer plan in planner.cpp (make_plan).
#include <cmath>
#include <functional>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include <cstdio>
#include <nvtx3/nvToolsExt.h>

#include "comm.hpp"
#include "internal.hpp"
#include "kernels/gemm.cuh"
#include "kernels/kernels.hpp"

using namespace pds;

struct ProfRec {
  int klass;
  cudaEvent_t a, b;
  double flops, bytes;
};

struct pds_saved {
  int strategy;
  int64_t s;
  const int* segs = nullptr;     // varlen table of the forward (R-VARLEN), reused by the backward
  const void* x;
  char* mem;
  int64_t bytes;
  BufPlan plan;
  char* at(const char* n) const { return mem + plan.saved_off(n); }
};

struct pds_group {
  LoopGroup g;
};

struct pds_ctx {
  pds_model m{};
  int P = 1, rank = 0, device = 0;
  Comm* comm = nullptr;
  // rope table (float2 [rope_pos][d/2])
  void* rope = nullptr;
  int64_t rope_pos = 0;
  // workspace
  char* ws = nullptr;
  int64_t ws_cap = 0;
  // saved arena: cached blocks by size
  std::multimap<int64_t, char*> free_blocks;
  int64_t saved_live = 0;
  // planner
  Bundle bundle;
  double capacity = 0, gamma = 0;
  uint32_t enabled = (1u << PDS_N_STRATEGIES) - 1;
  std::map<std::pair<int, int64_t>, std::pair<std::vector<uint8_t>, bool>> cache;
  std::vector<uint8_t> prev;
  // varlen packing (R-VARLEN, pds_set_varlen): the device segment table of the current
  // setting (NULL: one sequence) for seq_len = varlen_tokens; every table stays alive
  // until the context is destroyed (a saved set may still point at an older one)
  const int* segs = nullptr;
  int64_t varlen_tokens = 0;
  std::vector<int*> seg_tables;
  // debug taps
  void* tap_o = nullptr;
  void* tap_z = nullptr;
  // host-buffer steps (pds_layer_step_host): two staging sets of x, dy, y, dx used by
  // alternate calls, an upload and a download stream
  char* stage = nullptr;
  int64_t stage_cap = 0;       // bytes of one set
  int stage_next = 0;
  bool stage_used[2] = {false, false};
  cudaStream_t up_st = nullptr, down_st = nullptr;
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr}, ev_y = nullptr, ev_dx = nullptr;
  // side stream for collectives overlapped with compute (METP wave prefetch, TS tiles)
  cudaStream_t comm_st = nullptr;
  // tile-overlapped collectives (P > 1): device words [0, 8) = chunk-landed flags of the
  // all-gathers, [8, 16) = per-chunk store counters of the GEMMs feeding a
  // reduce-scatter, [16, 24) = per-block counters of the GEMMs feeding an all-to-all;
  // host-side epoch / running targets
  uint32_t* sync = nullptr;
  uint32_t ag_epoch = 0, rs_count = 0, a2a_count = 0;
  int overlap = 1;
  std::vector<cudaEvent_t> sync_pool;
  // comm log (JSON lines {"primitive", "bytes", "participants"}, the oracle
  // grid's convention: bytes this rank sends), pds_comm_log / pds_comm_log_read
  bool comm_log_on = false;
  std::string comm_log;
  // profiling
  bool prof = false;
  std::vector<ProfRec> pending;
  std::vector<cudaEvent_t> ev_pool;
  double acc_ms[5] = {0}, acc_flops[5] = {0}, acc_bytes[5] = {0};
  int64_t acc_n[5] = {0};

  ~pds_ctx() {
    for (auto& r : pending) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : ev_pool) cudaEventDestroy(e);
    for (auto& kv : free_blocks) cudaFree(kv.second);
    if (ws) cudaFree(ws);
    if (rope) cudaFree(rope);
    if (stage) cudaFree(stage);
    for (cudaEvent_t e : {ev_in[0], ev_in[1], ev_done[0], ev_done[1], ev_y, ev_dx})
      if (e) cudaEventDestroy(e);
    if (up_st) cudaStreamDestroy(up_st);
    if (down_st) cudaStreamDestroy(down_st);
    if (comm_st) cudaStreamDestroy(comm_st);
    if (sync) cudaFree(sync);
    for (int* t : seg_tables) cudaFree(t);
    for (auto e : sync_pool) cudaEventDestroy(e);
    delete comm;
  }
  cudaEvent_t ev() {
    if (!ev_pool.empty()) {
      cudaEvent_t e = ev_pool.back();
      ev_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};

namespace {

enum { K_GEMM = 0, K_ATTN_F = 1, K_ATTN_B = 2, K_NORM = 3, K_COMM = 4 };

// NVTX range per launch class (SURVEY §5 tracing): visible in nsys / ncu --nvtx; a
// no-op without an attached tool
const char* const kProfName[5] = {"pds:gemm", "pds:attn_fwd", "pds:attn_bwd", "pds:elementwise", "pds:comm"};
const char* const kLayerName[PDS_N_STRATEGIES][2] = {
    {"pds_layer_fwd MegatronTS", "pds_layer_bwd MegatronTS"}, {"pds_layer_fwd UlyssesZ", "pds_layer_bwd UlyssesZ"},
    {"pds_layer_fwd METP", "pds_layer_bwd METP"}, {"pds_layer_fwd MegatronCZ", "pds_layer_bwd MegatronCZ"},
    {"pds_layer_fwd METP-full", "pds_layer_bwd METP-full"}, {"pds_layer_fwd ColossalZ", "pds_layer_bwd ColossalZ"}};

struct Prof {
  pds_ctx* c;
  cudaStream_t st;
  int k;
  double fl, by;
  cudaEvent_t a = nullptr;
  Prof(pds_ctx* c_, cudaStream_t s_, int k_, double f_, double b_) : c(c_), st(s_), k(k_), fl(f_), by(b_) {
    nvtxRangePushA(kProfName[k]);
    if (c->prof) {
      a = c->ev();
      cudaEventRecord(a, st);
    }
  }
  ~Prof() {
    nvtxRangePop();
    if (a) {
      cudaEvent_t b = c->ev();
      cudaEventRecord(b, st);
      c->pending.push_back(ProfRec{k, a, b, fl, by});
    }
  }
};

pds_status kerr(int rc, const char* what) {
  if (rc == 0) return PDS_OK;
  set_error(std::string(what) + ": " + cudaGetErrorString((cudaError_t)rc));
  return rc == (int)cudaErrorMemoryAllocation ? PDS_ENOMEM : PDS_ECUDA;
}

struct Exec {
  pds_ctx* c;
  cudaStream_t st;
  const pds_model& m;
  int P, r;
  // s, sl: TOKEN ROWS (all / this rank) of the [s, b, h] layout = positions x b; every
  // GEMM, norm and collective counts rows.  sq, sp: positions (attention, RoPE).
  int64_t b, sq, sp, s, sl, h, F, nl, d, hl, Fl;
  // Llama variant (R-GQA / R-SWIGLU): nkl local key/value heads, qw / qwf the local /
  // full Q|K|V widths (3 hl / 3 h for MHA), f1w / f1wf the local / full FC1 output
  // widths (Fl / F; 2 Fl / 2 F with SwiGLU's interleaved [gate | up])
  int64_t nkl, qw, qwf, f1w, f1wf;
  bool swi;
  const int* segs;                   // varlen segment table (R-VARLEN) or NULL
  Exec(pds_ctx* c_, cudaStream_t st_, int64_t s_, const int* segs_ = nullptr)
      : c(c_), st(st_), m(c_->m), P(c_->P), r(c_->rank), b(c_->m.batch), sq(s_), sp(s_ / c_->P),
        s(s_ * c_->m.batch), sl(s_ / c_->P * c_->m.batch), h(c_->m.h), F(c_->m.ffn),
        nl(c_->m.n_heads / c_->P), d(c_->m.h / c_->m.n_heads), hl(c_->m.h / c_->P), Fl(c_->m.ffn / c_->P) {
    segs = segs_;
    nkl = (c_->m.n_kv_heads > 0 ? c_->m.n_kv_heads : c_->m.n_heads) / c_->P;
    qw = (nl + 2 * nkl) * d;
    qwf = qw * c_->P;
    swi = c_->m.ffn_act == 1;
    f1w = swi ? 2 * Fl : Fl;
    f1wf = swi ? 2 * F : F;
  }
  int fc1_epi() const { return swi ? EPI_SWIGLU : EPI_GELU; }
  int dfc1_epi() const { return swi ? EPI_DSWIGLU : EPI_DGELU; }

  // overlap settings armed for the next gemm() (ag_next / rs_arm / a2a_arm); a store
  // counter's running host target advances only once that GEMM has been launched, so
  // a failed launch never leaves a later stream wait behind an unreachable value
  GemmArgs nxt;
  bool has_nxt = false;
  cudaEvent_t nxt_join = nullptr;
  uint32_t* nxt_count = nullptr;
  uint32_t nxt_count_value = 0;

  pds_status gemm(GemmArgs g) {
    // algorithmic bytes: A and B once, C by epilogue (fp32 += reads and writes; GELU /
    // dGELU add the bf16 aux streams)
    const double mn = (double)g.M * g.N;
    const double cb = g.epi == EPI_F32_ACC ? 8.0 : g.epi == EPI_F32 ? 4.0 : g.epi == EPI_GELU ? 4.0
                    : g.epi == EPI_DGELU ? 6.0 : g.epi == EPI_SWIGLU ? 3.0 : g.epi == EPI_DSWIGLU ? 12.0 : 2.0;
    if (has_nxt) {
      g.wait_flags = nxt.wait_flags; g.flag_epoch = nxt.flag_epoch; g.done_ctr = nxt.done_ctr;
      g.chunk_rows = nxt.chunk_rows; g.m_rot_rows = nxt.m_rot_rows; g.sm_reserve = nxt.sm_reserve;
      g.chunk_cols = nxt.chunk_cols; g.n_rot_cols = nxt.n_rot_cols;
      has_nxt = false;
      nxt = GemmArgs();
    }
    {
      Prof p(c, st, K_GEMM, 2.0 * g.M * g.N * g.K, 2.0 * ((double)g.M + g.N) * g.K + cb * mn);
      PDS_TRY(kerr(gemm_launch(g, st), "gemm"));
    }
    if (nxt_count) {
      *nxt_count = nxt_count_value;
      nxt_count = nullptr;
    }
    if (nxt_join) {                      // the all-gather this GEMM consumed, joined
      cudaEvent_t ev = nxt_join;
      nxt_join = nullptr;
      PDS_TRY(wait(st, ev));
    }
    return PDS_OK;
  }

  // ---- tile-overlapped MegatronTS collectives ----
  bool overlap() const { return P > 1 && c->overlap && !c->comm->trivial(); }
  pds_status sync_init() {
    if (c->sync) return PDS_OK;
    PDS_CUDA(cudaMalloc(&c->sync, 32 * sizeof(uint32_t)));
    PDS_CUDA(cudaMemsetAsync(c->sync, 0, 32 * sizeof(uint32_t), st));
    return PDS_OK;
  }
  // AG of buf [P][count] (this rank's chunk already at slot r) on the side stream, chunk
  // by chunk, consumed tile by tile by the next gemm(), whose A operand is buf
  pds_status ag_next(void* buf, int64_t count, int64_t rows = 0) {
    if (!rows) rows = sl;                    // rows per rank chunk (METP: one wave's)
    PDS_TRY(sync_init());
    cudaStream_t cs = comm_stream();
    PDS_TRY(link(st, cs));
    pds_status rc = PDS_OK;
    Comm* cm = c->comm->side(&rc);
    if (!cm) return rc;
    const uint32_t epoch = ++c->ag_epoch;
    log_comm("AllGather", (double)count * 2 * (P - 1));
    {
      Prof p(c, cs, K_COMM, 0, (double)count * 2 * (P - 1));
      PDS_TRY(cm->all_gather_flagged(buf, count, DT_BF16, st, cs, c->sync, epoch));
    }
    nxt = GemmArgs();
    nxt.wait_flags = c->sync; nxt.flag_epoch = epoch;
    nxt.chunk_rows = rows; nxt.m_rot_rows = (int64_t)r * rows;
    nxt.sm_reserve = cm->overlap_sm_reserve();
    has_nxt = true;
    nxt_join = mark(cs);
    return PDS_OK;
  }
  // arm the next gemm() (output [P][sl][ncols], all rows) to count its stores per chunk,
  // computing the chunk sent first (r+1) first and its own chunk last
  uint32_t rs_target = 0;
  pds_status rs_arm(int64_t ncols, int64_t rows = 0) {
    if (!rows) rows = sl;
    PDS_TRY(sync_init());
    PDS_TRY(link(st, comm_stream()));        // the receive buffer's readers are done
    pds_status rc = PDS_OK;
    Comm* cm = c->comm->side(&rc);
    if (!cm) return rc;
    rs_target = c->rs_count + (uint32_t)(rows * ncols / 8);     // counted in units of 8 elements
    nxt_count = &c->rs_count;
    nxt_count_value = rs_target;
    nxt = GemmArgs();
    nxt.done_ctr = c->sync + 8;
    nxt.chunk_rows = rows; nxt.m_rot_rows = (int64_t)((r + 1) % P) * rows;
    nxt.sm_reserve = cm->overlap_sm_reserve();
    has_nxt = true;
    return PDS_OK;
  }
  // arm the next gemm() (column-blocked output [P][sl][blk], block j for rank j) to
  // count its stores per block, computing the block sent first (r+1) first
  uint32_t a2a_target = 0;
  pds_status a2a_arm(int64_t blk) {
    PDS_TRY(sync_init());
    PDS_TRY(link(st, comm_stream()));        // the receive buffer's readers are done
    pds_status rc = PDS_OK;
    Comm* cm = c->comm->side(&rc);
    if (!cm) return rc;
    a2a_target = c->a2a_count + (uint32_t)(sl * blk / 8);
    nxt_count = &c->a2a_count;
    nxt_count_value = a2a_target;
    nxt = GemmArgs();
    nxt.done_ctr = c->sync + 16;
    nxt.chunk_cols = blk; nxt.n_rot_cols = (int64_t)((r + 1) % P) * blk;
    nxt.sm_reserve = cm->overlap_sm_reserve();
    has_nxt = true;
    return PDS_OK;
  }
  // after the armed gemm(): the All-to-All, each block leaving as soon as it is stored
  pds_status a2a_run(const char* send, char* recv, int64_t count) {
    cudaStream_t cs = comm_stream();
    pds_status rc = PDS_OK;
    Comm* cm = c->comm->side(&rc);
    if (!cm) return rc;
    log_comm("AllToAll", (double)count * 2 * (P - 1));
    {
      Prof p(c, cs, K_COMM, 0, (double)count * 2 * (P - 1));
      PDS_TRY(cm->all_to_all_gated(send, recv, count, DT_BF16, st, cs, c->sync + 16, a2a_target));
    }
    return link(cs, st);
  }
  // after the armed gemm(): send each finished chunk of `partial` to its owner, receive
  // the peers' partials of this rank's chunk into recv [P][count], and sum them (rank
  // order, fp32) into partial + r*count: the reduce-scatter, overlapped with the GEMM
  pds_status rs_run(char* partial, char* recv, int64_t count) {
    cudaStream_t cs = comm_stream();
    pds_status rc = PDS_OK;
    Comm* cm = c->comm->side(&rc);
    if (!cm) return rc;
    log_comm("ReduceScatter", (double)count * 2 * (P - 1));
    {
      Prof p(c, cs, K_COMM, 0, (double)count * 2 * (P - 1));
      PDS_TRY(cm->reduce_scatter_gated(partial, recv, count, DT_BF16, st, cs, c->sync + 8, rs_target));
    }
    PDS_TRY(link(cs, st));
    const int64_t b = count * 2;
    const void* srcs[8];
    for (int j = 0; j < P; ++j) srcs[j] = j == r ? partial + j * b : recv + j * b;
    Prof p(c, st, K_NORM, 0, (double)count * 2 * (P + 1));
    return kerr(sum_bf16_p(srcs, P, partial + r * b, count, st), "sum_bf16_p");
  }
  // C[M,N] = A * B^T helpers
  static GemmArgs G(const void* A, int64_t lda, int a_mn, const void* B, int64_t ldb, int b_mn, int64_t M,
                    int64_t N, int64_t K, void* C, int64_t ldc, int epi = EPI_BF16) {
    GemmArgs g;
    g.A = A; g.lda = lda; g.a_mn = a_mn; g.B = B; g.ldb = ldb; g.b_mn = b_mn;
    g.M = (int)M; g.N = (int)N; g.K = (int)K; g.C = C; g.ldc = ldc; g.epi = epi;
    return g;
  }
  // hq / hk: the Q and the K (= V) widths of one [Q | K | V] column group (the local
  // head group for TS / METP / UlyssesZ, all heads for MegatronCZ / ColossalZ)
  GemmArgs rope(GemmArgs g, int64_t hq, int64_t hk, int64_t seg, int64_t seg_stride, int64_t seg_base) {
    g.epi = EPI_ROPE;
    g.rope = reinterpret_cast<const float2*>(c->rope);
    g.rope_d = (int)d;
    g.rope_hq = (int)hq;
    g.rope_hk = (int)hk;
    g.seg = seg; g.seg_stride = seg_stride; g.seg_base = seg_base;
    g.rope_b = (int)b;                 // row -> position: the mapped row / b
    g.rope_segs = segs;                // varlen: positions restart at every sequence
    return g;
  }
  pds_status norm_fwd(const void* x, const void* res, const void* g, int64_t rows, void* x1, void* u, void* rstd) {
    Prof p(c, st, K_NORM, 0, (double)rows * h * (res ? 8 : 4) + rows * 4);
    return kerr(rmsnorm_fwd(x, res, g, rows, (int)h, m.norm_eps, x1, u, rstd, st), "rmsnorm_fwd");
  }
  pds_status norm_bwd(const void* du, const void* x, const void* rstd, const void* g, const void* dres,
                      int64_t rows, void* dx, float* dgp, float* dg) {
    Prof p(c, st, K_NORM, 0, (double)rows * h * (dres ? 8 : 6));
    return kerr(rmsnorm_bwd(du, x, rstd, g, dres, rows, (int)h, dx, dgp, dg, st), "rmsnorm_bwd");
  }
  pds_status apply(const void* x, const void* rstd, const void* g, int64_t rows, void* u) {
    Prof p(c, st, K_NORM, 0, (double)rows * h * 4);
    return kerr(apply_norm(x, rstd, g, rows, (int)h, u, st), "apply_norm");
  }
  pds_status add(const void* a, const void* b, void* out, int64_t n) {
    Prof p(c, st, K_NORM, 0, (double)n * 6);
    return kerr(add_bf16(a, b, out, n, st), "add_bf16");
  }
  // attention over the sq positions of each of the b sequences: sequence bi is every
  // b-th row of the [s, b, .] buffers (row stride b x ld), LSE / D [b][heads][sq]
  pds_status attn_f(const void* qkv, void* out, void* lse) {
    const double fl = b * 4.0 * nl * d * (m.causal ? 0.5 * sq * sq : (double)sq * sq);
    Prof p(c, st, K_ATTN_F, fl, 0);
    for (int64_t bi = 0; bi < b; ++bi)
      PDS_TRY(kerr(attn_fwd(static_cast<const char*>(qkv) + bi * qw * 2, qw * b, (int)sq, (int)nl, (int)d,
                            m.causal, static_cast<char*>(out) + bi * hl * 2, hl * b,
                            static_cast<float*>(lse) + bi * nl * sq, st, (int)nkl, segs), "attn_fwd"));
    return PDS_OK;
  }
  // sc: the fused backward's scratch (an fp32 dQ accumulator of sc_bytes >= nl sq d 4,
  // a workspace region that is free during the attention backward) and its counters;
  // NULL selects the split kernels
  pds_status attn_b(const void* qkv, const void* out, const void* lse, const void* dout, void* dqkv, float* dd,
                    void* sc = nullptr, int64_t sc_bytes = 0, int* ctr = nullptr, void* dsb = nullptr,
                    int64_t dsb_bytes = 0) {
    const double fl = b * 10.0 * nl * d * (m.causal ? 0.5 * sq * sq : (double)sq * sq);
    Prof p(c, st, K_ATTN_B, fl, 0);
    float* acc = sc && ctr && sc_bytes >= nl * sq * d * 4 ? static_cast<float*>(sc) : nullptr;
    for (int64_t bi = 0; bi < b; ++bi)
      PDS_TRY(kerr(attn_bwd(static_cast<const char*>(qkv) + bi * qw * 2, qw * b,
                            static_cast<const char*>(out) + bi * hl * 2, hl * b,
                            static_cast<const float*>(lse) + bi * nl * sq, static_cast<const char*>(dout) + bi * hl * 2,
                            (int)sq, (int)nl, (int)d, m.causal, static_cast<char*>(dqkv) + bi * qw * 2, c->rope,
                            dd + bi * nl * sq, st, acc, acc ? ctr : nullptr, (int)nkl, segs, dsb, dsb_bytes),
                   "attn_bwd"));
    return PDS_OK;
  }
  // collectives
  pds_status ag(const void* send, void* recv, int64_t count, DType dt = DT_BF16) {
    log_comm("AllGather", (double)count * dt_size(dt) * (P - 1));
    Prof p(c, st, K_COMM, 0, (double)count * dt_size(dt) * (P - 1));
    return c->comm->all_gather(send, recv, count, dt, st);
  }
  // all_gather on another stream (the caller orders it with link())
  pds_status ag_on(cudaStream_t s2, const void* send, void* recv, int64_t count) {
    pds_status rc = PDS_OK;
    Comm* cm = s2 == st ? c->comm : c->comm->side(&rc);
    if (!cm) return rc;
    log_comm("AllGather", (double)count * 2 * (P - 1));
    Prof p(c, s2, K_COMM, 0, (double)count * 2 * (P - 1));
    return cm->all_gather(send, recv, count, DT_BF16, s2);
  }
  cudaStream_t comm_stream() {
    if (!c->comm_st) cudaStreamCreateWithFlags(&c->comm_st, cudaStreamNonBlocking);
    return c->comm_st;
  }
  // an event marking everything enqueued on `s` so far; consume it with wait()
  cudaEvent_t mark(cudaStream_t s) {
    cudaEvent_t ev;
    if (c->sync_pool.empty()) {
      cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    } else {
      ev = c->sync_pool.back();
      c->sync_pool.pop_back();
    }
    cudaEventRecord(ev, s);
    return ev;
  }
  pds_status wait(cudaStream_t s, cudaEvent_t ev) {
    PDS_CUDA(cudaStreamWaitEvent(s, ev, 0));
    c->sync_pool.push_back(ev);
    return PDS_OK;
  }
  cudaStream_t side_stream() { return c->comm->trivial() ? st : comm_stream(); }
  // `to` waits for everything enqueued on `from` so far
  pds_status link(cudaStream_t from, cudaStream_t to) {
    if (from == to) return PDS_OK;
    cudaEvent_t ev;
    if (c->sync_pool.empty()) {
      PDS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    } else {
      ev = c->sync_pool.back();
      c->sync_pool.pop_back();
    }
    PDS_CUDA(cudaEventRecord(ev, from));
    PDS_CUDA(cudaStreamWaitEvent(to, ev, 0));
    c->sync_pool.push_back(ev);       // the wait captured this record; the event may be reused
    return PDS_OK;
  }
  pds_status rs(const void* send, void* recv, int64_t count, DType dt = DT_BF16) {
    log_comm("ReduceScatter", (double)count * dt_size(dt) * (P - 1));
    Prof p(c, st, K_COMM, 0, (double)count * dt_size(dt) * (P - 1));
    return c->comm->reduce_scatter(send, recv, count, dt, st);
  }
  pds_status p2p(const P2P* sends, int ns, const P2P* recvs, int nr, cudaStream_t on, const char* prim = "SendRecv") {
    pds_status rc = PDS_OK;
    Comm* cm = on == st ? c->comm : c->comm->side(&rc);
    if (!cm) return rc;
    double bytes = 0;
    for (int i = 0; i < ns; ++i)
      if (sends[i].peer != r) bytes += (double)sends[i].bytes;
    log_comm(prim, bytes);
    Prof p(c, on, K_COMM, 0, bytes);
    return cm->p2p(sends, ns, recvs, nr, on);
  }
  pds_status a2a(const void* send, void* recv, int64_t count) {
    log_comm("AllToAll", (double)count * 2 * (P - 1));
    Prof p(c, st, K_COMM, 0, (double)count * 2 * (P - 1));
    return c->comm->all_to_all(send, recv, count, DT_BF16, st);
  }
  pds_status dgamma(float* dgl, const pds_grads* g) {
    log_comm("AllReduce", 2.0 * (P - 1) / P * 2 * h * 4);       // ring all-reduce payload
    {
      Prof p(c, st, K_COMM, 0, 2.0 * h * 4 * 2 * (P - 1));
      PDS_TRY(c->comm->all_reduce(dgl, 2 * h, DT_F32, st));
    }
    PDS_TRY(kerr(add_f32(dgl, g->dg1, h, st), "add_f32"));
    return kerr(add_f32(dgl + h, g->dg2, h, st), "add_f32");
  }
  pds_status tap(void* dst, const void* src, int64_t n) {
    if (!dst) return PDS_OK;
    PDS_CUDA(cudaMemcpyAsync(dst, src, n * 2, cudaMemcpyDeviceToDevice, st));
    return PDS_OK;
  }
  // one comm-log record: the bytes this rank sends (oracle/grid.py's payload convention)
  void log_comm(const char* prim, double bytes) {
    if (!c->comm_log_on || P == 1) return;
    char buf[160];
    std::snprintf(buf, sizeof buf, "{\"primitive\": \"%s\", \"bytes\": %.0f, \"participants\": %d}\n", prim, bytes, P);
    c->comm_log += buf;
  }
};

#define B16(p) (reinterpret_cast<char*>(p))

// Every GEMM is issued TN (both operands K-major), the layout the tcgen05 GEMM runs
// at full rate: weight operands that the math needs MN-major are transposed into
// `wt` per call (weights are small), and the token-major activations of the dW
// GEMMs (contraction over tokens) into `ta` / `tb`.
struct TN {
  Exec& e;
  char *ta, *tb, *wt;
  // C[M,N] (+)= A[M,K] B[N,K]^T with both operands K-major
  pds_status mm(const void* A, int64_t lda, const void* B, int64_t ldb, int64_t M, int64_t N, int64_t K, void* C,
                int64_t ldc, int epi = EPI_BF16) {
    return e.gemm(Exec::G(A, lda, 0, B, ldb, 0, M, N, K, C, ldc, epi));
  }
  // X [rows][cols] (rows optionally remapped) -> dst [cols][rows]
  pds_status tr(const void* X, int64_t ldx, int64_t rows, int64_t cols, void* dst, int64_t seg = 0,
                int64_t stride = 0, int64_t base = 0) {
    Prof p(e.c, e.st, K_NORM, 0, 4.0 * rows * cols);
    return kerr(transpose_bf16(X, ldx, rows, cols, dst, rows, seg, stride, base, e.st), "transpose");
  }
  // C[M,N] += Xa^T Xb over T tokens: Xa [T][M], Xb [T][N] token-major (dW GEMM)
  pds_status dw(const void* Xa, int64_t lda, const void* Xb, int64_t ldb, int64_t T, int64_t M, int64_t N, void* C,
                int epi = EPI_F32_ACC, int64_t seg = 0, int64_t stride = 0, int64_t base = 0) {
    PDS_TRY(tr(Xa, lda, T, M, ta, seg, stride, base));
    PDS_TRY(tr(Xb, ldb, T, N, tb));
    return mm(ta, T, tb, T, M, N, T, C, N, epi);
  }
  // C[M,N] = X[M,K] W[K,N] for a weight stored [K][N]: transpose W into wt [N][K]
  pds_status xw(const void* X, int64_t ldx, const void* W, int64_t ldw, int64_t M, int64_t N, int64_t K, void* C,
                int64_t ldc, int64_t aseg = 0, int64_t astride = 0, int64_t abase = 0, int64_t arows = 0) {
    PDS_TRY(tr(W, ldw, K, N, wt));
    GemmArgs g = Exec::G(X, ldx, 0, wt, K, 0, M, N, K, C, ldc);
    g.a_seg = aseg; g.a_stride = astride; g.a_base = abase; g.a_rows = arows;
    return e.gemm(g);
  }
};

// ================================================================== MegatronTS
pds_status ts_fwd(Exec& e, const void* x, const pds_weights* w, void* y, pds_saved* sv, char* ws) {
  const BufPlan& bp = sv->plan;
  char* gather = ws + bp.ws_off("gather");
  char* partial = ws + bp.ws_off("partial");
  char* f0 = ws + bp.ws_off("f0");
  TN tn{e, ws + bp.ws_off("ta"), ws + bp.ws_off("tb"), ws + bp.ws_off("wt")};
  const int64_t slot = e.r * e.sl * e.h * 2;
  // P > 1: every AG runs chunk by chunk on the side stream while the GEMM that reads it
  // computes the chunks already there (ag_next), and every RS sends each chunk of the
  // GEMM's output as soon as its tiles are stored (rs_arm / rs_run), the gather buffer
  // (free by then) receiving the peers' partials
  const bool ov = e.overlap();
  const int64_t n = e.sl * e.h;
  PDS_TRY(e.norm_fwd(x, nullptr, w->g1, e.sl, nullptr, gather + slot, sv->at("rstd1")));
  PDS_TRY(ov ? e.ag_next(gather, n) : e.ag(gather + slot, gather, n));                // AG(u)
  PDS_TRY(e.gemm(e.rope(Exec::G(gather, e.h, 0, w->w_qkv_t, e.h, 0, e.s, e.qw, e.h, sv->at("qkv"), e.qw),
                        e.hl, e.nkl * e.d, 0, 0, 0)));                                                // Eq. 1 + RoPE
  PDS_TRY(e.attn_f(sv->at("qkv"), sv->at("a"), sv->at("lse")));                          // Eq. 2
  if (ov) PDS_TRY(e.rs_arm(e.h));
  PDS_TRY(tn.xw(sv->at("a"), e.hl, w->w_proj, e.h, e.s, e.h, e.hl, partial, e.h));      // Eq. 3
  PDS_TRY(ov ? e.rs_run(partial, gather, n) : e.rs(partial, partial + slot, n));        // RS(o)
  PDS_TRY(e.tap(e.c->tap_o, partial + slot, e.sl * e.h));
  PDS_TRY(e.norm_fwd(x, partial + slot, w->g2, e.sl, sv->at("x1"), gather + slot, sv->at("rstd2")));
  PDS_TRY(ov ? e.ag_next(gather, n) : e.ag(gather + slot, gather, n));                // AG(v)
  GemmArgs fc1 = Exec::G(gather, e.h, 0, w->w_in_t, e.h, 0, e.s, e.f1w, e.h, sv->at("h"), e.f1w, e.fc1_epi());
  fc1.aux_out = f0; fc1.ld_aux = e.Fl;
  PDS_TRY(e.gemm(fc1));                                                                 // Eq. 4 (GELU / SwiGLU)
  if (ov) PDS_TRY(e.rs_arm(e.h));
  PDS_TRY(tn.xw(f0, e.Fl, w->w_out, e.h, e.s, e.h, e.Fl, partial, e.h));
  PDS_TRY(ov ? e.rs_run(partial, gather, n) : e.rs(partial, partial + slot, n));        // RS(z)
  PDS_TRY(e.tap(e.c->tap_z, partial + slot, e.sl * e.h));
  return e.add(sv->at("x1"), partial + slot, y, e.sl * e.h);
}

pds_status ts_bwd(Exec& e, const void* dy, pds_saved* sv, const pds_weights* w, const pds_grads* g, void* dx,
                  char* ws) {
  const BufPlan& bp = sv->plan;
  char* gather = ws + bp.ws_off("gather");
  char* partial = ws + bp.ws_off("partial");
  char* f0 = ws + bp.ws_off("f0");
  char* f1 = ws + bp.ws_off("f1");
  float* dd = reinterpret_cast<float*>(ws + bp.ws_off("dd"));
  float* dgp = reinterpret_cast<float*>(ws + bp.ws_off("dgp"));
  float* dgl = reinterpret_cast<float*>(ws + bp.ws_off("dgl"));
  TN tn{e, ws + bp.ws_off("ta"), ws + bp.ws_off("tb"), ws + bp.ws_off("wt")};
  const int64_t slot = e.r * e.sl * e.h * 2;
  PDS_CUDA(cudaMemsetAsync(dgl, 0, 2 * e.h * 4, e.st));
  // P > 1: the re-gathers of v and u (for dW_in and dW_qkv) go into a second gather
  // buffer on the side stream, overlapping the dG / dW_out GEMMs resp. the attention
  // backward; P = 1 keeps one buffer and program order (the gathers are identities).
  const bool pre = bp.has_ws("gather2");
  char* g2 = pre ? ws + bp.ws_off("gather2") : gather;
  const cudaStream_t cs = pre ? e.side_stream() : e.st;
  cudaEvent_t ev_v = nullptr, ev_u = nullptr;
  // tile-overlapped AG / RS as in the forward (P > 1); the side stream carries the
  // flagged gathers first, then the re-gathers
  const bool ov = e.overlap();
  const int64_t n = e.sl * e.h;
  if (ov) {
    PDS_CUDA(cudaMemcpyAsync(gather + slot, dy, n * 2, cudaMemcpyDeviceToDevice, e.st));
    PDS_TRY(e.ag_next(gather, n));                                                    // AG(dz)
  }
  if (pre) {
    PDS_TRY(e.apply(sv->at("x1"), sv->at("rstd2"), w->g2, e.sl, g2 + slot));
    PDS_TRY(e.link(e.st, cs));
    PDS_TRY(e.ag_on(cs, g2 + slot, g2, e.sl * e.h));                                  // AG(v) re-gather
    ev_v = e.mark(cs);
  }
  if (!ov) PDS_TRY(e.ag(dy, gather, n));                                                // AG(dz)
  // dH (row-major, for dV) plus the two operands the dW GEMMs need K-major, straight
  // from the epilogue: dH^T into f0, G^T into ta (G itself is never stored)
  GemmArgs dgel = Exec::G(gather, e.h, 0, w->w_out, e.h, 0, e.s, e.Fl, e.h, f1, e.f1w, e.dfc1_epi());
  dgel.aux_in = sv->at("h"); dgel.ld_aux = e.Fl; dgel.ld_aux_in = e.f1w;
  dgel.aux_t = tn.ta; dgel.c_t = f0; dgel.ld_t = e.s;
  PDS_TRY(e.gemm(dgel));                                                                // dH, dH^T, G^T
  PDS_TRY(tn.tr(gather, e.h, e.s, e.h, tn.tb));
  PDS_TRY(tn.mm(tn.ta, e.s, tn.tb, e.s, e.Fl, e.h, e.s, g->dw_out, e.h, EPI_F32_ACC));     // dW_out += G^T dZ
  if (pre) {
    PDS_TRY(e.wait(e.st, ev_v));
  } else {
    PDS_TRY(e.apply(sv->at("x1"), sv->at("rstd2"), w->g2, e.sl, gather + slot));
    PDS_TRY(e.ag(gather + slot, gather, e.sl * e.h));                                 // AG(v) re-gather
  }
  PDS_TRY(tn.tr(g2, e.h, e.s, e.h, tn.tb));
  PDS_TRY(tn.mm(f0, e.s, tn.tb, e.s, e.f1w, e.h, e.s, g->dw_in_t, e.h, EPI_F32_ACC));     // dW_in^T += dH^T V
  if (pre) {
    PDS_TRY(e.apply(sv->x, sv->at("rstd1"), w->g1, e.sl, g2 + slot));
    PDS_TRY(e.link(e.st, cs));
    PDS_TRY(e.ag_on(cs, g2 + slot, g2, e.sl * e.h));                                  // AG(u) re-gather
    ev_u = e.mark(cs);
  }
  if (ov) PDS_TRY(e.rs_arm(e.h));
  PDS_TRY(tn.xw(f1, e.f1w, w->w_in_t, e.h, e.s, e.h, e.f1w, partial, e.h));             // dV = dH W_in^T
  PDS_TRY(ov ? e.rs_run(partial, gather, n) : e.rs(partial, partial + slot, n));        // RS(dv)
  PDS_TRY(e.norm_bwd(partial + slot, sv->at("x1"), sv->at("rstd2"), w->g2, dy, e.sl, dx, dgp, dgl + e.h));
  if (ov) {
    PDS_CUDA(cudaMemcpyAsync(gather + slot, dx, n * 2, cudaMemcpyDeviceToDevice, e.st));
    PDS_TRY(e.ag_next(gather, n));                                                    // AG(dx1)
  } else {
    PDS_TRY(e.ag(dx, gather, n));                                                       // AG(dx1)
  }
  PDS_TRY(tn.mm(gather, e.h, w->w_proj, e.h, e.s, e.hl, e.h, f1, e.hl));                 // dA
  PDS_TRY(tn.dw(sv->at("a"), e.hl, gather, e.h, e.s, e.hl, e.h, g->dw_proj));            // dW_proj += A^T dX1
  PDS_TRY(e.attn_b(sv->at("qkv"), sv->at("a"), sv->at("lse"), f1, f0, dd, tn.ta, bp.ws_size("ta"),
                   reinterpret_cast<int*>(ws + bp.ws_off("actr")), bp.has_ws("dsb") ? ws + bp.ws_off("dsb") : nullptr,
                   bp.ws_size("dsb")));                     // dQKV (RoPE^T)
  if (pre) {
    PDS_TRY(e.wait(e.st, ev_u));
  } else {
    PDS_TRY(e.apply(sv->x, sv->at("rstd1"), w->g1, e.sl, gather + slot));
    PDS_TRY(e.ag(gather + slot, gather, e.sl * e.h));                                 // AG(u) re-gather
  }
  PDS_TRY(tn.dw(f0, e.qw, g2, e.h, e.s, e.qw, e.h, g->dw_qkv_t));                       // dW_qkv^T += dQKV^T U
  if (ov) PDS_TRY(e.rs_arm(e.h));
  PDS_TRY(tn.xw(f0, e.qw, w->w_qkv_t, e.h, e.s, e.h, e.qw, partial, e.h));              // dU = dQKV W_qkv^T
  PDS_TRY(ov ? e.rs_run(partial, gather, n) : e.rs(partial, partial + slot, n));        // RS(du)
  PDS_TRY(e.norm_bwd(partial + slot, sv->x, sv->at("rstd1"), w->g1, dx, e.sl, dx, dgp, dgl));
  return e.dgamma(dgl, g);
}

// ================================================================== UlyssesZ
// ZeRO3 weight gathers (rows contiguous).  The first weight a pass needs
// is gathered on the compute stream; the others are prefetched on the side stream
// while the compute stream works, each consumed through its own event.
pds_status uz_fwd(Exec& e, const void* x, const pds_weights* w, void* y, pds_saved* sv, char* ws) {
  const BufPlan& bp = sv->plan;
  const cudaStream_t cs = e.side_stream();
  PDS_TRY(e.link(e.st, cs));                 // gather buffers free (previous layer done with them)
  PDS_TRY(e.ag(w->w_qkv_t, ws + bp.ws_off("wqkv"), e.qw * e.h));
  PDS_TRY(e.ag_on(cs, w->w_proj, ws + bp.ws_off("wproj"), e.hl * e.h));
  cudaEvent_t ev_proj = e.mark(cs);
  PDS_TRY(e.ag_on(cs, w->w_in_t, ws + bp.ws_off("win"), e.f1w * e.h));
  PDS_TRY(e.ag_on(cs, w->w_out, ws + bp.ws_off("wout"), e.Fl * e.h));
  cudaEvent_t ev_ffn = e.mark(cs);
  char* wqkv = ws + bp.ws_off("wqkv");
  char* wproj = ws + bp.ws_off("wproj");
  char* win = ws + bp.ws_off("win");
  char* wout = ws + bp.ws_off("wout");
  char* u1 = ws + bp.ws_off("u1");
  char* s1 = ws + bp.ws_off("s1");
  char* r1 = ws + bp.ws_off("r1");
  char* f0 = ws + bp.ws_off("f0");
  TN tn{e, ws + bp.ws_off("ta"), ws + bp.ws_off("tb"), ws + bp.ws_off("wt")};
  PDS_TRY(e.norm_fwd(x, nullptr, w->g1, e.sl, nullptr, u1, sv->at("rstd1")));
  // local QKV for all heads, head-group-major columns, written straight into the A2A
  // send layout [P][s/P][3h/P]; RoPE at global positions r*s/P + t
  GemmArgs q = e.rope(Exec::G(u1, e.h, 0, wqkv, e.h, 0, e.sl, e.qwf, e.h, s1, e.qw), e.hl, e.nkl * e.d, 0, 0,
                      e.r * e.sl);
  q.blk_w = (int)e.qw;
  q.blk_stride = e.sl * e.qw;
  // P > 1: block j of the packed output leaves for rank j as soon as its tiles are stored
  const bool ov = e.overlap();
  if (ov) PDS_TRY(e.a2a_arm(e.qw));
  PDS_TRY(e.gemm(q));
  PDS_TRY(ov ? e.a2a_run(s1, sv->at("qkv"), e.sl * e.qw)
             : e.a2a(s1, sv->at("qkv"), e.sl * e.qw));                                   // A2A seq -> heads
  PDS_TRY(e.attn_f(sv->at("qkv"), sv->at("a"), sv->at("lse")));
  PDS_TRY(e.a2a(sv->at("a"), r1, e.sl * e.hl));                                        // A2A heads -> seq
  {
    Prof p(e.c, e.st, K_NORM, 0, 4.0 * e.sl * e.h);
    PDS_TRY(kerr(unpack_blocks(r1, e.P, e.sl, e.hl, sv->at("afull"), e.h, e.st), "unpack"));
  }
  PDS_TRY(e.wait(e.st, ev_proj));
  PDS_TRY(tn.xw(sv->at("afull"), e.h, wproj, e.h, e.sl, e.h, e.h, u1, e.h));          // O
  PDS_TRY(e.tap(e.c->tap_o, u1, e.sl * e.h));
  PDS_TRY(e.norm_fwd(x, u1, w->g2, e.sl, sv->at("x1"), s1, sv->at("rstd2")));
  PDS_TRY(e.wait(e.st, ev_ffn));
  GemmArgs fc1 = Exec::G(s1, e.h, 0, win, e.h, 0, e.sl, e.f1wf, e.h, sv->at("h"), e.f1wf, e.fc1_epi());
  fc1.aux_out = f0; fc1.ld_aux = e.F;
  PDS_TRY(e.gemm(fc1));
  PDS_TRY(tn.xw(f0, e.F, wout, e.h, e.sl, e.h, e.F, u1, e.h));                          // Z
  PDS_TRY(e.tap(e.c->tap_z, u1, e.sl * e.h));
  return e.add(sv->at("x1"), u1, y, e.sl * e.h);
}

pds_status uz_dw(Exec& e, char* dw, int64_t rows_full, void* grad) {
  // ZeRO3: reduce-scatter the full local fp32 dW into spec shards, then accumulate
  const int64_t cnt = rows_full / e.P * e.h;
  char* mine = dw + e.r * cnt * 4;
  PDS_TRY(e.rs(dw, mine, cnt, DT_F32));
  return kerr(add_f32(mine, grad, cnt, e.st), "add_f32");
}

pds_status uz_bwd(Exec& e, const void* dy, pds_saved* sv, const pds_weights* w, const pds_grads* g, void* dx,
                  char* ws) {
  const BufPlan& bp = sv->plan;
  const cudaStream_t cs = e.side_stream();
  PDS_TRY(e.link(e.st, cs));
  PDS_TRY(e.ag(w->w_out, ws + bp.ws_off("wout"), e.Fl * e.h));
  PDS_TRY(e.ag_on(cs, w->w_in_t, ws + bp.ws_off("win"), e.f1w * e.h));
  cudaEvent_t ev_in = e.mark(cs);
  PDS_TRY(e.ag_on(cs, w->w_proj, ws + bp.ws_off("wproj"), e.hl * e.h));
  cudaEvent_t ev_proj = e.mark(cs);
  PDS_TRY(e.ag_on(cs, w->w_qkv_t, ws + bp.ws_off("wqkv"), e.qw * e.h));
  cudaEvent_t ev_qkv = e.mark(cs);
  char* wqkv = ws + bp.ws_off("wqkv");
  char* wproj = ws + bp.ws_off("wproj");
  char* win = ws + bp.ws_off("win");
  char* wout = ws + bp.ws_off("wout");
  char* dw = ws + bp.ws_off("dw");
  char* u1 = ws + bp.ws_off("u1");
  char* s1 = ws + bp.ws_off("s1");
  char* r1 = ws + bp.ws_off("r1");
  char* f0 = ws + bp.ws_off("f0");
  char* f1 = ws + bp.ws_off("f1");
  char* x3 = ws + bp.ws_off("x3");
  char* x4 = ws + bp.ws_off("x4");
  char* v2 = ws + bp.ws_off("v2");
  float* dd = reinterpret_cast<float*>(ws + bp.ws_off("dd"));
  float* dgp = reinterpret_cast<float*>(ws + bp.ws_off("dgp"));
  float* dgl = reinterpret_cast<float*>(ws + bp.ws_off("dgl"));
  TN tn{e, ws + bp.ws_off("ta"), ws + bp.ws_off("tb"), ws + bp.ws_off("wt")};
  PDS_CUDA(cudaMemsetAsync(dgl, 0, 2 * e.h * 4, e.st));
  GemmArgs dgel = Exec::G(dy, e.h, 0, wout, e.h, 0, e.sl, e.F, e.h, f1, e.f1wf, e.dfc1_epi());
  dgel.aux_in = sv->at("h"); dgel.ld_aux = e.F; dgel.ld_aux_in = e.f1wf;
  dgel.aux_t = tn.ta; dgel.c_t = f0; dgel.ld_t = e.sl;                                 // G^T, dH^T
  PDS_TRY(e.gemm(dgel));
  PDS_TRY(tn.tr(dy, e.h, e.sl, e.h, tn.tb));
  PDS_TRY(tn.mm(tn.ta, e.sl, tn.tb, e.sl, e.F, e.h, e.sl, dw, e.h, EPI_F32));           // dW_out (full, local)
  PDS_TRY(uz_dw(e, dw, e.F, g->dw_out));
  PDS_TRY(e.apply(sv->at("x1"), sv->at("rstd2"), w->g2, e.sl, u1));
  PDS_TRY(tn.tr(u1, e.h, e.sl, e.h, tn.tb));
  PDS_TRY(tn.mm(f0, e.sl, tn.tb, e.sl, e.f1wf, e.h, e.sl, dw, e.h, EPI_F32));           // dW_in^T (full, local)
  PDS_TRY(uz_dw(e, dw, e.f1wf, g->dw_in_t));
  PDS_TRY(e.wait(e.st, ev_in));
  PDS_TRY(tn.xw(f1, e.f1wf, win, e.h, e.sl, e.h, e.f1wf, v2, e.h));
  PDS_TRY(e.norm_bwd(v2, sv->at("x1"), sv->at("rstd2"), w->g2, dy, e.sl, dx, dgp, dgl + e.h));
  PDS_TRY(e.wait(e.st, ev_proj));
  GemmArgs dafull = Exec::G(dx, e.h, 0, wproj, e.h, 0, e.sl, e.h, e.h, s1, e.hl);
  dafull.blk_w = (int)e.hl;
  dafull.blk_stride = e.sl * e.hl;
  const bool ov = e.overlap();       // P > 1: A2A(dO) block by block, under the dW_proj work too
  if (ov) PDS_TRY(e.a2a_arm(e.hl));
  PDS_TRY(e.gemm(dafull));                                                              // packed for A2A
  if (ov) PDS_TRY(e.a2a_run(s1, r1, e.sl * e.hl));                                     // A2A(dO)
  PDS_TRY(tn.dw(sv->at("afull"), e.h, dx, e.h, e.sl, e.h, e.h, dw, EPI_F32));
  PDS_TRY(uz_dw(e, dw, e.h, g->dw_proj));
  if (!ov) PDS_TRY(e.a2a(s1, r1, e.sl * e.hl));                                         // A2A(dO)
  PDS_TRY(e.attn_b(sv->at("qkv"), sv->at("a"), sv->at("lse"), r1, x3, dd, tn.ta, bp.ws_size("ta"),
                   reinterpret_cast<int*>(ws + bp.ws_off("actr")), bp.has_ws("dsb") ? ws + bp.ws_off("dsb") : nullptr,
                   bp.ws_size("dsb")));
  PDS_TRY(e.a2a(x3, r1, e.sl * e.qw));                                                 // A2A(dQKV)
  {
    Prof p(e.c, e.st, K_NORM, 0, 4.0 * e.sl * e.qwf);
    PDS_TRY(kerr(unpack_blocks(r1, e.P, e.sl, e.qw, x4, e.qwf, e.st), "unpack"));
  }
  PDS_TRY(e.apply(sv->x, sv->at("rstd1"), w->g1, e.sl, u1));
  PDS_TRY(tn.dw(x4, e.qwf, u1, e.h, e.sl, e.qwf, e.h, dw, EPI_F32));
  PDS_TRY(uz_dw(e, dw, e.qwf, g->dw_qkv_t));
  PDS_TRY(e.wait(e.st, ev_qkv));
  PDS_TRY(tn.xw(x4, e.qwf, wqkv, e.h, e.sl, e.h, e.qwf, v2, e.h));
  PDS_TRY(e.norm_bwd(v2, sv->x, sv->at("rstd1"), w->g1, dx, e.sl, dx, dgp, dgl));
  return e.dgamma(dgl, g);
}

// ================================================================== MegatronCZ
// Megatron-LM CP + ZeRO3 (reading R-CZ): ZeRO3 weight gathers
// as in UlyssesZ, every GEMM local on the rank's s/P rows, and the context-parallel
// attention as zigzag-balanced ring attention (below).  W_qkv^T is gathered part by
// part (the Q, K, V rows of every spec shard) into [Q all; K all; V all], so the local
// QKV GEMM yields all heads; its gradient is reduce-scattered part by part back into
// the spec layout.
// GQA (R-GQA): the K and V parts are n_kv d / P rows per shard, n_kv d in the gather.
pds_status cz_wqkv(Exec& e, const pds_weights* w, char* wqkv, cudaStream_t on) {
  const int64_t hkl = e.nkl * e.d, hk = hkl * e.P;
  const int64_t src_off[3] = {0, e.hl * e.h, (e.hl + hkl) * e.h};   // within the spec shard
  const int64_t dst_off[3] = {0, e.h * e.h, (e.h + hk) * e.h};      // [Q all; K all; V all]
  const int64_t cnt[3] = {e.hl * e.h, hkl * e.h, hkl * e.h};
  for (int i = 0; i < 3; ++i) {
    const char* src = static_cast<const char*>(w->w_qkv_t) + src_off[i] * 2;
    PDS_TRY(on == e.st ? e.ag(src, wqkv + dst_off[i] * 2, cnt[i]) : e.ag_on(on, src, wqkv + dst_off[i] * 2, cnt[i]));
  }
  return PDS_OK;
}

// ---------------------------------------------------------------- ring attention (R-CZ)
// Zigzag placement of the attention (DESIGN.md R-CZ): the s positions are 2P half-chunks
// of c = s/(2P); rank r computes the queries of half-chunks r and 2P-1-r ("zig rows":
// [half-chunk r ; half-chunk 2P-1-r], c*b rows each, b sequences interleaved as in the
// boundary layout).  Every other tensor of the layer stays on the boundary rows.
struct Zig {
  int P, r;
  int64_t c, cb;                                      // positions / rows per half-chunk
  int zz(int j) const { return j < P ? j : 2 * P - 1 - j; }
  int hc(int i) const { return i == 0 ? r : 2 * P - 1 - r; }    // half-chunk of zig half i
};

// boundary rows X [2 cb][cols] -> zig rows Z (to_zig) or back (!to_zig), bf16
pds_status zig_exchange(Exec& e, const Zig& z, char* X, char* Z, int64_t cols, bool to_zig) {
  const int64_t bytes = z.cb * cols * 2;
  P2P snd[2], rcv[2];
  for (int i = 0; i < 2; ++i) {
    const int own = 2 * z.r + i;                      // boundary half-chunks 2r, 2r+1
    const int mine = z.hc(i);                         // zig half-chunks r, 2P-1-r
    if (to_zig) {
      snd[i] = P2P{z.zz(own), own, X + i * bytes, bytes};
      rcv[i] = P2P{mine / 2, mine, Z + i * bytes, bytes};
    } else {
      snd[i] = P2P{mine / 2, mine, Z + i * bytes, bytes};
      rcv[i] = P2P{z.zz(own), own, X + i * bytes, bytes};
    }
  }
  return e.p2p(snd, 2, rcv, 2, e.st);
}

// the ring: send `cur` to rank r+1, receive rank r-1's block into `nxt`
pds_status ring_pass(Exec& e, const char* cur, char* nxt, int64_t bytes, cudaStream_t on) {
  P2P snd{(e.r + 1) % e.P, 0, const_cast<char*>(cur), bytes};
  P2P rcv{(e.r - 1 + e.P) % e.P, 0, nxt, bytes};
  return e.p2p(&snd, 1, &rcv, 1, on, "RingPass");
}

pds_status cz_fwd(Exec& e, const void* x, const pds_weights* w, void* y, pds_saved* sv, char* ws) {
  const BufPlan& bp = sv->plan;
  const cudaStream_t cs = e.side_stream();
  const int64_t n = e.m.n_heads, h = e.h;
  const int64_t hk = e.nkl * e.d * e.P, qw = e.qwf;      // K (V) width, [Q | K | V] width (GQA: n_kv d)
  const Zig z{e.P, e.r, e.sp / 2, e.sl / 2};
  char* wqkv = ws + bp.ws_off("wqkv");
  char* wproj = ws + bp.ws_off("wproj");
  char* win = ws + bp.ws_off("win");
  char* wout = ws + bp.ws_off("wout");
  char* u1 = ws + bp.ws_off("u1");
  char* qkvb = ws + bp.ws_off("qkvb");
  char* kvb[2] = {ws + bp.ws_off("kv0"), ws + bp.ws_off("kv1")};
  float* oacc = reinterpret_cast<float*>(ws + bp.ws_off("acc"));
  char* op = ws + bp.ws_off("op");
  char* oz = ws + bp.ws_off("oz");
  float* lp = reinterpret_cast<float*>(ws + bp.ws_off("lp"));
  char* v2 = ws + bp.ws_off("v2");
  char* f0 = ws + bp.ws_off("f0");
  char* qkvz = sv->at("qkv");                        // saved: zig rows, post-RoPE [Q | K | V]
  float* lse = reinterpret_cast<float*>(sv->at("lse"));   // saved: [b][2 zig halves][n][c]
  TN tn{e, ws + bp.ws_off("ta"), ws + bp.ws_off("tb"), ws + bp.ws_off("wt")};
  PDS_TRY(e.link(e.st, cs));                 // gather buffers free (previous layer done with them)
  PDS_TRY(cz_wqkv(e, w, wqkv, e.st));
  PDS_TRY(e.ag_on(cs, w->w_proj, wproj, e.hl * h));
  cudaEvent_t ev_proj = e.mark(cs);
  PDS_TRY(e.ag_on(cs, w->w_in_t, win, e.f1w * h));
  PDS_TRY(e.ag_on(cs, w->w_out, wout, e.Fl * h));
  cudaEvent_t ev_ffn = e.mark(cs);
  PDS_TRY(e.norm_fwd(x, nullptr, w->g1, e.sl, nullptr, u1, sv->at("rstd1")));
  // local Q/K/V of all heads ([Q (h) | K (hk) | V (hk)] column blocks), RoPE at global positions
  PDS_TRY(e.gemm(e.rope(Exec::G(u1, h, 0, wqkv, h, 0, e.sl, qw, h, qkvb, qw), h, hk, 0, 0, e.r * e.sl)));
  PDS_TRY(zig_exchange(e, z, qkvb, qkvz, qw, true));                                     // -> zig rows
  PDS_CUDA(cudaMemcpy2DAsync(kvb[0], 2 * hk * 2, qkvz + h * 2, qw * 2, 2 * hk * 2, e.sl, cudaMemcpyDeviceToDevice,
                             e.st));
  // P ring steps; step k holds the K/V of rank r - k (its zig half-chunks), the next
  // block is received on the side stream while this one is computed
  bool first[2] = {true, true};
  for (int k = 0; k < e.P; ++k) {
    const int src = (e.r - k + e.P) % e.P;
    char* kv = kvb[k & 1];
    cudaEvent_t ev_next = nullptr;
    if (k + 1 < e.P) {
      PDS_TRY(e.link(e.st, cs));
      PDS_TRY(ring_pass(e, kv, kvb[(k + 1) & 1], e.sl * 2 * hk * 2, cs));
      ev_next = e.mark(cs);
    }
    const Zig zs{e.P, src, z.c, z.cb};
    for (int ai = 0; ai < 2; ++ai)
      for (int bi = 0; bi < 2; ++bi) {
        const int qa = z.hc(ai), kb = zs.hc(bi);
        if (e.m.causal && kb > qa) continue;          // every key after every query
        const int diag = e.m.causal && kb == qa;
        {
          Prof p(e.c, e.st, K_ATTN_F, e.b * 4.0 * n * e.d * (diag ? 0.5 * z.c * z.c : (double)z.c * z.c), 0);
          for (int64_t j = 0; j < e.b; ++j)
            PDS_TRY(kerr(attn_fwd_pair(qkvz + ((ai * z.cb) + j) * qw * 2, e.b * qw,
                                       kv + ((bi * z.cb) + j) * 2 * hk * 2, e.b * 2 * hk, 0, (int)hk, (int)z.c,
                                       (int)z.c, (int)n, (int)e.d, diag, op + j * h * 2, e.b * h, lp + j * n * z.c,
                                       e.st, (int)(e.nkl * e.P)),
                         "attn_fwd_pair"));
        }
        Prof p(e.c, e.st, K_NORM, 0, (double)z.cb * h * 10);
        for (int64_t j = 0; j < e.b; ++j)
          PDS_TRY(kerr(attn_merge(oacc + ((ai * z.cb) + j) * h, e.b * h, lse + (j * 2 + ai) * n * z.c, z.c,
                                  op + j * h * 2, e.b * h, lp + j * n * z.c, z.c, (int)z.c, (int)n, (int)e.d,
                                  first[ai], nullptr, 0, e.st), "attn_merge"));
        first[ai] = false;
      }
    if (ev_next) PDS_TRY(e.wait(e.st, ev_next));
  }
  {
    Prof p(e.c, e.st, K_NORM, 0, (double)e.sl * h * 6);
    PDS_TRY(kerr(rope_t_f32_bf16(oacc, h, (int)e.sl, (int)h, (int)e.d, nullptr, 0, 0, (int)z.cb, (int)e.b, oz, h,
                                 e.st), "o convert"));
  }
  PDS_TRY(zig_exchange(e, z, sv->at("a"), oz, h, false));                               // -> boundary rows
  PDS_TRY(e.wait(e.st, ev_proj));
  PDS_TRY(tn.xw(sv->at("a"), h, wproj, h, e.sl, h, h, u1, h));                          // O
  PDS_TRY(e.tap(e.c->tap_o, u1, e.sl * h));
  PDS_TRY(e.norm_fwd(x, u1, w->g2, e.sl, sv->at("x1"), v2, sv->at("rstd2")));
  PDS_TRY(e.wait(e.st, ev_ffn));
  GemmArgs fc1 = Exec::G(v2, h, 0, win, h, 0, e.sl, e.f1wf, h, sv->at("h"), e.f1wf, e.fc1_epi());
  fc1.aux_out = f0; fc1.ld_aux = e.F;
  PDS_TRY(e.gemm(fc1));
  PDS_TRY(tn.xw(f0, e.F, wout, h, e.sl, h, e.F, u1, h));                                // Z
  PDS_TRY(e.tap(e.c->tap_z, u1, e.sl * h));
  return e.add(sv->at("x1"), u1, y, e.sl * h);
}

pds_status cz_bwd(Exec& e, const void* dy, pds_saved* sv, const pds_weights* w, const pds_grads* g, void* dx,
                  char* ws) {
  const BufPlan& bp = sv->plan;
  const cudaStream_t cs = e.side_stream();
  const int64_t n = e.m.n_heads, h = e.h;
  const int64_t hk = e.nkl * e.d * e.P, qw = e.qwf;
  const Zig z{e.P, e.r, e.sp / 2, e.sl / 2};
  char* wqkv = ws + bp.ws_off("wqkv");
  char* wproj = ws + bp.ws_off("wproj");
  char* win = ws + bp.ws_off("win");
  char* wout = ws + bp.ws_off("wout");
  char* dw = ws + bp.ws_off("dw");
  char* u1 = ws + bp.ws_off("u1");
  char* qkvb = ws + bp.ws_off("qkvb");
  char* kvb[2] = {ws + bp.ws_off("kv0"), ws + bp.ws_off("kv1")};
  float* dkvb[2] = {reinterpret_cast<float*>(ws + bp.ws_off("dkv0")), reinterpret_cast<float*>(ws + bp.ws_off("dkv1"))};
  float* dqacc = reinterpret_cast<float*>(ws + bp.ws_off("acc"));
  char* doz = ws + bp.ws_off("op");
  char* oz = ws + bp.ws_off("oz");
  char* dqkvz = ws + bp.ws_off("dqkvz");
  char* f0 = ws + bp.ws_off("f0");
  char* f1 = ws + bp.ws_off("f1");
  char* v2 = ws + bp.ws_off("v2");
  char* da = ws + bp.ws_off("da");
  float* dd = reinterpret_cast<float*>(ws + bp.ws_off("dd"));
  float* dgp = reinterpret_cast<float*>(ws + bp.ws_off("dgp"));
  float* dgl = reinterpret_cast<float*>(ws + bp.ws_off("dgl"));
  const char* qkvz = sv->at("qkv");
  const float* lse = reinterpret_cast<const float*>(sv->at("lse"));
  TN tn{e, ws + bp.ws_off("ta"), ws + bp.ws_off("tb"), ws + bp.ws_off("wt")};
  PDS_TRY(e.link(e.st, cs));
  PDS_TRY(e.ag(w->w_out, wout, e.Fl * h));
  PDS_TRY(e.ag_on(cs, w->w_in_t, win, e.f1w * h));
  cudaEvent_t ev_in = e.mark(cs);
  PDS_TRY(e.ag_on(cs, w->w_proj, wproj, e.hl * h));
  cudaEvent_t ev_proj = e.mark(cs);
  PDS_TRY(cz_wqkv(e, w, wqkv, cs));
  cudaEvent_t ev_qkv = e.mark(cs);
  PDS_CUDA(cudaMemsetAsync(dgl, 0, 2 * h * 4, e.st));
  // FFN: local with full weights (as UlyssesZ)
  GemmArgs dgel = Exec::G(dy, h, 0, wout, h, 0, e.sl, e.F, h, f1, e.f1wf, e.dfc1_epi());
  dgel.aux_in = sv->at("h"); dgel.ld_aux = e.F; dgel.ld_aux_in = e.f1wf;
  dgel.aux_t = tn.ta; dgel.c_t = f0; dgel.ld_t = e.sl;                                 // G^T, dH^T
  PDS_TRY(e.gemm(dgel));
  PDS_TRY(tn.tr(dy, h, e.sl, h, tn.tb));
  PDS_TRY(tn.mm(tn.ta, e.sl, tn.tb, e.sl, e.F, h, e.sl, dw, h, EPI_F32));               // dW_out (full, local)
  PDS_TRY(uz_dw(e, dw, e.F, g->dw_out));
  PDS_TRY(e.apply(sv->at("x1"), sv->at("rstd2"), w->g2, e.sl, u1));
  PDS_TRY(tn.tr(u1, h, e.sl, h, tn.tb));
  PDS_TRY(tn.mm(f0, e.sl, tn.tb, e.sl, e.f1wf, h, e.sl, dw, h, EPI_F32));               // dW_in^T (full, local)
  PDS_TRY(uz_dw(e, dw, e.f1wf, g->dw_in_t));
  PDS_TRY(e.wait(e.st, ev_in));
  PDS_TRY(tn.xw(f1, e.f1wf, win, h, e.sl, h, e.f1wf, v2, h));
  PDS_TRY(e.norm_bwd(v2, sv->at("x1"), sv->at("rstd2"), w->g2, dy, e.sl, dx, dgp, dgl + h));
  PDS_TRY(e.wait(e.st, ev_proj));
  PDS_TRY(e.gemm(Exec::G(dx, h, 0, wproj, h, 0, e.sl, h, h, da, h)));                  // dA = dX1 W_proj^T
  PDS_TRY(tn.dw(sv->at("a"), h, dx, h, e.sl, h, h, dw, EPI_F32));
  PDS_TRY(uz_dw(e, dw, h, g->dw_proj));
  // ring attention backward on the zig rows: O and dO to zig rows, D = rowsum(dO o O)
  PDS_TRY(zig_exchange(e, z, sv->at("a"), oz, h, true));
  PDS_TRY(zig_exchange(e, z, da, doz, h, true));
  {
    Prof p(e.c, e.st, K_NORM, 0, (double)e.sl * h * 4);
    for (int64_t j = 0; j < e.b; ++j)
      for (int ai = 0; ai < 2; ++ai)
        PDS_TRY(kerr(attn_dot(oz + ((ai * z.cb) + j) * h * 2, e.b * h, doz + ((ai * z.cb) + j) * h * 2, (int)z.c,
                              (int)n, (int)e.d, dd + (j * 2 + ai) * n * z.c, e.st), "attn_dot"));
  }
  PDS_CUDA(cudaMemsetAsync(dqacc, 0, e.sl * h * 4, e.st));
  PDS_CUDA(cudaMemsetAsync(dkvb[0], 0, e.sl * 2 * hk * 4, e.st));
  PDS_CUDA(cudaMemcpy2DAsync(kvb[0], 2 * hk * 2, qkvz + h * 2, qw * 2, 2 * hk * 2, e.sl, cudaMemcpyDeviceToDevice,
                             e.st));
  int cur = 0;                                     // dK/dV accumulator of the block in hand
  for (int k = 0; k < e.P; ++k) {
    const int src = (e.r - k + e.P) % e.P;
    char* kv = kvb[k & 1];
    cudaEvent_t ev_next = nullptr;
    if (k + 1 < e.P) {
      PDS_TRY(e.link(e.st, cs));
      PDS_TRY(ring_pass(e, kv, kvb[(k + 1) & 1], e.sl * 2 * hk * 2, cs));
      ev_next = e.mark(cs);
    }
    const Zig zs{e.P, src, z.c, z.cb};
    for (int ai = 0; ai < 2; ++ai)
      for (int bi = 0; bi < 2; ++bi) {
        const int qa = z.hc(ai), kb = zs.hc(bi);
        if (e.m.causal && kb > qa) continue;
        const int diag = e.m.causal && kb == qa;
        Prof p(e.c, e.st, K_ATTN_B, e.b * 10.0 * n * e.d * (diag ? 0.5 * z.c * z.c : (double)z.c * z.c), 0);
        for (int64_t j = 0; j < e.b; ++j)
          PDS_TRY(kerr(attn_bwd_pair(qkvz + ((ai * z.cb) + j) * qw * 2, e.b * qw,
                                     kv + ((bi * z.cb) + j) * 2 * hk * 2, e.b * 2 * hk, 0, (int)hk,
                                     doz + ((ai * z.cb) + j) * h * 2, e.b * h, lse + (j * 2 + ai) * n * z.c,
                                     dd + (j * 2 + ai) * n * z.c, (int)z.c, (int)z.c, (int)n, (int)e.d, diag,
                                     dqacc + ((ai * z.cb) + j) * h, e.b * h,
                                     dkvb[cur] + ((bi * z.cb) + j) * 2 * hk, e.b * 2 * hk, e.st,
                                     (int)(e.nkl * e.P)), "attn_bwd_pair"));
      }
    // the accumulator travels with its block: P passes bring it home
    if (e.P > 1) {
      PDS_TRY(ring_pass(e, reinterpret_cast<char*>(dkvb[cur]), reinterpret_cast<char*>(dkvb[cur ^ 1]),
                        e.sl * 2 * hk * 4, e.st));
      cur ^= 1;
    }
    if (ev_next) PDS_TRY(e.wait(e.st, ev_next));
  }
  {
    // RoPE^T at the zig positions, bf16, [dQ | dK | dV] zig rows
    Prof p(e.c, e.st, K_NORM, 0, (double)e.sl * qw * 6);
    const int64_t b0 = z.hc(0) * z.c, b1 = z.hc(1) * z.c;
    PDS_TRY(kerr(rope_t_f32_bf16(dqacc, h, (int)e.sl, (int)h, (int)e.d, e.c->rope, b0, b1, (int)z.cb, (int)e.b,
                                 dqkvz, qw, e.st), "dq rope_t"));
    PDS_TRY(kerr(rope_t_f32_bf16(dkvb[cur], 2 * hk, (int)e.sl, (int)hk, (int)e.d, e.c->rope, b0, b1, (int)z.cb,
                                 (int)e.b, dqkvz + h * 2, qw, e.st), "dk rope_t"));
    PDS_TRY(kerr(rope_t_f32_bf16(dkvb[cur] + hk, 2 * hk, (int)e.sl, (int)hk, (int)e.d, nullptr, 0, 0, (int)z.cb,
                                 (int)e.b, dqkvz + (h + hk) * 2, qw, e.st), "dv convert"));
  }
  PDS_TRY(zig_exchange(e, z, qkvb, dqkvz, qw, false));                                  // dQKV -> boundary
  char* dqkv = qkvb;
  PDS_TRY(e.apply(sv->x, sv->at("rstd1"), w->g1, e.sl, u1));
  PDS_TRY(tn.dw(dqkv, qw, u1, h, e.sl, qw, h, dw, EPI_F32));                            // [Q; K; V] all rows
  {                                   // ZeRO3 RS part by part into the spec shard [Q_r; K_r; V_r]
    const int64_t hkl = e.nkl * e.d;
    const int64_t part_off[3] = {0, h * h, (h + hk) * h};          // rows of [Q all; K all; V all]
    const int64_t shard_off[3] = {0, e.hl * h, (e.hl + hkl) * h};  // rows of the spec shard
    const int64_t cnts[3] = {e.hl * h, hkl * h, hkl * h};
    for (int i = 0; i < 3; ++i) {
      char* part = dw + part_off[i] * 4;
      char* mine = part + e.r * cnts[i] * 4;
      PDS_TRY(e.rs(part, mine, cnts[i], DT_F32));
      PDS_TRY(kerr(add_f32(mine, static_cast<char*>(g->dw_qkv_t) + shard_off[i] * 4, cnts[i], e.st), "add_f32"));
    }
  }
  PDS_TRY(e.wait(e.st, ev_qkv));
  PDS_TRY(tn.xw(dqkv, qw, wqkv, h, e.sl, h, qw, v2, h));                                // dU
  PDS_TRY(e.norm_bwd(v2, sv->x, sv->at("rstd1"), w->g1, dx, e.sl, dx, dgp, dgl));
  return e.dgamma(dgl, g);
}

// ================================================================== ColossalZ (R-COL)
// Colossal-AI sequence parallelism (Ring Self-Attention) + ZeRO3 weights:
// weights and GEMMs as MegatronCZ on the boundary rows; the keys, then the values, pass
// around the ring of contiguous chunks; every rank materialises the scores of its rows
// against all s keys ([b][n][s/P][s] fp32, softmax -> bf16 probabilities saved for the
// backward: the quadratic memory that makes the paper exclude it).
// Per (sequence, head, key block) one tcgen05 GEMM for each product.
struct ColBufs {
  char* qkv;            // saved [s/P b][3h] post-RoPE
  char* probs;          // saved [b][n][sp][s]
  float* scores;        // ws [b][n][sp][s] fp32
};

// block j (the rank whose K / V is in hand) of the key axis: columns [j sp, (j+1) sp)
pds_status col_ring(Exec& e, const char* first, int64_t col_off, char* kr[2],
                    const std::function<pds_status(int k, int j, const char* blk)>& step) {
  const int64_t hk = e.nkl * e.d * e.P;                   // a K (V) block's width (GQA)
  PDS_CUDA(cudaMemcpy2DAsync(kr[0], hk * 2, first + col_off * 2, e.qwf * 2, hk * 2, e.sl, cudaMemcpyDeviceToDevice,
                             e.st));
  for (int k = 0; k < e.P; ++k) {
    const int j = (e.r - k + e.P) % e.P;
    PDS_TRY(step(k, j, kr[k & 1]));
    if (k + 1 < e.P) PDS_TRY(ring_pass(e, kr[k & 1], kr[(k + 1) & 1], e.sl * hk * 2, e.st));
  }
  return PDS_OK;
}

pds_status col_fwd(Exec& e, const void* x, const pds_weights* w, void* y, pds_saved* sv, char* ws) {
  const BufPlan& bp = sv->plan;
  const cudaStream_t cs = e.side_stream();
  const int64_t n = e.m.n_heads, h = e.h, d = e.d, sp = e.sp, sq = e.sq, b = e.b;
  const int64_t hk = e.nkl * d * e.P, qw = e.qwf, grp = n / (e.nkl * e.P);   // GQA widths
  char* wqkv = ws + bp.ws_off("wqkv");
  char* wproj = ws + bp.ws_off("wproj");
  char* win = ws + bp.ws_off("win");
  char* wout = ws + bp.ws_off("wout");
  char* u1 = ws + bp.ws_off("u1");
  float* scores = reinterpret_cast<float*>(ws + bp.ws_off("scores"));
  char* kr[2] = {ws + bp.ws_off("kr0"), ws + bp.ws_off("kr1")};
  float* oacc = reinterpret_cast<float*>(ws + bp.ws_off("acc"));
  char* v2 = ws + bp.ws_off("v2");
  char* f0 = ws + bp.ws_off("f0");
  char* qkv = sv->at("qkv");
  char* probs = sv->at("probs");
  TN tn{e, ws + bp.ws_off("ta"), ws + bp.ws_off("tb"), ws + bp.ws_off("wt")};
  PDS_TRY(e.link(e.st, cs));
  PDS_TRY(cz_wqkv(e, w, wqkv, e.st));
  PDS_TRY(e.ag_on(cs, w->w_proj, wproj, e.hl * h));
  cudaEvent_t ev_proj = e.mark(cs);
  PDS_TRY(e.ag_on(cs, w->w_in_t, win, e.f1w * h));
  PDS_TRY(e.ag_on(cs, w->w_out, wout, e.Fl * h));
  cudaEvent_t ev_ffn = e.mark(cs);
  PDS_TRY(e.norm_fwd(x, nullptr, w->g1, e.sl, nullptr, u1, sv->at("rstd1")));
  PDS_TRY(e.gemm(e.rope(Exec::G(u1, h, 0, wqkv, h, 0, e.sl, qw, h, qkv, qw), h, hk, 0, 0, e.r * e.sl)));
  // ring of K: scores of the own rows against key block j, per sequence and head
  PDS_TRY(col_ring(e, qkv, h, kr, [&](int, int j, const char* kb) -> pds_status {
    for (int64_t q = 0; q < b; ++q)
      for (int64_t hd = 0; hd < n; ++hd)
        PDS_TRY(e.gemm(Exec::G(qkv + (q * qw + hd * d) * 2, b * qw, 0, kb + (q * hk + hd / grp * d) * 2, b * hk, 0,
                               sp, sp, d, scores + ((q * n + hd) * sp * sq + j * sp), sq, EPI_F32)));
    return PDS_OK;
  }));
  {
    Prof p(e.c, e.st, K_NORM, 0, (double)b * n * sp * sq * 6);
    PDS_TRY(kerr(rsa_softmax(scores, sq, (int)(b * n * sp), (int)sq, (int)sp, e.r * sp, e.m.causal,
                             1.0f / std::sqrt((float)d), probs, sq, e.st), "rsa_softmax"));
  }
  // ring of V: O += P_j V_j
  PDS_CUDA(cudaMemsetAsync(oacc, 0, e.sl * h * 4, e.st));
  PDS_TRY(col_ring(e, qkv, h + hk, kr, [&](int, int j, const char* vb) -> pds_status {
    for (int64_t q = 0; q < b; ++q)
      for (int64_t hd = 0; hd < n; ++hd)
        PDS_TRY(e.gemm(Exec::G(probs + ((q * n + hd) * sp * sq + j * sp) * 2, sq, 0, vb + (q * hk + hd / grp * d) * 2,
                               b * hk, 1, sp, d, sp, oacc + q * h + hd * d, b * h, EPI_F32_ACC)));
    return PDS_OK;
  }));
  {
    Prof p(e.c, e.st, K_NORM, 0, (double)e.sl * h * 6);
    PDS_TRY(kerr(rope_t_f32_bf16(oacc, h, (int)e.sl, (int)h, (int)d, nullptr, 0, 0, (int)e.sl, (int)b, sv->at("a"),
                                 h, e.st), "o convert"));
  }
  PDS_TRY(e.wait(e.st, ev_proj));
  PDS_TRY(tn.xw(sv->at("a"), h, wproj, h, e.sl, h, h, u1, h));                          // O
  PDS_TRY(e.tap(e.c->tap_o, u1, e.sl * h));
  PDS_TRY(e.norm_fwd(x, u1, w->g2, e.sl, sv->at("x1"), v2, sv->at("rstd2")));
  PDS_TRY(e.wait(e.st, ev_ffn));
  GemmArgs fc1 = Exec::G(v2, h, 0, win, h, 0, e.sl, e.f1wf, h, sv->at("h"), e.f1wf, e.fc1_epi());
  fc1.aux_out = f0; fc1.ld_aux = e.F;
  PDS_TRY(e.gemm(fc1));
  PDS_TRY(tn.xw(f0, e.F, wout, h, e.sl, h, e.F, u1, h));                                // Z
  PDS_TRY(e.tap(e.c->tap_z, u1, e.sl * h));
  return e.add(sv->at("x1"), u1, y, e.sl * h);
}

pds_status col_bwd(Exec& e, const void* dy, pds_saved* sv, const pds_weights* w, const pds_grads* g, void* dx,
                   char* ws) {
  const BufPlan& bp = sv->plan;
  const cudaStream_t cs = e.side_stream();
  const int64_t n = e.m.n_heads, h = e.h, d = e.d, sp = e.sp, sq = e.sq, b = e.b;
  const int64_t hk = e.nkl * d * e.P, qw = e.qwf, grp = n / (e.nkl * e.P);   // GQA widths
  char* wqkv = ws + bp.ws_off("wqkv");
  char* wproj = ws + bp.ws_off("wproj");
  char* win = ws + bp.ws_off("win");
  char* wout = ws + bp.ws_off("wout");
  char* dw = ws + bp.ws_off("dw");
  char* u1 = ws + bp.ws_off("u1");
  float* dp = reinterpret_cast<float*>(ws + bp.ws_off("scores"));
  char* ds = ws + bp.ws_off("ds");
  char* kr[2] = {ws + bp.ws_off("kr0"), ws + bp.ws_off("kr1")};
  float* dqacc = reinterpret_cast<float*>(ws + bp.ws_off("acc"));
  float* dacc[2] = {reinterpret_cast<float*>(ws + bp.ws_off("dacc0")), reinterpret_cast<float*>(ws + bp.ws_off("dacc1"))};
  char* dqkv = ws + bp.ws_off("dqkv");
  char* f0 = ws + bp.ws_off("f0");
  char* f1 = ws + bp.ws_off("f1");
  char* v2 = ws + bp.ws_off("v2");
  char* da = ws + bp.ws_off("da");
  float* dd = reinterpret_cast<float*>(ws + bp.ws_off("dd"));
  float* dgp = reinterpret_cast<float*>(ws + bp.ws_off("dgp"));
  float* dgl = reinterpret_cast<float*>(ws + bp.ws_off("dgl"));
  const char* qkv = sv->at("qkv");
  const char* probs = sv->at("probs");
  TN tn{e, ws + bp.ws_off("ta"), ws + bp.ws_off("tb"), ws + bp.ws_off("wt")};
  PDS_TRY(e.link(e.st, cs));
  PDS_TRY(e.ag(w->w_out, wout, e.Fl * h));
  PDS_TRY(e.ag_on(cs, w->w_in_t, win, e.f1w * h));
  cudaEvent_t ev_in = e.mark(cs);
  PDS_TRY(e.ag_on(cs, w->w_proj, wproj, e.hl * h));
  cudaEvent_t ev_proj = e.mark(cs);
  PDS_TRY(cz_wqkv(e, w, wqkv, cs));
  cudaEvent_t ev_qkv = e.mark(cs);
  PDS_CUDA(cudaMemsetAsync(dgl, 0, 2 * h * 4, e.st));
  GemmArgs dgel = Exec::G(dy, h, 0, wout, h, 0, e.sl, e.F, h, f1, e.f1wf, e.dfc1_epi());
  dgel.aux_in = sv->at("h"); dgel.ld_aux = e.F; dgel.ld_aux_in = e.f1wf;
  dgel.aux_t = tn.ta; dgel.c_t = f0; dgel.ld_t = e.sl;
  PDS_TRY(e.gemm(dgel));
  PDS_TRY(tn.tr(dy, h, e.sl, h, tn.tb));
  PDS_TRY(tn.mm(tn.ta, e.sl, tn.tb, e.sl, e.F, h, e.sl, dw, h, EPI_F32));               // dW_out (full, local)
  PDS_TRY(uz_dw(e, dw, e.F, g->dw_out));
  PDS_TRY(e.apply(sv->at("x1"), sv->at("rstd2"), w->g2, e.sl, u1));
  PDS_TRY(tn.tr(u1, h, e.sl, h, tn.tb));
  PDS_TRY(tn.mm(f0, e.sl, tn.tb, e.sl, e.f1wf, h, e.sl, dw, h, EPI_F32));               // dW_in^T (full, local)
  PDS_TRY(uz_dw(e, dw, e.f1wf, g->dw_in_t));
  PDS_TRY(e.wait(e.st, ev_in));
  PDS_TRY(tn.xw(f1, e.f1wf, win, h, e.sl, h, e.f1wf, v2, h));
  PDS_TRY(e.norm_bwd(v2, sv->at("x1"), sv->at("rstd2"), w->g2, dy, e.sl, dx, dgp, dgl + h));
  PDS_TRY(e.wait(e.st, ev_proj));
  PDS_TRY(e.gemm(Exec::G(dx, h, 0, wproj, h, 0, e.sl, h, h, da, h)));                  // dA = dO of attention
  PDS_TRY(tn.dw(sv->at("a"), h, dx, h, e.sl, h, h, dw, EPI_F32));
  PDS_TRY(uz_dw(e, dw, h, g->dw_proj));
  {
    Prof p(e.c, e.st, K_NORM, 0, (double)e.sl * h * 4);
    for (int64_t q = 0; q < b; ++q)
      PDS_TRY(kerr(attn_dot(sv->at("a") + q * h * 2, b * h, da + q * h * 2, (int)sp, (int)n, (int)d, dd + q * n * sp,
                            e.st), "attn_dot"));
  }
  // ring of V: dP_j = dO V_j^T, dV_j += P_j^T dO (the accumulator travels with V_j)
  PDS_CUDA(cudaMemsetAsync(dacc[0], 0, e.sl * hk * 4, e.st));
  int cur = 0;
  PDS_TRY(col_ring(e, qkv, h + hk, kr, [&](int, int j, const char* vb) -> pds_status {
    for (int64_t q = 0; q < b; ++q)
      for (int64_t hd = 0; hd < n; ++hd) {         // a value head's dV sums its query group (GQA)
        PDS_TRY(e.gemm(Exec::G(da + (q * h + hd * d) * 2, b * h, 0, vb + (q * hk + hd / grp * d) * 2, b * hk, 0, sp,
                               sp, d, dp + ((q * n + hd) * sp * sq + j * sp), sq, EPI_F32)));
        PDS_TRY(e.gemm(Exec::G(probs + ((q * n + hd) * sp * sq + j * sp) * 2, sq, 1, da + (q * h + hd * d) * 2,
                               b * h, 1, sp, d, sp, dacc[cur] + q * hk + hd / grp * d, b * hk, EPI_F32_ACC)));
      }
    if (e.P > 1) {
      PDS_TRY(ring_pass(e, reinterpret_cast<char*>(dacc[cur]), reinterpret_cast<char*>(dacc[cur ^ 1]),
                        e.sl * hk * 4, e.st));
      cur ^= 1;
    }
    return PDS_OK;
  }));
  // dV (home after P passes) -> the V columns of dQKV
  {
    Prof p(e.c, e.st, K_NORM, 0, (double)e.sl * h * 6);
    PDS_TRY(kerr(rope_t_f32_bf16(dacc[cur], hk, (int)e.sl, (int)hk, (int)d, nullptr, 0, 0, (int)e.sl, (int)b,
                                 dqkv + (h + hk) * 2, qw, e.st), "dv convert"));
  }
  {
    Prof p(e.c, e.st, K_NORM, 0, (double)b * n * sp * sq * 8);
    for (int64_t q = 0; q < b; ++q)
      PDS_TRY(kerr(rsa_dsoftmax(probs + q * n * sp * sq * 2, sq, dp + q * n * sp * sq, sq, dd + q * n * sp,
                                (int)(n * sp), (int)sq, 1.0f / std::sqrt((float)d), ds + q * n * sp * sq * 2, sq, e.st),
                   "rsa_dsoftmax"));
  }
  // ring of K: dQ += dS_j K_j, dK_j += dS_j^T Q (the accumulator travels with K_j)
  PDS_CUDA(cudaMemsetAsync(dqacc, 0, e.sl * h * 4, e.st));
  PDS_CUDA(cudaMemsetAsync(dacc[cur], 0, e.sl * hk * 4, e.st));
  PDS_TRY(col_ring(e, qkv, h, kr, [&](int, int j, const char* kb) -> pds_status {
    for (int64_t q = 0; q < b; ++q)
      for (int64_t hd = 0; hd < n; ++hd) {
        const char* dsb = ds + ((q * n + hd) * sp * sq + j * sp) * 2;
        PDS_TRY(e.gemm(Exec::G(dsb, sq, 0, kb + (q * hk + hd / grp * d) * 2, b * hk, 1, sp, d, sp,
                               dqacc + q * h + hd * d, b * h, EPI_F32_ACC)));
        PDS_TRY(e.gemm(Exec::G(dsb, sq, 1, qkv + (q * qw + hd * d) * 2, b * qw, 1, sp, d, sp,
                               dacc[cur] + q * hk + hd / grp * d, b * hk, EPI_F32_ACC)));
      }
    if (e.P > 1) {
      PDS_TRY(ring_pass(e, reinterpret_cast<char*>(dacc[cur]), reinterpret_cast<char*>(dacc[cur ^ 1]),
                        e.sl * hk * 4, e.st));
      cur ^= 1;
    }
    return PDS_OK;
  }));
  {
    Prof p(e.c, e.st, K_NORM, 0, (double)e.sl * (h + hk) * 6);
    const int64_t b0 = e.r * sp;
    PDS_TRY(kerr(rope_t_f32_bf16(dqacc, h, (int)e.sl, (int)h, (int)d, e.c->rope, b0, b0, (int)e.sl, (int)b, dqkv,
                                 qw, e.st), "dq rope_t"));
    PDS_TRY(kerr(rope_t_f32_bf16(dacc[cur], hk, (int)e.sl, (int)hk, (int)d, e.c->rope, b0, b0, (int)e.sl, (int)b,
                                 dqkv + h * 2, qw, e.st), "dk rope_t"));
  }
  PDS_TRY(e.apply(sv->x, sv->at("rstd1"), w->g1, e.sl, u1));
  PDS_TRY(tn.dw(dqkv, qw, u1, h, e.sl, qw, h, dw, EPI_F32));
  const int64_t hkl = e.nkl * d;
  const int64_t part_off[3] = {0, h * h, (h + hk) * h};            // rows of [Q all; K all; V all]
  const int64_t shard_off[3] = {0, e.hl * h, (e.hl + hkl) * h};    // rows of the spec shard
  const int64_t cnts[3] = {e.hl * h, hkl * h, hkl * h};
  for (int i = 0; i < 3; ++i) {
    char* part = dw + part_off[i] * 4;
    char* mine = part + e.r * cnts[i] * 4;
    PDS_TRY(e.rs(part, mine, cnts[i], DT_F32));
    PDS_TRY(kerr(add_f32(mine, static_cast<char*>(g->dw_qkv_t) + shard_off[i] * 4, cnts[i], e.st), "add_f32"));
  }
  PDS_TRY(e.wait(e.st, ev_qkv));
  PDS_TRY(tn.xw(dqkv, qw, wqkv, h, e.sl, h, qw, v2, h));                                // dU
  PDS_TRY(e.norm_bwd(v2, sv->x, sv->at("rstd1"), w->g1, dx, e.sl, dx, dgp, dgl));
  return e.dgamma(dgl, g);
}

// ================================================================== METP (R-METP)
int64_t metp_c(const Exec& e) { return e.m.metp_chunks > 0 ? e.m.metp_chunks : e.P; }

pds_status metp_fwd(Exec& e, const void* x, const pds_weights* w, void* y, pds_saved* sv, char* ws) {
  const BufPlan& bp = sv->plan;
  const int64_t c = metp_c(e), wr = e.sl / c, W = e.P * wr;   // wave rows per rank / gathered
  char* ul = ws + bp.ws_off("ul");
  char* vl = ws + bp.ws_off("vl");
  char* wg = ws + bp.ws_off("wg");
  char* pw = ws + bp.ws_off("pw");
  char* hw = ws + bp.ws_off("hw");
  char* gw = ws + bp.ws_off("gw");
  char* wt = ws + bp.ws_off("wt");
  TN tn{e, ws + bp.ws_off("ta"), ws + bp.ws_off("tb"), wt};
  const int64_t row = e.h * 2;
  const int64_t slot = e.r * wr * e.h * 2;
  const char* xb = static_cast<const char*>(x);
  // metp_recompute = full: Q/K/V live in the workspace (recomputed in bwd), not saved
  char* qkv = bp.has_ws("qkv") ? ws + bp.ws_off("qkv") : sv->at("qkv");
  // Wave gathers run on a side stream one wave ahead of the GEMMs ("asynchronous
  // ring-based execution"): AG(k+1) into one of two buffers while the
  // GEMM of wave k reads the other.  At P = 1 the gathers are identities.
  char* gb[2] = {wg, ws + bp.ws_off("wg2")};
  const cudaStream_t cs = e.c->comm->trivial() ? e.st : e.comm_stream();
  auto waves = [&](const char* src, auto&& gemm_wave) -> pds_status {
    PDS_TRY(e.link(e.st, cs));                                   // src rows are ready
    PDS_TRY(e.ag_on(cs, src, gb[0], wr * e.h));
    for (int64_t k = 0; k < c; ++k) {
      PDS_TRY(e.link(cs, e.st));                                 // wave k gathered
      if (k + 1 < c) PDS_TRY(e.ag_on(cs, src + (k + 1) * wr * row, gb[(k + 1) & 1], wr * e.h));
      PDS_TRY(gemm_wave(k, gb[k & 1]));
      if (k + 2 < c) PDS_TRY(e.link(e.st, cs));                  // buffer k & 1 free again
    }
    return PDS_OK;
  };
  PDS_TRY(e.norm_fwd(x, nullptr, w->g1, e.sl, nullptr, ul, sv->at("rstd1")));
  PDS_TRY(waves(ul, [&](int64_t k, char* buf) -> pds_status {   // QKV waves: rows land at global positions
    GemmArgs q = e.rope(Exec::G(buf, e.h, 0, w->w_qkv_t, e.h, 0, W, e.qw, e.h, qkv, e.qw),
                        e.hl, e.nkl * e.d, wr, e.sl, k * wr);
    q.c_seg = wr; q.c_stride = e.sl; q.c_base = k * wr;
    return e.gemm(q);
  }));
  PDS_TRY(e.attn_f(qkv, sv->at("a"), sv->at("lse")));             // query-chunk x KV-chunk loop
  PDS_TRY(tn.tr(w->w_proj, e.h, e.hl, e.h, wt));                 // W_proj^T, reused by every wave
  // P > 1: each wave's RS leaves tile by tile while its GEMM runs (as in TS, §7); the
  // wave-gather buffers, free during the projection waves, receive the peers' partials
  const bool ov = e.overlap();
  for (int64_t k = 0; k < c; ++k) {   // projection waves (A rows read through the TMA row remap)
    GemmArgs pj = Exec::G(sv->at("a"), e.hl, 0, wt, e.hl, 0, W, e.h, e.hl, pw, e.h);
    pj.a_seg = wr; pj.a_stride = e.sl; pj.a_base = k * wr; pj.a_rows = e.s;
    if (ov) PDS_TRY(e.rs_arm(e.h, wr));
    PDS_TRY(e.gemm(pj));
    PDS_TRY(ov ? e.rs_run(pw, gb[k & 1], wr * e.h) : e.rs(pw, pw + slot, wr * e.h));
    if (e.c->tap_o) PDS_TRY(e.tap(static_cast<char*>(e.c->tap_o) + k * wr * row, pw + slot, wr * e.h));
    PDS_TRY(e.norm_fwd(xb + k * wr * row, pw + slot, w->g2, wr, sv->at("x1") + k * wr * row, vl + k * wr * row,
                       sv->at("rstd2") + k * wr * 4));
  }
  PDS_TRY(tn.tr(w->w_out, e.h, e.Fl, e.h, wt));                  // W_out^T, reused by every wave
  return waves(vl, [&](int64_t k, char* buf) -> pds_status {     // FFN waves
    GemmArgs fc1 = Exec::G(buf, e.h, 0, w->w_in_t, e.h, 0, W, e.f1w, e.h, hw, e.f1w, e.fc1_epi());
    fc1.aux_out = gw; fc1.ld_aux = e.Fl;
    PDS_TRY(e.gemm(fc1));
    if (ov) PDS_TRY(e.rs_arm(e.h, wr));
    PDS_TRY(tn.mm(gw, e.Fl, wt, e.Fl, W, e.h, e.Fl, pw, e.h));
    PDS_TRY(ov ? e.rs_run(pw, buf, wr * e.h) : e.rs(pw, pw + slot, wr * e.h));   // buf: consumed by FC1
    if (e.c->tap_z) PDS_TRY(e.tap(static_cast<char*>(e.c->tap_z) + k * wr * row, pw + slot, wr * e.h));
    return e.add(sv->at("x1") + k * wr * row, pw + slot, static_cast<char*>(y) + k * wr * row, wr * e.h);
  });
}

pds_status metp_bwd(Exec& e, const void* dy, pds_saved* sv, const pds_weights* w, const pds_grads* g, void* dx,
                    char* ws) {
  const BufPlan& bp = sv->plan;
  const int64_t c = metp_c(e), wr = e.sl / c, W = e.P * wr;
  char* ul = ws + bp.ws_off("ul");
  char* vl = ws + bp.ws_off("vl");
  char* wg = ws + bp.ws_off("wg");
  char* wg2 = ws + bp.ws_off("wg2");
  char* pw = ws + bp.ws_off("pw");
  char* hw = ws + bp.ws_off("hw");
  char* gw = ws + bp.ws_off("gw");
  char* dhw = ws + bp.ws_off("dhw");
  char* da = ws + bp.ws_off("da");
  char* dqkv = ws + bp.ws_off("dqkv");
  char* wt = ws + bp.ws_off("wt");
  float* dd = reinterpret_cast<float*>(ws + bp.ws_off("dd"));
  float* dgp = reinterpret_cast<float*>(ws + bp.ws_off("dgp"));
  float* dgl = reinterpret_cast<float*>(ws + bp.ws_off("dgl"));
  TN tn{e, ws + bp.ws_off("ta"), ws + bp.ws_off("tb"), wt};
  const int64_t row = e.h * 2;
  const int64_t slot = e.r * wr * e.h * 2;
  const char* dyb = static_cast<const char*>(dy);
  const char* xb = static_cast<const char*>(sv->x);
  char* dxb = static_cast<char*>(dx);
  PDS_CUDA(cudaMemsetAsync(dgl, 0, 2 * e.h * 4, e.st));
  const bool ov = e.overlap();       // P > 1: wave AG / RS overlapped with the wave GEMMs' tiles
  PDS_TRY(tn.tr(w->w_in_t, e.h, e.f1w, e.h, wt));                // W_in (= (W_in^T)^T) for dV, every wave
  for (int64_t k = 0; k < c; ++k) {   // FFN backward waves, recomputing v, H, G
    const int64_t o = k * wr;
    PDS_TRY(e.apply(sv->at("x1") + o * row, sv->at("rstd2") + o * 4, w->g2, wr, vl));
    if (ov) {                          // tile-overlapped wave gathers (§7)
      PDS_CUDA(cudaMemcpyAsync(wg2 + slot, vl, wr * row, cudaMemcpyDeviceToDevice, e.st));
      PDS_TRY(e.ag_next(wg2, wr * e.h, wr));                                             // AG(v)
      PDS_TRY(tn.mm(wg2, e.h, w->w_in_t, e.h, W, e.f1w, e.h, hw, e.f1w));               // H recompute
      PDS_CUDA(cudaMemcpyAsync(wg + slot, dyb + o * row, wr * row, cudaMemcpyDeviceToDevice, e.st));
      PDS_TRY(e.ag_next(wg, wr * e.h, wr));                                              // AG(dz)
    } else {
      PDS_TRY(e.ag(dyb + o * row, wg, wr * e.h));                                       // AG(dz)
      PDS_TRY(e.ag(vl, wg2, wr * e.h));                                                  // AG(v)
      PDS_TRY(tn.mm(wg2, e.h, w->w_in_t, e.h, W, e.f1w, e.h, hw, e.f1w));               // H recompute
    }
    GemmArgs dgel = Exec::G(wg, e.h, 0, w->w_out, e.h, 0, W, e.Fl, e.h, dhw, e.f1w, e.dfc1_epi());
    dgel.aux_in = hw; dgel.ld_aux = e.Fl; dgel.ld_aux_in = e.f1w;
    dgel.aux_t = tn.ta; dgel.c_t = gw; dgel.ld_t = W;                                  // G^T, dH^T
    PDS_TRY(e.gemm(dgel));
    PDS_TRY(tn.tr(wg, e.h, W, e.h, tn.tb));
    PDS_TRY(tn.mm(tn.ta, W, tn.tb, W, e.Fl, e.h, W, g->dw_out, e.h, EPI_F32_ACC));      // dW_out += G^T dZ
    PDS_TRY(tn.tr(wg2, e.h, W, e.h, tn.tb));
    PDS_TRY(tn.mm(gw, W, tn.tb, W, e.f1w, e.h, W, g->dw_in_t, e.h, EPI_F32_ACC));       // dW_in^T += dH^T V
    if (ov) PDS_TRY(e.rs_arm(e.h, wr));
    PDS_TRY(tn.mm(dhw, e.f1w, wt, e.f1w, W, e.h, e.f1w, pw, e.h));
    PDS_TRY(ov ? e.rs_run(pw, wg, wr * e.h) : e.rs(pw, pw + slot, wr * e.h));            // RS(dv)
    PDS_TRY(e.norm_bwd(pw + slot, sv->at("x1") + o * row, sv->at("rstd2") + o * 4, w->g2, dyb + o * row, wr,
                       dxb + o * row, dgp, dgl + e.h));
  }
  for (int64_t k = 0; k < c; ++k) {   // projection backward waves
    const int64_t o = k * wr;
    if (ov) {
      PDS_CUDA(cudaMemcpyAsync(wg + slot, dxb + o * row, wr * row, cudaMemcpyDeviceToDevice, e.st));
      PDS_TRY(e.ag_next(wg, wr * e.h, wr));                                              // AG(dx1)
    } else {
      PDS_TRY(e.ag(dxb + o * row, wg, wr * e.h));                                        // AG(dx1)
    }
    GemmArgs dA = Exec::G(wg, e.h, 0, w->w_proj, e.h, 0, W, e.hl, e.h, da, e.hl);
    dA.c_seg = wr; dA.c_stride = e.sl; dA.c_base = o;
    PDS_TRY(e.gemm(dA));
    PDS_TRY(tn.dw(sv->at("a"), e.hl, wg, e.h, W, e.hl, e.h, g->dw_proj, EPI_F32_ACC, wr, e.sl, o));
  }
  char* qkv = sv->plan.has_ws("qkv") ? ws + bp.ws_off("qkv") : sv->at("qkv");
  if (bp.has_ws("qkv")) {             // full: Q/K/V recomputed from per-wave re-gathers of u
    for (int64_t k = 0; k < c; ++k) {
      const int64_t o = k * wr;
      PDS_TRY(e.apply(xb + o * row, sv->at("rstd1") + o * 4, w->g1, wr, ul));
      PDS_TRY(e.ag(ul, wg, wr * e.h));                                                   // AG(u) recompute
      GemmArgs q = e.rope(Exec::G(wg, e.h, 0, w->w_qkv_t, e.h, 0, W, e.qw, e.h, qkv, e.qw),
                          e.hl, e.nkl * e.d, wr, e.sl, o);
      q.c_seg = wr; q.c_stride = e.sl; q.c_base = o;
      PDS_TRY(e.gemm(q));
    }
  }
  // the dQ accumulator borrows ul + vl (adjacent, 2u, free between the waves)
  const int64_t ulv = bp.ws_off("vl") == bp.ws_off("ul") + bp.ws_size("ul") ? 2 * bp.ws_size("ul") : bp.ws_size("ul");
  PDS_TRY(e.attn_b(qkv, sv->at("a"), sv->at("lse"), da, dqkv, dd, ul, ulv,
                   reinterpret_cast<int*>(ws + bp.ws_off("actr")), bp.has_ws("dsb") ? ws + bp.ws_off("dsb") : nullptr,
                   bp.ws_size("dsb")));
  PDS_TRY(tn.tr(w->w_qkv_t, e.h, e.qw, e.h, wt));                // W_qkv for dU, every wave
  for (int64_t k = 0; k < c; ++k) {   // QKV backward waves
    const int64_t o = k * wr;
    PDS_TRY(e.apply(xb + o * row, sv->at("rstd1") + o * 4, w->g1, wr, ul));
    PDS_TRY(e.ag(ul, wg, wr * e.h));                                                     // AG(u)
    PDS_TRY(tn.dw(dqkv, e.qw, wg, e.h, W, e.qw, e.h, g->dw_qkv_t, EPI_F32_ACC, wr, e.sl, o));
    GemmArgs du = Exec::G(dqkv, e.qw, 0, wt, e.qw, 0, W, e.h, e.qw, pw, e.h);
    du.a_seg = wr; du.a_stride = e.sl; du.a_base = o; du.a_rows = e.s;
    if (ov) PDS_TRY(e.rs_arm(e.h, wr));
    PDS_TRY(e.gemm(du));
    PDS_TRY(ov ? e.rs_run(pw, wg2, wr * e.h) : e.rs(pw, pw + slot, wr * e.h));           // RS(du)
    PDS_TRY(e.norm_bwd(pw + slot, xb + o * row, sv->at("rstd1") + o * 4, w->g1, dxb + o * row, wr, dxb + o * row,
                       dgp, dgl));
  }
  return e.dgamma(dgl, g);
}

// ------------------------------------------------------------------ ctx helpers
pds_status ensure_ws(pds_ctx* c, int64_t bytes, cudaStream_t st) {
  if (bytes <= c->ws_cap) return PDS_OK;
  PDS_CUDA(cudaStreamSynchronize(st));
  if (c->ws) PDS_CUDA(cudaFree(c->ws));
  c->ws = nullptr;
  c->ws_cap = 0;
  PDS_CUDA(cudaMalloc(&c->ws, bytes));
  c->ws_cap = bytes;
  return PDS_OK;
}

pds_status ensure_rope(pds_ctx* c, int64_t s, cudaStream_t st) {
  if (s <= c->rope_pos) return PDS_OK;
  const int64_t d = c->m.h / c->m.n_heads;
  const int64_t n = std::max<int64_t>(s, 2 * c->rope_pos);
  PDS_CUDA(cudaStreamSynchronize(st));
  if (c->rope) PDS_CUDA(cudaFree(c->rope));
  c->rope = nullptr;
  PDS_CUDA(cudaMalloc(&c->rope, n * (d / 2) * 8));
  c->rope_pos = n;
  return kerr(rope_table(c->rope, n, (int)d, c->m.rope_theta, st), "rope_table");
}

pds_status alloc_saved(pds_ctx* c, int64_t bytes, char** out) {
  auto it = c->free_blocks.find(bytes);
  if (it != c->free_blocks.end()) {
    *out = it->second;
    c->free_blocks.erase(it);
    return PDS_OK;
  }
  cudaError_t e = cudaMalloc(out, bytes);
  if (e == cudaErrorMemoryAllocation && !c->free_blocks.empty()) {
    cudaGetLastError();
    cudaDeviceSynchronize();
    for (auto& kv : c->free_blocks) cudaFree(kv.second);
    c->free_blocks.clear();
    e = cudaMalloc(out, bytes);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error(std::string("saved arena cudaMalloc(") + std::to_string(bytes) + "): " + cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? PDS_ENOMEM : PDS_ECUDA;
  }
  return PDS_OK;
}

pds_status check_layer(pds_ctx* c, uint8_t strategy, int64_t s) {
  if (!c) PDS_FAIL(PDS_EINVAL, "NULL ctx");
  if (c->device < 0) PDS_FAIL(PDS_ESTATE, "host-only planner context (device < 0) runs no layer");
  if (strategy >= PDS_N_STRATEGIES) PDS_FAIL(PDS_ESTRATEGY, "unknown strategy id " + std::to_string(strategy));
  return PDS_OK;
}

}  // namespace

// ================================================================== C ABI
extern "C" pds_status pds_nccl_unique_id(void* out128);

static pds_status ctx_common(pds_ctx* c, const pds_model* m, int P, int rank, int device) {
  if (!m) PDS_FAIL(PDS_EINVAL, "NULL model");
  if (P < 1 || P > 8) PDS_FAIL(PDS_EINVAL, "P must be in [1, 8]");
  if (rank < 0 || rank >= P) PDS_FAIL(PDS_EINVAL, "rank out of range");
  c->m = *m;
  if (c->m.norm_eps <= 0) c->m.norm_eps = 1e-5f;
  if (c->m.rope_theta <= 0) c->m.rope_theta = 10000.0;
  c->P = P;
  c->rank = rank;
  c->device = device;
  BufPlan probe;
  PDS_TRY(make_plan(c->m, P, PDS_MEGATRON_TS, (int64_t)128 * P, &probe));   // validates dims
  if (device < 0) {            // host-only planner context: no CUDA call, capacity from the bundle
    c->capacity = 0;
    return PDS_OK;
  }
  PDS_CUDA(cudaSetDevice(device));
  size_t fr = 0, tot = 0;
  PDS_CUDA(cudaMemGetInfo(&fr, &tot));
  c->capacity = (double)tot;
  return PDS_OK;
}

extern "C" pds_status pds_create(const pds_model* model, int32_t P, int32_t rank, int32_t device,
                                 const void* nccl_unique_id, pds_ctx** out) {
  if (!out) PDS_FAIL(PDS_EINVAL, "NULL out");
  std::unique_ptr<pds_ctx> c(new pds_ctx());
  PDS_TRY(ctx_common(c.get(), model, P, rank, device));
  if (device < 0) {            // planner only (pds_plan / pds_cost_eval): no communicator
    if (nccl_unique_id) PDS_FAIL(PDS_EINVAL, "a host-only context (device < 0) takes no NCCL id");
    *out = c.release();
    return PDS_OK;
  }
  if (P == 1 && !nccl_unique_id) {
    c->comm = make_self_comm();
  } else {       // P = 1 with an id: a one-rank NCCL communicator (exercises the NCCL path)
    if (!nccl_unique_id) PDS_FAIL(PDS_EINVAL, "P > 1 needs an NCCL unique id");
    pds_status st = PDS_OK;
    c->comm = make_nccl_comm(P, rank, nccl_unique_id, &st);
    if (st != PDS_OK) return st;
    // The tile-overlapped collectives (persistent GEMMs polling flags that a CTA-capped
    // NCCL side communicator sets) have run on one GPU only (loopback, one-rank NCCL);
    // with real peers they are opt-in until tests/test_multigpu_nccl.py has passed on
    // the hardware: PDS_OVERLAP=1 or pds_set_overlap(ctx, 1).
    const char* ov = getenv("PDS_OVERLAP");
    if (P > 1) c->overlap = ov && atoi(ov) != 0;
  }
  *out = c.release();
  return PDS_OK;
}

extern "C" pds_status pds_group_create(int32_t P, pds_group** out) {
  if (!out || P < 1 || P > 8) PDS_FAIL(PDS_EINVAL, "pds_group_create: bad args");
  pds_group* g = new pds_group();
  g->g.P = P;
  g->g.ptr.assign(P, nullptr);
  g->g.ready.resize(P);
  g->g.done.resize(P);
  for (int i = 0; i < P; ++i) {
    cudaEventCreateWithFlags(&g->g.ready[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&g->g.done[i], cudaEventDisableTiming);
  }
  *out = g;
  return PDS_OK;
}

extern "C" pds_status pds_group_destroy(pds_group* g) {
  if (!g) return PDS_OK;
  for (auto e : g->g.ready) cudaEventDestroy(e);
  for (auto e : g->g.done) cudaEventDestroy(e);
  delete g;
  return PDS_OK;
}

extern "C" pds_status pds_create_loopback(const pds_model* model, pds_group* g, int32_t rank, int32_t device,
                                          pds_ctx** out) {
  if (!out || !g) PDS_FAIL(PDS_EINVAL, "NULL argument");
  std::unique_ptr<pds_ctx> c(new pds_ctx());
  PDS_TRY(ctx_common(c.get(), model, g->g.P, rank, device));
  pds_status st = PDS_OK;
  c->comm = g->g.P == 1 ? make_self_comm() : make_loop_comm(&g->g, rank, &st);
  if (st != PDS_OK) return st;
  *out = c.release();
  return PDS_OK;
}

extern "C" pds_status pds_destroy(pds_ctx* c) {
  if (!c) return PDS_OK;
  if (c->device >= 0) {
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
  }
  delete c;
  return PDS_OK;
}

extern "C" pds_status pds_reserve(pds_ctx* c, int64_t max_seq_len, uint32_t mask) {
  if (!c) PDS_FAIL(PDS_EINVAL, "NULL ctx");
  if (c->device < 0) PDS_FAIL(PDS_ESTATE, "host-only planner context (device < 0)");
  int64_t need = 0;
  for (int i = 0; i < PDS_N_STRATEGIES; ++i) {
    if (!(mask >> i & 1)) continue;
    BufPlan bp;
    PDS_TRY(make_plan(c->m, c->P, i, max_seq_len, &bp));
    need = std::max(need, bp.ws_bytes);
  }
  PDS_CUDA(cudaSetDevice(c->device));
  PDS_TRY(ensure_ws(c, need, 0));
  return ensure_rope(c, max_seq_len, 0);
}

extern "C" pds_status pds_release_cache(pds_ctx* c) {
  if (!c) PDS_FAIL(PDS_EINVAL, "NULL ctx");
  if (c->device < 0) return PDS_OK;
  PDS_CUDA(cudaSetDevice(c->device));
  PDS_CUDA(cudaDeviceSynchronize());
  for (auto& kv : c->free_blocks) cudaFree(kv.second);
  c->free_blocks.clear();
  if (c->ws) cudaFree(c->ws);
  c->ws = nullptr;
  c->ws_cap = 0;
  if (c->stage) cudaFree(c->stage);
  c->stage = nullptr;
  c->stage_cap = 0;
  c->stage_used[0] = c->stage_used[1] = false;
  return PDS_OK;
}

extern "C" pds_status pds_comm_log(pds_ctx* c, int32_t on) {
  if (!c) PDS_FAIL(PDS_EINVAL, "NULL ctx");
  c->comm_log_on = on != 0;
  c->comm_log.clear();
  return PDS_OK;
}

extern "C" pds_status pds_comm_log_read(pds_ctx* c, char* buf, int64_t cap, int64_t* len_out) {
  if (!c || !len_out) PDS_FAIL(PDS_EINVAL, "NULL ctx / len_out");
  *len_out = (int64_t)c->comm_log.size();
  if (buf && cap > 0) {
    const int64_t n = std::min<int64_t>(cap - 1, (int64_t)c->comm_log.size());
    std::memcpy(buf, c->comm_log.data(), (size_t)n);
    buf[n] = 0;
  }
  return PDS_OK;
}

extern "C" pds_status pds_set_varlen(pds_ctx* c, int32_t n_seqs, const int64_t* lens) {
  if (!c) PDS_FAIL(PDS_EINVAL, "NULL ctx");
  if (n_seqs < 0 || (n_seqs > 0 && !lens)) PDS_FAIL(PDS_EINVAL, "pds_set_varlen: bad n_seqs / lens");
  if (n_seqs == 0) {
    c->segs = nullptr;
    c->varlen_tokens = 0;
    return PDS_OK;
  }
  if (c->m.batch != 1) PDS_FAIL(PDS_EINVAL, "varlen packing replaces the batch: batch must be 1");
  if (c->device < 0) PDS_FAIL(PDS_ESTATE, "host-only planner context (device < 0)");
  int64_t T = 0;
  std::vector<int> tab;
  for (int i = 0; i < n_seqs; ++i) {
    if (lens[i] <= 0 || lens[i] % 256)
      PDS_FAIL(PDS_EDIVISIBILITY, "varlen: sequence " + std::to_string(i) + " length " + std::to_string(lens[i]) +
                                      " must be a positive multiple of 256 (caller pads, R-VARLEN)");
    const int lo = (int)(T / 128), hi = (int)((T + lens[i]) / 128);
    for (int blk = lo; blk < hi; ++blk) {
      tab.push_back(lo);
      tab.push_back(hi);
    }
    T += lens[i];
  }
  int* d = nullptr;
  PDS_CUDA(cudaSetDevice(c->device));
  PDS_CUDA(cudaMalloc(&d, tab.size() * sizeof(int)));
  c->seg_tables.push_back(d);
  PDS_CUDA(cudaMemcpy(d, tab.data(), tab.size() * sizeof(int), cudaMemcpyHostToDevice));
  c->segs = d;
  c->varlen_tokens = T;
  return PDS_OK;
}

extern "C" pds_status pds_set_overlap(pds_ctx* c, int32_t on) {
  if (!c) PDS_FAIL(PDS_EINVAL, "pds_set_overlap: null ctx");
  c->overlap = on ? 1 : 0;
  return PDS_OK;
}

extern "C" pds_status pds_debug_taps(pds_ctx* c, void* o_out, void* z_out) {
  if (!c) PDS_FAIL(PDS_EINVAL, "NULL ctx");
  c->tap_o = o_out;
  c->tap_z = z_out;
  return PDS_OK;
}

extern "C" pds_status pds_layer_fwd(pds_ctx* c, uint8_t strategy, int64_t seq_len, const void* x,
                                    const pds_weights* w, void* y, pds_saved** saved, void* stream) {
  PDS_TRY(check_layer(c, strategy, seq_len));
  if (!x || !w || !y) PDS_FAIL(PDS_EINVAL, "NULL x / w / y");
  if (!w->w_qkv_t || !w->w_proj || !w->w_in_t || !w->w_out || !w->g1 || !w->g2)
    PDS_FAIL(PDS_EINVAL, "NULL weight pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  BufPlan bp;
  PDS_TRY(make_plan(c->m, c->P, strategy, seq_len, &bp));
  if (c->segs) {
    if (seq_len != c->varlen_tokens)
      PDS_FAIL(PDS_EINVAL, "varlen: seq_len=" + std::to_string(seq_len) + " != the packed total " +
                               std::to_string(c->varlen_tokens) + " (pds_set_varlen)");
    if (strategy == PDS_MEGATRON_CZ || strategy == PDS_COLOSSAL_Z)
      PDS_FAIL(PDS_ENOTIMPL, "varlen packing runs on MegatronTS, UlyssesZ, METP and METP-full only");
  }
  PDS_CUDA(cudaSetDevice(c->device));
  PDS_TRY(ensure_ws(c, bp.ws_bytes, st));
  PDS_TRY(ensure_rope(c, seq_len, st));
  std::unique_ptr<pds_saved> sv(new pds_saved());
  sv->strategy = strategy;
  sv->s = seq_len;
  sv->segs = c->segs;
  sv->x = x;
  sv->plan = bp;
  sv->bytes = bp.saved_bytes;
  PDS_TRY(alloc_saved(c, bp.saved_bytes, &sv->mem));
  Exec e(c, st, seq_len, sv->segs);
  pds_status rc;
  nvtxRangePushA(kLayerName[strategy][0]);
  switch (strategy) {
    case PDS_MEGATRON_TS: rc = ts_fwd(e, x, w, y, sv.get(), c->ws); break;
    case PDS_ULYSSES_Z: rc = uz_fwd(e, x, w, y, sv.get(), c->ws); break;
    case PDS_MEGATRON_CZ: rc = cz_fwd(e, x, w, y, sv.get(), c->ws); break;
    case PDS_COLOSSAL_Z: rc = col_fwd(e, x, w, y, sv.get(), c->ws); break;
    default: rc = metp_fwd(e, x, w, y, sv.get(), c->ws); break;
  }
  nvtxRangePop();
  c->tap_o = c->tap_z = nullptr;
  if (rc != PDS_OK || !saved) {
    c->free_blocks.emplace(sv->bytes, sv->mem);
    return rc;
  }
  c->saved_live += sv->bytes;
  *saved = sv.release();
  return PDS_OK;
}

extern "C" pds_status pds_layer_bwd(pds_ctx* c, uint8_t strategy, const void* dy, pds_saved* saved,
                                    const pds_weights* w, const pds_grads* g, void* dx, void* stream) {
  PDS_TRY(check_layer(c, strategy, saved ? saved->s : 0));
  if (!dy || !saved || !w || !g || !dx) PDS_FAIL(PDS_EINVAL, "NULL argument");
  if (!g->dw_qkv_t || !g->dw_proj || !g->dw_in_t || !g->dw_out || !g->dg1 || !g->dg2)
    PDS_FAIL(PDS_EINVAL, "NULL gradient pointer");
  if (saved->strategy != strategy)
    PDS_FAIL(PDS_ESTATE, "bwd strategy " + std::to_string(strategy) + " != fwd strategy " +
                             std::to_string(saved->strategy));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  PDS_CUDA(cudaSetDevice(c->device));
  PDS_TRY(ensure_ws(c, saved->plan.ws_bytes, st));
  Exec e(c, st, saved->s, saved->segs);
  pds_status rc;
  nvtxRangePushA(kLayerName[strategy][1]);
  switch (strategy) {
    case PDS_MEGATRON_TS: rc = ts_bwd(e, dy, saved, w, g, dx, c->ws); break;
    case PDS_ULYSSES_Z: rc = uz_bwd(e, dy, saved, w, g, dx, c->ws); break;
    case PDS_MEGATRON_CZ: rc = cz_bwd(e, dy, saved, w, g, dx, c->ws); break;
    case PDS_COLOSSAL_Z: rc = col_bwd(e, dy, saved, w, g, dx, c->ws); break;
    default: rc = metp_bwd(e, dy, saved, w, g, dx, c->ws); break;
  }
  nvtxRangePop();
  c->saved_live -= saved->bytes;
  c->free_blocks.emplace(saved->bytes, saved->mem);
  delete saved;
  return rc;
}

// One layer fwd + bwd with HOST activations.  Uploads run on an upload stream, the
// y / dx downloads on a download stream, and consecutive calls alternate between two
// staging sets, so call k+1's uploads overlap call k's compute and call k's
// downloads overlap call k+1's compute.  pds_host_drain orders `stream` after every
// outstanding download.
extern "C" pds_status pds_layer_step_host(pds_ctx* c, uint8_t strategy, int64_t seq_len, const void* x_host,
                                          const void* dy_host, const pds_weights* w, const pds_grads* g,
                                          void* y_host, void* dx_host, void* stream) {
  PDS_TRY(check_layer(c, strategy, seq_len));
  if (!x_host || !dy_host || !y_host || !dx_host) PDS_FAIL(PDS_EINVAL, "NULL host buffer");
  if (seq_len <= 0 || seq_len % c->P) PDS_FAIL(PDS_EDIVISIBILITY, "seq_len not divisible by P");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  PDS_CUDA(cudaSetDevice(c->device));
  const int64_t nb = seq_len / c->P * c->m.batch * c->m.h * 2;   // one local [s/P, b, h] bf16 activation
  const int64_t slot = (nb + 255) / 256 * 256;
  if (!c->up_st) {
    PDS_CUDA(cudaStreamCreateWithFlags(&c->up_st, cudaStreamNonBlocking));
    PDS_CUDA(cudaStreamCreateWithFlags(&c->down_st, cudaStreamNonBlocking));
    for (cudaEvent_t* e : {&c->ev_in[0], &c->ev_in[1], &c->ev_done[0], &c->ev_done[1], &c->ev_y, &c->ev_dx})
      PDS_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  }
  if (c->stage_cap < 4 * slot) {
    PDS_CUDA(cudaDeviceSynchronize());                   // every outstanding step is done with the old sets
    if (c->stage) PDS_CUDA(cudaFree(c->stage));
    c->stage = nullptr;
    c->stage_cap = 0;
    c->stage_used[0] = c->stage_used[1] = false;
    cudaError_t e = cudaMalloc(&c->stage, 2 * 4 * slot);
    if (e != cudaSuccess) {
      cudaGetLastError();
      PDS_FAIL(e == cudaErrorMemoryAllocation ? PDS_ENOMEM : PDS_ECUDA,
               std::string("staging cudaMalloc: ") + cudaGetErrorString(e));
    }
    c->stage_cap = 4 * slot;
  }
  const int b = c->stage_next;
  c->stage_next ^= 1;
  char* base = c->stage + b * c->stage_cap;
  char *x = base, *dy = base + slot, *y = base + 2 * slot, *dx = base + 3 * slot;
  // uploads: set b is free once the call that last used it has downloaded dx
  if (c->stage_used[b]) PDS_CUDA(cudaStreamWaitEvent(c->up_st, c->ev_done[b], 0));
  PDS_CUDA(cudaMemcpyAsync(x, x_host, nb, cudaMemcpyHostToDevice, c->up_st));
  PDS_CUDA(cudaMemcpyAsync(dy, dy_host, nb, cudaMemcpyHostToDevice, c->up_st));
  PDS_CUDA(cudaEventRecord(c->ev_in[b], c->up_st));
  PDS_CUDA(cudaStreamWaitEvent(st, c->ev_in[b], 0));
  pds_saved* sv = nullptr;
  PDS_TRY(pds_layer_fwd(c, strategy, seq_len, x, w, y, &sv, stream));
  PDS_CUDA(cudaEventRecord(c->ev_y, st));
  PDS_CUDA(cudaStreamWaitEvent(c->down_st, c->ev_y, 0));
  PDS_CUDA(cudaMemcpyAsync(y_host, y, nb, cudaMemcpyDeviceToHost, c->down_st));
  PDS_TRY(pds_layer_bwd(c, strategy, dy, sv, w, g, dx, stream));
  PDS_CUDA(cudaEventRecord(c->ev_dx, st));
  PDS_CUDA(cudaStreamWaitEvent(c->down_st, c->ev_dx, 0));
  PDS_CUDA(cudaMemcpyAsync(dx_host, dx, nb, cudaMemcpyDeviceToHost, c->down_st));
  PDS_CUDA(cudaEventRecord(c->ev_done[b], c->down_st));
  c->stage_used[b] = true;
  return PDS_OK;
}

extern "C" pds_status pds_host_drain(pds_ctx* c, void* stream) {
  if (!c) PDS_FAIL(PDS_EINVAL, "NULL ctx");
  if (!c->down_st) return PDS_OK;
  cudaEvent_t ev;
  PDS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  PDS_CUDA(cudaEventRecord(ev, c->down_st));
  PDS_CUDA(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), ev, 0));
  PDS_CUDA(cudaEventDestroy(ev));
  return PDS_OK;
}

extern "C" pds_status pds_saved_release(pds_ctx* c, pds_saved* saved) {
  if (!c || !saved) PDS_FAIL(PDS_EINVAL, "NULL argument");
  c->saved_live -= saved->bytes;
  c->free_blocks.emplace(saved->bytes, saved->mem);
  delete saved;
  return PDS_OK;
}

// ------------------------------------------------------------------ planner with ctx
extern "C" pds_status pds_load_costs(pds_ctx* c, const char* path) {
  if (!c || !path) PDS_FAIL(PDS_EINVAL, "NULL argument");
  Bundle b;
  PDS_TRY(load_bundle(path, &b));
  if (b.P != c->P || b.h != c->m.h || b.n != c->m.n_heads || b.ffn != c->m.ffn)
    PDS_FAIL(PDS_EINVAL, "bundle (P, h, n, ffn) does not match the context");
  const int kv_b = b.n_kv > 0 ? b.n_kv : b.n, kv_c = c->m.n_kv_heads > 0 ? c->m.n_kv_heads : c->m.n_heads;
  if (kv_b != kv_c || b.act != c->m.ffn_act)
    PDS_FAIL(PDS_EINVAL, "bundle (n_kv, ffn_act) does not match the context");
  c->bundle = b;
  c->cache.clear();
  c->prev.clear();
  c->capacity = b.capacity > 0 ? b.capacity - b.reserve : c->capacity;
  return PDS_OK;
}

extern "C" pds_status pds_set_capacity(pds_ctx* c, double capacity, double gamma) {
  if (!c || capacity <= 0 || gamma < 0 || gamma >= 1) PDS_FAIL(PDS_EINVAL, "bad capacity / gamma");
  c->capacity = capacity;
  c->gamma = gamma;
  c->cache.clear();
  return PDS_OK;
}

extern "C" pds_status pds_set_enabled(pds_ctx* c, uint32_t mask) {
  const uint32_t all = (1u << PDS_N_STRATEGIES) - 1;
  if (!c || !(mask & all)) PDS_FAIL(PDS_EINVAL, "empty strategy mask");
  c->enabled = mask & all;
  c->cache.clear();
  c->prev.clear();
  return PDS_OK;
}

// T_pi(s) from the bundle (Eq. 9) and M_pi(s) = persistent + saved bytes of one
// layer (exact plan); w = its workspace (one per plan, reading R-22)
static pds_status costs(pds_ctx* c, int64_t s, double* t, double* mm, int* branch, double* w) {
  if (!c->bundle.loaded) PDS_FAIL(PDS_ENOCOSTS, "no cost bundle loaded (pds_load_costs)");
  for (int i = 0; i < PDS_N_STRATEGIES; ++i) {
    t[i] = c->bundle.strat[i].present ? bundle_time(c->bundle, i, s, branch ? &branch[i] : nullptr) : 1e300;
    int64_t saved = 0, tr = 0, pers = 0;
    pds_status rc = pds_mem_bytes(&c->m, c->P, (uint8_t)i, s, &saved, &tr, &pers);
    if (rc != PDS_OK) {
      mm[i] = 1e300;
      if (w) w[i] = 1e300;
      continue;
    }
    mm[i] = (double)(saved + pers);
    if (w) w[i] = (double)tr;
  }
  return PDS_OK;
}

extern "C" pds_status pds_cost_eval(pds_ctx* c, int64_t s, double* t_layer, double* m_layer, int32_t* branch) {
  if (!c || !t_layer || !m_layer) PDS_FAIL(PDS_EINVAL, "NULL argument");
  double t[PDS_N_STRATEGIES], mm[PDS_N_STRATEGIES];
  int br[PDS_N_STRATEGIES] = {};
  PDS_TRY(costs(c, s, t, mm, br, nullptr));
  for (int i = 0; i < PDS_N_STRATEGIES; ++i) {
    t_layer[i] = t[i];
    m_layer[i] = mm[i];
    if (branch) branch[i] = br[i];
  }
  return PDS_OK;
}

extern "C" pds_status pds_plan(pds_ctx* c, int64_t s, uint8_t* out, int32_t L, uint32_t* flags_out) {
  if (!c || !out) PDS_FAIL(PDS_EINVAL, "NULL argument");
  if (L <= 0) PDS_FAIL(PDS_EINVAL, "L must be >= 1");
  uint32_t flags = 0;
  std::vector<uint8_t> plan;
  double t[PDS_N_STRATEGIES], mm[PDS_N_STRATEGIES], ws[PDS_N_STRATEGIES];
  const auto key = std::make_pair(c->m.batch, s);
  auto it = c->cache.find(key);
  bool need_costs = true;
  if (it != c->cache.end() && (int)it->second.first.size() == L) {
    plan = it->second.first;
    flags |= PDS_PLAN_CACHED | (it->second.second ? PDS_PLAN_INFEASIBLE : 0u);
  } else {
    PDS_TRY(costs(c, s, t, mm, nullptr, ws));
    need_costs = false;
    uint8_t en[PDS_N_STRATEGIES];
    for (int i = 0; i < PDS_N_STRATEGIES; ++i) en[i] = (c->enabled >> i & 1) && c->bundle.strat[i].present && mm[i] < 1e299;
    const double cap = c->capacity;
    bool inf = false, early = false;
    bool any = false;
    for (int i = 0; i < PDS_N_STRATEGIES; ++i) any |= en[i] != 0;
    if (!any) PDS_FAIL(PDS_ESTRATEGY, "no enabled strategy is valid at this seq_len");
    alg1(L, PDS_N_STRATEGIES, t, mm, ws, en, cap, plan, &inf, &early, nullptr);
    flags |= (inf ? PDS_PLAN_INFEASIBLE : 0u) | (early ? PDS_PLAN_EARLY : 0u);
    c->cache[key] = std::make_pair(plan, inf);
  }
  // smoothing (R-19) exactly as pds_plan_ex: keep the previous plan if it is valid,
  // feasible and within (1 + gamma) of the new one (gamma = 0: only exact time ties)
  if ((int)c->prev.size() == L && c->prev != plan) {
    if (need_costs) PDS_TRY(costs(c, s, t, mm, nullptr, ws));
    bool valid = true;
    for (uint8_t p : c->prev) valid &= (c->enabled >> p & 1) && mm[p] < 1e299;
    const double cap = c->capacity;
    if (valid && plan_feasible(c->prev.data(), L, mm, ws, cap, nullptr) &&
        plan_time(c->prev.data(), L, t) <= (1.0 + c->gamma) * plan_time(plan.data(), L, t)) {
      plan = c->prev;
      flags |= PDS_PLAN_SMOOTHED;
      flags &= ~PDS_PLAN_INFEASIBLE;
    }
  }
  c->prev = plan;
  std::memcpy(out, plan.data(), (size_t)L);
  if (flags_out) *flags_out = flags;
  return PDS_OK;
}

// ------------------------------------------------------------------ profiling
extern "C" pds_status pds_profile_enable(pds_ctx* c, int32_t on) {
  if (!c) PDS_FAIL(PDS_EINVAL, "NULL ctx");
  c->prof = on != 0;
  return PDS_OK;
}

static void drain(pds_ctx* c) {
  for (auto& r : c->pending) {
    cudaEventSynchronize(r.b);
    float ms = 0;
    cudaEventElapsedTime(&ms, r.a, r.b);
    c->acc_ms[r.klass] += ms;
    c->acc_n[r.klass] += 1;
    c->acc_flops[r.klass] += r.flops;
    c->acc_bytes[r.klass] += r.bytes;
    c->ev_pool.push_back(r.a);
    c->ev_pool.push_back(r.b);
  }
  c->pending.clear();
}

extern "C" pds_status pds_profile_read(pds_ctx* c, int32_t k, double* ms, int64_t* n, double* flops, double* bytes) {
  if (!c || k < 0 || k > 4) PDS_FAIL(PDS_EINVAL, "bad profile class");
  drain(c);
  if (ms) *ms = c->acc_ms[k];
  if (n) *n = c->acc_n[k];
  if (flops) *flops = c->acc_flops[k];
  if (bytes) *bytes = c->acc_bytes[k];
  return PDS_OK;
}

extern "C" pds_status pds_profile_reset(pds_ctx* c) {
  if (!c) PDS_FAIL(PDS_EINVAL, "NULL ctx");
  drain(c);
  for (int k = 0; k < 5; ++k) c->acc_ms[k] = c->acc_flops[k] = c->acc_bytes[k] = 0, c->acc_n[k] = 0;
  return PDS_OK;
}
