/* paradyse.h — C ABI of the B200-native ParaDySe hot path (arXiv 2511.13198).
 *
 * The calls follow the paper's statement of the problem:
 *   - pds_plan(seq_len) -> layer-wise strategy vector Pi* (Eqs. 5-6, PAPER.md:112-116,
 *     Algorithm 1, cost model Eq. 9);
 *   - pds_layer_fwd / pds_layer_bwd(strategy, shard): one Transformer layer
 *     f_{pi,MHA} then f_{pi,FFN} (Eqs. 7-8) over the unified
 *     boundary layout of Table 2's "Specification" row.
 *
 * Conventions (all calls):
 *   - Every call returns pds_status (0 = OK).  No exception crosses the ABI.  On
 *     error, pds_last_error() returns a thread-local message naming the offending
 *     argument / axis / value.
 *   - Device pointers are plain CUDA device addresses (the caller owns them, e.g.
 *     torch tensors passed by data_ptr).  Host pointers are marked "host".
 *   - Streams are cudaStream_t passed as void* (NULL = legacy default stream).  All
 *     device work of a call is enqueued on that stream; calls do not synchronise
 *     the host unless stated.
 *   - Dtypes: activations / weights bf16; weight gradients fp32, ACCUMULATED (+=).
 *   - Boundary activation layout: [s/P, b, h] row-major bf16, rank r holding
 *     global positions [r*s/P, (r+1)*s/P) (reading R-10); token row t*b + j is
 *     position t of sequence j.  b >= 1 independent equal-length sequences (no
 *     attention across them, reading Q-35); b < 1 -> PDS_EINVAL.
 *   - Weight shards (spec layout, reading R-9), rank r of P, n heads, d = h/n, F = ffn:
 *       w_qkv_t [3h/P, h]  rows: Q rows of head group r (heads [r n/P, (r+1) n/P)),
 *                          then its K rows, then its V rows  ((3h/p x h)^T of Table 2)
 *       w_proj  [h/P, h]   rows [r h/P, (r+1) h/P) of W_proj
 *       w_in_t  [F/P, h]   rows [r F/P, (r+1) F/P) of W_in^T   ((4h/p x h)^T)
     Llama variant: w_qkv_t [(n + 2 n_kv) d / P, h] = the Q rows of head group r, then
       the K rows of KV group r (n_kv/P heads), then its V rows; SwiGLU w_in_t [2F/P, h]
       = rows [r 2F/P, (r+1) 2F/P) of [W_gate | W_up]^T with its rows interleaved in
       blocks of 64 (gate rows 64j..64j+63, then up rows 64j..64j+63), so every shard
       and every row-wise gather holds whole (gate, up) pairs; 64 | F/P.
 *       w_out   [F/P, h]   rows [r F/P, (r+1) F/P) of W_out
 *       g1, g2  [h]        RMSNorm gains, replicated
 *   - Divisibility (P | s, P | n, 128 | s/P, metp_chunks | s/P) is a hard error
 *     (PDS_EDIVISIBILITY), never padded: the caller pads (reading R-15).
 */
#ifndef PARADYSE_H
#define PARADYSE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PDS_OK = 0,
  PDS_EINVAL = -1,         /* bad argument (NULL pointer, L = 0, P = 0, ...)           */
  PDS_EDIVISIBILITY = -2,  /* s, n or chunk count not divisible as required            */
  PDS_ESTRATEGY = -3,      /* unknown / disabled strategy id                           */
  PDS_ENOMEM = -4,         /* device allocation failed (cudaErrorMemoryAllocation)     */
  PDS_ECUDA = -5,          /* any other CUDA error                                     */
  PDS_ENCCL = -6,          /* NCCL error                                               */
  PDS_ESTATE = -7,         /* call order / state error (e.g. bwd strategy != fwd)      */
  PDS_ENOCOSTS = -8,       /* pds_plan without a loaded cost bundle                    */
  PDS_ENOTIMPL = -9        /* feature outside this build (e.g. head dim not 64 / 128)  */
} pds_status;

/* Strategy ids, stored as uint8_t in plans. */
typedef enum {
  PDS_MEGATRON_TS = 0,     /* Megatron-LM TP+SP                    */
  PDS_ULYSSES_Z = 1,       /* DeepSpeed Ulysses + ZeRO3 weight gathering*/
  PDS_METP = 2,            /* METP-style chunked, memory-bounded (R-11)  */
  PDS_MEGATRON_CZ = 3,     /* Megatron-LM CP + ZeRO3: zigzag-balanced ring attention
                              (reading R-CZ)                            */
  PDS_METP_FULL = 4,       /* METP with Q/K/V also recomputed in bwd (saved 3u + 2l +
                              lam instead of 6u + ..., SURVEY O-6): the planner's
                              deepest memory saver, chosen per layer   */
  PDS_COLOSSAL_Z = 5       /* Colossal-AI SP (Ring Self-Attention) + ZeRO3 (PAPER.md:220,
                              reading R-COL): the score matrix of the own rows is
                              materialised, memory quadratic in s     */
} pds_strategy;
#define PDS_N_STRATEGIES 6

/* pds_plan flags */
#define PDS_PLAN_INFEASIBLE 1u  /* no plan satisfies Eq. 6; least-memory fallback returned */
#define PDS_PLAN_CACHED 2u      /* served from the (b, s) dictionary D     */
#define PDS_PLAN_EARLY 4u       /* early termination (R-18)             */
#define PDS_PLAN_SMOOTHED 8u    /* previous plan retained by gamma-smoothing (R-19)       */

/* Model configuration C = (h, n, L) plus the north_star additions. */
typedef struct {
  int32_t h;              /* hidden size                                     */
  int32_t n_heads;        /* attention heads n (d = h / n, d in {64, 128})   */
  int32_t ffn;            /* FFN width F (4h in the paper, Eq. 4)            */
  int32_t n_layers;       /* L                                               */
  int32_t batch;          /* b >= 1 equal-length sequences (reading Q-35)    */
  float norm_eps;         /* RMSNorm epsilon (1e-5, R-2)                     */
  double rope_theta;      /* RoPE base (10000, R-3)                          */
  int32_t causal;         /* 1 = causal mask (north_star), 0 = none          */
  int32_t metp_chunks;    /* METP wave count c (0 -> P)                      */
  int32_t metp_recompute; /* what PDS_METP recomputes in bwd: 0 = the FFN
                              intermediates (R-11); 1 = also Q/K/V (then
                              PDS_METP behaves as PDS_METP_FULL); else EINVAL.
                              PDS_METP_FULL always recomputes Q/K/V.          */
  /* Llama variant (the paper's LLaMA, Table 4, PAPER.md:317;
   * readings R-GQA / R-SWIGLU), on every strategy. */
  int32_t n_kv_heads;     /* key/value heads (GQA): 0 -> n_heads (MHA); must
                              divide n_heads and be divisible by P           */
  int32_t ffn_act;        /* 0 = GELU (Eq. 4), 1 = SwiGLU: FFN(v) = (SiLU(v W_gate)
                              * (v W_up)) W_down with ffn = the width of W_down  */
} pds_model;

typedef struct pds_ctx pds_ctx;     /* opaque: rank, P, comm, streams, arenas, costs, plan cache */
typedef struct pds_group pds_group; /* opaque: in-process loopback group (P virtual ranks on    */
                                    /* one device; used by single-GPU multi-rank parity tests) */
typedef struct pds_saved pds_saved; /* opaque: one layer's saved activations (ctx-owned)        */

/* Spec-layout weight shards (bf16, device) and their fp32 gradients (device, +=). */
typedef struct { const void *w_qkv_t, *w_proj, *w_in_t, *w_out, *g1, *g2; } pds_weights;
typedef struct { void *dw_qkv_t, *dw_proj, *dw_in_t, *dw_out, *dg1, *dg2; } pds_grads;

/* ------------------------------------------------------------------ context */
/* Writes a 128-byte NCCL unique id (host) — rank 0 calls this and broadcasts it
 * (e.g. via torch.distributed) before every rank calls pds_create. */
pds_status pds_nccl_unique_id(void* out128);

/* Create the per-rank context on `device`.  P = 1 and nccl_unique_id = NULL: no
 * communicator (collectives are identities).  Otherwise nccl_unique_id (host, 128 B)
 * must be the same on all ranks and the NCCL communicator is created collectively
 * (blocks until all ranks join); P = 1 with an id gives a one-rank NCCL
 * communicator, which runs the NCCL code path on a single GPU.
 * device < 0 (any P in [1, 8], nccl_unique_id = NULL): a HOST-ONLY planner context —
 * no CUDA or NCCL call is made; pds_load_costs / pds_set_capacity / pds_set_enabled /
 * pds_plan / pds_cost_eval work as on a device context (capacity from the bundle or
 * pds_set_capacity), every layer / reserve call returns PDS_ESTATE.
 * With NCCL and P > 1 the tile-overlapped collectives (pds_set_overlap) start OFF
 * unless the environment sets PDS_OVERLAP=1 (not yet validated with real peers). */
pds_status pds_create(const pds_model* model, int32_t P, int32_t rank, int32_t device,
                      const void* nccl_unique_id, pds_ctx** out);

/* Loopback: P virtual ranks in one process on one device; rank r's calls must run
 * on their own host thread (collectives rendezvous on a host barrier). */
pds_status pds_group_create(int32_t P, pds_group** out);
pds_status pds_group_destroy(pds_group* g);
pds_status pds_create_loopback(const pds_model* model, pds_group* g, int32_t rank,
                               int32_t device, pds_ctx** out);
pds_status pds_destroy(pds_ctx* ctx);

/* Optional: pre-allocate workspace for sequences up to max_seq_len (global) for the
 * strategies in strategy_mask (bit i = strategy i); otherwise grown on demand. */
pds_status pds_reserve(pds_ctx* ctx, int64_t max_seq_len, uint32_t strategy_mask);

/* Free the context's cached device memory (idle saved-arena blocks, workspace) so a
 * following call starts from an empty pool.  Live pds_saved sets are untouched. */
pds_status pds_release_cache(pds_ctx* ctx);

/* ------------------------------------------------------------------ planner (host only) */
/* Load a calibrated cost bundle (text, "pds_bundle 1" format, see DESIGN.md §Cost
 * bundle): per strategy an exported random forest (RF, interpolation) and an AIC-
 * selected polynomial (PR, extrapolation) for T_pi(s), plus s_profile_max (Eq. 9). */
pds_status pds_load_costs(pds_ctx* ctx, const char* bundle_path);
/* Device capacity (bytes) the plan must stay strictly below (Eq. 6) and the
 * smoothing ratio gamma.  Defaults: after pds_load_costs, the
 * bundle's recorded `capacity` minus its `reserve` (the device the bundle was
 * calibrated on); before any bundle, cudaMemGetInfo's total (0 on a host-only
 * context); gamma = 0.  Either call clears the (b, s) dictionary. */
pds_status pds_set_capacity(pds_ctx* ctx, double capacity_bytes, double gamma);
/* Enable / disable strategies (bit mask; default: all). */
pds_status pds_set_enabled(pds_ctx* ctx, uint32_t strategy_mask);

/* Pi*(b, s): writes L strategy ids to strategy_out (host, L bytes) — always a full
 * plan (totality); *flags_out (nullable) gets PDS_PLAN_* bits.
 * T_pi(s) from the bundle (Eq. 9), M_pi(s) from pds_mem_bytes (exact model: saved
 * + persistent per layer, plus the plan's largest workspace, R-22), Algorithm 1
 * with the readings R-17..R-24, dictionary D keyed by (b, s). */
pds_status pds_plan(pds_ctx* ctx, int64_t seq_len, uint8_t* strategy_out, int32_t L,
                    uint32_t* flags_out);

/* Stateless Algorithm 1 on explicit per-layer costs (host arrays of n_strat):
 * t_layer[i], m_layer[i] for strategy i, w_layer[i] (nullable) the strategy's
 * workspace, enabled[i] in {0,1}; a plan is feasible iff
 * sum_l m[pi_l] + max_l w[pi_l] < capacity (strict; Eq. 6 with reading R-22: one
 * workspace per plan, reused by every layer; w_layer = NULL gives the paper's
 * sum m < capacity).  prev_plan (nullable, L bytes) enables smoothing with gamma.
 * counters_out (nullable, 3 x int64): layer memory checks, candidate plans
 * generated, cache hits (always 0 here).  Bit-exact contract with the oracle. */
pds_status pds_plan_ex(int32_t L, int32_t n_strat, const double* t_layer, const double* m_layer,
                       const double* w_layer, const uint8_t* enabled, double capacity, double gamma,
                       const uint8_t* prev_plan, uint8_t* strategy_out, uint32_t* flags_out,
                       int64_t* counters_out);

/* T_pi(s) and M_pi(s) for every strategy (host arrays of PDS_N_STRATEGIES entries):
 * t_layer[i] = Eq. 9 (RF iff s <= s_profile_max of strategy i, else PR; 1e300 for a
 * strategy absent from the bundle), m_layer[i] = persistent + saved bytes of one layer
 * (1e300 where the strategy is invalid at this s, e.g. divisibility);
 * branch_out (nullable, host int32[PDS_N_STRATEGIES]): 0 = RF, 1 = PR. */
pds_status pds_cost_eval(pds_ctx* ctx, int64_t seq_len, double* t_layer, double* m_layer,
                         int32_t* branch_out);

/* Exact per-rank memory model of this implementation:
 * saved activations per layer, the strategy's workspace peak, and the persistent
 * bytes per layer (bf16 weight shards + fp32 gradient shards).  Host only. */
pds_status pds_mem_bytes(const pds_model* model, int32_t P, uint8_t strategy, int64_t seq_len,
                         int64_t* saved_per_layer, int64_t* transient_peak,
                         int64_t* persistent_per_layer);

/* ------------------------------------------------------------------ the layer */
/* y = f_{pi,FFN}(f_{pi,MHA}(x)) with residuals and pre-norms,
 * x, y: local [s/P, b, h] bf16 shards of a length-seq_len global sequence.
 * *saved receives the layer's saved activations (ctx arena, LIFO across layers);
 * pass saved = NULL for a forward-only call.  x must stay valid until the
 * matching bwd (it is referenced, not copied). */
pds_status pds_layer_fwd(pds_ctx* ctx, uint8_t strategy, int64_t seq_len, const void* x,
                         const pds_weights* w, void* y, pds_saved** saved, void* stream);
/* dx = VJP of the layer at dy; weight gradients accumulated (+=) into g (fp32).
 * `strategy` must equal the forward's (else PDS_ESTATE).  Consumes `saved`. */
pds_status pds_layer_bwd(pds_ctx* ctx, uint8_t strategy, const void* dy, pds_saved* saved,
                         const pds_weights* w, const pds_grads* g, void* dx, void* stream);
/* End-to-end step with HOST activations (the call a user without device buffers
 * makes): x_host, dy_host (host, [s/P, b, h] bf16) are uploaded into library-owned
 * staging, one layer fwd + bwd runs as pds_layer_fwd / pds_layer_bwd on `stream`,
 * and y_host, dx_host (host, same layout) receive the results; weight gradients are
 * accumulated into g as in pds_layer_bwd.  Asynchronous: uploads and downloads run
 * on context-owned copy streams and consecutive calls alternate between two staging
 * sets, so a call's transfers overlap the neighbouring calls' compute.  Host buffers
 * must be page-locked for the overlap and must stay untouched until
 * pds_host_drain(ctx, stream) has been enqueued and `stream` has reached it; the
 * compute of every call is ordered on `stream`.  Errors: as pds_layer_fwd /
 * pds_layer_bwd; staging allocation failure -> PDS_ENOMEM. */
pds_status pds_layer_step_host(pds_ctx* ctx, uint8_t strategy, int64_t seq_len, const void* x_host,
                               const void* dy_host, const pds_weights* w, const pds_grads* g,
                               void* y_host, void* dx_host, void* stream);
/* Orders `stream` after every transfer of the pds_layer_step_host calls issued so
 * far (after it, synchronising `stream` makes all y_host / dx_host valid). */
pds_status pds_host_drain(pds_ctx* ctx, void* stream);
/* Release a saved set without running backward. */
pds_status pds_saved_release(pds_ctx* ctx, pds_saved* saved);
/* Comm log: on = 1 clears and starts recording every collective of this
 * rank's layer calls as a JSON line {"primitive": "AllGather" | "ReduceScatter" |
 * "AllToAll" | "AllReduce" | "SendRecv" | "RingPass", "bytes": B, "participants": P}
 * with B the bytes this rank sends (the oracle grid's payload convention, SPEC.md:109;
 * nothing at P = 1); on = 0 stops.  pds_comm_log_read copies the log (NUL-terminated,
 * truncated to cap - 1 bytes; buf may be NULL) and returns its full length in *len_out.
 * Host-side bookkeeping only; every layer call also opens NVTX ranges
 * ("pds_layer_fwd <strategy>", and "pds:gemm" / "pds:attn_fwd" / ... per launch). */
pds_status pds_comm_log(pds_ctx* ctx, int32_t on);
pds_status pds_comm_log_read(pds_ctx* ctx, char* buf, int64_t cap, int64_t* len_out);
/* Varlen packing (reading R-VARLEN): the following layer calls of
 * this context treat their seq_len tokens as n_seqs independent sequences packed back to
 * back in the boundary layout (rank r holds tokens [r T/P, (r+1) T/P) of the packed
 * stream, T = sum lens); attention never crosses a sequence boundary (causal or not) and
 * RoPE positions restart at each sequence's first token.  lens: host int64[n_seqs], each
 * a positive multiple of 256 (PDS_EDIVISIBILITY otherwise: the caller pads each
 * sequence); the layer calls must pass seq_len = T (PDS_EINVAL otherwise).  n_seqs = 0
 * restores one sequence.  Requires batch = 1 (PDS_EINVAL); MegatronTS, UlyssesZ, METP,
 * METP-full (MegatronCZ / ColossalZ: PDS_ENOTIMPL).  A forward's setting is kept with
 * its saved set, so the matching backward uses it whatever was set since.  Blocking
 * (uploads a small table). */
pds_status pds_set_varlen(pds_ctx* ctx, int32_t n_seqs, const int64_t* lens);

/* Tile-level overlap of the MegatronTS collectives (P > 1): every
 * all-gather feeding a column-parallel GEMM (QKV, FC1; bwd dGELU, dA) runs chunk by
 * chunk on a side stream while the GEMM polls per tile for the chunks it needs, and
 * every reduce-scatter after a row-parallel GEMM (proj, FC2; bwd dV, dU) sends each
 * chunk as soon as the GEMM has stored it ("communication overlapped with GEMM tiles",
 * north_star; the AG / RS of PAPER.md:203); METP does the same per wave, and
 * UlyssesZ sends each head-group block of its sequence -> head All-to-Alls as soon
 * as the packing GEMM has stored it.  on = 1 or 0 (plain in-order collectives);
 * default 1 for the loopback group, 0 for an NCCL communicator with P > 1 unless
 * PDS_OVERLAP=1 (see pds_create).  Results are bit-identical either way.  Ignored at
 * P = 1. */
pds_status pds_set_overlap(pds_ctx* ctx, int32_t on);
/* Debug taps: the next pds_layer_fwd also writes the sublayer deltas O (attention
 * block output) and Z (FFN output), local [s/P, b, h] bf16 (reading R-34).  NULL
 * pointers disable. */
pds_status pds_debug_taps(pds_ctx* ctx, void* o_out, void* z_out);

/* ------------------------------------------------------------------ measurement */
/* Per-kernel-class device timing with CUDA events on the launching stream.
 * Classes: 0 GEMM, 1 attention fwd, 2 attention bwd, 3 norm/elementwise,
 * 4 collectives.  read: total ms, launches, algorithmic flops and bytes. */
pds_status pds_profile_enable(pds_ctx* ctx, int32_t on);
pds_status pds_profile_read(pds_ctx* ctx, int32_t klass, double* ms, int64_t* launches,
                            double* flops, double* bytes);
pds_status pds_profile_reset(pds_ctx* ctx);

/* Development aid: copies `rows` x 8 clock64 stamps of one dQ-kernel CTA's timeline
 * (host int64) from a library built with -DPDS_TRACE; PDS_ENOTIMPL otherwise. */
pds_status pds_debug_trace(int64_t* host_out, int32_t rows);

/* ------------------------------------------------------------------ kernel-level entry points
 * Per-stage parity (fp32-accumulate path, reading R-14).  Device pointers, stream-
 * ordered, no context needed. */
/* C[M,N] (op)= A * B^T with A [M][K] (a_mn = 0) or [K][M] (a_mn = 1), B [N][K]
 * (b_mn = 0) or [K][N] (b_mn = 1); epi: 0 bf16 store, 1 fp32 +=, 2 fp32 store,
 * 3 GELU (C = H bf16, aux_out = GELU(H)), 4 dGELU (aux_in = H; C = acc * GELU'(H),
 * aux_out = GELU(H)). */
pds_status pds_k_gemm(const void* A, int64_t lda, int32_t a_mn, const void* B, int64_t ldb,
                      int32_t b_mn, int32_t M, int32_t N, int32_t K, void* C, int64_t ldc,
                      int32_t epi, const void* aux_in, void* aux_out, int64_t ld_aux,
                      void* stream);
/* The collective-overlap protocol of the MegatronTS GEMMs (pds_set_overlap), bf16
 * C = A B^T with both operands K-major.  M splits into chunks of chunk_rows (a
 * multiple of 32 dividing M).  wait_flags (nullable, device uint32 [M/chunk_rows]):
 * a CTA loads A rows of chunk c only once (int32)(wait_flags[c] - flag_epoch) >= 0
 * (traps after > 30 s).  done_ctr (nullable, device uint32 [M/chunk_rows]): grows by
 * the number of elements stored in chunk c divided by 8, so it has grown by
 * chunk_rows*N/8 when the chunk is complete.  m_rot_rows: first row of the tile order (wraps).  sm_reserve:
 * SMs left idle.  Bad chunking -> PDS_EINVAL. */
pds_status pds_k_gemm_sync(const void* A, int64_t lda, const void* B, int64_t ldb, int32_t M,
                           int32_t N, int32_t K, void* C, int64_t ldc, const uint32_t* wait_flags,
                           uint32_t flag_epoch, uint32_t* done_ctr, int64_t chunk_rows,
                           int64_t m_rot_rows, int32_t sm_reserve, void* stream);
/* Stream memory operations (no SM): *addr := value after the stream's prior work;
 * block the stream until (int32)(*addr - value) >= 0.  addr: device memory. */
pds_status pds_k_stream_write32(void* stream, uint32_t* addr, uint32_t value);
pds_status pds_k_stream_wait32(void* stream, const uint32_t* addr, uint32_t value);
/* QKV GEMM with fused RoPE on the Q and K columns: C [M, N] where columns form
 * groups of 3*hq ([Q | K | V], hq = heads*d); row r has global position
 * (r / seg) * seg_stride + seg_base + r % seg.  rope: [positions][d/2] float2. */
pds_status pds_k_gemm_rope(const void* A, int64_t lda, const void* B, int64_t ldb, int32_t M,
                           int32_t N, int32_t K, void* C, int64_t ldc, const void* rope,
                           int32_t d, int32_t hq, int64_t seg, int64_t seg_stride,
                           int64_t seg_base, void* stream);
/* cos/sin table [n_pos][d/2] (float2), angles t * theta^(-2k/d) formed and
 * range-reduced in fp64 (reading R-3). */
pds_status pds_k_rope_table(void* table, int64_t n_pos, int32_t d, double theta, void* stream);
/* RMSNorm forward over rows of h: if residual != NULL, x1 = x + residual is
 * written to x1_out and normalised; u = g * x1 * rstd; rstd fp32 [rows]. */
pds_status pds_k_rmsnorm_fwd(const void* x, const void* residual, const void* g, int64_t rows,
                             int32_t h, float eps, void* x1_out, void* u_out, void* rstd_out,
                             void* stream);
/* RMSNorm backward: dx = r (a - xhat mean(a xhat)) (+ dres if != NULL), a = du g;
 * dg_partial fp32 [gridrows][h] reduced into dg (fp32 [h], +=). */
pds_status pds_k_rmsnorm_bwd(const void* du, const void* x, const void* rstd, const void* g,
                             const void* dres, int64_t rows, int32_t h, void* dx, void* dg,
                             void* stream);
/* Causal (or full) attention forward over qkv [s][ld] laid out [Q | K | V] blocks
 * of heads*d: out [s][ld_out] (head i at column i*d), lse fp32 [heads][s]. */
pds_status pds_k_attn_fwd(const void* qkv, int64_t ld, int32_t s, int32_t heads, int32_t d,
                          int32_t causal, void* out, int64_t ld_out, void* lse, void* stream);
/* Attention backward: dqkv [s][ld] (pre-RoPE positions handled by caller), from
 * qkv (post-RoPE Q, K), out, lse, dout.  Two implementations (pds_set_attn_bwd):
 * the split dK/dV + dQ kernels (default; d in {64, 128}, causal or not) and the fused
 * kernel (d = 128, causal: one kernel for dQ, dK, dV, 5 matmuls per block pair, dQ
 * summed over key blocks through an fp32 accumulator in a fixed order, so the result is
 * deterministic; scratch heads * s * 128 fp32 cached by this entry point). */
pds_status pds_k_attn_bwd(const void* qkv, int64_t ld, const void* out, int64_t ld_out,
                          const void* lse, const void* dout, int32_t s, int32_t heads, int32_t d,
                          int32_t causal, void* dqkv, void* stream);
/* Llama variant (readings R-GQA / R-SWIGLU).
 * GQA attention: qkv [s][ld] laid out [Q (heads*d) | K (kv_heads*d) | V (kv_heads*d)];
 * query head i attends with key / value head i / (heads / kv_heads).  out [s][ld_out],
 * lse fp32 [heads][s] as pds_k_attn_fwd; the backward writes dqkv in qkv's layout, a
 * key / value head's gradient summed over its query group (split kernels; the dK/dV
 * kernel walks the group's query heads in one TMEM accumulation).  kv_heads must
 * divide heads (PDS_EINVAL otherwise); kv_heads = heads is pds_k_attn_fwd/bwd. */
pds_status pds_k_attn_fwd_gqa(const void* qkv, int64_t ld, int32_t s, int32_t heads, int32_t kv_heads,
                              int32_t d, int32_t causal, void* out, int64_t ld_out, void* lse, void* stream);
pds_status pds_k_attn_bwd_gqa(const void* qkv, int64_t ld, const void* out, int64_t ld_out,
                              const void* lse, const void* dout, int32_t s, int32_t heads, int32_t kv_heads,
                              int32_t d, int32_t causal, void* dqkv, void* stream);
/* SwiGLU GEMM epilogues.  bwd = 0 (FC1): C [M, N] bf16 = H = A B^T, whose columns are
 * interleaved in 64-blocks [gate_j | up_j] (N % 128 == 0), and g_out [M, N/2] (row
 * stride ld_g) = SiLU(bf16 gate) * bf16 up.  bwd = 1 (dG GEMM): the accumulator is dG
 * [M, N] (N % 64 == 0); h_in = H [M, 2N] (row stride ld_h); C [M, 2N] = dH in H's
 * layout (dgate = dG up SiLU'(gate), dup = dG SiLU(gate)); optional g_out [M, N] = G,
 * c_t [2N][ld_t] = dH^T, g_t [N][ld_t] = G^T (the dW GEMMs' K-major operands).
 * Device pointers; PDS_EINVAL on a missing buffer or a misaligned N. */
pds_status pds_k_gemm_swiglu(const void* A, int64_t lda, const void* B, int64_t ldb, int32_t M, int32_t N,
                             int32_t K, int32_t bwd, void* C, int64_t ldc, const void* h_in, int64_t ld_h,
                             void* g_out, int64_t ld_g, void* c_t, void* g_t, int64_t ld_t, void* stream);
/* QKV GEMM + RoPE with GQA column groups [Q (hq) | K (hk) | V (hk)] repeated every
 * hq + 2 hk columns; row r at position r. */
pds_status pds_k_gemm_rope_gqa(const void* A, int64_t lda, const void* B, int64_t ldb, int32_t M,
                               int32_t N, int32_t K, void* C, int64_t ldc, const void* rope, int32_t d,
                               int32_t hq, int32_t hk, void* stream);
/* Query-row-range attention (a rank's rows of an all-gathered context; the layer's
 * MegatronCZ uses the ring pairs below instead): the query rows [qlo, qlo + qn) of the s
 * positions of qkv [s][ld] against every key (causal: keys <= the query position).
 * out [qn][ld_out] and lse fp32 [heads][qn] hold the local rows.  Backward: from the
 * local out / lse / dout, dQ of rows [qlo, qlo + qn) and the dK / dV contributions of
 * those queries to every key row, into dqkv [s][ld]; under the causal mask key rows
 * >= qlo + qn are not written (the caller zeroes dqkv first).  qlo, qn multiples of
 * 128, qlo + qn <= s, else PDS_EINVAL. */
pds_status pds_k_attn_fwd_rows(const void* qkv, int64_t ld, int32_t s, int32_t heads, int32_t d,
                               int32_t causal, int32_t qlo, int32_t qn, void* out, int64_t ld_out,
                               void* lse, void* stream);
pds_status pds_k_attn_bwd_rows(const void* qkv, int64_t ld, const void* out, int64_t ld_out,
                               const void* lse, const void* dout, int32_t s, int32_t heads, int32_t d,
                               int32_t causal, int32_t qlo, int32_t qn, void* dqkv, void* stream);

/* Ring attention (MegatronCZ, reading R-CZ): one (query block, key block) pair with
 * queries q [sq][ld_q] (head i at column i*d) and keys / values at columns kcol / vcol
 * (+ i*d) of kv [sk][ld_kv].  causal = the diagonal pair (sq == sk, aligned positions);
 * otherwise every key is visible.  out [sq][ld_out] bf16 and lse fp32 [heads][sq] are the
 * pair's own softmax result.  sq, sk multiples of 128, else PDS_EINVAL. */
pds_status pds_k_attn_fwd_pair(const void* q, int64_t ld_q, const void* kv, int64_t ld_kv, int32_t kcol,
                               int32_t vcol, int32_t sq, int32_t sk, int32_t heads, int32_t d, int32_t causal,
                               void* out, int64_t ld_out, void* lse, void* stream);
/* Its backward given the MERGED row statistics lse, Dd (fp32 [heads][sq]; Dd =
 * rowsum(dO o O), pds_k_attn_dot): dQ * (1/sqrt d) is ADDED to dq_acc [sq][ld_dqa] fp32
 * and dK * (1/sqrt d) / dV to dkv_acc [sk][ld_dkva] fp32 (dK at column i*d, dV at
 * heads*d + i*d); no RoPE^T (the caller's, at the rows' positions). */
pds_status pds_k_attn_bwd_pair(const void* q, int64_t ld_q, const void* kv, int64_t ld_kv, int32_t kcol,
                               int32_t vcol, const void* dout, int64_t ld_out, const void* lse, const void* Dd,
                               int32_t sq, int32_t sk, int32_t heads, int32_t d, int32_t causal, void* dq_acc,
                               int64_t ld_dqa, void* dkv_acc, int64_t ld_dkva, void* stream);
/* Log-sum-exp merge of a pair result (o_p bf16 [rows][ld_op], l_p fp32 [heads][lstride_p])
 * into the running one (o_acc fp32 [rows][ld_oacc], l_acc fp32 [heads][lstride_acc]);
 * first = 1: the running result is empty.  out (nullable): also the bf16 O. */
pds_status pds_k_attn_merge(void* o_acc, int64_t ld_oacc, void* l_acc, int64_t lstride_acc, const void* o_p,
                            int64_t ld_op, const void* l_p, int64_t lstride_p, int32_t rows, int32_t heads,
                            int32_t d, int32_t first, void* out, int64_t ld_out, void* stream);
/* D = rowsum(dO o O) per (head, row): Dd fp32 [heads][s]. */
pds_status pds_k_attn_dot(const void* out, int64_t ld_out, const void* dout, int32_t s, int32_t heads, int32_t d,
                          void* Dd, void* stream);

/* Attention backward implementation, process wide: 0 = the split dK/dV + dQ kernels
 * (default), 1 = the fused kernel where it applies (d = 128, causal, all query rows;
 * slower on B200: its dQ reduction through L2 is the bottleneck).
 * Affects pds_layer_bwd and pds_k_attn_bwd; any other mode is PDS_EINVAL. */
pds_status pds_set_attn_bwd(int32_t mode);

const char* pds_last_error(void);
const char* pds_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PARADYSE_H */
