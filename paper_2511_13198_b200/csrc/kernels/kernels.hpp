// Launchers of the non-GEMM kernels (all return 0 or a cudaError_t value).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pds {
// clock64 timeline of one dQ-kernel CTA (trace builds, -DPDS_TRACE); -1 otherwise
int attn_debug_trace(long long* host_out, int rows);
// qkv rows packed [Q (heads) | K (kv_heads) | V (kv_heads)]; kv_heads = 0: heads (MHA),
// else GQA with query head i on key / value head i / (heads / kv_heads)
int attn_fwd(const void* qkv, int64_t ld, int s, int heads, int d, int causal, void* out, int64_t ld_out,
             void* lse, cudaStream_t st, int kv_heads = 0, const int* segs = nullptr);
// dqacc (heads * s * d fp32) and ctr (heads * s / 128 + 1 ints) select the fused
// one-kernel backward (d = 128, causal, MHA); NULL keeps the split dK/dV + dQ kernels
int attn_bwd(const void* qkv, int64_t ld, const void* out, int64_t ld_out, const void* lse, const void* dout,
             int s, int heads, int d, int causal, void* dqkv, const void* rope, float* Dd, cudaStream_t st,
             float* dqacc = nullptr, int* ctr = nullptr, int kv_heads = 0, const int* segs = nullptr,
             void* dsbuf = nullptr, int64_t ds_bytes = 0);
// dS-through-HBM backward: the dsbuf bytes attn_bwd uses for a causal d = 128
// attention over s positions with at most `budget` bytes (whole KV groups of heads, s^2 bf16
// each); 0 when the path does not apply (then the split kernels run)
int64_t attn_ds_bytes(int64_t s, int heads, int kv_heads, int d, int causal, int64_t budget);
// varlen packing (R-VARLEN): segs int32 [2 * s / 128] on the device, for every 128-row
// block the [first, last + 1) block range of the sequence it belongs to (sequences are
// 256-row aligned); attention stays inside each sequence and RoPE positions restart at
// its first row; NULL = one sequence
bool attn_bwd_fused_applies(int d, int causal);
int attn_bwd_mode();
void set_attn_bwd_mode(int mode);
// context parallelism: queries [qlo, qlo + qn) against all s keys (attention.cu)
int attn_fwd_rows(const void* qkv, int64_t ld, int s, int heads, int d, int causal, int qlo, int qn, void* out,
                  int64_t ld_out, void* lse, cudaStream_t st);
int attn_bwd_rows(const void* qkv, int64_t ld, const void* out, int64_t ld_out, const void* lse,
                  const void* dout, int s, int heads, int d, int causal, int qlo, int qn, void* dqkv,
                  const void* rope, float* Dd, cudaStream_t st);
// ring attention (MegatronCZ, attn_tc.cu / attention.cu): one (query block, key block)
// pair with separate query and key / value buffers, its backward in fp32-accumulate
// mode, the log-sum-exp merge of pair results, the RoPE^T + bf16 conversion of the
// accumulated gradients, and D = rowsum(dO o O)
int attn_fwd_pair(const void* q, int64_t ld_q, const void* kv, int64_t ld_kv, int kcol, int vcol, int sq, int sk,
                  int heads, int d, int causal, void* out, int64_t ld_out, void* lse, cudaStream_t st,
                  int kv_heads = 0);
int attn_bwd_pair(const void* q, int64_t ld_q, const void* kv, int64_t ld_kv, int kcol, int vcol, const void* dout,
                  int64_t ld_out, const void* lse, const float* Dd, int sq, int sk, int heads, int d, int causal,
                  float* dq_acc, int64_t ld_dqa, float* dkv_acc, int64_t ld_dkva, cudaStream_t st,
                  int kv_heads = 0);
int attn_merge(float* o_acc, int64_t ld_oacc, float* l_acc, int64_t lstride_acc, const void* o_p, int64_t ld_op,
               const float* l_p, int64_t lstride_p, int rows, int heads, int d, int first, void* out, int64_t ld_out,
               cudaStream_t st);
int rope_t_f32_bf16(const float* src, int64_t ld_src, int rows, int cols, int d, const void* rope, int64_t base0,
                    int64_t base1, int half, int b, void* dst, int64_t ld_dst, cudaStream_t st);
int attn_dot(const void* out, int64_t ld_out, const void* dout, int s, int heads, int d, float* Dd, cudaStream_t st);
// Ring Self-Attention (ColossalZ, attention.cu): row softmax of materialised fp32 scores
// (causal by position pos0 + row % rows_per_head), and dS = scale * P o (dP - D)
int rsa_softmax(const float* S, int64_t lds, int rows, int cols, int rows_per_head, int64_t pos0, int causal,
                float scale, void* Pr, int64_t ldp, cudaStream_t st);
int rsa_dsoftmax(const void* Pr, int64_t ldp, const float* dP, int64_t lddp, const float* D, int rows, int cols,
                 float scale, void* dS, int64_t ldds, cudaStream_t st);
int rmsnorm_fwd(const void* x, const void* res, const void* g, int64_t rows, int h, float eps, void* x1_out,
                void* u_out, void* rstd, cudaStream_t st);
int rmsnorm_bwd_grid(int64_t rows);
int rmsnorm_bwd(const void* du, const void* x, const void* rstd, const void* g, const void* dres, int64_t rows,
                int h, void* dx, float* dg_part, float* dg, cudaStream_t st);
int apply_norm(const void* x, const void* rstd, const void* g, int64_t rows, int h, void* u, cudaStream_t st);
int add_bf16(const void* a, const void* b, void* c, int64_t n, cudaStream_t st);
int add_f32(const void* a, void* acc, int64_t n, cudaStream_t st);
int sum_bf16_p(const void* const* srcs, int P, void* dst, int64_t n, cudaStream_t st);
int sum_f32_p(const void* const* srcs, int P, void* dst, int64_t n, cudaStream_t st);
// dst[c][r] = src[map(r)][c], map(r) = (r / seg) * stride + base + r % seg (seg = 0: identity)
int transpose_bf16(const void* src, int64_t ld_src, int64_t rows, int64_t cols, void* dst, int64_t ld_dst,
                   int64_t seg, int64_t stride, int64_t base, cudaStream_t st);
int rope_table(void* t, int64_t n_pos, int d, double theta, cudaStream_t st);
// dst[t][j*cw + c] = src[j][t][c]  (A2A receive buffer -> row-major columns), bf16
int unpack_blocks(const void* src, int P, int64_t rows, int64_t cw, void* dst, int64_t ld_dst, cudaStream_t st);
}  // namespace pds
