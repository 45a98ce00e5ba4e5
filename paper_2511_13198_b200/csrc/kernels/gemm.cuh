// Host-visible description of the tcgen05 GEMM and its fused epilogues.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pds {

// C[M,N] (op)= A[M,K] * B[N,K]^T   with fp32 accumulation in TMEM.
//   A K-major : A stored [M][K] (row stride lda elements)
//   A MN-major: A stored [K][M] (row stride lda)      -- i.e. C = A_stored^T * ...
//   B K-major : B stored [N][K] (row stride ldb)
//   B MN-major: B stored [K][N] (row stride ldb)
enum GemmEpi : int {
  EPI_BF16 = 0,      // C bf16 = acc
  EPI_F32_ACC = 1,   // C fp32 += acc            (weight gradients)
  EPI_F32 = 2,       // C fp32 = acc
  EPI_GELU = 3,      // C bf16 = H = acc ; aux_out bf16 = GELU(bf16(H))
  EPI_DGELU = 4,     // aux_in = H (bf16): C bf16 = acc * GELU'(H) ; aux_out bf16 = GELU(H)
  EPI_ROPE = 5,      // C bf16 = acc with RoPE applied to the Q/K columns
  // SwiGLU (Llama variant, R-SWIGLU): the FC1 output's columns are interleaved in
  // blocks of 64, [gate_j | up_j] per 128 (N % 128 == 0, every tile holds whole pairs)
  EPI_SWIGLU = 6,    // C bf16 = H = acc [M, N] ; aux_out bf16 [M, N/2] = SiLU(bf16 gate) * bf16 up
  EPI_ROPE_T = 8,    // C bf16 [M, d] = RoPE^T(epi_scale * acc) at position = row (the attention dQ
                     // from dS K); N == d == 128
  EPI_DSWIGLU = 7,   // acc = dG [M, N]; aux_in = H [M, 2N] (row stride ld_aux_in): C bf16 [M, 2N]
                     // = dH (dgate = dG up SiLU'(gate), dup = dG SiLU(gate)) in H's layout;
                     // aux_out [M, N] = G; c_t = dH^T [2N][ld_t]; aux_t = G^T [N][ld_t]
};

struct GemmArgs {
  const void* A = nullptr;
  int64_t lda = 0;
  int a_mn = 0;
  const void* B = nullptr;
  int64_t ldb = 0;
  int b_mn = 0;
  int M = 0, N = 0, K = 0;
  void* C = nullptr;
  int64_t ldc = 0;
  int epi = EPI_BF16;
  // output column blocking (Ulysses pack): column c goes to
  //   C + (c / blk_w) * blk_stride + row * ldc + (c % blk_w)     (blk_w = 0: off)
  int blk_w = 0;
  int64_t blk_stride = 0;
  // GELU / dGELU aux tensors, same [M, N] indexing (row stride ld_aux)
  const void* aux_in = nullptr;
  void* aux_out = nullptr;
  int64_t ld_aux = 0;
  int64_t ld_aux_in = 0;          // EPI_DSWIGLU: row stride of aux_in (0: ld_aux)
  // RoPE: columns laid out in groups of hq + 2 hk = [Q | K | V] (hq = q heads * d,
  // hk = kv heads * d; rope_hk = 0: hk = hq, MHA); the Q and K columns are rotated;
  // position of row r: ((r / seg) * seg_stride + seg_base + (r % seg)) / rope_b
  const float2* rope = nullptr;   // [positions][d/2] (cos, sin)
  int rope_d = 0;
  int rope_hq = 0;
  int rope_hk = 0;
  int rope_b = 1;                 // rows per position (batch b, layout [s, b, h]): pos = mapped row / b
  const int* rope_segs = nullptr; // varlen packing (R-VARLEN): pos -= rope_segs[2 (pos / 128)] * 128
  int64_t seg = 0, seg_stride = 0, seg_base = 0;
  // Row remaps of the STORED matrices (seg = 0: identity): logical row r lives at
  // storage row (r / seg) * stride + base + r % seg.  For A/B this is the TMA outer
  // coordinate (a tile never crosses a segment: seg % tile rows == 0); for C the
  // output row.  Used by METP waves to read / write position-ordered buffers.
  int64_t a_seg = 0, a_stride = 0, a_base = 0;
  int64_t b_seg = 0, b_stride = 0, b_base = 0;
  int64_t c_seg = 0, c_stride = 0, c_base = 0;
  // storage row counts of A / B when remapped (0: the logical extent)
  int64_t a_rows = 0, b_rows = 0;
  // EPI_DGELU only: transposed bf16 copies of C (dH^T) and of the aux output (G^T),
  // [N][ld_t] (element (r, c) at c * ld_t + r); aux_out may then be NULL.  They feed
  // the dW GEMMs, which take both operands K-major (K = tokens).
  void* c_t = nullptr;
  void* aux_t = nullptr;
  int64_t ld_t = 0;
  // Tile-level overlap with a collective (MegatronTS over P ranks).  The
  // M rows split into chunks of chunk_rows, one per rank.
  //   wait_flags  AG -> GEMM: before a CTA loads A rows of chunk c it waits until
  //               (int32)(wait_flags[c] - flag_epoch) >= 0, i.e. the all-gather has
  //               landed chunk c (K-major A, no A remap).  Bounded spin, then trap.
  //   done_ctr    GEMM -> RS: after an epilogue warp has stored its rows of chunk c it
  //               adds the number of elements stored / 8 to done_ctr[c] (release), so
  //               the chunk is complete once the counter has grown by chunk_rows * N / 8.
  //   m_rot_rows  tiles are issued starting at this row, wrapping over M, so the chunk
  //               that is local (AG) or sent first (RS) is computed first.
  //   sm_reserve  SMs left free for the collective's kernels during this GEMM.
  const uint32_t* wait_flags = nullptr;
  uint32_t flag_epoch = 0;
  uint32_t* done_ctr = nullptr;
  int64_t chunk_rows = 0;
  int64_t m_rot_rows = 0;
  int sm_reserve = 0;
  // GEMM -> All-to-All (UlyssesZ, column-blocked output): chunk_cols > 0 makes done_ctr
  // count per block of chunk_cols LOGICAL output columns (block j goes to rank j), so
  // block j is complete once done_ctr[j] has grown by M * chunk_cols / 8; n_rot_cols: first
  // column of the tile order (wraps).
  int64_t chunk_cols = 0;
  int64_t n_rot_cols = 0;
  // Batched GEMM (1-CTA kernel only): `batch` independent problems of the same shape; problem
  // z reads A rows shifted by z * a_boff (MN-major A: the stored K rows), B columns shifted by
  // z * b_boff (MN-major B) and writes C columns shifted by z * c_boff.  k_causal: the tile of
  // rows [m0, m0 + 128) only runs the K blocks below m0 + 128 (a causal contraction: K index
  // <= M index).  epi_scale: EPI_ROPE_T's scale.
  int batch = 1;
  int64_t a_boff = 0, b_boff = 0, c_boff = 0;
  int b_grp = 1;                  // B's shift is (z / b_grp) * b_boff (GQA: query heads per K head)
  int64_t b_cols = 0;             // MN-major B: stored column extent (0: N)
  int k_causal = 0;
  float epi_scale = 1.0f;
};

// returns 0 on success, a cudaError_t value otherwise
int gemm_launch(const GemmArgs& g, cudaStream_t st);
int gemm_num_sms();

}  // namespace pds
