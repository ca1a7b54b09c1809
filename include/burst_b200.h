/*
 * burst-b200 C ABI: the drop-in boundary between the burstsim-compatible Python
 * host code (paper_2509_19836_b200/) and the sm_100a kernels.
 *
 * Every entry point replaces one NumPy einsum loop of the reference
 * (`burstsim`, /root/reference/pkg/src/burstsim):
 *
 *   bb_attn_fwd_step        distributed.py:180-188  one ring step of distributed_forward
 *                           (masked S, step LSE, normalised O_step, lse_merge, rescale-add)
 *   bb_attn_bwd_step        distributed.py:288-295  one ring step of burst_backward
 *                           (and :239-247 ring_backward: same math, different owners)
 *   bb_attn_bwd_preprocess  distributed.py:274-275  D = rowsum_hadamard(dO, O), numerics.py:86-92
 *   bb_permute_rows         distributed.py:104-130  shard_rows / gather_rows / make_device_states
 *   bb_lmhead_fused         lmhead.py:41-93         fused_lmhead_loss (loss, dH, dW)
 *   bb_gemm_bf16_rows       oracle.py:60-65 +       project_qkv with shard_rows' permutation
 *                           distributed.py:104-117  fused into the GEMM store; also the output
 *                           oracle.py:29-44         projection O W_attn back to token order
 *   bb_fill_u32             distributed.py:172-173  the zero / -inf initialisation of O, lse and
 *                           (and :270-272)          the gradient accumulators
 *   bb_add_rows_f32         distributed.py:293-295  adding a peer's dQ (dK/dV) partial to the
 *                                                   owner's accumulator
 *   bb_matmul_f64 ...       numerics.py:35-116      the reference's float64 tile math
 *   bb_xent_f64             oracle.py:129-154       (matmul, row_logsumexp, lse_merge,
 *                                                   exp_shifted, exp_gap, rowsum_hadamard)
 *                                                   and naive_lmhead_loss's softmax - onehot
 *   bb_ipc_* / bb_arena_* / fabric.py:180-226       a ring step's payload transfer (copy
 *   bb_copy_async / bb_flag_*                       engines over NVLink + stream-ordered flags)
 *
 * Conventions: plain device pointers and sizes, no torch types.  Token ids and
 * devices are 1-based (burstsim README "Conventions").  All functions take a
 * cudaStream_t as `void*` (NULL = legacy default stream), never allocate (except
 * bb_arena_alloc), never synchronise, and return 0 on success or a BB_ERR_* code; the message is
 * available from bb_last_error() (thread-local).  No C++ exception crosses
 * this boundary.
 */
#ifndef BURST_B200_H
#define BURST_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BB_OK 0
#define BB_ERR_INVALID 1     /* argument / shape / divisibility error (Python: ValueError) */
#define BB_ERR_CUDA 2        /* CUDA runtime or driver failure */
#define BB_ERR_UNSUPPORTED 3 /* valid request outside what the kernels implement */

/* Layout kinds: partitioning.py:38-43 */
#define BB_LAYOUT_CONTIGUOUS 0
#define BB_LAYOUT_ZIGZAG 1
#define BB_LAYOUT_STRIPED 2
#define BB_LAYOUT_BLOCK_STRIPED 3

/* Mask kinds: masks.py:19-24 */
#define BB_MASK_FULL 0
#define BB_MASK_CAUSAL 1
#define BB_MASK_SLIDING_WINDOW 2
#define BB_MASK_BLOCK_SPARSE 3

/* ShardLayout (partitioning.py:46-76): token -> device assignment. */
typedef struct bb_layout {
  int32_t kind;
  int32_t devices;   /* G */
  int64_t seq_len;   /* N */
  int64_t block_len; /* block_striped only */
} bb_layout;

/* MaskSpec (masks.py:28-40).  block_mask is a device pointer to a
 * num_blocks x num_blocks uint8 0/1 matrix (block_sparse only).  row_span /
 * col_span (optional, may be NULL) are device int32 [num_blocks][2] arrays with
 * the first and last nonzero column of each block row / row of each block
 * column ([-1, -1] if empty): the kernels use them to bound, per CTA, the tiles
 * they consider instead of scanning the whole shard. */
typedef struct bb_mask {
  int32_t kind;
  int32_t reserved;
  int64_t window;     /* sliding_window width w: allowed iff 0 <= q-k < w */
  int64_t block_len;  /* block_sparse block length */
  int64_t num_blocks; /* block_sparse side = N / block_len */
  const uint8_t* block_mask;
  const int32_t* row_span;
  const int32_t* col_span;
} bb_mask;

/* One forward ring step: device `q_device` folds key shard `k_device` into its
 * running (O, lse).  Q/K/V are bf16 token-major [rows, heads, head_dim]; the
 * running state is f32 O [n_q, hq, head_dim] and lse [hq, n_q], initialised by
 * the caller to 0 / -inf (distributed.py:172-173).  Rows with no allowed key in
 * this step are left untouched (exp(-inf) identity, numerics.py:62-69).
 * A key shard above 524288 rows (zigzag / contiguous layouts) is run as launches over
 * its consecutive-id sub-shards; bb_attn_bwd_step does the same for query shards. */
typedef struct bb_attn_fwd_args {
  const void* q;
  const void* k;
  const void* v;
  float* o;
  float* lse;
  int64_t n_q;
  int64_t n_k;
  int32_t hq;
  int32_t hkv;       /* hq % hkv == 0 (GQA groups) */
  int32_t head_dim;  /* padded head dim the tensors are laid out with: 64 or 128 */
  float softmax_scale; /* 1/sqrt(d) of the *unpadded* head dim (oracle.py:75) */
  int32_t q_device;
  int32_t k_device;
  bb_layout layout;
  bb_mask mask;
  /* Optional (NULL = off): also store bf16(O) [n_q, hq, head_dim] after this step's merge,
   * for every row < n_q (rows this step does not touch are copied from O).  Passed on the
   * last ring step, it fuses the cast the output projection's bf16 GEMM needs
   * (bb_gemm_bf16_rows, AttentionParams.w_attn, oracle.py:29-44). */
  void* o_bf16;
} bb_attn_fwd_args;

/* One backward ring step (K/V-stationary kernel).  Accumulates, in f32:
 *   dq[n_q,hq,d]  += dS K * scale       (circulating dQ_j in burst_backward)
 *   dk[n_k,hkv,d] += dS^T Q * scale     (resident dK_i)
 *   dv[n_k,hkv,d] += P^T dO              (resident dV_i)
 * with P = exp(S - lse_j) and dS = P o (dO V^T - D_j) (distributed.py:288-295).
 * lse and delta are f32 [hq, n_q]. */
typedef struct bb_attn_bwd_args {
  const void* q;
  const void* k;
  const void* v;
  const void* dout;
  const float* lse;
  const float* delta;
  float* dq;
  float* dk;
  float* dv;
  int64_t n_q;
  int64_t n_k;
  int32_t hq;
  int32_t hkv;
  int32_t head_dim;
  float softmax_scale;
  int32_t q_device;
  int32_t k_device;
  bb_layout layout;
  bb_mask mask;
  /* kv heads [kv_head_begin, kv_head_end) only (their q heads, dK/dV rows and dQ
   * columns); kv_head_end == 0 means all hkv heads.  Lets the ring split a step's
   * work so a gradient transfer can overlap the other half. */
  int32_t kv_head_begin;
  int32_t kv_head_end;
} bb_attn_bwd_args;

int bb_attn_fwd_step(const bb_attn_fwd_args* args, void* stream);
int bb_attn_bwd_step(const bb_attn_bwd_args* args, void* stream);

/* delta[h, r] = sum_c dout[r,h,c] * o[r,h,c]  (dout bf16, o f32). */
int bb_attn_bwd_preprocess(const void* dout, const float* o, float* delta, int64_t n, int32_t heads,
                           int32_t head_dim, void* stream);

/* Row permutation over rows of `row_bytes` bytes (multiple of 16).
 * scatter == 0: dst[r] = src[index[r]];  scatter != 0: dst[index[r]] = src[r].
 * index holds 0-based row numbers (token_id - 1). */
int bb_permute_rows(void* dst, const void* src, const int64_t* index, int64_t n_rows,
                    int64_t row_bytes, int32_t scatter, void* stream);

/* Fill `count` 32-bit words (4-byte aligned; 16-byte stores when 16-byte aligned and
 * count % 4 == 0) with `value`: the zeroed
 * gradient accumulators and the -inf running lse of a ring pass (distributed.py:172-173,
 * 270-272), at the copy rate of cudaMemsetAsync. */
int bb_fill_u32(void* dst, uint32_t value, int64_t count, void* stream);

/* dst[r, c] += src[r, c] for r < rows, c < cols over row strides dst_ld / src_ld (floats;
 * cols and strides multiples of 4, 16-byte aligned): folding a gradient partial that
 * arrived from a peer into the owner's accumulator (distributed.py:293-295, the
 * circulating dQ's additions), whole or restricted to a head range. */
int bb_add_rows_f32(float* dst, const float* src, int64_t rows, int64_t cols, int64_t dst_ld, int64_t src_ld,
                    void* stream);

/* Cast f32 -> bf16 with optional zero padding of the last dimension
 * (cols_in -> cols_out, cols_out >= cols_in); rows are contiguous. */
int bb_cast_pad_bf16(void* dst, const float* src, int64_t rows, int32_t cols_in, int32_t cols_out,
                     void* stream);

/* Fused LM head + cross entropy (lmhead.py:41-93): h bf16 [n, dim], w bf16
 * [vocab, dim], targets int64 [n].  Writes loss f32 [n] (per-token nats, the
 * caller sums), dh f32 [n, dim]; ACCUMULATES dw f32 [vocab, dim] (so sequence
 * shards / row tiles reduce into one buffer).  rows_per_tile is B_s: logits of
 * one row tile (B_s x vocab) are the only logits-class buffer alive, retained
 * between forward and backward (no recompute).  vocab_per_tile
 * (B_v) does not change values (tests/test_lmhead.py:73-81); the kernels tile
 * the vocabulary in 256-column UMMA tiles. */
typedef struct bb_lmhead_args {
  const void* h;
  const void* w;
  const int64_t* targets;
  int64_t n;
  int64_t vocab;
  int64_t dim;
  int64_t rows_per_tile;
  int64_t vocab_per_tile;
  float* loss;
  float* dh;
  float* dw;
  void* workspace;
  int64_t workspace_bytes;
} bb_lmhead_args;

int64_t bb_lmhead_workspace_bytes(int64_t n, int64_t vocab, int64_t dim, int64_t rows_per_tile);
int bb_lmhead_fused(const bb_lmhead_args* args, void* stream);

/* Dense tcgen05 GEMM used by the LM head, exported for tests:
 * C[M,N] (+)= A[M,K] * B[N,K]^T.  a_mn/b_mn select MN-major storage
 * (A stored [K][M], B stored [K][N]); otherwise K-major ([M][K], [N][K]).
 * accumulate != 0 adds into C. */
int bb_gemm_bf16(const void* a, const void* b, float* c, int64_t m, int64_t n, int64_t k,
                 int32_t a_mn, int32_t b_mn, int32_t accumulate, void* stream);

/* Projection GEMM with the layout permutation and the bf16 cast fused into its store
 * (replaces oracle.project_qkv's matmul + shard_rows' row gather, oracle.py:60-65,
 * distributed.py:104-117): C[row_map[i], :] = bf16(A[i, :] . B^T) for i < m, with A
 * bf16 [m, k] K-major and B bf16 [n, k] (b_mn == 0) or [k, n] (b_mn != 0); row_map
 * (device int64 [m], may be NULL = identity) sends token row i to its shard-major row. */
int bb_gemm_bf16_rows(const void* a, const void* b, void* c, const int64_t* row_map, int64_t m, int64_t n, int64_t k,
                      int32_t b_mn, void* stream);

/* ---- Peer fabric for the one-process-per-GPU ring (csrc/bb_fabric.cu) ----
 * Replaces the reference's payload "send" of a ring step (TransferStep /
 * MessageLog, fabric.py:180-226; distributed.py:176-177, 283-286) with a
 * copy-engine push over NVLink into the receiver's arena plus a stream-ordered
 * flag.  An arena is one cudaMalloc (zero-filled) exported by CUDA IPC; peers
 * open it once.  bb_copy_async is a D2D cudaMemcpyAsync (peer pointers go over
 * NVLink on the copy engines, no SM work).  bb_flag_write stores `value` to a
 * 32-bit word (local or peer) after all earlier work of `stream`;
 * bb_flag_wait blocks `stream` until the local word is >= value. */
int32_t bb_ipc_handle_bytes(void);
int bb_arena_alloc(int64_t bytes, void** ptr_out);
int bb_arena_free(void* ptr);
int bb_ipc_export(const void* ptr, void* handle_out);
int bb_ipc_import(const void* handle, void** ptr_out);
int bb_ipc_close(void* ptr);
int bb_copy_async(void* dst, const void* src, int64_t bytes, void* stream);
int bb_flag_write(void* flag, uint32_t value, void* stream);
int bb_flag_wait(const void* flag, uint32_t value, void* stream);

/* ---- float64 tile math (burstsim/numerics.py, oracle.py:129-154) ----
 * Device pointers to float64; -inf is an exact sentinel as in the reference
 * (numerics.py:62-69,101-116).  bb_matmul_f64: C[m,n] (row-major, contiguous)
 * = sum_k A[i*sa0 + k*sa1] * B[k*sb0 + j*sb1], k ascending (transposes are
 * stride swaps).  bb_row_logsumexp_f64: rows of `cols` at stride `lds`, all -inf
 * rows give -inf.  bb_lse_merge_f64: np.logaddexp.  bb_exp_shifted_f64:
 * exp(s - lse[:,None]), rows with lse == -inf give 0.  bb_exp_gap_f64: exp(a-b),
 * a == -inf gives 0.  bb_rowsum_hadamard_f64: out[i] = sum_j a[i,j] b[i,j].
 * bb_xent_f64: loss[r] = lse[r] - logits[r, y_r], g = exp(logits - lse) - onehot(y)
 * (0-based targets, checked by the caller). */
int bb_matmul_f64(const double* a, int64_t sa0, int64_t sa1, const double* b, int64_t sb0, int64_t sb1,
                  double* c, int64_t m, int64_t n, int64_t k, void* stream);
/* In place: s[i] = allowed[i] ? s[i] / root : -inf (masked_scores, oracle.py:66-75; root = sqrt(d),
 * divided like the reference's `/ np.sqrt(d)`). */
int bb_scale_mask_f64(double* s, const uint8_t* allowed, double root, int64_t n, void* stream);
int bb_row_logsumexp_f64(const double* s, int64_t rows, int64_t cols, int64_t lds, double* out, void* stream);
int bb_lse_merge_f64(const double* a, const double* b, double* out, int64_t n, void* stream);
int bb_exp_shifted_f64(const double* s, const double* lse, double* out, int64_t rows, int64_t cols, void* stream);
int bb_exp_gap_f64(const double* a, const double* b, double* out, int64_t n, void* stream);
int bb_rowsum_hadamard_f64(const double* a, const double* b, double* out, int64_t rows, int64_t cols, void* stream);
int bb_xent_f64(const double* logits, const double* lse, const int64_t* targets, int64_t rows, int64_t vocab,
                double* loss, double* g, void* stream);

const char* bb_last_error(void);
/* Diagnostics: with BB_PROBE=1 in the environment, kernels record per-phase
 * clock64() stamps of CTA (0,0) for its first tiles; copies n int64 to host. */
int bb_debug_probe(int64_t* host_out, int32_t n);
/* Test hook: the shard size (rows, multiple of 128; 0 = the default 524288) above which
 * bb_attn_fwd_step (key shard) and bb_attn_bwd_step (query shard) split a zigzag or contiguous
 * shard into sub-shards of a contiguous layout with more devices and launch every sub-shard
 * pair -- how one call takes a shard larger than the kernels' class tables (a 1M-token
 * sequence on one or two GPUs).  Process-wide. */
int bb_debug_set_split_rows(int64_t rows);

/* Mask realisation dump for tests (replaces nothing in the reference; it exposes what the
 * kernels compute in place of local_pair_mask, partitioning.py:120-169).  For the ring step
 * (q_device, k_device) with n_q query and n_k key rows, writes classes[qt * n_kt + kt]
 * (device int8, 0 skip / 1 full / 2 partial) exactly as attn_fwd_kernel (view 0) or
 * attn_bwd_kernel (view 1) classify the 128x128 tile, and, if `allowed` is not NULL,
 * allowed[q * n_k + k] (device uint8, n_q x n_k) = the element mask that kernel applies. */
int bb_debug_mask_tiles(const bb_layout* layout, const bb_mask* mask, int32_t q_device, int32_t k_device,
                        int64_t n_q, int64_t n_k, int32_t view, int8_t* classes, uint8_t* allowed, void* stream);
int32_t bb_abi_version(void);
/* Number of kernel launches issued by this library since load (for bench). */
int64_t bb_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* BURST_B200_H */
