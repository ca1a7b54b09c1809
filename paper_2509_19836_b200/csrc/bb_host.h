// Host-side plumbing shared by the kernel translation units: error state,
// launch accounting and TMA tensor-map construction (driver entry point is
// resolved through cudart so the library has no link-time libcuda dependency
// and loads on GPU-less hosts).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "../../include/burst_b200.h"

namespace bb {

int set_error(int code, const char* fmt, ...);
int check_cuda(cudaError_t err, const char* what);
int check_launch(const char* what);  // cudaGetLastError after a launch; counts it

extern std::atomic<int64_t> g_launches;

// 2-D bf16 tensor map: `inner` contiguous elements per row, `outer` rows,
// `row_stride_bytes` between rows; SWIZZLE_128B box {box_inner, box_outer}.
bool make_tmap_bf16_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                       uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer);

bool make_tmap_2d(CUtensorMap* map, const void* base, CUtensorMapDataType dtype, uint64_t inner, uint64_t outer,
                  uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer,
                  CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_128B);

int num_sms();

// BB_PROBE=1 in the environment: device buffer kernels write phase timestamps into.
long long* debug_probe_buffer();

// ---- launchers (one per kernel family) ----
enum GemmEpilogue { GEMM_STORE = 0, GEMM_ACCUM = 1, GEMM_LOGITS = 2, GEMM_BF16 = 3 };

struct LogitsEpilogue {
  const int64_t* targets;  // [M] vocab ids for the rows of this tile
  float* part_max;         // [M][n_tiles]
  float* part_sum;         // [M][n_tiles]
  float* tgt_logit;        // [M]
};

int launch_gemm(const void* a, const void* b, float* c, int64_t m, int64_t n, int64_t k,
                int64_t lda, int64_t ldb, int64_t ldc, bool a_mn, bool b_mn, int epilogue,
                const LogitsEpilogue* le, bool raster_m_fast, cudaStream_t stream);
int gemm_n_tile();
// C16[row_map ? row_map[i] : i, :] = bf16(A[i, :] . B^T); A K-major, B K-major or MN-major.
int launch_gemm_bf16(const void* a, const void* b, void* c16, const int64_t* row_map, int64_t m, int64_t n, int64_t k,
                     int64_t lda, int64_t ldb, int64_t ldc, bool b_mn, cudaStream_t stream);

// lse_ld: row length of the lse (and delta) arrays; a.n_q unless bb_api.cu launches a sub-shard
int launch_attn_fwd(const bb_attn_fwd_args& a, cudaStream_t stream, int64_t lse_ld);
int launch_attn_bwd(const bb_attn_bwd_args& a, cudaStream_t stream, int64_t lse_ld);
// diagnostics buffer (BB_PROBE=1): [0, 4096) per-phase clocks of one CTA, then 8 words per CTA
// (SM id, globaltimer at entry / end of prologue / epilogue start / exit) from 4096 on
constexpr int kProbeEntries = 65536;
// largest shard (rows) one launch takes: the kernels' class tables hold 4096 tiles of 128
constexpr int64_t MAX_SHARD_ROWS = 4096 * 128;

int launch_matmul_f64(const double* a, int64_t sa0, int64_t sa1, const double* b, int64_t sb0, int64_t sb1,
                      double* c, int64_t m, int64_t n, int64_t k, cudaStream_t st);
int launch_scale_mask_f64(double* s, const uint8_t* allowed, double scale, int64_t n, cudaStream_t st);
int launch_row_lse_f64(const double* s, int64_t rows, int64_t cols, int64_t lds, double* out, cudaStream_t st);
int launch_lse_merge_f64(const double* a, const double* b, double* out, int64_t n, cudaStream_t st);
int launch_exp_shifted_f64(const double* s, const double* lse, double* out, int64_t rows, int64_t cols,
                           cudaStream_t st);
int launch_exp_gap_f64(const double* a, const double* b, double* out, int64_t n, cudaStream_t st);
int launch_rowsum_hadamard_f64(const double* a, const double* b, double* out, int64_t rows, int64_t cols,
                               cudaStream_t st);
int launch_xent_f64(const double* logits, const double* lse, const int64_t* targets, int64_t rows, int64_t vocab,
                    double* loss, double* g, cudaStream_t st);

}  // namespace bb
