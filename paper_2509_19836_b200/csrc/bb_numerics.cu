// Float64 tile math of burstsim/numerics.py on the device (the reference's public
// numerics API, SURVEY §8a row "numerics.*"): every kernel keeps -inf exact, as
// numerics.py:62-69,101-116 do, and fixes its accumulation order so results are
// bit-identical run to run (numerics.py:1-11).
//   matmul_f64        numerics.py:35-45   C = A B, strided operands (transposes are free)
//   row_lse_f64       numerics.py:48-59   per-row logsumexp; all -inf rows give -inf
//   lse_merge_f64     numerics.py:62-69   np.logaddexp semantics
//   exp_shifted_f64   numerics.py:101-107 exp(s - lse[:, None]); lse == -inf rows give 0
//   exp_gap_f64       numerics.py:110-116 exp(a - b); a == -inf gives 0
//   rowsum_hadamard   numerics.py:86-92   out[i] = sum_j a[i,j] b[i,j]
//   scale_mask_f64    oracle.py:66-75     masked_scores: S / sqrt(d), masked entries -inf
//   xent_f64          oracle.py:129-154   loss = lse - logit[y], g = softmax - onehot(y)
// All are HBM-bound (one read of each operand, one write) except matmul, which runs on the
// FP64 pipe with a 64x64 CTA tile staged in shared memory.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <algorithm>

#include "bb_host.h"

namespace bb {
namespace {

constexpr int kWarps = 8;  // 256-thread CTAs, one warp per row for the row reductions

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffff, v, s));
  return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(0xffffffff, v, s);
  return v;
}

__global__ void row_lse_kernel(const double* __restrict__ s, int64_t rows, int64_t cols, int64_t lds,
                               double* __restrict__ out) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const double* row = s + r * lds;
  double m = -CUDART_INF;
  for (int64_t c = lane; c < cols; c += 32) m = fmax(m, row[c]);
  m = warp_max(m);
  if (m == -CUDART_INF) {
    if (lane == 0) out[r] = -CUDART_INF;
    return;
  }
  double acc = 0.0;
  for (int64_t c = lane; c < cols; c += 32) acc += exp(row[c] - m);
  acc = warp_sum(acc);
  if (lane == 0) out[r] = m + log(acc);
}

// np.logaddexp: equal arguments (incl. -inf, -inf) give a + ln 2 (-inf stays -inf);
// otherwise max + log1p(exp(-|a - b|)).
__global__ void lse_merge_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                 double* __restrict__ out, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = a[i], y = b[i];
  double r;
  if (x == y) {
    r = x + CUDART_LN2;
  } else {
    const double t = x - y;
    if (t > 0.0) r = x + log1p(exp(-t));
    else if (t <= 0.0) r = y + log1p(exp(t));
    else r = t;  // NaN propagates
  }
  out[i] = r;
}

__global__ void exp_shifted_kernel(const double* __restrict__ s, const double* __restrict__ lse,
                                   double* __restrict__ out, int64_t rows, int64_t cols) {
  const int64_t total = rows * cols;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double l = lse[i / cols];
    out[i] = (l == -CUDART_INF) ? 0.0 : exp(s[i] - l);
  }
}

__global__ void exp_gap_kernel(const double* __restrict__ a, const double* __restrict__ b,
                               double* __restrict__ out, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = a[i];
  out[i] = (x == -CUDART_INF) ? 0.0 : exp(x - b[i]);
}

__global__ void rowsum_hadamard_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                       double* __restrict__ out, int64_t rows, int64_t cols) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  double acc = 0.0;
  for (int64_t c = lane; c < cols; c += 32) acc = fma(a[r * cols + c], b[r * cols + c], acc);
  acc = warp_sum(acc);
  if (lane == 0) out[r] = acc;
}

// One warp per row: loss[r] = lse[r] - logits[r, y]; g[r, :] = exp(logits - lse) - onehot(y).
__global__ void xent_kernel(const double* __restrict__ logits, const double* __restrict__ lse,
                            const int64_t* __restrict__ targets, int64_t rows, int64_t vocab,
                            double* __restrict__ loss, double* __restrict__ g) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const double l = lse[r];
  const int64_t y = targets[r];
  const double* row = logits + r * vocab;
  for (int64_t c = lane; c < vocab; c += 32) {
    double p = (l == -CUDART_INF) ? 0.0 : exp(row[c] - l);
    if (c == y) p -= 1.0;
    g[r * vocab + c] = p;
  }
  if (lane == 0) loss[r] = -row[y] + l;
}

// s[i] = allowed[i] ? s[i] / root : -inf, in place (oracle.py:73-75 after the Q K^T product;
// a division like the reference's `/ np.sqrt(d)`, not a multiply by its reciprocal).
__global__ void scale_mask_kernel(double* __restrict__ s, const uint8_t* __restrict__ allowed, double root,
                                  int64_t n) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    s[i] = allowed[i] ? s[i] / root : -CUDART_INF;
}

// C[m, n] = sum_k A[m, k] B[k, n] in float64, k ascending for every element.
// 64x64 output tile per 256-thread CTA, 4x4 per thread, K staged 16 at a time.
constexpr int kTm = 64, kTn = 64, kTk = 16;

__global__ void __launch_bounds__(256) matmul_f64_kernel(const double* __restrict__ a, int64_t sa0, int64_t sa1,
                                                         const double* __restrict__ b, int64_t sb0, int64_t sb1,
                                                         double* __restrict__ c, int64_t m, int64_t n, int64_t k) {
  __shared__ double as[kTk][kTm + 1];
  __shared__ double bs[kTk][kTn + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * kTm, n0 = static_cast<int64_t>(blockIdx.x) * kTn;
  double acc[4][4] = {};
  for (int64_t k0 = 0; k0 < k; k0 += kTk) {
    for (int i = threadIdx.x; i < kTk * kTm; i += 256) {
      // A tile: consecutive threads walk m when A is column-major (sa0 == 1), else k.
      const int kk = (sa0 == 1) ? i / kTm : i % kTk;
      const int mm = (sa0 == 1) ? i % kTm : i / kTk;
      const int64_t gm = m0 + mm, gk = k0 + kk;
      as[kk][mm] = (gm < m && gk < k) ? a[gm * sa0 + gk * sa1] : 0.0;
    }
    for (int i = threadIdx.x; i < kTk * kTn; i += 256) {
      const int kk = (sb1 == 1) ? i / kTn : i % kTk;
      const int nn = (sb1 == 1) ? i % kTn : i / kTk;
      const int64_t gn = n0 + nn, gk = k0 + kk;
      bs[kk][nn] = (gn < n && gk < k) ? b[gk * sb0 + gn * sb1] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kTk; ++kk) {
      double av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = as[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gm = m0 + ty + 16 * i;
    if (gm >= m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gn = n0 + tx + 16 * j;
      if (gn < n) c[gm * n + gn] = acc[i][j];
    }
  }
}

inline unsigned blocks_for(int64_t items, int per_block) {
  return static_cast<unsigned>((items + per_block - 1) / per_block);
}

}  // namespace

int launch_matmul_f64(const double* a, int64_t sa0, int64_t sa1, const double* b, int64_t sb0, int64_t sb1,
                      double* c, int64_t m, int64_t n, int64_t k, cudaStream_t st) {
  if (m < 0 || n < 0 || k < 0) return set_error(BB_ERR_INVALID, "bb_matmul_f64: negative extent");
  if (m == 0 || n == 0) return BB_OK;
  if (k == 0) return check_cuda(cudaMemsetAsync(c, 0, sizeof(double) * m * n, st), "bb_matmul_f64 memset");
  if (m > 65535LL * kTm) return set_error(BB_ERR_UNSUPPORTED, "bb_matmul_f64: m %lld too large", (long long)m);
  dim3 grid(blocks_for(n, kTn), blocks_for(m, kTm));
  matmul_f64_kernel<<<grid, 256, 0, st>>>(a, sa0, sa1, b, sb0, sb1, c, m, n, k);
  return check_launch("matmul_f64_kernel");
}

int launch_scale_mask_f64(double* s, const uint8_t* allowed, double scale, int64_t n, cudaStream_t st) {
  if (n == 0) return BB_OK;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 16);
  scale_mask_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(s, allowed, scale, n);
  return check_launch("scale_mask_kernel");
}

int launch_row_lse_f64(const double* s, int64_t rows, int64_t cols, int64_t lds, double* out, cudaStream_t st) {
  if (rows == 0) return BB_OK;
  row_lse_kernel<<<blocks_for(rows, kWarps), 32 * kWarps, 0, st>>>(s, rows, cols, lds, out);
  return check_launch("row_lse_kernel");
}

int launch_lse_merge_f64(const double* a, const double* b, double* out, int64_t n, cudaStream_t st) {
  if (n == 0) return BB_OK;
  lse_merge_kernel<<<blocks_for(n, 256), 256, 0, st>>>(a, b, out, n);
  return check_launch("lse_merge_kernel");
}

int launch_exp_shifted_f64(const double* s, const double* lse, double* out, int64_t rows, int64_t cols,
                           cudaStream_t st) {
  if (rows == 0 || cols == 0) return BB_OK;
  const int64_t blocks = std::min<int64_t>((rows * cols + 255) / 256, int64_t(num_sms()) * 16);
  exp_shifted_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(s, lse, out, rows, cols);
  return check_launch("exp_shifted_kernel");
}

int launch_exp_gap_f64(const double* a, const double* b, double* out, int64_t n, cudaStream_t st) {
  if (n == 0) return BB_OK;
  exp_gap_kernel<<<blocks_for(n, 256), 256, 0, st>>>(a, b, out, n);
  return check_launch("exp_gap_kernel");
}

int launch_rowsum_hadamard_f64(const double* a, const double* b, double* out, int64_t rows, int64_t cols,
                               cudaStream_t st) {
  if (rows == 0) return BB_OK;
  rowsum_hadamard_kernel<<<blocks_for(rows, kWarps), 32 * kWarps, 0, st>>>(a, b, out, rows, cols);
  return check_launch("rowsum_hadamard_kernel");
}

int launch_xent_f64(const double* logits, const double* lse, const int64_t* targets, int64_t rows, int64_t vocab,
                    double* loss, double* g, cudaStream_t st) {
  if (rows == 0) return BB_OK;
  xent_kernel<<<blocks_for(rows, kWarps), 32 * kWarps, 0, st>>>(logits, lse, targets, rows, vocab, loss, g);
  return check_launch("xent_kernel");
}

}  // namespace bb
