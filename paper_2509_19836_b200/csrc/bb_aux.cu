// HBM-bound helper kernels on the hot path.
//   attn_bwd_preprocess : D = rowsum(dO o O) once per backward (distributed.py:274-275)
//   permute_rows        : shard_rows / gather_rows row permutations (distributed.py:104-130)
//   cast_pad_bf16       : f32 -> bf16 staging of caller inputs with head-dim padding
//   lmhead_reduce       : streaming-LSE combine + loss = lse - <h, w_y> (lmhead.py:79-81)
//   lmhead_dlogits      : softmax - onehot in place over the retained logits (lmhead.py:86-89)
//   fill_u32            : zero / -inf initialisation of the ring's accumulators
//   add_rows            : folding a peer's gradient partial into the owner's accumulator
#include <algorithm>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "bb_host.h"

namespace bb {
namespace {

// One warp per (row, head): coalesced 16-byte loads along head_dim.
__global__ void preprocess_kernel(const __nv_bfloat16* __restrict__ dout, const float* __restrict__ o,
                                  float* __restrict__ delta, int64_t n, int32_t heads, int32_t d) {
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= n * heads) return;
  const int64_t r = gw / heads;
  const int32_t h = static_cast<int32_t>(gw % heads);
  const __nv_bfloat16* dr = dout + gw * d;
  const float* orow = o + gw * d;
  float acc = 0.f;
  for (int c = lane * 4; c < d; c += 128) {
    const float4 ov = *reinterpret_cast<const float4*>(orow + c);
    const __nv_bfloat162 d01 = *reinterpret_cast<const __nv_bfloat162*>(dr + c);
    const __nv_bfloat162 d23 = *reinterpret_cast<const __nv_bfloat162*>(dr + c + 2);
    acc += __low2float(d01) * ov.x + __high2float(d01) * ov.y + __low2float(d23) * ov.z +
           __high2float(d23) * ov.w;
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffff, acc, s);
  if (lane == 0) delta[static_cast<int64_t>(h) * n + r] = acc;
}

// One warp per row, int4 (16 B) moves.
__global__ void permute_kernel(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src,
                               const int64_t* __restrict__ index, int64_t n_rows, int64_t row_bytes,
                               int scatter) {
  const int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= n_rows) return;
  const int64_t other = index[r];
  const int4* s = reinterpret_cast<const int4*>(src + (scatter ? r : other) * row_bytes);
  int4* d = reinterpret_cast<int4*>(dst + (scatter ? other : r) * row_bytes);
  const int64_t n16 = row_bytes / 16;
  for (int64_t i = lane; i < n16; i += 32) d[i] = s[i];
}

__global__ void cast_pad_kernel(__nv_bfloat16* __restrict__ dst, const float* __restrict__ src,
                                int64_t rows, int32_t cin, int32_t cout) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows * cout) return;
  const int64_t r = i / cout;
  const int32_t c = static_cast<int32_t>(i % cout);
  dst[i] = __float2bfloat16_rn(c < cin ? src[r * cin + c] : 0.f);
}

__global__ void lmhead_reduce_kernel(const float* __restrict__ part_max, const float* __restrict__ part_sum,
                                     const float* __restrict__ tgt_logit, int64_t rows, int32_t tiles,
                                     float* __restrict__ lse_out, float* __restrict__ loss) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  float m = -INFINITY;
  for (int t = 0; t < tiles; ++t) m = fmaxf(m, part_max[r * tiles + t]);
  float s = 0.f;
  for (int t = 0; t < tiles; ++t) s += part_sum[r * tiles + t] * expf(part_max[r * tiles + t] - m);
  const float lse = m + logf(s);
  lse_out[r] = lse;
  loss[r] = lse - tgt_logit[r];
}

// g = exp(logit - lse) - [col == y], written as bf16 (UMMA operand of dH / dW).
__global__ void lmhead_dlogits_kernel(const float* __restrict__ logits, const float* __restrict__ lse,
                                      const int64_t* __restrict__ targets, int64_t rows, int64_t vocab,
                                      int64_t ldg, __nv_bfloat16* __restrict__ g) {
  const int64_t r = blockIdx.y;
  const int64_t c0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
  if (r >= rows || c0 >= vocab) return;
  const float l = lse[r];
  const int64_t y = targets[r];
  const float* src = logits + r * ldg + c0;
  __nv_bfloat16* dst = g + r * ldg + c0;
  if (c0 + 4 <= vocab && (ldg % 4) == 0) {
    const float4 x = *reinterpret_cast<const float4*>(src);
    float v0 = __expf(x.x - l), v1 = __expf(x.y - l), v2 = __expf(x.z - l), v3 = __expf(x.w - l);
    if (y == c0) v0 -= 1.f;
    if (y == c0 + 1) v1 -= 1.f;
    if (y == c0 + 2) v2 -= 1.f;
    if (y == c0 + 3) v3 -= 1.f;
    reinterpret_cast<__nv_bfloat162*>(dst)[0] = __floats2bfloat162_rn(v0, v1);
    reinterpret_cast<__nv_bfloat162*>(dst)[1] = __floats2bfloat162_rn(v2, v3);
  } else {
    for (int64_t c = c0; c < c0 + 4 && c < vocab; ++c) {
      float v = __expf(src[c - c0] - l);
      if (y == c) v -= 1.f;
      dst[c - c0] = __float2bfloat16_rn(v);
    }
  }
}

// Fill with a 32-bit pattern (0 for the gradient accumulators, -inf for the running lse):
// 16-byte stores, a grid of a few CTAs per SM striding over the buffer.  (torch's fill_
// reaches ~3.6 TB/s on a 4 GB buffer; this is the ~6.5 TB/s of cudaMemsetAsync.)
__global__ void fill_u32_kernel(uint4* __restrict__ dst, uint32_t v, int64_t n4) {
  const uint4 x = make_uint4(v, v, v, v);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n4; i += 4 * stride) {
    dst[i] = x;
    dst[i + stride] = x;
    dst[i + 2 * stride] = x;
    dst[i + 3 * stride] = x;
  }
  for (; i < n4; i += stride) dst[i] = x;
}

__global__ void fill_u32_scalar_kernel(uint32_t* __restrict__ dst, uint32_t v, int64_t n) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = v;
}

// dst[r, :cols] += src[r, :cols] over row-strided float matrices (the ring's gradient folds,
// whole accumulators or a head range of them); 16-byte accesses, 4 in flight per thread.
__global__ void add_rows_kernel(float4* __restrict__ dst, const float4* __restrict__ src, int64_t rows,
                                int64_t cols4, int64_t dld4, int64_t sld4) {
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    float4* d = dst + r * dld4;
    const float4* s = src + r * sld4;
    int64_t c = threadIdx.x;
    for (; c + 3 * blockDim.x < cols4; c += 4 * blockDim.x) {
      float4 a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = d[c + u * blockDim.x];
        b[u] = s[c + u * blockDim.x];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        d[c + u * blockDim.x] = make_float4(a[u].x + b[u].x, a[u].y + b[u].y, a[u].z + b[u].z, a[u].w + b[u].w);
    }
    for (; c < cols4; c += blockDim.x) {
      const float4 a = d[c], b = s[c];
      d[c] = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
    }
  }
}

}  // namespace

int launch_preprocess(const void* dout, const float* o, float* delta, int64_t n, int32_t heads, int32_t d,
                      cudaStream_t st) {
  if (d % 4 != 0) return set_error(BB_ERR_UNSUPPORTED, "preprocess: head_dim %d not a multiple of 4", d);
  const int64_t warps = n * heads;
  const int threads = 256;
  const int64_t blocks = (warps * 32 + threads - 1) / threads;
  preprocess_kernel<<<static_cast<unsigned>(blocks), threads, 0, st>>>(
      static_cast<const __nv_bfloat16*>(dout), o, delta, n, heads, d);
  return check_launch("preprocess_kernel");
}

int launch_permute(void* dst, const void* src, const int64_t* index, int64_t n_rows, int64_t row_bytes,
                   int scatter, cudaStream_t st) {
  if (row_bytes % 16) return set_error(BB_ERR_INVALID, "permute_rows: row_bytes %lld not a multiple of 16", (long long)row_bytes);
  if (n_rows == 0) return BB_OK;
  const int threads = 256;
  const int64_t blocks = (n_rows * 32 + threads - 1) / threads;
  permute_kernel<<<static_cast<unsigned>(blocks), threads, 0, st>>>(
      static_cast<uint8_t*>(dst), static_cast<const uint8_t*>(src), index, n_rows, row_bytes, scatter);
  return check_launch("permute_kernel");
}

int launch_cast_pad(void* dst, const float* src, int64_t rows, int32_t cin, int32_t cout, cudaStream_t st) {
  const int64_t total = rows * cout;
  if (total == 0) return BB_OK;
  const int threads = 256;
  cast_pad_kernel<<<static_cast<unsigned>((total + threads - 1) / threads), threads, 0, st>>>(
      static_cast<__nv_bfloat16*>(dst), src, rows, cin, cout);
  return check_launch("cast_pad_kernel");
}

int launch_lmhead_reduce(const float* pmax, const float* psum, const float* tgt, int64_t rows, int32_t tiles,
                         float* lse, float* loss, cudaStream_t st) {
  const int threads = 256;
  lmhead_reduce_kernel<<<static_cast<unsigned>((rows + threads - 1) / threads), threads, 0, st>>>(
      pmax, psum, tgt, rows, tiles, lse, loss);
  return check_launch("lmhead_reduce_kernel");
}

int launch_lmhead_dlogits(const float* logits, const float* lse, const int64_t* targets, int64_t rows,
                          int64_t vocab, int64_t ldg, void* g, cudaStream_t st) {
  const int threads = 256;
  dim3 grid(static_cast<unsigned>((vocab / 4 + threads) / threads), static_cast<unsigned>(rows));
  lmhead_dlogits_kernel<<<grid, threads, 0, st>>>(logits, lse, targets, rows, vocab, ldg,
                                                  static_cast<__nv_bfloat16*>(g));
  return check_launch("lmhead_dlogits_kernel");
}

int launch_fill_u32(void* dst, uint32_t value, int64_t count, cudaStream_t st) {
  if (count <= 0) return BB_OK;
  if (reinterpret_cast<uintptr_t>(dst) & 3) return set_error(BB_ERR_INVALID, "fill_u32: buffer not 4-byte aligned");
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int threads = 512;
  if ((reinterpret_cast<uintptr_t>(dst) & 15) || (count & 3)) {  // small / odd buffers: word stores
    const int64_t blocks = std::min<int64_t>(static_cast<int64_t>(sms) * 4, (count + threads - 1) / threads);
    fill_u32_scalar_kernel<<<static_cast<unsigned>(blocks), threads, 0, st>>>(static_cast<uint32_t*>(dst), value, count);
    return check_launch("fill_u32_scalar_kernel");
  }
  const int64_t n4 = count / 4;
  const int64_t blocks = std::min<int64_t>(static_cast<int64_t>(sms) * 4, (n4 + threads - 1) / threads);
  fill_u32_kernel<<<static_cast<unsigned>(blocks), threads, 0, st>>>(static_cast<uint4*>(dst), value, n4);
  return check_launch("fill_u32_kernel");
}

int launch_add_rows(float* dst, const float* src, int64_t rows, int64_t cols, int64_t dst_ld, int64_t src_ld,
                    cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return BB_OK;
  if ((reinterpret_cast<uintptr_t>(dst) & 15) || (reinterpret_cast<uintptr_t>(src) & 15) || (cols & 3) ||
      (dst_ld & 3) || (src_ld & 3) || dst_ld < cols || src_ld < cols)
    return set_error(BB_ERR_INVALID, "add_rows: rows must be 16-byte aligned float4 runs (cols %lld, ld %lld / %lld)",
                     (long long)cols, (long long)dst_ld, (long long)src_ld);
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>(static_cast<int64_t>(sms) * 8, rows);
  add_rows_kernel<<<static_cast<unsigned>(blocks), threads, 0, st>>>(
      reinterpret_cast<float4*>(dst), reinterpret_cast<const float4*>(src), rows, cols / 4, dst_ld / 4, src_ld / 4);
  return check_launch("add_rows_kernel");
}

}  // namespace bb
