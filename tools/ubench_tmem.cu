// Micro-benchmark: tcgen05.ld / tcgen05.st throughput per SM (bytes per clock) at 4 / 8 / 16
// warps, the numbers that bound how fast the softmax warps can drain S (and dP) from TMEM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I. -o ubench_tmem tools/ubench_tmem.cu
#include <cstdint>
#include <cstdio>

#include "paper_2509_19836_b200/csrc/bb_ptx.cuh"

using namespace bb;

template <int MODE>  // 0: ld x32 (+wait per ld), 1: 4 x ld x32 then one wait, 2: st x32, 3: ld x32 + MUFU on it
__global__ void __launch_bounds__(512, 1) tmem_bench(float* out, long long* cyc, int iters) {
  __shared__ uint32_t slot;
  const uint32_t warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t lane_base = ((warp & 3) * 32) << 16;
  const uint32_t col0 = (warp >> 2) * 128;  // 4 column groups of 128
  float acc = 0.f;
  float v[32];
  for (int i = 0; i < 32; ++i) v[i] = i * 0.001f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0 || MODE == 3) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        tmem_ld32(tmem + lane_base + col0 + c * 32, v);
        tmem_ld_wait();
        if (MODE == 3) {
#pragma unroll
          for (int i = 0; i < 32; ++i) acc += ex2_approx(v[i]);
        } else {
          acc += v[c];
        }
      }
    } else if (MODE == 1) {
      float a[32], b[32], c2[32], d[32];
      tmem_ld32(tmem + lane_base + col0 + 0, a);
      tmem_ld32(tmem + lane_base + col0 + 32, b);
      tmem_ld32(tmem + lane_base + col0 + 64, c2);
      tmem_ld32(tmem + lane_base + col0 + 96, d);
      tmem_ld_wait();
      acc += a[it & 31] + b[(it + 1) & 31] + c2[(it + 2) & 31] + d[(it + 3) & 31];
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        v[c] += 1.f;
        tmem_st32(tmem + lane_base + col0 + c * 32, v);
      }
      tmem_st_wait();
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + v[3];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 512 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 2000;
  const char* names[] = {"tcgen05.ld x32 + wait", "4 x ld x32, one wait", "tcgen05.st x32", "ld x32 + 32 MUFU"};
  for (int warps : {4, 8, 16}) {
    for (int mode = 0; mode < 4; ++mode) {
      long long h = 0;
      for (int rep = 0; rep < 2; ++rep) {
        switch (mode) {
          case 0: tmem_bench<0><<<148, warps * 32>>>(out, cyc, iters); break;
          case 1: tmem_bench<1><<<148, warps * 32>>>(out, cyc, iters); break;
          case 2: tmem_bench<2><<<148, warps * 32>>>(out, cyc, iters); break;
          case 3: tmem_bench<3><<<148, warps * 32>>>(out, cyc, iters); break;
        }
        cudaError_t e = cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) {
          printf("error %s\n", cudaGetErrorString(e));
          return 1;
        }
      }
      const double bytes = double(iters) * 4 * 32 * 4 * 32 * warps;  // 4 x (32 lanes x 32 cols x 4 B) per warp-iter
      printf("warps/SM %2d  %-24s %.1f B/clk/SM  (%.0f clk per 64 KB)\n", warps, names[mode], bytes / double(h),
             65536.0 / (bytes / double(h)));
    }
  }
  return 0;
}
