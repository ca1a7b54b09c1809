// Micro-benchmarks of the per-element softmax ops on sm_100a (clock64 per warp).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench tools/ubench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// exp2 on the FMA pipe: 2^x = 2^floor(x) * p(frac), degree-3 minimax (FA4-style)
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -127.f);
  const float fl = floorf(x);
  const float f = x - fl;
  float p = fmaf(0.0555041086648216f, f, 0.2402264923172231f);
  p = fmaf(p, f, 0.6931471805599453f);
  p = fmaf(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + (static_cast<int>(fl) << 23));
}
__device__ __forceinline__ uint32_t pack(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ uint32_t pack_int(float a, float b) {  // round-to-nearest-even via integer ops
  uint32_t ua = __float_as_uint(a), ub = __float_as_uint(b);
  ua += 0x7FFFu + ((ua >> 16) & 1u);
  ub += 0x7FFFu + ((ub >> 16) & 1u);
  return __byte_perm(ua, ub, 0x7632);
}

template <int MODE>
__global__ void bench(float* out, long long* cyc, int iters) {
  float v[32];
  for (int i = 0; i < 32; ++i) v[i] = -0.01f * (threadIdx.x % 7 + i);
  uint32_t acc = 0;
  float facc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if (MODE == 0) v[i] = ex2(v[i]) - 1.0f;
      if (MODE == 1) v[i] = ex2_poly(v[i]) - 1.0f;
      if (MODE == 2 && (i & 1)) acc ^= pack(v[i - 1], v[i]);
      if (MODE == 3 && (i & 1)) acc ^= pack_int(v[i - 1], v[i]);
      if (MODE == 4) v[i] = fmaf(v[i], 1.0001f, -0.5f);
    }
    if (MODE >= 2) v[it & 31] += __uint_as_float(acc & 0x3f800000u) * 1e-30f;
  }
  long long t1 = clock64();
  for (int i = 0; i < 32; ++i) facc += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = facc + acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 2000;
  const char* names[] = {"MUFU.EX2", "ex2 poly (FMA pipe)", "F2FP bf16x2 pack", "int-op bf16x2 pack", "FFMA"};
  for (int warps : {4, 8, 16}) {
    for (int mode = 0; mode < 5; ++mode) {
      long long h = 0;
      for (int rep = 0; rep < 2; ++rep) {
        switch (mode) {
          case 0: bench<0><<<148, warps * 32>>>(out, cyc, iters); break;
          case 1: bench<1><<<148, warps * 32>>>(out, cyc, iters); break;
          case 2: bench<2><<<148, warps * 32>>>(out, cyc, iters); break;
          case 3: bench<3><<<148, warps * 32>>>(out, cyc, iters); break;
          case 4: bench<4><<<148, warps * 32>>>(out, cyc, iters); break;
        }
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      }
      const double elems = double(iters) * 32 * warps * 32;  // per SM
      printf("warps/SM %2d  %-22s %.2f elements/clk/SM\n", warps, names[mode], elems / double(h));
    }
  }
  return 0;
}
