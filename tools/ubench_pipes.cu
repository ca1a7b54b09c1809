// Pipe-assignment micro-benchmark for the softmax inner loop on sm_100a: throughput (per SM per
// clock) of MUFU.EX2, F2FP (bf16x2 pack), FRND, the FMA-pipe exp2 polynomial, and their mixes,
// each with 32 independent chains per thread so latency is hidden.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_pipes_bin tools/ubench_pipes.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t f2fp(float a, float b) {
  uint32_t r;
  asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}
// 2^x on the FMA pipe without FRND: floor via a round-down add of 1.5*2^23, cubic on the fraction,
// exponent inserted with an integer multiply-add.
__device__ __forceinline__ float ex2_fma(float x) {
  x = fmaxf(x, -126.f);
  float j;
  asm volatile("add.rm.f32 %0, %1, 0f4B400000;" : "=f"(j) : "f"(x));
  const float fl = j - 12582912.f;
  const float f = x - fl;
  float p = fmaf(0.0555041086648216f, f, 0.2402264923172231f);
  p = fmaf(p, f, 0.6931471805599453f);
  p = fmaf(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(j) << 23));
}

__device__ __forceinline__ uint32_t ex2_h2(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t ex2_bf2(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

template <int MODE>
__global__ void __launch_bounds__(512) pipes(float* out, long long* cyc, int iters) {
  float v[32];
  uint32_t u = 0;
  for (int i = 0; i < 32; ++i) v[i] = -0.001f * (threadIdx.x % 7 + i);
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      if (MODE == 0) {  // MUFU only
        v[i] = ex2(v[i]);
        v[i + 1] = ex2(v[i + 1]);
      } else if (MODE == 1) {  // F2FP only
        const uint32_t r = f2fp(v[i], v[i + 1]);
        v[i] = __uint_as_float(r);
      } else if (MODE == 2) {  // MUFU + F2FP (the softmax mix: 1 pack per 2 exps)
        const float a = ex2(v[i]), b = ex2(v[i + 1]);
        const uint32_t r = f2fp(a, b);
        v[i] = __uint_as_float(r);
        v[i + 1] = b;
      } else if (MODE == 3) {  // FRND only
        v[i] = floorf(v[i]) + 0.5f;
        v[i + 1] = floorf(v[i + 1]) + 0.5f;
      } else if (MODE == 4) {  // FMA-pipe exp2
        v[i] = ex2_fma(v[i]);
        v[i + 1] = ex2_fma(v[i + 1]);
      } else if (MODE == 5) {  // 3 MUFU : 1 poly, + F2FP
        const float a = (i & 6) == 6 ? ex2_fma(v[i]) : ex2(v[i]);
        const float b = ex2(v[i + 1]);
        v[i] = __uint_as_float(f2fp(a, b));
        v[i + 1] = b;
      } else if (MODE == 6) {  // MUFU + int rounding pack (round half up: +0x8000, PRMT)
        const float a = ex2(v[i]), b = ex2(v[i + 1]);
        const uint32_t r = __byte_perm(__float_as_uint(a) + 0x8000u, __float_as_uint(b) + 0x8000u, 0x7632);
        v[i] = __uint_as_float(r);
        v[i + 1] = b;
      } else if (MODE == 8) {  // MUFU f16x2: 2 exps per lane per instruction
        v[i] = __uint_as_float(ex2_h2(__float_as_uint(v[i])));
      } else if (MODE == 9) {  // MUFU bf16x2
        v[i] = __uint_as_float(ex2_bf2(__float_as_uint(v[i])));
      } else if (MODE == 7) {  // FFMA + FADD per element (the scale and the row sum)
        v[i] = fmaf(v[i], 1.0001f, -0.5f);
        v[i + 1] = v[i + 1] + v[i];
      }
    }
    u += __float_as_uint(v[0]) ^ it;
  }
  const long long t1 = clock64();
  float acc = 0.f;
  for (int i = 0; i < 32; ++i) acc += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + u;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 512 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 4000;
  const char* names[] = {"MUFU.EX2", "F2FP pack", "MUFU + F2FP", "FRND", "ex2 FMA-pipe", "3 MUFU:1 poly + F2FP",
                         "MUFU + int pack", "FFMA + FADD", "MUFU f16x2 (2/lane)", "MUFU bf16x2 (2/lane)"};
  for (int warps : {4, 8, 16}) {
    for (int mode = 0; mode < 10; ++mode) {
      long long h = 0;
      for (int rep = 0; rep < 2; ++rep) {
        switch (mode) {
          case 0: pipes<0><<<148, warps * 32>>>(out, cyc, iters); break;
          case 1: pipes<1><<<148, warps * 32>>>(out, cyc, iters); break;
          case 2: pipes<2><<<148, warps * 32>>>(out, cyc, iters); break;
          case 3: pipes<3><<<148, warps * 32>>>(out, cyc, iters); break;
          case 4: pipes<4><<<148, warps * 32>>>(out, cyc, iters); break;
          case 5: pipes<5><<<148, warps * 32>>>(out, cyc, iters); break;
          case 6: pipes<6><<<148, warps * 32>>>(out, cyc, iters); break;
          case 7: pipes<7><<<148, warps * 32>>>(out, cyc, iters); break;
          case 8: pipes<8><<<148, warps * 32>>>(out, cyc, iters); break;
          case 9: pipes<9><<<148, warps * 32>>>(out, cyc, iters); break;
        }
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      }
      const double elems = double(iters) * 32 * warps * 32;  // elements (value slots) per SM
      printf("warps/SM %2d  %-22s %6.2f elements/clk/SM  (%5.0f clk per 16384)\n", warps, names[mode],
             elems / double(h), 16384.0 * double(h) / elems);
    }
  }
  return 0;
}
