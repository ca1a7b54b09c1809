// Micro-benchmark of the forward softmax exp pass in isolation (registers only): x = s*c - m,
// e = 2^x (MUFU), row-sum, bf16x2 pack — for COLS score columns per thread, W warps per SM.
// Reports SM clocks per 128x128 tile (16384 elements); the MUFU floor is 1024.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I. -o tools/ubench_softmax_bin tools/ubench_softmax.cu
#include <cstdint>
#include <cstdio>

#include "paper_2509_19836_b200/csrc/bb_ptx.cuh"

using namespace bb;


template <int COLS, int MODE>
__global__ void __launch_bounds__(COLS == 128 ? 256 : 512, 1) sm_bench(float* out, long long* cyc, int iters, float sl2) {
  float s[COLS];
  for (int i = 0; i < COLS; ++i) s[i] = -0.01f * ((threadIdx.x * 7 + i * 13) % 97);
  float l_run = 0.f;
  uint32_t sink = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const float neg_m = -0.5f - 1e-7f * it;
    float acc8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    uint32_t pk[COLS / 2];
    if (MODE >= 2) {  // packed fp32x2: FFMA2 for the scale, FADD2 for the row sums
      float2 a4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      const float2 c2 = make_float2(sl2, sl2), m2 = make_float2(neg_m, neg_m);
#pragma unroll
      for (int c = 0; c < COLS; c += 8) {
        float2 e[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 x = __ffma2_rn(make_float2(s[c + 2 * i], s[c + 2 * i + 1]), c2, m2);
          if (MODE == 3 && i == 3) {
            e[i] = ex2_poly2(x);
          } else {
            e[i] = make_float2(ex2_approx(x.x), ex2_approx(x.y));
          }
          a4[i] = __fadd2_rn(a4[i], e[i]);
          pk[c / 2 + i] = pack_bf16(e[i].x, e[i].y);
        }
      }
      acc8[0] = a4[0].x + a4[0].y;
      acc8[1] = a4[1].x + a4[1].y;
      acc8[2] = a4[2].x + a4[2].y;
      acc8[3] = a4[3].x + a4[3].y;
    } else
#pragma unroll
    for (int c = 0; c < COLS; c += 8) {
      float e[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float x = fmaf(s[c + i], sl2, neg_m);
        e[i] = (MODE == 1 && (i & 3) == 3) ? ex2_poly(x) : ex2_approx(x);
        acc8[i] += e[i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) pk[c / 2 + i] = pack_bf16(e[2 * i], e[2 * i + 1]);
    }
    l_run += ((acc8[0] + acc8[1]) + (acc8[2] + acc8[3])) + ((acc8[4] + acc8[5]) + (acc8[6] + acc8[7]));
#pragma unroll
    for (int i = 0; i < COLS / 2; ++i) sink ^= pk[i];
    s[0] += 1e-9f * __uint_as_float(sink & 0x3f800000u);  // keep the loop from being hoisted
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = l_run + sink;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int COLS, int MODE>
void run(int warps, float* out, long long* cyc) {
  const int iters = 2000;
  long long h = 0;
  for (int rep = 0; rep < 2; ++rep) {
    sm_bench<COLS, MODE><<<148, warps * 32>>>(out, cyc, iters, 0.127f);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  }
  const double elems = double(iters) * COLS * warps * 32;
  const char* names[] = {"MUFU", "3:1 poly", "x2 MUFU", "x2 3:1 poly"};
  printf("COLS %3d  warps/SM %2d  %-12s %6.0f clk per 16384 elements\n", COLS, warps, names[MODE],
         16384.0 * double(h) / elems);
}


// The forward softmax body as in attn_fwd_kernel, on a fake S tile resident in TMEM:
// tcgen05.ld of the 128-column row, 3-input-max tree, exp pass (x2 packed), tcgen05.st of P.
template <int MODE>
__global__ void __launch_bounds__(384, 1) sm_tmem_bench(float* out, long long* cyc, int iters, float sl2, int nwarps) {
  __shared__ uint32_t slot;
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t quad = warp & 3;
  const uint32_t t_lane = (quad * 32) << 16;
  const uint32_t sbuf = ((warp >> 2) & 1) * 128;
  {  // fill S with something finite
    float v[32];
    for (int i = 0; i < 32; ++i) v[i] = -0.01f * ((lane * 7 + i * 13) % 97);
    for (int c = 0; c < 4; ++c) tmem_st32(tmem + t_lane + sbuf + c * 32, v);
    tmem_st_wait();
  }
  __syncthreads();
  float l_run = 0.f;
  const long long t0 = clock64();
  if (warp < nwarps) {
    for (int it = 0; it < iters; ++it) {
      float s[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(tmem + t_lane + sbuf + c * 32, *reinterpret_cast<float(*)[32]>(&s[c * 32]));
      tmem_ld_wait();
      float mx8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mx8[i] = fmax3(s[i], s[i + 8], s[i + 16]);
#pragma unroll
      for (int c = 24; c < 120; c += 16)
#pragma unroll
        for (int i = 0; i < 8; ++i) mx8[i] = fmax3(mx8[i], s[c + i], s[c + 8 + i]);
#pragma unroll
      for (int i = 0; i < 8; ++i) mx8[i] = fmaxf(mx8[i], s[120 + i]);
      const float mx = fmax3(fmax3(mx8[0], mx8[1], mx8[2]), fmax3(mx8[3], mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]));
      const float neg_m = -mx * sl2;
      float2 acc4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      const float2 c2 = make_float2(sl2, sl2), m2 = make_float2(neg_m, neg_m);
#pragma unroll
      for (int c = 0; c < 128; c += 32) {
        uint32_t pk[16];
#pragma unroll
        for (int h = 0; h < 32; h += 8)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 x = __ffma2_rn(make_float2(s[c + h + 2 * i], s[c + h + 2 * i + 1]), c2, m2);
            const float2 e = (MODE == 1 && i == 3) ? ex2_poly2(x) : make_float2(ex2_approx(x.x), ex2_approx(x.y));
            acc4[i] = __fadd2_rn(acc4[i], e);
            pk[h / 2 + i] = pack_bf16(e.x, e.y);
          }
        if (MODE != 2) tmem_st16(tmem + t_lane + sbuf + 64 + c / 2, pk);  // P into the upper half
        else l_run += __uint_as_float(pk[it & 15] & 0x3f000000u);
      }
      l_run += (acc4[0].x + acc4[0].y) + (acc4[1].x + acc4[1].y) + (acc4[2].x + acc4[2].y) + (acc4[3].x + acc4[3].y);
      tmem_st_wait();
    }
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = l_run;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int MODE>
void run_tmem(int warps, float* out, long long* cyc) {
  const int iters = 1000;
  long long h = 0;
  for (int rep = 0; rep < 2; ++rep) {
    sm_tmem_bench<MODE><<<148, 384>>>(out, cyc, iters, 0.127f, warps);
    cudaError_t e = cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return; }
  }
  const double elems = double(iters) * 128 * warps * 32;
  const char* names[] = {"tmem x2 MUFU", "tmem x2 3:1 poly", "tmem no STTM"};
  printf("TMEM-resident softmax  warps %2d  %-18s %6.0f clk per 16384 elements\n", warps, names[MODE], 16384.0 * double(h) / elems);
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 512 * 4);
  cudaMalloc(&cyc, 148 * 8);
  for (int w : {4, 8, 16}) {
    if (w <= 8) run<128, 0>(w, out, cyc);
    run<64, 0>(w, out, cyc);
    if (w <= 8) run<128, 1>(w, out, cyc);
    run<64, 1>(w, out, cyc);
    if (w <= 8) run<128, 2>(w, out, cyc);
    run<64, 2>(w, out, cyc);
    if (w <= 8) run<128, 3>(w, out, cyc);
    run<64, 3>(w, out, cyc);
  }
  for (int w : {4, 8}) {
    run_tmem<0>(w, out, cyc);
    run_tmem<1>(w, out, cyc);
    run_tmem<2>(w, out, cyc);
  }
  return 0;
}
