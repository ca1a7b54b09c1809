// Throughput of the backward kernel's dQ drain path: TMA bulk tensor reduce-add (fp32) of
// 128-row x 32-column boxes from shared memory into global memory, per SM, with every SM
// busy.  Variants: each CTA adds into its own L2-resident rows; all CTAs add into the same
// rows (the contention the K/V-stationary backward creates); rows spread over 2 GB (HBM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I. -o tools/ubench_reduce_bin tools/ubench_reduce.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>

#include "paper_2509_19836_b200/csrc/bb_ptx.cuh"

using namespace bb;

// mode 0: own rows (L2), 1: shared rows, 2: spread over the whole buffer (HBM)
template <int INFLIGHT>
__global__ void __launch_bounds__(128, 1) red_kernel(const __grid_constant__ CUtensorMap map, long long* out,
                                                     int iters, int mode, int rows_total) {
  extern __shared__ __align__(1024) uint8_t smem[];
  for (int i = threadIdx.x; i < 65536 / 4; i += 128) reinterpret_cast<float*>(smem)[i] = 1.0f;
  fence_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      int row;
      if (mode == 0)
        row = (blockIdx.x * 4 + (i & 3)) * 128;
      else if (mode == 1)
        row = (i & 15) * 128;
      else
        row = ((blockIdx.x * 977 + i * 131) % (rows_total / 128)) * 128;
      const int slot = i & 3;  // 4 x 16 KB staging slots
      tma_reduce_add_2d(&map, smem + slot * 16384, 0, row);
      tma_reduce_add_2d(&map, smem + slot * 16384, 32, row);  // same data, next 32 columns
      bulk_commit();
      bulk_wait_read<INFLIGHT>();
    }
    bulk_wait<0>();
    out[blockIdx.x] = clock64() - t0;
  }
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q{};
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  const int cols = 128;                       // fp32 per row (one head's dQ row)
  const int rows = (1 << 30) / (cols * 4);    // 1 GB
  float* buf;
  cudaMalloc(&buf, size_t(rows) * cols * 4);
  cudaMemset(buf, 0, size_t(rows) * cols * 4);
  CUtensorMap map;
  cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(cols) * 4};
  cuuint32_t box[2] = {32, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d (enc %p)\n", int(cr), (void*)enc);
  long long* out;
  cudaMalloc(&out, 148 * 8);
  const int iters = 2000;
  const char* names[3] = {"own rows (L2)", "shared rows", "spread (HBM)"};
  for (int grid : {1, 148}) {
    for (int mode = 0; mode < 3; ++mode) {
      for (int infl : {0, 1, 3}) {
        auto k = infl == 0 ? red_kernel<0> : infl == 1 ? red_kernel<1> : red_kernel<3>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        k<<<grid, 128, 65536>>>(map, out, 20, mode, rows);
        cudaError_t e0 = cudaDeviceSynchronize();
        if (e0 != cudaSuccess) { printf("warmup: %s\n", cudaGetErrorString(e0)); return 1; }
        cudaEventRecord(a);
        k<<<grid, 128, 65536>>>(map, out, iters, mode, rows);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        long long h[148];
        cudaMemcpy(h, out, grid * 8, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
        const double bytes = double(grid) * iters * 32768;
        printf("grid %3d %-14s in-flight %d: %6.1f B/clk/SM  chip %7.1f GB/s\n", grid, names[mode], infl + 1,
               double(iters) * 32768 / double(mx), bytes / (ms * 1e-3) / 1e9);
      }
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
