// tcgen05.mma issue/execution rate vs N (M=128, K=16 per instruction, bf16 SS and TS):
// one thread issues NI instructions back to back, one commit at the end; clock64 from the
// first issue to the commit's mbarrier completing.  Reports cycles per instruction next to
// the nominal 128*N/256 (8192 flop/clk/SM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I. -o tools/ubench_mma_rate_bin tools/ubench_mma_rate.cu
#include <cstdint>
#include <cstdio>

#include "paper_2509_19836_b200/csrc/bb_ptx.cuh"

using namespace bb;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) rate(long long* out, int ni) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const uint32_t warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 98304 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  fence_async_smem();
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_bf16(128, N, false, false);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 16384);
    const long long t0 = clock64();
    for (int i = 0; i < ni; i += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t off = ((i + u) & 3) * 32;
        if (TS)
          umma_ts(tmem + 256, tmem + ((i + u) & 7) * 8, sw128_desc(b + off, 16, 1024), idesc, 1);
        else
          umma_ss(tmem, sw128_desc(a + off, 16, 1024), sw128_desc(b + off, 16, 1024), idesc, 1);
      }
    }
    const long long t1 = clock64();
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t2 = clock64();
    out[blockIdx.x * 2] = t1 - t0;
    out[blockIdx.x * 2 + 1] = t2 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int N, bool TS>
void run(long long* out) {
  const int ni = 256;
  cudaFuncSetAttribute(rate<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304);
  long long h[2] = {0, 0};
  for (int rep = 0; rep < 3; ++rep) {
    rate<N, TS><<<148, 128, 98304>>>(out, ni);
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
  }
  printf("M=128 N=%3d %s: %6.1f clk/instr to issue, %6.1f clk/instr to complete (nominal %d)\n", N, TS ? "TS" : "SS",
         double(h[0]) / ni, double(h[1]) / ni, 128 * N / 256);
}

int main() {
  long long* out;
  cudaMalloc(&out, 148 * 16);
  run<64, false>(out);
  run<128, false>(out);
  run<256, false>(out);
  run<64, true>(out);
  run<128, true>(out);
  run<256, true>(out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
