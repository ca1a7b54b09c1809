// Micro-benchmark: tcgen05.mma issue cost and queueing on sm_100a.  One thread issues groups of
// 8 SS MMAs (M=128, N=128, K=16 bf16 -> 128x128x128 per group, the attention tile) and records
// clock64 after each group's issue and after each group's commit barrier completes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I. -o tools/ubench_mma_bin tools/ubench_mma.cu
#include <cstdint>
#include <cstdio>

#include "paper_2509_19836_b200/csrc/bb_ptx.cuh"

using namespace bb;

constexpr int GROUPS = 16;

__global__ void __launch_bounds__(128, 1) mma_bench(long long* out, int n_ts, int sts_load, int n256) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[GROUPS];
  __shared__ uint32_t slot;
  const uint32_t warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 65536 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    for (int g = 0; g < GROUPS; ++g) mbar_init(&bars[g], 1);
    fence_barrier_init();
  }
  fence_async_smem();
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  long long t_issue[GROUPS], t_done[GROUPS];
  __shared__ volatile int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if (warp >= 1 && sts_load) {  // smem store traffic (16 B/lane) into a separate 32 KB region
    uint4* dst = reinterpret_cast<uint4*>(smem + 98304);
    uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
    int i = 0;
    while (!stop) {
#pragma unroll
      for (int u = 0; u < 16; ++u) dst[((i + u) * 96 + threadIdx.x - 32) & 2047] = v;
      i += 16;
    }
  }
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_bf16(128, 128, false, false);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    const long long t0 = clock64();
    for (int g = 0; g < GROUPS; ++g) {
      const uint32_t d = tmem + (n256 ? (g & 1) * 256 : (g & 3) * 128);
      if (n256) {
        constexpr uint32_t idesc256 = idesc_bf16(128, 256, false, false);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          umma_ss(d, sw128_desc(a + ks * 32, 16, 1024), sw128_desc(b + ks * 32, 16, 1024), idesc256, ks > 0);
      } else if (g < n_ts) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          umma_ts(d, tmem + 256 + ks * 8 + 0 * (g & 1), sw128_desc(b + (ks >> 2) * 16384 + (ks & 3) * 32, 16, 1024),
                  idesc, ks > 0);
      } else {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const uint32_t off = (ks >> 2) * 16384 + (ks & 3) * 32;
          umma_ss(d, sw128_desc(a + off, 16, 1024), sw128_desc(b + off, 16, 1024), idesc, ks > 0);
        }
      }
      umma_commit(&bars[g]);
      t_issue[g] = clock64() - t0;
    }
    for (int g = 0; g < GROUPS; ++g) {
      mbar_wait(&bars[g], 0);
      t_done[g] = clock64() - t0;
    }
    for (int g = 0; g < GROUPS; ++g) {
      out[blockIdx.x * 2 * GROUPS + g] = t_issue[g];
      out[blockIdx.x * 2 * GROUPS + GROUPS + g] = t_done[g];
    }
    stop = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
  long long* out;
  cudaMalloc(&out, 148 * 2 * GROUPS * 8);
  cudaFuncSetAttribute(mma_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 65536);
  struct Cfg { int n_ts, sts, n256; const char* name; };
  const Cfg cfgs[] = {{0, 0, 0, "SS N=128"}, {GROUPS, 0, 0, "TS N=128"}, {0, 1, 0, "SS N=128 + STS load"},
                      {GROUPS, 1, 0, "TS N=128 + STS load"}, {0, 0, 1, "SS N=256 (4 k-steps/group)"},
                      {0, 1, 1, "SS N=256 + STS load"}};
  for (const Cfg& cf : cfgs) {
    const int n_ts = cf.n_ts;
    for (int rep = 0; rep < 2; ++rep) mma_bench<<<148, 128, 65536 + 65536>>>(out, cf.n_ts, cf.sts, cf.n256);
    long long h[2 * GROUPS];
    cudaError_t e = cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      return 1;
    }
    (void)n_ts;
    printf("%s\n  issued:", cf.name);
    for (int g = 0; g < GROUPS; ++g) printf(" %lld", h[g]);
    printf("\n  done:  ");
    for (int g = 0; g < GROUPS; ++g) printf(" %lld", h[GROUPS + g]);
    printf("\n  per group (steady): %.0f clk\n", double(h[2 * GROUPS - 1] - h[GROUPS + 3]) / (GROUPS - 4));
  }
  return 0;
}
