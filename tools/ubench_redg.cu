// red.global.add.v4.f32 throughput per SM (all 148 SMs busy) for the access patterns a dQ
// drain can produce from tcgen05.ld fragments, against the L2-resident dQ rows of a tile.
//   pattern 0: each lane owns a row (lane stride 512 B), 16 B per lane per instruction
//   pattern 1: a warp instruction covers 512 contiguous bytes of one row
//   pattern 2: lane pairs cover one 32 B sector, 16 rows per instruction
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_redg_bin tools/ubench_redg.cu
#include <cstdio>
#include <cstdint>

template <int PAT>
__global__ void redk(float* buf, long long* out, int iters, int nwarps) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (warp >= nwarps) return;
  float* tile = buf + size_t(blockIdx.x) * 128 * 128;  // one 64 KB dQ tile per CTA
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const int c = (i * nwarps + warp);  // instruction index within the tile sweep
    float* a;
    if (PAT == 0) {
      const int row = (c / 32) * 32 % 128 + lane;
      a = tile + row * 128 + (c % 32) * 4;
    } else if (PAT == 1) {
      const int row = c % 128;
      a = tile + row * 128 + lane * 4;
    } else {
      const int row = (c % 8) * 16 + lane / 2;
      a = tile + row * 128 + ((c / 8) % 16) * 8 + (lane & 1) * 4;
    }
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(a), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f)
                 : "memory");
  }
  __syncwarp();
  if (lane == 0 && warp == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
  float* buf;
  cudaMalloc(&buf, size_t(148) * 128 * 128 * 4);
  cudaMemset(buf, 0, size_t(148) * 128 * 128 * 4);
  long long* out;
  cudaMalloc(&out, 148 * 8);
  for (int nw : {4, 8}) {
    for (int pat = 0; pat < 3; ++pat) {
      auto k = pat == 0 ? redk<0> : pat == 1 ? redk<1> : redk<2>;
      const int iters = 4096;
      k<<<148, 256>>>(buf, out, 64, nw);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      k<<<148, 256>>>(buf, out, iters, nw);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      long long h[148];
      cudaMemcpy(h, out, 148 * 8, cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      const double bytes = double(iters) * nw * 512;
      printf("warps %d pattern %d: %6.1f B/clk/SM, chip %7.1f GB/s\n", nw, pat, bytes / mx, 148 * bytes / (ms * 1e-3) / 1e9);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
