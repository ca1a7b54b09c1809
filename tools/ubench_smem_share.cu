// Does tcgen05.mma operand fetch share the SM's shared-memory bandwidth with STS / LDS /
// bulk-copy (TMA) traffic?  One thread issues NI M=128 x N x K=16 bf16 MMAs back to back
// (SS or TS, optionally cta_group::2) while 8 other warps stream STS.128 / LDS.128 or one
// warp streams 16 KB bulk copies into shared memory.  Reports MMA cycles per instruction and
// the side traffic's bytes per clock, alone and together.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I. -o tools/ubench_smem_share_bin tools/ubench_smem_share.cu
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>

#include "paper_2509_19836_b200/csrc/bb_ptx.cuh"

using namespace bb;

enum Side { NONE = 0, STS = 1, LDS = 2, BULK = 3, TRED = 4, REDG = 5, TMLD = 6, LDSB = 7 };

constexpr int OPS = 65536;       // A/B operand region
constexpr int SIDE = 65536;      // side-traffic region
constexpr int SMEM = OPS + SIDE;

template <int N, bool TS, int SIDE_KIND, bool MMA>
__global__ void __launch_bounds__(384, 1) kern(long long* out, const uint4* gsrc, int ni, int nside,
                                               const __grid_constant__ CUtensorMap rmap, float* gred) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bbar;
  __shared__ uint32_t slot;
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < SMEM / 4; i += 384) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bbar, 1);
    fence_barrier_init();
  }
  fence_async_smem();
  if (warp == 2) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  long long* o = out + blockIdx.x * 4;
  if (warp == 0 && lane == 0 && MMA) {
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
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t2 = clock64();
    o[0] = t2 - t0;
  }
  if (SIDE_KIND == STS && warp >= 4) {
    const long long t0 = clock64();
    uint8_t* base = smem + OPS;
    const uint32_t t = threadIdx.x - 128;
    const uint4 v = make_uint4(t, t + 1, t + 2, t + 3);
    for (int i = 0; i < nside; ++i) {
      asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(smem_u32(base + ((t * 16 + i * 4096) & (SIDE - 1)))),
                   "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
    }
    __syncwarp();
    const long long t1 = clock64();
    if (threadIdx.x == 128) o[1] = t1 - t0;
  }
  if (SIDE_KIND == LDS && warp >= 4) {
    const long long t0 = clock64();
    const uint8_t* base = smem + OPS;
    const uint32_t t = threadIdx.x - 128;
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (int i = 0; i < nside; ++i) {
      uint4 x;
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w)
                   : "r"(smem_u32(base + ((t * 16 + i * 4096) & (SIDE - 1)))) : "memory");
      acc.x ^= x.x;
      acc.y += x.y;
      acc.z ^= x.z;
      acc.w += x.w;
    }
    __syncwarp();
    const long long t1 = clock64();
    if (threadIdx.x == 128) o[1] = t1 - t0;
    if (acc.x == 0x12345 && acc.y == 7) o[3] = acc.z + acc.w;
  }
  if (SIDE_KIND == BULK && warp == 1 && lane == 0) {
    // nside bulk copies of 16 KB each, 4 in flight (64 KB region), L2-resident source
    const long long t0 = clock64();
    uint8_t* base = smem + OPS;
    for (int i = 0; i < nside; i += 4) {
      mbar_expect_tx(&bbar, 4 * 16384);
      for (int u = 0; u < 4; ++u) bulk_load(base + u * 16384, gsrc + (((i + u) & 15) * 1024), 16384, &bbar);
      mbar_wait(&bbar, (i / 4) & 1);
    }
    const long long t1 = clock64();
    o[1] = t1 - t0;
  }
  if (SIDE_KIND == TRED && warp == 1 && lane == 0) {
    // TMA bulk reduce-add of 16 KB [128 x 32 fp32] boxes from shared memory, 2 in flight
    const long long t0 = clock64();
    for (int i = 0; i < nside; ++i) {
      tma_reduce_add_2d(&rmap, smem + OPS + (i & 1) * 16384, (i & 3) * 32, blockIdx.x * 128);
      bulk_commit();
      bulk_wait_read<1>();
    }
    bulk_wait<0>();
    o[1] = clock64() - t0;
  }
  if (SIDE_KIND == REDG && warp >= 4) {
    // red.global.add.v4.f32 straight from registers: each thread owns one 512 B row
    const long long t0 = clock64();
    const uint32_t t = threadIdx.x - 128;
    float* row = gred + (size_t(blockIdx.x) * 256 + t) * 128;
    for (int i = 0; i < nside; ++i) {
      float* a = row + (i & 31) * 4;
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(a), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f)
                   : "memory");
    }
    __syncwarp();
    const long long t1 = clock64();
    if (threadIdx.x == 128) o[1] = t1 - t0;
  }
  if (SIDE_KIND == TMLD && warp >= 4) {
    const long long t0 = clock64();
    const uint32_t q = warp & 3;
    float acc = 0.f;
    for (int i = 0; i < nside; ++i) {
      float v[32];
      tmem_ld32(tmem + ((q * 32) << 16) + 384 + (i & 3) * 32, v);
      tmem_ld_wait();
      acc += v[0] + v[31];
    }
    __syncwarp();
    const long long t1 = clock64();
    if (threadIdx.x == 128) o[1] = t1 - t0;
    if (acc == 12345.f) o[3] = 1;
  }
  if (SIDE_KIND == LDSB && warp >= 4) {
    const long long t0 = clock64();
    const uint8_t* base = smem + OPS;
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (int i = 0; i < nside; ++i) {
      uint4 x;
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w)
                   : "r"(smem_u32(base + ((i * 16) & (SIDE - 1)))) : "memory");
      acc.x ^= x.x;
      acc.y += x.y;
    }
    __syncwarp();
    const long long t1 = clock64();
    if (threadIdx.x == 128) o[1] = t1 - t0;
    if (acc.x == 0x12345 && acc.y == 7) o[3] = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

CUtensorMap g_rmap;
float* g_red;
template <int N, bool TS, int SK, bool MMA>
void run(const char* name, long long* out, const uint4* g, int ni, int nside) {
  auto k = kern<N, TS, SK, MMA>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  long long h[4] = {0, 0, 0, 0};
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(out, 0, 148 * 32);
    k<<<148, 384, SMEM>>>(out, g, ni, nside, g_rmap, g_red);
    cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
  }
  double side_bytes = SK == STS || SK == LDS || SK == REDG || SK == LDSB ? 256.0 * 16 * nside : SK == BULK || SK == TRED ? 16384.0 * nside : SK == TMLD ? 256.0 * 128 * nside : 0;
  printf("%-34s mma %7.1f clk/instr (nominal %3d)   side %7.1f B/clk (%lld clk)\n", name,
         MMA ? double(h[0]) / ni : 0.0, 128 * N / 256, h[1] ? side_bytes / double(h[1]) : 0.0, h[1]);
}

int main() {
  long long* out;
  uint4* g;
  cudaMalloc(&out, 148 * 32);
  cudaMalloc(&g, 16 * 16384);
  cudaMemset(g, 0, 16 * 16384);
  const int ni = 2048;
  {
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q{};
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
    float* buf;
    const int rows = 148 * 128;
    cudaMalloc(&buf, size_t(rows) * 128 * 4);
    cudaMemset(buf, 0, size_t(rows) * 128 * 4);
    cuuint64_t dims[2] = {128, cuuint64_t(rows)};
    cuuint64_t strides[1] = {512};
    cuuint32_t box[2] = {32, 128};
    cuuint32_t es[2] = {1, 1};
    enc(&g_rmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaMalloc(&g_red, size_t(148) * 256 * 128 * 4);
    cudaMemset(g_red, 0, size_t(148) * 256 * 128 * 4);
  }
  // side traffic sized to last about as long as the MMA stream
  run<128, false, NONE, true>("SS N=128 alone", out, g, ni, 0);
  run<128, false, STS, false>("STS alone", out, g, ni, 4096);
  run<128, false, STS, true>("SS N=128 + STS", out, g, ni, 4096);
  run<128, false, LDS, false>("LDS alone", out, g, ni, 4096);
  run<128, false, LDS, true>("SS N=128 + LDS", out, g, ni, 4096);
  run<128, false, BULK, false>("bulk alone", out, g, ni, 1024);
  run<128, false, BULK, true>("SS N=128 + bulk", out, g, ni, 1024);
  run<128, true, NONE, true>("TS N=128 alone", out, g, ni, 0);
  run<128, true, STS, true>("TS N=128 + STS", out, g, ni, 4096);
  run<128, true, BULK, true>("TS N=128 + bulk", out, g, ni, 1024);
  run<256, false, NONE, true>("SS N=256 alone", out, g, ni / 2, 0);
  run<256, false, STS, true>("SS N=256 + STS", out, g, ni / 2, 4096);
  run<256, false, BULK, true>("SS N=256 + bulk", out, g, ni / 2, 1024);
  run<128, false, TRED, false>("TMA reduce alone", out, g, ni, 256);
  run<128, false, TRED, true>("SS N=128 + TMA reduce", out, g, ni, 256);
  run<128, false, REDG, false>("red.global.v4 alone", out, g, ni, 1024);
  run<128, false, REDG, true>("SS N=128 + red.global.v4", out, g, ni, 1024);
  run<128, false, TMLD, false>("tcgen05.ld alone", out, g, ni, 2048);
  run<128, false, TMLD, true>("SS N=128 + tcgen05.ld", out, g, ni, 2048);
  run<128, false, LDSB, false>("LDS broadcast alone", out, g, ni, 4096);
  run<128, false, LDSB, true>("SS N=128 + LDS broadcast", out, g, ni, 4096);
  run<64, false, NONE, true>("SS N=64 alone", out, g, ni * 2, 0);
  run<64, false, STS, true>("SS N=64 + STS", out, g, ni * 2, 4096);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
