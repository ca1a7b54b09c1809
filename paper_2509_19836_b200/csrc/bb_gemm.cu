// Warp-specialised tcgen05 GEMM for the fused LM head (lmhead.py:76-91).
//
//   C[M,N] (+)= A[M,K] * B[N,K]^T,  bf16 operands, fp32 accumulation in TMEM.
//
// Tile 128 x 256 x 64, 4-stage TMA -> smem ring, one elected thread issues
// tcgen05.mma (M=128, N=256, K=16 per instruction), four epilogue warps drain
// TMEM with tcgen05.ld.  Persistent (one CTA per SM) with the accumulator
// double-buffered in TMEM, so each tile's epilogue overlaps the next main loop.  Operands may be K-major or MN-major (SWIZZLE_128B
// either way), which lets the three LM-head contractions run without any
// transposed copies:
//   logits = H  . W^T   (A=H  K-major,  B=W K-major)   lmhead.py:78
//   dH     = G  . W     (A=G  K-major,  B=W MN-major)  lmhead.py:90
//   dW    += G^T. H     (A=G  MN-major, B=H MN-major)  lmhead.py:91
// The LOGITS epilogue also emits per-(row, vocab tile) (max, sum exp) partials
// and the target logit, i.e. the streaming LSE of lmhead.py:79-81.
#include <cuda_runtime.h>

#include "bb_host.h"
#include "bb_ptx.cuh"

namespace bb {
namespace {

#ifndef BB_GEMM_PAIR
#define BB_GEMM_PAIR 1
#endif
constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr uint32_t A_BYTES = BM * BK * 2;  // 16 KB
constexpr uint32_t B_BYTES = BN * BK * 2;  // 32 KB
constexpr uint32_t SMEM_BYTES = STAGES * (A_BYTES + B_BYTES) + 1024 /*align*/ + 256;
constexpr int THREADS = 256;

struct GemmArgs {
  int64_t m, n, k, ldc;
  float* c;
  __nv_bfloat16* c16;       // GEMM_BF16: bf16 output, row grow written to row row_map[grow]
  const int64_t* row_map;   // (identity when null)
  LogitsEpilogue le;
  int tiles_m, tiles_n;
  bool raster_m_fast;
  bool pair;  // CTA-pair kernel (cta_group::2, 256 x 256 tiles)
};

// Persistent: one CTA per SM walks tiles blockIdx.x, +gridDim.x, ...; the accumulator is
// double-buffered in TMEM (2 x 256 columns) so tile i+1's main loop runs while the epilogue
// warps drain tile i.
template <bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                const GemmArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;  // [2]
  uint64_t* acc_empty = acc_full + 2;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int n_tiles = p.tiles_m * p.tiles_n;
  const int num_k = static_cast<int>((p.k + BK - 1) / BK);
  const uint32_t warp = warp_id(), lane = lane_id();
  auto tile_mn = [&](int tile, int& m0, int& n0, int& tn) {
    const int tm = p.raster_m_fast ? tile % p.tiles_m : tile / p.tiles_n;
    tn = p.raster_m_fast ? tile / p.tiles_m : tile % p.tiles_n;
    m0 = tm * BM;
    n0 = tn * BN;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tma_a);
    tma_prefetch(&tma_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 128);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (elect_one()) {
      uint32_t kc = 0;  // k-blocks issued so far (ring position)
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        int m0, n0, tn;
        tile_mn(tile, m0, n0, tn);
        for (int kb = 0; kb < num_k; ++kb, ++kc) {
          const int s = kc % STAGES;
          const uint32_t ph = (kc / STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], A_BYTES + B_BYTES);
          const int k0 = kb * BK;
          uint8_t* a_dst = sA + s * A_BYTES;
          uint8_t* b_dst = sB + s * B_BYTES;
          if (!A_MN) {
            tma_load_2d(a_dst, &tma_a, &full[s], k0, m0);
          } else {
            tma_load_2d(a_dst, &tma_a, &full[s], m0, k0);
            tma_load_2d(a_dst + 8192, &tma_a, &full[s], m0 + 64, k0);
          }
          if (!B_MN) {
            tma_load_2d(b_dst, &tma_b, &full[s], k0, n0);
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) tma_load_2d(b_dst + i * 8192, &tma_b, &full[s], n0 + 64 * i, k0);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t idesc = idesc_bf16(BM, BN, A_MN, B_MN);
    uint32_t kc = 0;
    int it = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
      const int buf = it & 1;
      mbar_wait(&acc_empty[buf], ((it >> 1) & 1) ^ 1);  // epilogue has drained this buffer
      tc_fence_after();
      const uint32_t acc = tmem + buf * BN;
      for (int kb = 0; kb < num_k; ++kb, ++kc) {
        const int s = kc % STAGES;
        const uint32_t ph = (kc / STAGES) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a_base = smem_u32(sA + s * A_BYTES);
          const uint32_t b_base = smem_u32(sB + s * B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ad = A_MN ? sw128_desc(a_base + kk * 2048, 8192, 1024)
                                     : sw128_desc(a_base + kk * 32, 16, 1024);
            const uint64_t bd = B_MN ? sw128_desc(b_base + kk * 2048, 8192, 1024)
                                     : sw128_desc(b_base + kk * 32, 16, 1024);
            umma_ss(acc, ad, bd, idesc, (kb | kk) != 0);
          }
          umma_commit(&empty[s]);
          if (kb == num_k - 1) umma_commit(&acc_full[buf]);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: TMEM -> registers -> global ----------------
    const uint32_t quad = warp & 3;
    const int row = quad * 32 + lane;
    int it = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
      int m0, n0, tn;
      tile_mn(tile, m0, n0, tn);
      const int buf = it & 1;
      const int64_t grow = m0 + row;
      mbar_wait(&acc_full[buf], (it >> 1) & 1);
      tc_fence_after();
      const bool row_ok = grow < p.m;
      float run_max = -INFINITY, run_sum = 0.f;
      int64_t tgt = -1;
      if (EPI == GEMM_LOGITS && row_ok) tgt = p.le.targets[grow] - n0;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        float v[32];
        tmem_ld32(tmem + ((quad * 32) << 16) + buf * BN + c * 32, v);
        tmem_ld_wait();
        if (c == BN / 32 - 1) {  // the whole accumulator is in registers: hand the buffer back
          tc_fence_before();
          mbar_arrive(&acc_empty[buf]);
        }
        const int64_t col0 = n0 + c * 32;
        if (!row_ok || col0 >= p.n) continue;
        if (EPI == GEMM_BF16) {  // cast + row permutation fused into the store
          __nv_bfloat16* d16 = p.c16 + (p.row_map ? p.row_map[grow] : grow) * p.ldc + col0;
          if (col0 + 32 <= p.n && (p.ldc % 8) == 0) {
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = pack_bf16(v[2 * i], v[2 * i + 1]);
#pragma unroll
            for (int i = 0; i < 4; ++i)
              reinterpret_cast<uint4*>(d16)[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
          } else {
            for (int i = 0; i < 32 && col0 + i < p.n; ++i) d16[i] = __float2bfloat16_rn(v[i]);
          }
          continue;
        }
        float* dst = p.c ? p.c + grow * p.ldc + col0 : nullptr;
        const bool full_chunk = col0 + 32 <= p.n;
        if (EPI == GEMM_LOGITS) {
          float cmax = -INFINITY;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (full_chunk || col0 + i < p.n) cmax = fmaxf(cmax, v[i]);
          const float nmax = fmaxf(run_max, cmax);
          float s = 0.f;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (full_chunk || col0 + i < p.n) s += __expf(v[i] - nmax);
          run_sum = run_sum * __expf(run_max - nmax) + s;
          run_max = nmax;
          const int64_t t = tgt - c * 32;
          if (t >= 0 && t < 32) {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (i == t) p.le.tgt_logit[grow] = v[i];
          }
        }
        if (dst) {
          if (full_chunk && (p.ldc % 4) == 0) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              float4* d4 = reinterpret_cast<float4*>(dst + i);
              if (EPI == GEMM_ACCUM) {
                float4 o = *d4;
                o.x += v[i];
                o.y += v[i + 1];
                o.z += v[i + 2];
                o.w += v[i + 3];
                *d4 = o;
              } else {
                *d4 = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
              }
            }
          } else {
            for (int i = 0; i < 32 && col0 + i < p.n; ++i) {
              if (EPI == GEMM_ACCUM)
                dst[i] += v[i];
              else
                dst[i] = v[i];
            }
          }
        }
      }
      if (EPI == GEMM_LOGITS && row_ok) {
        p.le.part_max[grow * p.tiles_n + tn] = run_max;
        p.le.part_sum[grow * p.tiles_n + tn] = run_sum;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}


// ---------------------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of two CTAs computes a 256 x 256 tile.  Each CTA
// loads its own 128 rows of A and half (128 rows) of the B tile, the leader issues
// M=256 x N=256 MMAs that read both CTAs' smem, and each CTA's TMEM holds its 128 rows of
// the accumulator.  Per SM this streams 32 KB per 512 MMA cycles instead of 48 KB, which is
// what the L2 can feed at full tensor rate (the single-CTA tile is L2-bound).
constexpr int STAGES2 = 6;
constexpr uint32_t B2_BYTES = 128 * BK * 2;  // this CTA's half of the B tile
constexpr uint32_t SMEM2_BYTES = STAGES2 * (A_BYTES + B2_BYTES) + 1024 + 256;

template <bool A_MN, bool B_MN, int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                 const GemmArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES2 * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES2 * B2_BYTES);
  uint64_t* empty = full + STAGES2;
  uint64_t* acc_full = empty + STAGES2;  // [2]
  uint64_t* acc_empty = acc_full + 2;    // [2] (leader: both CTAs' epilogues arrive)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  const int tiles_m2 = (p.tiles_m + 1) / 2;  // 256-row pair tiles
  const int n_tiles = tiles_m2 * p.tiles_n;
  const int num_k = static_cast<int>((p.k + BK - 1) / BK);
  const uint32_t warp = warp_id(), lane = lane_id();
  auto tile_mn = [&](int tile, int& m0, int& n0, int& tn) {
    const int tm = p.raster_m_fast ? tile % tiles_m2 : tile / p.tiles_n;
    tn = p.raster_m_fast ? tile / tiles_m2 : tile % p.tiles_n;
    m0 = tm * 2 * BM + static_cast<int>(rank) * BM;  // this CTA's 128 rows
    n0 = tn * BN;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tma_a);
    tma_prefetch(&tma_b);
    for (int s = 0; s < STAGES2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 256);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised, TMEM allocated in both
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs; bytes counted on the leader's full[s]) -------
    if (elect_one()) {
      uint32_t kc = 0;
      for (int tile = pair; tile < n_tiles; tile += n_pairs) {
        int m0, n0, tn;
        tile_mn(tile, m0, n0, tn);
        const int nb = n0 + static_cast<int>(rank) * 128;  // this CTA's half of the B tile
        for (int kb = 0; kb < num_k; ++kb, ++kc) {
          const int s = kc % STAGES2;
          const uint32_t ph = (kc / STAGES2) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          if (leader) mbar_expect_tx(&full[s], 2 * (A_BYTES + B2_BYTES));
          const uint32_t fb = mapa_smem(&full[s], 0);
          const int k0 = kb * BK;
          uint8_t* a_dst = sA + s * A_BYTES;
          uint8_t* b_dst = sB + s * B2_BYTES;
          if (!A_MN) {
            tma_load_2d_pair(a_dst, &tma_a, fb, k0, m0);
          } else {
            tma_load_2d_pair(a_dst, &tma_a, fb, m0, k0);
            tma_load_2d_pair(a_dst + 8192, &tma_a, fb, m0 + 64, k0);
          }
          if (!B_MN) {
            tma_load_2d_pair(b_dst, &tma_b, fb, k0, nb);
          } else {
            tma_load_2d_pair(b_dst, &tma_b, fb, nb, k0);
            tma_load_2d_pair(b_dst + 8192, &tma_b, fb, nb + 64, k0);
          }
        }
      }
    }
  } else if (warp == 1 && leader) {
    // ---------------- MMA issuer (leader only) ----------------
    constexpr uint32_t idesc = idesc_bf16(2 * BM, BN, A_MN, B_MN);
    uint32_t kc = 0;
    int it = 0;
    for (int tile = pair; tile < n_tiles; tile += n_pairs, ++it) {
      const int buf = it & 1;
      mbar_wait(&acc_empty[buf], ((it >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t acc = tmem + buf * BN;
      for (int kb = 0; kb < num_k; ++kb, ++kc) {
        const int s = kc % STAGES2;
        const uint32_t ph = (kc / STAGES2) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a_base = smem_u32(sA + s * A_BYTES);
          const uint32_t b_base = smem_u32(sB + s * B2_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ad = A_MN ? sw128_desc(a_base + kk * 2048, 8192, 1024)
                                     : sw128_desc(a_base + kk * 32, 16, 1024);
            const uint64_t bd = B_MN ? sw128_desc(b_base + kk * 2048, 8192, 1024)
                                     : sw128_desc(b_base + kk * 32, 16, 1024);
            umma_ss_pair(acc, ad, bd, idesc, (kb | kk) != 0);
          }
          umma_commit_pair(&empty[s]);
          if (kb == num_k - 1) umma_commit_pair(&acc_full[buf]);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (both CTAs, own 128 rows) ----------------
    const uint32_t quad = warp & 3;
    const int row = quad * 32 + lane;
    const uint32_t acc_empty_leader0 = mapa_smem(&acc_empty[0], 0);
    const uint32_t acc_empty_leader1 = mapa_smem(&acc_empty[1], 0);
    int it = 0;
    for (int tile = pair; tile < n_tiles; tile += n_pairs, ++it) {
      int m0, n0, tn;
      tile_mn(tile, m0, n0, tn);
      const int buf = it & 1;
      const int64_t grow = m0 + row;
      mbar_wait(&acc_full[buf], (it >> 1) & 1);
      tc_fence_after();
      const bool row_ok = grow < p.m;
      float run_max = -INFINITY, run_sum = 0.f;
      int64_t tgt = -1;
      if (EPI == GEMM_LOGITS && row_ok) tgt = p.le.targets[grow] - n0;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        float v[32];
        tmem_ld32(tmem + ((quad * 32) << 16) + buf * BN + c * 32, v);
        tmem_ld_wait();
        if (c == BN / 32 - 1) {
          tc_fence_before();
          mbar_arrive_cluster(buf ? acc_empty_leader1 : acc_empty_leader0);
        }
        const int64_t col0 = n0 + c * 32;
        if (!row_ok || col0 >= p.n) continue;
        if (EPI == GEMM_BF16) {  // cast + row permutation fused into the store
          __nv_bfloat16* d16 = p.c16 + (p.row_map ? p.row_map[grow] : grow) * p.ldc + col0;
          if (col0 + 32 <= p.n && (p.ldc % 8) == 0) {
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = pack_bf16(v[2 * i], v[2 * i + 1]);
#pragma unroll
            for (int i = 0; i < 4; ++i)
              reinterpret_cast<uint4*>(d16)[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
          } else {
            for (int i = 0; i < 32 && col0 + i < p.n; ++i) d16[i] = __float2bfloat16_rn(v[i]);
          }
          continue;
        }
        float* dst = p.c ? p.c + grow * p.ldc + col0 : nullptr;
        const bool full_chunk = col0 + 32 <= p.n;
        if (EPI == GEMM_LOGITS) {
          float cmax = -INFINITY;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (full_chunk || col0 + i < p.n) cmax = fmaxf(cmax, v[i]);
          const float nmax = fmaxf(run_max, cmax);
          float s = 0.f;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (full_chunk || col0 + i < p.n) s += __expf(v[i] - nmax);
          run_sum = run_sum * __expf(run_max - nmax) + s;
          run_max = nmax;
          const int64_t t = tgt - c * 32;
          if (t >= 0 && t < 32) {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (i == t) p.le.tgt_logit[grow] = v[i];
          }
        }
        if (dst) {
          if (full_chunk && (p.ldc % 4) == 0) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              float4* d4 = reinterpret_cast<float4*>(dst + i);
              if (EPI == GEMM_ACCUM) {
                float4 o = *d4;
                o.x += v[i];
                o.y += v[i + 1];
                o.z += v[i + 2];
                o.w += v[i + 3];
                *d4 = o;
              } else {
                *d4 = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
              }
            }
          } else {
            for (int i = 0; i < 32 && col0 + i < p.n; ++i) {
              if (EPI == GEMM_ACCUM)
                dst[i] += v[i];
              else
                dst[i] = v[i];
            }
          }
        }
      }
      if (EPI == GEMM_LOGITS && row_ok) {
        p.le.part_max[grow * p.tiles_n + tn] = run_max;
        p.le.part_sum[grow * p.tiles_n + tn] = run_sum;
      }
    }
  }

  tc_fence_before();
  cluster_sync();  // both CTAs done with TMEM and with each other's barriers
  if (warp == 2) tmem_dealloc_pair<512>(tmem);
}

template <bool A_MN, bool B_MN, int EPI>
int launch_impl(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& args, cudaStream_t st) {
  auto kern = gemm_kernel<A_MN, B_MN, EPI>;
  static uint64_t attr_done = 0;  // per device: the attribute is per-context
  int dev = 0;
  cudaGetDevice(&dev);
  if (!((attr_done >> dev) & 1)) {
    if (check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES),
                   "gemm smem attribute"))
      return BB_ERR_CUDA;
    attr_done |= uint64_t(1) << dev;
  }
  static int sms[64] = {0};
  if (!sms[dev & 63]) cudaDeviceGetAttribute(&sms[dev & 63], cudaDevAttrMultiProcessorCount, dev);
  if (args.pair) {
    auto kern2 = gemm2_kernel<A_MN, B_MN, EPI>;
    static uint64_t attr2_done = 0;
    if (!((attr2_done >> dev) & 1)) {
      if (check_cuda(cudaFuncSetAttribute(kern2, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2_BYTES),
                     "gemm2 smem attribute"))
        return BB_ERR_CUDA;
      attr2_done |= uint64_t(1) << dev;
    }
    const int pairs = ((args.tiles_m + 1) / 2) * args.tiles_n;
    const int max_pairs = sms[dev & 63] / 2;
    const int grid = 2 * (pairs < max_pairs ? pairs : max_pairs);
    kern2<<<grid, THREADS, SMEM2_BYTES, st>>>(ta, tb, args);
    return check_launch("gemm2_kernel");
  }
  const int tiles = args.tiles_m * args.tiles_n;
  const int grid = tiles < sms[dev & 63] ? tiles : sms[dev & 63];
  kern<<<grid, THREADS, SMEM_BYTES, st>>>(ta, tb, args);
  return check_launch("gemm_kernel");
}

}  // namespace

int gemm_n_tile() { return BN; }

int launch_gemm_bf16(const void* a, const void* b, void* c16, const int64_t* row_map, int64_t m, int64_t n, int64_t k,
                     int64_t lda, int64_t ldb, int64_t ldc, bool b_mn, cudaStream_t stream) {
  if (m <= 0 || n <= 0 || k <= 0) return set_error(BB_ERR_INVALID, "gemm: empty problem %lld x %lld x %lld", (long long)m, (long long)n, (long long)k);
  if ((lda * 2) % 16 || (ldb * 2) % 16)
    return set_error(BB_ERR_INVALID, "gemm: leading dimensions must be multiples of 8 elements");
  CUtensorMap ta, tb;
  const bool pair = BB_GEMM_PAIR && m >= 2 * BM;
  bool ok = make_tmap_bf16_2d(&ta, a, k, m, lda * 2, 64, BM);
  ok = ok && (b_mn ? make_tmap_bf16_2d(&tb, b, n, k, ldb * 2, 64, 64)
                   : make_tmap_bf16_2d(&tb, b, k, n, ldb * 2, 64, pair ? 128 : BN));
  if (!ok) return BB_ERR_CUDA;
  GemmArgs args{};
  args.m = m;
  args.n = n;
  args.k = k;
  args.ldc = ldc;
  args.c16 = static_cast<__nv_bfloat16*>(c16);
  args.row_map = row_map;
  args.tiles_m = static_cast<int>((m + BM - 1) / BM);
  args.tiles_n = static_cast<int>((n + BN - 1) / BN);
  args.raster_m_fast = false;
  args.pair = pair;
  return b_mn ? launch_impl<false, true, GEMM_BF16>(ta, tb, args, stream)
              : launch_impl<false, false, GEMM_BF16>(ta, tb, args, stream);
}

int launch_gemm(const void* a, const void* b, float* c, int64_t m, int64_t n, int64_t k, int64_t lda,
                int64_t ldb, int64_t ldc, bool a_mn, bool b_mn, int epilogue, const LogitsEpilogue* le,
                bool raster_m_fast, cudaStream_t stream) {
  if (m <= 0 || n <= 0 || k <= 0) return set_error(BB_ERR_INVALID, "gemm: empty problem %lld x %lld x %lld", (long long)m, (long long)n, (long long)k);
  if ((lda * 2) % 16 || (ldb * 2) % 16)
    return set_error(BB_ERR_INVALID, "gemm: leading dimensions must be multiples of 8 elements");
  CUtensorMap ta, tb;
  const bool pair = BB_GEMM_PAIR && m >= 2 * BM;
  bool ok = a_mn ? make_tmap_bf16_2d(&ta, a, m, k, lda * 2, 64, 64)
                 : make_tmap_bf16_2d(&ta, a, k, m, lda * 2, 64, BM);
  ok = ok && (b_mn ? make_tmap_bf16_2d(&tb, b, n, k, ldb * 2, 64, 64)
                   : make_tmap_bf16_2d(&tb, b, k, n, ldb * 2, 64, pair ? 128 : BN));
  if (!ok) return BB_ERR_CUDA;
  GemmArgs args{};
  args.m = m;
  args.n = n;
  args.k = k;
  args.ldc = ldc;
  args.c = c;
  if (le) args.le = *le;
  args.tiles_m = static_cast<int>((m + BM - 1) / BM);
  args.tiles_n = static_cast<int>((n + BN - 1) / BN);
  args.raster_m_fast = raster_m_fast;
  // CTA pairs need the B tile split in two 128-row TMA boxes (K-major: box rows 128)
  args.pair = BB_GEMM_PAIR && m >= 2 * BM;
  if (epilogue == GEMM_LOGITS) {
    if (a_mn || b_mn || !le) return set_error(BB_ERR_INVALID, "gemm: logits epilogue needs K-major operands");
    return launch_impl<false, false, GEMM_LOGITS>(ta, tb, args, stream);
  }
  const bool acc = epilogue == GEMM_ACCUM;
  if (!a_mn && !b_mn) return acc ? launch_impl<false, false, GEMM_ACCUM>(ta, tb, args, stream)
                                 : launch_impl<false, false, GEMM_STORE>(ta, tb, args, stream);
  if (!a_mn && b_mn) return acc ? launch_impl<false, true, GEMM_ACCUM>(ta, tb, args, stream)
                                : launch_impl<false, true, GEMM_STORE>(ta, tb, args, stream);
  if (a_mn && !b_mn) return acc ? launch_impl<true, false, GEMM_ACCUM>(ta, tb, args, stream)
                                : launch_impl<true, false, GEMM_STORE>(ta, tb, args, stream);
  return acc ? launch_impl<true, true, GEMM_ACCUM>(ta, tb, args, stream)
             : launch_impl<true, true, GEMM_STORE>(ta, tb, args, stream);
}

}  // namespace bb
