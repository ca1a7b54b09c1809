// One backward ring step of BurstAttention on sm_100a.
//
// The same kernel serves both reference backward passes, which differ only in
// which buffers circulate (distributed.py:207-299):
//   burst_backward (:288-295): K_i/V_i resident, (Q_j, dQ_j, dO_j, D_j, Lse_j) visit;
//   ring_backward  (:239-247): Q_i resident, (K_j, V_j, dK_j, dV_j) visit.
// Per (query shard, key shard) pair it accumulates in fp32
//   P   = exp(S - lse)            (S = Q K^T * scale, masked)
//   dV += P^T dO,  dP = dO V^T,  dS = P o (dP - D)
//   dK += dS^T Q * scale,  dQ += dS K * scale.
//
// CTA = one 128-key tile x one kv head, K/V-stationary (the BurstAttention
// backward's own data flow); it sweeps every (query head of the GQA group,
// 128-row query tile) pair that the mask does not fully hide.
//   warp 0     TMA: K, V once; Q_i, dO_i per query tile
//   warp 1     MMA: S^T = K Q^T, dP^T = V dO^T (M=keys), dV += P^T dO,
//              dK += dS^T Q, dQ = dS K (M=queries, dS^T read MN-major)
//   warp 2     TMEM allocator
//   warps 4-7  one thread per TMEM lane: P^T / dS^T into SWIZZLE_128B smem,
//              dQ tile -> fp32 atomics, final dK / dV read-modify-write.
// TMEM: S^T [0,128) (reused by the dQ tile), dP^T [128,256), dV, dK.
#include <cuda_runtime.h>

#include "bb_host.h"
#include "bb_mask.cuh"
#include "bb_ptx.cuh"

namespace bb {
namespace {

constexpr int BWD_THREADS = 256;

template <int D>
struct BwdSmem {
  static constexpr uint32_t TILE = 128 * D * 2;
  static constexpr uint32_t PTILE = 128 * 128 * 2;
  static constexpr uint32_t K_OFF = 0;
  static constexpr uint32_t V_OFF = K_OFF + TILE;
  static constexpr uint32_t Q_OFF = V_OFF + TILE;
  static constexpr uint32_t DO_OFF = Q_OFF + TILE;
  static constexpr uint32_t P_OFF = DO_OFF + TILE;
  static constexpr uint32_t DS_OFF = P_OFF + PTILE;
  static constexpr uint32_t VEC_OFF = DS_OFF + PTILE;  // lse2[2][128], delta[2][128]
  static constexpr uint32_t BAR_OFF = VEC_OFF + 4 * 128 * 4;
  static constexpr uint32_t BYTES = BAR_OFF + 256;
};

struct BwdParams {
  const float* lse;
  const float* delta;
  float* dq;
  float* dk;
  float* dv;
  int64_t n_q, n_k;
  int32_t hq, hkv;
  float scale, scale_log2;
  int32_t q_device, k_device;
  bb_layout layout;
  bb_mask mask;
};

__device__ __forceinline__ int32_t bwd_class(const BwdParams& p, int64_t qt, int64_t c0) {
  const int64_t r0 = qt * 128, r1 = min(r0 + 128, p.n_q);
  const int64_t c1 = min(c0 + 128, p.n_k);
  return classify_tile(p.layout, p.mask, p.q_device, r0, r1, p.k_device, c0, c1, c1 - c0 == 128);
}

template <int D>
__global__ void __launch_bounds__(BWD_THREADS, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                    const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo,
                    const BwdParams p) {
  using L = BwdSmem<D>;
  constexpr int PANELS = D / 64;
  constexpr uint32_t COL_S = 0, COL_DP = 128, COL_DV = 256, COL_DK = 256 + D, COL_DQ = 0;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023) != 0) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* kv_full = bars + 0;
  uint64_t* qdo_full = bars + 1;
  uint64_t* qdo_empty = bars + 2;
  uint64_t* sdp_full = bars + 3;
  uint64_t* p_full = bars + 4;
  uint64_t* ds_full = bars + 5;
  uint64_t* dq_full = bars + 6;
  uint64_t* dq_free = bars + 7;
  uint64_t* acc_full = bars + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 9);
  float* lse2_s = reinterpret_cast<float*>(smem + L::VEC_OFF);  // [2][128]
  float* delta_s = lse2_s + 256;                                  // [2][128]

  const int kv_head = blockIdx.y;
  const int group = p.hq / p.hkv;
  const int64_t n_kt = (p.n_k + 127) / 128;
  const int64_t c0 = static_cast<int64_t>(n_kt - 1 - blockIdx.x) * 128;
  const int64_t n_qt = (p.n_q + 127) / 128;
  const int64_t n_work = group * n_qt;  // (query head in group, query tile) pairs
  const uint32_t warp = warp_id(), lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tq);
    tma_prefetch(&tk);
    tma_prefetch(&tv);
    tma_prefetch(&tdo);
    mbar_init(kv_full, 1);
    mbar_init(qdo_full, 1);
    mbar_init(qdo_empty, 1);
    mbar_init(sdp_full, 1);
    mbar_init(p_full, 128);
    mbar_init(ds_full, 128);
    mbar_init(dq_full, 1);
    mbar_init(dq_free, 128);
    mbar_init(acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (elect_one()) {
      mbar_expect_tx(kv_full, 2 * L::TILE);
      for (int pn = 0; pn < PANELS; ++pn) {
        tma_load_2d(smem + L::K_OFF + pn * 16384, &tk, kv_full, kv_head * D + pn * 64, static_cast<int32_t>(c0));
        tma_load_2d(smem + L::V_OFF + pn * 16384, &tv, kv_full, kv_head * D + pn * 64, static_cast<int32_t>(c0));
      }
      uint32_t it = 0;
      for (int64_t w = 0; w < n_work; ++w) {
        const int64_t qt = w % n_qt;
        const int h = kv_head * group + static_cast<int>(w / n_qt);
        if (bwd_class(p, qt, c0) == TILE_SKIP) continue;
        mbar_wait(qdo_empty, (it & 1) ^ 1);
        mbar_expect_tx(qdo_full, 2 * L::TILE);
        for (int pn = 0; pn < PANELS; ++pn) {
          tma_load_2d(smem + L::Q_OFF + pn * 16384, &tq, qdo_full, h * D + pn * 64, static_cast<int32_t>(qt * 128));
          tma_load_2d(smem + L::DO_OFF + pn * 16384, &tdo, qdo_full, h * D + pn * 64, static_cast<int32_t>(qt * 128));
        }
        ++it;
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_st = idesc_bf16(128, 128, false, false);  // S^T, dP^T: both K-major
    constexpr uint32_t idesc_acc = idesc_bf16(128, D, false, true);    // dV, dK: B (dO / Q) MN-major
    constexpr uint32_t idesc_dq = idesc_bf16(128, D, true, true);      // dQ: A = dS (MN), B = K (MN)
    const uint32_t k_base = smem_u32(smem + L::K_OFF), v_base = smem_u32(smem + L::V_OFF);
    const uint32_t q_base = smem_u32(smem + L::Q_OFF), do_base = smem_u32(smem + L::DO_OFF);
    const uint32_t p_base = smem_u32(smem + L::P_OFF), ds_base = smem_u32(smem + L::DS_OFF);
    mbar_wait(kv_full, 0);
    uint32_t it = 0;
    for (int64_t w = 0; w < n_work; ++w) {
      const int64_t qt = w % n_qt;
      if (bwd_class(p, qt, c0) == TILE_SKIP) continue;
      mbar_wait(qdo_full, it & 1);
      if (it > 0) mbar_wait(dq_free, (it - 1) & 1);  // S^T columns double as the dQ tile
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t off = (ks >> 2) * 16384 + (ks & 3) * 32;
          umma_ss(tmem + COL_S, sw128_desc(k_base + off, 16, 1024), sw128_desc(q_base + off, 16, 1024), idesc_st, ks > 0);
        }
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t off = (ks >> 2) * 16384 + (ks & 3) * 32;
          umma_ss(tmem + COL_DP, sw128_desc(v_base + off, 16, 1024), sw128_desc(do_base + off, 16, 1024), idesc_st, ks > 0);
        }
        umma_commit(sdp_full);
      }
      __syncwarp();
      mbar_wait(p_full, it & 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {  // K = 128 query rows
          const uint64_t ad = sw128_desc(p_base + (ks >> 2) * 16384 + (ks & 3) * 32, 16, 1024);
          const uint64_t bd = sw128_desc(do_base + ks * 2048, 16384, 1024);
          umma_ss(tmem + COL_DV, ad, bd, idesc_acc, (it | ks) != 0);
        }
      }
      __syncwarp();
      mbar_wait(ds_full, it & 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const uint64_t ad = sw128_desc(ds_base + (ks >> 2) * 16384 + (ks & 3) * 32, 16, 1024);
          const uint64_t bd = sw128_desc(q_base + ks * 2048, 16384, 1024);
          umma_ss(tmem + COL_DK, ad, bd, idesc_acc, (it | ks) != 0);
        }
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {  // K = 128 keys
          const uint64_t ad = sw128_desc(ds_base + ks * 2048, 16384, 1024);
          const uint64_t bd = sw128_desc(k_base + ks * 2048, 16384, 1024);
          umma_ss(tmem + COL_DQ, ad, bd, idesc_dq, ks > 0);
        }
        umma_commit(dq_full);
        umma_commit(qdo_empty);
      }
      __syncwarp();
      ++it;
    }
    if (elect_one()) umma_commit(acc_full);
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------ P / dS / dQ / epilogue
    const uint32_t quad = warp & 3;
    const int row = quad * 32 + lane;  // key row for S^T / dP^T; query row for dQ
    const uint32_t t_lane = (quad * 32) << 16;
    const int64_t krow = c0 + row;
    const bool key_ok = krow < p.n_k;
    const int64_t k_id = key_ok ? token_id(p.layout, p.k_device, krow) : 0;
    uint8_t* p_tile = smem + L::P_OFF;
    uint8_t* ds_tile = smem + L::DS_OFF;
    uint32_t it = 0;
    for (int64_t w = 0; w < n_work; ++w) {
      const int64_t qt = w % n_qt;
      const int h = kv_head * group + static_cast<int>(w / n_qt);
      const int32_t cls = bwd_class(p, qt, c0);
      if (cls == TILE_SKIP) continue;
      const int64_t r0 = qt * 128;
      float* lse2 = lse2_s + (it & 1) * 128;
      float* dlt = delta_s + (it & 1) * 128;
      {
        const int64_t r = r0 + row;
        float l2 = INFINITY, dd = 0.f;
        if (r < p.n_q) {
          const float l = p.lse[static_cast<int64_t>(h) * p.n_q + r];
          l2 = (l == -INFINITY) ? INFINITY : l * 1.4426950408889634f;
          dd = p.delta[static_cast<int64_t>(h) * p.n_q + r];
        }
        lse2[row] = l2;
        dlt[row] = dd;
      }
      named_bar_sync(1, 128);
      mbar_wait(sdp_full, it & 1);
      tc_fence_after();
      // P^T = exp2(S^T * scale*log2e - lse2[q])  -> smem (K-major rows = keys)
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        float s[32];
        tmem_ld32(tmem + t_lane + COL_S + c * 32, s);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int qc = c * 32 + i;
          bool ok = key_ok;
          if (cls == TILE_PARTIAL && ok) {
            const int64_t qr = r0 + qc;
            ok = qr < p.n_q && pair_allowed(p.mask, token_id(p.layout, p.q_device, qr), k_id);
          }
          s[i] = ok ? ex2_approx(fmaf(s[i], p.scale_log2, -lse2[qc])) : 0.f;
        }
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 v;
          v.x = pack_bf16(s[i + 0], s[i + 1]);
          v.y = pack_bf16(s[i + 2], s[i + 3]);
          v.z = pack_bf16(s[i + 4], s[i + 5]);
          v.w = pack_bf16(s[i + 6], s[i + 7]);
          *reinterpret_cast<uint4*>(p_tile + sw128_offset(row, c * 32 + i, 16384)) = v;
        }
      }
      fence_async_smem();
      tc_fence_before();
      mbar_arrive(p_full);
      // dS^T = P^T o (dP^T - D[q])  (P re-read as the bf16 values the dV MMA consumed)
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        float dp[32];
        tmem_ld32(tmem + t_lane + COL_DP + c * 32, dp);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          const uint32_t off = sw128_offset(row, c * 32 + i, 16384);
          const uint4 pv = *reinterpret_cast<const uint4*>(p_tile + off);
          const uint32_t pw[4] = {pv.x, pv.y, pv.z, pv.w};
          float ds[8];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&pw[e]);
            ds[2 * e] = __low2float(b) * (dp[i + 2 * e] - dlt[c * 32 + i + 2 * e]);
            ds[2 * e + 1] = __high2float(b) * (dp[i + 2 * e + 1] - dlt[c * 32 + i + 2 * e + 1]);
          }
          uint4 v;
          v.x = pack_bf16(ds[0], ds[1]);
          v.y = pack_bf16(ds[2], ds[3]);
          v.z = pack_bf16(ds[4], ds[5]);
          v.w = pack_bf16(ds[6], ds[7]);
          *reinterpret_cast<uint4*>(ds_tile + off) = v;
        }
      }
      fence_async_smem();
      tc_fence_before();
      mbar_arrive(ds_full);
      // dQ tile (TMEM lane = query row) -> fp32 atomics into the circulating dQ.
      mbar_wait(dq_full, it & 1);
      tc_fence_after();
      {
        const int64_t qr = r0 + row;
        float* dst = p.dq + (qr * p.hq + h) * static_cast<int64_t>(D);
#pragma unroll 1
        for (int c = 0; c < D / 32; ++c) {
          float g[32];
          tmem_ld32(tmem + t_lane + COL_DQ + c * 32, g);
          tmem_ld_wait();
          if (qr < p.n_q) {
#pragma unroll
            for (int i = 0; i < 32; i += 4)
              atomicAdd(reinterpret_cast<float4*>(dst + c * 32 + i),
                        make_float4(g[i] * p.scale, g[i + 1] * p.scale, g[i + 2] * p.scale, g[i + 3] * p.scale));
          }
        }
      }
      tc_fence_before();
      mbar_arrive(dq_free);
      ++it;
    }
    // dK (scaled) and dV accumulate into the resident fp32 buffers.
    if (it > 0) {
      mbar_wait(acc_full, 0);
      tc_fence_after();
      float* dk_row = p.dk + (krow * p.hkv + kv_head) * static_cast<int64_t>(D);
      float* dv_row = p.dv + (krow * p.hkv + kv_head) * static_cast<int64_t>(D);
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        float a[32], b[32];
        tmem_ld32(tmem + t_lane + COL_DK + c * 32, a);
        tmem_ld32(tmem + t_lane + COL_DV + c * 32, b);
        tmem_ld_wait();
        if (key_ok) {
          float4* k4 = reinterpret_cast<float4*>(dk_row + c * 32);
          float4* v4 = reinterpret_cast<float4*>(dv_row + c * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float4 x = k4[i], y = v4[i];
            x.x += a[4 * i] * p.scale;
            x.y += a[4 * i + 1] * p.scale;
            x.z += a[4 * i + 2] * p.scale;
            x.w += a[4 * i + 3] * p.scale;
            y.x += b[4 * i];
            y.y += b[4 * i + 1];
            y.z += b[4 * i + 2];
            y.w += b[4 * i + 3];
            k4[i] = x;
            v4[i] = y;
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

template <int D>
int launch_bwd_d(const bb_attn_bwd_args& a, cudaStream_t st) {
  CUtensorMap tq, tk, tv, tdo;
  const uint64_t qrow = static_cast<uint64_t>(a.hq) * D * 2, krow = static_cast<uint64_t>(a.hkv) * D * 2;
  if (!make_tmap_bf16_2d(&tq, a.q, static_cast<uint64_t>(a.hq) * D, a.n_q, qrow, 64, 128) ||
      !make_tmap_bf16_2d(&tdo, a.dout, static_cast<uint64_t>(a.hq) * D, a.n_q, qrow, 64, 128) ||
      !make_tmap_bf16_2d(&tk, a.k, static_cast<uint64_t>(a.hkv) * D, a.n_k, krow, 64, 128) ||
      !make_tmap_bf16_2d(&tv, a.v, static_cast<uint64_t>(a.hkv) * D, a.n_k, krow, 64, 128))
    return BB_ERR_CUDA;
  BwdParams p{};
  p.lse = a.lse;
  p.delta = a.delta;
  p.dq = a.dq;
  p.dk = a.dk;
  p.dv = a.dv;
  p.n_q = a.n_q;
  p.n_k = a.n_k;
  p.hq = a.hq;
  p.hkv = a.hkv;
  p.scale = a.softmax_scale;
  p.scale_log2 = a.softmax_scale * 1.4426950408889634f;
  p.q_device = a.q_device;
  p.k_device = a.k_device;
  p.layout = a.layout;
  p.mask = a.mask;
  auto kern = attn_bwd_kernel<D>;
  static uint64_t attr_done = 0;  // per device: the attribute is per-context
  int dev = 0;
  cudaGetDevice(&dev);
  if (!((attr_done >> dev) & 1)) {
    if (check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, BwdSmem<D>::BYTES),
                   "attn_bwd smem attribute"))
      return BB_ERR_CUDA;
    attr_done |= uint64_t(1) << dev;
  }
  dim3 grid(static_cast<unsigned>((a.n_k + 127) / 128), a.hkv);
  kern<<<grid, BWD_THREADS, BwdSmem<D>::BYTES, st>>>(tq, tk, tv, tdo, p);
  return check_launch("attn_bwd_kernel");
}

}  // namespace

int launch_attn_bwd(const bb_attn_bwd_args& a, cudaStream_t st) {
  if (a.head_dim == 128) return launch_bwd_d<128>(a, st);
  if (a.head_dim == 64) return launch_bwd_d<64>(a, st);
  return set_error(BB_ERR_UNSUPPORTED, "attn_bwd: head_dim %d (kernels take 64 or 128)", a.head_dim);
}

}  // namespace bb
