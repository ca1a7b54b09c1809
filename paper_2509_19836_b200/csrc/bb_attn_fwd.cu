// One forward ring step of BurstAttention on sm_100a (distributed.py:174-188).
//
// For query shard i (resident) and visiting key shard j it computes, per head,
//   S = Q K^T * scale  masked on global token ids (masks.py:89-104),
//   lse_step = row_logsumexp(S),  O_step = softmax(S) V,
// and folds them into the running (O, lse) with the exact lse_merge /
// exp_gap weights of distributed.py:184-188 -- the merge is the epilogue.
//
// CTA = 2 query tiles of 128 rows x one head; K/V tiles of 128 keys stream
// through a 3-slot TMA ring and are shared by both query tiles.
//   warp 0      TMA producer (Q once, then K_j, V_j)
//   warp 1      MMA issuer: S_k = Q_k K_j^T (SS, M=128,N=128) and
//               O_k += P_k V_j (SS, M=128, N=D, V MN-major) into TMEM
//   warp 2      TMEM allocator
//   warps 4-7   softmax for query tile 0, warps 8-11 for query tile 1:
//               one thread per row, online softmax in the log2 domain with a
//               lazy (threshold 8) rescale of the TMEM O accumulator, P written
//               to shared memory in the UMMA SWIZZLE_128B K-major layout.
// Tiles are classified from the closed-form id bounds (bb_mask.cuh): fully
// masked tiles are never loaded or multiplied, fully visible tiles skip the
// per-element predicate.
#include <cuda_runtime.h>

#include "bb_host.h"
#include "bb_mask.cuh"
#include "bb_ptx.cuh"

namespace bb {
namespace {

constexpr int FWD_THREADS = 384;
constexpr int KV_SLOTS = 3;
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 units: P may reach 2^8 before O is rescaled

template <int D>
struct FwdSmem {
  static constexpr uint32_t TILE = 128 * D * 2;  // one Q / K / V tile, D/64 panels of 16 KB
  static constexpr uint32_t PTILE = 128 * 128 * 2;
  static constexpr uint32_t Q_OFF = 0;
  static constexpr uint32_t P_OFF = Q_OFF + 2 * TILE;
  static constexpr uint32_t KV_OFF = P_OFF + 2 * PTILE;
  static constexpr uint32_t BAR_OFF = KV_OFF + KV_SLOTS * TILE;
  static constexpr uint32_t BYTES = BAR_OFF + 256;
};

struct FwdParams {
  float* o;
  float* lse;
  int64_t n_q, n_k;
  int32_t hq, hkv;
  float scale_log2;
  int32_t q_device, k_device;
  bb_layout layout;
  bb_mask mask;
  int32_t q_pairs;  // number of 256-row query blocks
};

__device__ __forceinline__ int32_t fwd_class(const FwdParams& p, int q, int64_t m0, int64_t j) {
  const int64_t r0 = m0 + 128 * q;
  const int64_t r1 = min(r0 + 128, p.n_q);
  const int64_t c0 = j * 128;
  const int64_t c1 = min(c0 + 128, p.n_k);
  return classify_tile(p.layout, p.mask, p.q_device, r0, r1, p.k_device, c0, c1, c1 - c0 == 128);
}

template <int D>
__global__ void __launch_bounds__(FWD_THREADS, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                    const __grid_constant__ CUtensorMap tv, const FwdParams p) {
  using L = FwdSmem<D>;
  constexpr int PANELS = D / 64;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023) != 0) __trap();

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;               // [3]
  uint64_t* kv_empty = bars + 4;              // [3]
  uint64_t* s_full = bars + 7;                // [2]
  uint64_t* p_full = bars + 9;                // [2]
  uint64_t* pv_done = bars + 11;              // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 13);

  const int head = blockIdx.y;
  const int kv_head = head / (p.hq / p.hkv);
  const int64_t m0 = static_cast<int64_t>(p.q_pairs - 1 - blockIdx.x) * 256;  // heavy rows first
  const int64_t n_kt = (p.n_k + 127) / 128;
  const uint32_t warp = warp_id(), lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tq);
    tma_prefetch(&tk);
    tma_prefetch(&tv);
    mbar_init(q_full, 1);
    for (int s = 0; s < KV_SLOTS; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int k = 0; k < 2; ++k) {
      mbar_init(&s_full[k], 1);
      mbar_init(&p_full[k], 128);
      mbar_init(&pv_done[k], 1);
    }
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
      const bool q1_live = m0 + 128 < p.n_q;
      mbar_expect_tx(q_full, (q1_live ? 2 : 1) * L::TILE);
      for (int q = 0; q < (q1_live ? 2 : 1); ++q)
        for (int pn = 0; pn < PANELS; ++pn)
          tma_load_2d(smem + L::Q_OFF + q * L::TILE + pn * 16384, &tq, q_full, head * D + pn * 64,
                      static_cast<int32_t>(m0 + 128 * q));
      uint32_t use = 0;
      for (int64_t j = 0; j < n_kt; ++j) {
        if (fwd_class(p, 0, m0, j) == TILE_SKIP && fwd_class(p, 1, m0, j) == TILE_SKIP) continue;
        for (int which = 0; which < 2; ++which, ++use) {
          const uint32_t s = use % KV_SLOTS, ph = (use / KV_SLOTS) & 1;
          mbar_wait(&kv_empty[s], ph ^ 1);
          mbar_expect_tx(&kv_full[s], L::TILE);
          for (int pn = 0; pn < PANELS; ++pn)
            tma_load_2d(smem + L::KV_OFF + s * L::TILE + pn * 16384, which ? &tv : &tk, &kv_full[s],
                        kv_head * D + pn * 64, static_cast<int32_t>(j * 128));
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_s = idesc_bf16(128, 128, false, false);
    constexpr uint32_t idesc_o = idesc_bf16(128, D, false, true);
    mbar_wait(q_full, 0);
    uint32_t use = 0, issued[2] = {0, 0};
    for (int64_t j = 0; j < n_kt; ++j) {
      const int32_t cls[2] = {fwd_class(p, 0, m0, j), fwd_class(p, 1, m0, j)};
      if (cls[0] == TILE_SKIP && cls[1] == TILE_SKIP) continue;
      const uint32_t sk = use % KV_SLOTS, phk = (use / KV_SLOTS) & 1;
      ++use;
      const uint32_t sv = use % KV_SLOTS, phv = (use / KV_SLOTS) & 1;
      ++use;
      mbar_wait(&kv_full[sk], phk);
      tc_fence_after();
      const uint32_t k_base = smem_u32(smem + L::KV_OFF + sk * L::TILE);
      for (int q = 0; q < 2; ++q) {
        if (cls[q] == TILE_SKIP) continue;
        if (elect_one()) {
          const uint32_t q_base = smem_u32(smem + L::Q_OFF + q * L::TILE);
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks) {
            const uint32_t off = (ks >> 2) * 16384 + (ks & 3) * 32;
            umma_ss(tmem + (q * 128u), sw128_desc(q_base + off, 16, 1024),
                    sw128_desc(k_base + off, 16, 1024), idesc_s, ks > 0);
          }
          umma_commit(&s_full[q]);
        }
        __syncwarp();
      }
      if (elect_one()) umma_commit(&kv_empty[sk]);
      __syncwarp();
      mbar_wait(&kv_full[sv], phv);
      tc_fence_after();
      const uint32_t v_base = smem_u32(smem + L::KV_OFF + sv * L::TILE);
      for (int q = 0; q < 2; ++q) {
        if (cls[q] == TILE_SKIP) continue;
        mbar_wait(&p_full[q], issued[q] & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t p_base = smem_u32(smem + L::P_OFF + q * L::PTILE);
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const uint64_t ad = sw128_desc(p_base + (ks >> 2) * 16384 + (ks & 3) * 32, 16, 1024);
            const uint64_t bd = sw128_desc(v_base + ks * 2048, 16384, 1024);
            umma_ss(tmem + (256u + q * D), ad, bd, idesc_o, (issued[q] | ks) != 0);
          }
          umma_commit(&pv_done[q]);
        }
        __syncwarp();
        ++issued[q];
      }
      if (elect_one()) umma_commit(&kv_empty[sv]);
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ softmax / correction / epilogue
    const int q = (warp - 4) >> 2;  // query tile of this warpgroup
    const uint32_t quad = warp & 3;
    const int row = quad * 32 + lane;
    const int64_t qrow = m0 + 128 * q + row;
    const bool row_ok = qrow < p.n_q;
    const int64_t q_id = row_ok ? token_id(p.layout, p.q_device, qrow) : 0;
    const uint32_t t_lane = (quad * 32) << 16;
    uint8_t* p_tile = smem + L::P_OFF + q * L::PTILE;
    const float sl2 = p.scale_log2;

    float m_run = -INFINITY, l_run = 0.f;
    uint32_t t = 0;
    for (int64_t j = 0; j < n_kt; ++j) {
      const int32_t cls = fwd_class(p, q, m0, j);
      if (cls == TILE_SKIP) continue;
      mbar_wait(&s_full[q], t & 1);
      tc_fence_after();
      float s[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(tmem + t_lane + (q * 128u) + c * 32, *reinterpret_cast<float(*)[32]>(&s[c * 32]));
      tmem_ld_wait();
      if (cls == TILE_PARTIAL) {
        const int64_t kv0 = j * 128;
#pragma unroll
        for (int c = 0; c < 128; ++c) {
          const int64_t kr = kv0 + c;
          bool ok = row_ok && kr < p.n_k;
          if (ok) ok = pair_allowed(p.mask, q_id, token_id(p.layout, p.k_device, kr));
          if (!ok) s[c] = -INFINITY;
        }
      }
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < 128; ++c) mx = fmaxf(mx, s[c]);
      const float m_tile = mx * sl2;
      const bool need = m_tile > m_run + RESCALE_THRESHOLD;
      float alpha = 1.f;
      if (need) {
        alpha = (m_run == -INFINITY) ? 0.f : ex2_approx(m_run - m_tile);
        m_run = m_tile;
        l_run *= alpha;
      }
      const float m_use = (m_run == -INFINITY) ? 0.f : m_run;
      float lsum = 0.f;
#pragma unroll
      for (int c = 0; c < 128; ++c) {
        s[c] = ex2_approx(fmaf(s[c], sl2, -m_use));
        lsum += s[c];
      }
      l_run += lsum;
      // The P buffer and the O accumulator are free once the previous P.V retired.
      if (t > 0) {
        mbar_wait(&pv_done[q], (t - 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffff, need)) {
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            float o[32];
            tmem_ld32(tmem + t_lane + (256u + q * D) + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] *= alpha;
            tmem_st32(tmem + t_lane + (256u + q * D) + c * 32, o);
          }
          tmem_st_wait();
        }
      }
#pragma unroll
      for (int c = 0; c < 128; c += 8) {
        uint4 v;
        v.x = pack_bf16(s[c + 0], s[c + 1]);
        v.y = pack_bf16(s[c + 2], s[c + 3]);
        v.z = pack_bf16(s[c + 4], s[c + 5]);
        v.w = pack_bf16(s[c + 6], s[c + 7]);
        *reinterpret_cast<uint4*>(p_tile + sw128_offset(row, c, 16384)) = v;
      }
      fence_async_smem();
      tc_fence_before();
      mbar_arrive(&p_full[q]);
      ++t;
    }

    if (t > 0) {
      mbar_wait(&pv_done[q], (t - 1) & 1);
      tc_fence_after();
      // lse_step in natural log: sum exp(S) = 2^m_run * l_run.
      const float lse_step = (l_run > 0.f) ? (m_run * 0.69314718055994531f + logf(l_run)) : -INFINITY;
      float w_step = 0.f, w_old = 0.f, lse_new = -INFINITY;
      bool write = row_ok && lse_step != -INFINITY;
      float* lse_ptr = p.lse + static_cast<int64_t>(head) * p.n_q + qrow;
      if (write) {
        const float lse_prev = *lse_ptr;
        if (lse_prev == -INFINITY) {
          lse_new = lse_step;
          w_step = 1.f / l_run;
        } else {
          const float hi = fmaxf(lse_prev, lse_step), lo = fminf(lse_prev, lse_step);
          lse_new = hi + log1pf(expf(lo - hi));
          w_step = expf(lse_step - lse_new) / l_run;
          w_old = expf(lse_prev - lse_new);
        }
        *lse_ptr = lse_new;
      }
      float* o_row = p.o + (qrow * p.hq + head) * static_cast<int64_t>(D);
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        float o[32];
        tmem_ld32(tmem + t_lane + (256u + q * D) + c * 32, o);
        tmem_ld_wait();
        if (write) {
          float4* dst = reinterpret_cast<float4*>(o_row + c * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float4 r = make_float4(o[4 * i] * w_step, o[4 * i + 1] * w_step, o[4 * i + 2] * w_step,
                                   o[4 * i + 3] * w_step);
            if (w_old != 0.f) {
              const float4 prev = dst[i];
              r.x += w_old * prev.x;
              r.y += w_old * prev.y;
              r.z += w_old * prev.z;
              r.w += w_old * prev.w;
            }
            dst[i] = r;
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
int launch_fwd_d(const bb_attn_fwd_args& a, cudaStream_t st) {
  CUtensorMap tq, tk, tv;
  const uint64_t qrow = static_cast<uint64_t>(a.hq) * D * 2, krow = static_cast<uint64_t>(a.hkv) * D * 2;
  if (!make_tmap_bf16_2d(&tq, a.q, static_cast<uint64_t>(a.hq) * D, a.n_q, qrow, 64, 128) ||
      !make_tmap_bf16_2d(&tk, a.k, static_cast<uint64_t>(a.hkv) * D, a.n_k, krow, 64, 128) ||
      !make_tmap_bf16_2d(&tv, a.v, static_cast<uint64_t>(a.hkv) * D, a.n_k, krow, 64, 128))
    return BB_ERR_CUDA;
  FwdParams p{};
  p.o = a.o;
  p.lse = a.lse;
  p.n_q = a.n_q;
  p.n_k = a.n_k;
  p.hq = a.hq;
  p.hkv = a.hkv;
  p.scale_log2 = a.softmax_scale * 1.4426950408889634f;
  p.q_device = a.q_device;
  p.k_device = a.k_device;
  p.layout = a.layout;
  p.mask = a.mask;
  p.q_pairs = static_cast<int32_t>((a.n_q + 255) / 256);
  auto kern = attn_fwd_kernel<D>;
  static uint64_t attr_done = 0;  // per device: the attribute is per-context
  int dev = 0;
  cudaGetDevice(&dev);
  if (!((attr_done >> dev) & 1)) {
    if (check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdSmem<D>::BYTES),
                   "attn_fwd smem attribute"))
      return BB_ERR_CUDA;
    attr_done |= uint64_t(1) << dev;
  }
  dim3 grid(p.q_pairs, a.hq);
  kern<<<grid, FWD_THREADS, FwdSmem<D>::BYTES, st>>>(tq, tk, tv, p);
  return check_launch("attn_fwd_kernel");
}

}  // namespace

int launch_attn_fwd(const bb_attn_fwd_args& a, cudaStream_t st) {
  if (a.head_dim == 128) return launch_fwd_d<128>(a, st);
  if (a.head_dim == 64) return launch_fwd_d<64>(a, st);
  return set_error(BB_ERR_UNSUPPORTED, "attn_fwd: head_dim %d (kernels take 64 or 128)", a.head_dim);
}

}  // namespace bb
