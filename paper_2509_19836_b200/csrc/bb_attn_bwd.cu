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
// backward's own data flow), sweeping every (query head of the GQA group,
// 128-row query tile) the mask does not fully hide.
//   warp 0      TMA: K, V once; Q_i (2 stages) and dO_i per query tile
//   warp 1      MMA: S^T = K Q^T, dP^T = V dO^T          (SS, M = keys)
//                    dV += P^T dO   with P^T read from TMEM (TS, no smem round trip)
//                    dK += dS^T Q, dQ = dS K               (SS; dS^T read MN-major)
//   warp 2      TMEM allocator
//   warps 4-11  two groups of 4 warps, each owning half of the 128 query columns
//               (group g: TMEM columns of its half, all 128 lanes):
//               P^T -> TMEM (bf16, in place over S^T), dS^T -> SWIZZLE_128B smem,
//               final dK / dV read-modify-write.
//   warps 12-15 dQ drain: dQ tile -> swizzled smem staging -> TMA bulk reduce-add (fp32)
//               into the circulating dQ, overlapped with the next tile's P / dS.
// TMEM: S^T / P^T [0,128), dP^T then dQ [128,256), dV [256,256+D), dK [256+D,256+2D).
#include <cuda_runtime.h>

#include <type_traits>

#include "bb_host.h"
#include "bb_mask.cuh"
#include "bb_ptx.cuh"

namespace bb {
namespace {

#ifndef BB_BWD_NG
#define BB_BWD_NG 2
#endif
constexpr int NG = BB_BWD_NG;
#ifndef BB_BWD_MC
#define BB_BWD_MC 0  // 2-CTA Q/dO multicast clusters: correct since the empty-range fix, but a wash (976 vs 968 full 32K, 952 vs 955 causal 128K)
#endif
constexpr bool MC = BB_BWD_MC;
#ifndef BB_BWD_DQ128
#define BB_BWD_DQ128 1
#endif
              // compute column groups (4 warps each)
constexpr int CPG = 128 / NG;              // query columns per group
constexpr int CH = CPG / 32;               // 32-column chunks per group
constexpr int NCOMP = NG * 128;            // compute threads
constexpr int BWD_THREADS = 128 + NCOMP + 128;  // control warps + compute + dQ drain
constexpr int MAX_QT = 4096;  // query tiles per shard the class table holds (n_q <= 524288)

template <int D>
struct BwdSmem {
  static constexpr uint32_t TILE = 128 * D * 2;
  static constexpr uint32_t K_OFF = 0;
  static constexpr uint32_t V_OFF = K_OFF + TILE;
  static constexpr uint32_t Q_OFF = V_OFF + TILE;    // 2 stages
  static constexpr uint32_t DO_OFF = Q_OFF + 2 * TILE;
  static constexpr uint32_t DS_OFF = DO_OFF + TILE;  // dS^T, 128 keys x 128 queries bf16
  static constexpr uint32_t STG_OFF = DS_OFF + 128 * 128 * 2;  // 2 x [128 x 32] fp32 dQ staging
  static constexpr uint32_t VEC_OFF = STG_OFF + 2 * 16384;     // [lse2 128 | delta 128]
  static constexpr uint32_t BAR_OFF = VEC_OFF + 256 * 4;
  static constexpr uint32_t CLS_OFF = BAR_OFF + 256;  // 2-bit tile class per query tile
  static constexpr uint32_t BYTES = CLS_OFF + MAX_QT / 4;
};

struct BwdParams {
  const float* lse;
  const float* delta;
  float* dq;
  float* dk;
  float* dv;
  int64_t n_q, n_k;
  int32_t hq, hkv;
  int32_t kv_head0;  // first kv head of this launch (grid.y covers the range)
  float scale, scale_log2;
  int32_t q_device, k_device;
  LayoutD layout;
  MaskD mask;
  long long* probe;  // diagnostics: per-phase clock64() of CTA (0,0), see bb_debug_probe
};

#define BB_PROBE(slot)                                                                 \
  do {                                                                                 \
    if (p.probe && blockIdx.x == 0 && blockIdx.y == 0 && it < 16) p.probe[it * 32 + (slot)] = clock64(); \
  } while (0)

__device__ __forceinline__ int32_t bwd_class(const BwdParams& p, int64_t qt, int64_t c0) {
  const int64_t r0 = qt * 128, r1 = min(r0 + 128, p.n_q);
  const int64_t c1 = min(c0 + 128, p.n_k);
  return classify_tile(p.layout, p.mask, p.q_device, r0, r1, p.k_device, c0, c1, c1 - c0 == 128);
}

template <int D>
__global__ void __launch_bounds__(BWD_THREADS, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                    const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo,
                    const __grid_constant__ CUtensorMap tdq, const BwdParams p) {
  using L = BwdSmem<D>;
  constexpr int PANELS = D / 64;
  constexpr uint32_t COL_S = 0, COL_DP = 128, COL_DV = 256, COL_DK = 256 + D;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023) != 0) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* kv_full = bars + 0;
  uint64_t* q_full = bars + 1;   // [2]
  uint64_t* q_empty = bars + 3;  // [2]
  uint64_t* do_full = bars + 5;
  uint64_t* do_empty = bars + 6;
  uint64_t* s_full = bars + 7;
  uint64_t* p_full = bars + 8;
  uint64_t* dp_full = bars + 9;
  uint64_t* ds_full = bars + 10;
  uint64_t* dq_full = bars + 11;
  uint64_t* dq_free = bars + 12;
  uint64_t* acc_full = bars + 13;
  // The dP^T / dQ columns are handed over in two 64-column halves: dQ half h (head dims
  // [64h, 64h+64)) and dP^T half g (query columns of compute group g) share TMEM columns
  // COL_DP + 64h, so dP_g(t+1) goes as soon as the drain has read dQ half g of tile t.
  //   dp_full[g] = bars 9 / 14, dq_full[h] = bars 11 / 15, dq_free[h] = bars 12 / 16
  uint64_t* dp_full2[2] = {bars + 9, bars + 14};
  uint64_t* dq_full2[2] = {bars + 11, bars + 15};
  uint64_t* dq_free2[2] = {bars + 12, bars + 16};
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 17);
  float* vec_s = reinterpret_cast<float*>(smem + L::VEC_OFF);

  const int kv_head = p.kv_head0 + static_cast<int>(blockIdx.y);
  const int group = p.hq / p.hkv;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 128;  // low key tiles carry the most work
  // MC: clusters of two adjacent key tiles share every Q / dO tile through a TMA multicast
  // (half the L2 reads); both CTAs walk the union of their query ranges, and a query tile
  // only one of them can see is computed by the other fully masked (P = 0).
  const uint32_t crank = MC ? cluster_ctarank() : 0;
  const int64_t c0p = c0 + (crank ? -128 : 128);  // the partner's key tile (MC)
  auto q_range = [&](int64_t kc, int64_t& lo, int64_t& hi) {
    lo = hi = 0;
    if (kc < 0 || kc >= p.n_k) return;
    active_runs(p.layout, p.mask, token_id(p.layout, p.k_device, kc),
                token_id(p.layout, p.k_device, min(kc + 128, p.n_k) - 1), p.q_device, p.n_q, false, lo, hi);
  };
  // Query tiles that can touch this key tile (two binary searches, every thread), then the
  // work items (query head of the GQA group, query tile in [q_lo, q_hi)).
  int64_t q_lo, q_hi;
  q_range(c0, q_lo, q_hi);
  if (MC) {
    int64_t p_lo, p_hi;
    q_range(c0p, p_lo, p_hi);
    if (p_hi > p_lo) {
      if (q_hi > q_lo) {
        q_lo = min(q_lo, p_lo);
        q_hi = max(q_hi, p_hi);
      } else {
        q_lo = p_lo;
        q_hi = p_hi;
      }
    }
  }
  const uint32_t nr = static_cast<uint32_t>(q_hi - q_lo);
  // Work item w packs (head-in-group << 16 | query-tile index): no divisions on the roles'
  // per-tile path (a u32 div/mod is a ~100-cycle dependent chain).  n_work = end sentinel.
  const int64_t n_work = static_cast<int64_t>(group) << 16;
  const uint32_t warp = warp_id(), lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tq);
    tma_prefetch(&tk);
    tma_prefetch(&tv);
    tma_prefetch(&tdo);
    tma_prefetch(&tdq);
    mbar_init(kv_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], MC ? 2 : 1);  // MC: both CTAs' MMAs must have read the slot
    }
    mbar_init(do_full, 1);
    mbar_init(do_empty, MC ? 2 : 1);
    mbar_init(s_full, 1);
    mbar_init(p_full, NCOMP);
    mbar_init(dp_full, 1);
    mbar_init(dp_full2[1], 1);
    mbar_init(dq_full2[1], 1);
    mbar_init(dq_free2[1], 128);
    mbar_init(ds_full, NCOMP);
    mbar_init(dq_full, 1);
    mbar_init(dq_free, 128);
    mbar_init(acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  // Classify this key tile against every query tile once (2 bits each); the warp roles then
  // look classes up instead of re-deriving them per tile (that inlined id arithmetic put
  // several KB of code on every role's per-tile path and stalled on instruction fetch).
  uint8_t* cls_tab = smem + L::CLS_OFF;
  for (uint32_t b = threadIdx.x; b < (nr + 3) / 4; b += BWD_THREADS) {
    uint32_t byte = 0;
    for (uint32_t k = 0; k < 4; ++k)
      if (4 * b + k < nr) {
        const int64_t qt = q_lo + 4 * b + k;
        int32_t cls = c0 < p.n_k ? bwd_class(p, qt, c0) : TILE_SKIP;
        if (MC && cls == TILE_SKIP && c0p >= 0 && c0p < p.n_k && bwd_class(p, qt, c0p) != TILE_SKIP)
          cls = TILE_PARTIAL;  // the partner needs this tile: compute it fully masked
        byte |= static_cast<uint32_t>(cls) << (2 * k);
      }
    cls_tab[b] = static_cast<uint8_t>(byte);
  }
  auto tile_cls = [&](uint32_t qt) {
    const uint32_t x = qt - static_cast<uint32_t>(q_lo);
    return static_cast<int32_t>((cls_tab[x >> 2] >> ((x & 3) * 2)) & 3);
  };
  tc_fence_before();
  if (MC)
    cluster_sync();  // the partner's multicasts may target this CTA's barriers from here on
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // Work items: (query head of the GQA group, query tile) in order, skipping masked tiles.
  // (nr == 0 must end at once: the class table is empty, and a head step must re-check the
  // range -- reading an unwritten table entry once sent two CTAs of a multicast cluster down
  // different item lists, a hang)
  auto next_active = [&](int64_t w) {
    if (nr == 0) return n_work;
    for (;;) {
      if ((w & 0xFFFF) >= nr) w = ((w >> 16) + 1) << 16;
      if (w >= n_work) return n_work;
      if (tile_cls(static_cast<uint32_t>(q_lo) + static_cast<uint32_t>(w & 0xFFFF)) != TILE_SKIP) return w;
      ++w;
    }
  };
  auto item_qt = [&](int64_t w) { return static_cast<uint32_t>(q_lo) + static_cast<uint32_t>(w & 0xFFFF); };
  auto item_head = [&](int64_t w) { return kv_head * group + static_cast<int>(w >> 16); };

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (elect_one()) {
      mbar_expect_tx(kv_full, 2 * L::TILE);
      for (int pn = 0; pn < PANELS; ++pn) {
        tma_load_2d(smem + L::K_OFF + pn * 16384, &tk, kv_full, kv_head * D + pn * 64, static_cast<int32_t>(c0));
        tma_load_2d(smem + L::V_OFF + pn * 16384, &tv, kv_full, kv_head * D + pn * 64, static_cast<int32_t>(c0));
      }
      uint32_t it = 0;
      for (int64_t w = next_active(0); w < n_work; w = next_active(w + 1), ++it) {
        const int32_t qrow0 = static_cast<int32_t>(item_qt(w) * 128);
        const int h = item_head(w);
        const uint32_t qs = it & 1;
        BB_PROBE(0);
        mbar_wait(&q_empty[qs], ((it >> 1) & 1) ^ 1);
        BB_PROBE(1);
        mbar_expect_tx(&q_full[qs], L::TILE);
        for (int pn = 0; pn < PANELS; ++pn) {
          if (!MC)
            tma_load_2d(smem + L::Q_OFF + qs * L::TILE + pn * 16384, &tq, &q_full[qs], h * D + pn * 64, qrow0);
          else if (crank == 0)
            tma_load_2d_mc(smem + L::Q_OFF + qs * L::TILE + pn * 16384, &tq, &q_full[qs], h * D + pn * 64, qrow0, 3);
        }
        mbar_wait(do_empty, (it & 1) ^ 1);
        BB_PROBE(2);
        mbar_expect_tx(do_full, L::TILE);
        for (int pn = 0; pn < PANELS; ++pn)
          if (!MC)
            tma_load_2d(smem + L::DO_OFF + pn * 16384, &tdo, do_full, h * D + pn * 64, qrow0);
          else if (crank == 0)
            tma_load_2d_mc(smem + L::DO_OFF + pn * 16384, &tdo, do_full, h * D + pn * 64, qrow0, 3);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    // Per tile t:  dV(t) [P(t) ready], S(t+1), dK(t) dQ(t) [dS(t) ready], dP(t+1) [dQ(t) drained].
    // S(t+1) goes out as soon as dV(t) has been issued (the tensor pipe is in order, so dV(t)
    // reads P(t) from the S columns before S(t+1) overwrites them); the compute warps then
    // start P(t+1) while dK(t)/dQ(t) run and the drain warps empty dQ(t).
    constexpr uint32_t idesc_st = idesc_bf16(128, 128, false, false);  // S^T, dP^T
    constexpr uint32_t idesc_acc = idesc_bf16(128, D, false, true);    // dV (TS), dK: B MN-major
    const uint32_t k_base = smem_u32(smem + L::K_OFF), v_base = smem_u32(smem + L::V_OFF);
    const uint32_t do_base = smem_u32(smem + L::DO_OFF), ds_base = smem_u32(smem + L::DS_OFF);
    auto issue_s = [&](uint32_t qs) {
      const uint32_t q_base = smem_u32(smem + L::Q_OFF + qs * L::TILE);
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t off = (ks >> 2) * 16384 + (ks & 3) * 32;
          umma_ss(tmem + COL_S, sw128_desc(k_base + off, 16, 1024), sw128_desc(q_base + off, 16, 1024), idesc_st, ks > 0);
        }
        umma_commit(s_full);
      }
      __syncwarp();
    };
    constexpr uint32_t idesc_st64 = idesc_bf16(128, 64, false, false);  // dP^T half: 64 query columns
    constexpr uint32_t idesc_dq64 = idesc_bf16(128, 64, true, true);    // dQ half: 64 head dims
    constexpr uint32_t idesc_dq = idesc_bf16(128, D, true, true);       // dQ: A = dS (MN), B = K (MN)
    auto issue_dp_half = [&](int g) {  // dP^T[:, 64g:64g+64] = V . dO[64g:64g+64]^T
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t off = (ks >> 2) * 16384 + (ks & 3) * 32;
          umma_ss(tmem + COL_DP + 64 * g, sw128_desc(v_base + off, 16, 1024),
                  sw128_desc(do_base + off + 8192 * g, 16, 1024), idesc_st64, ks > 0);
        }
        umma_commit(dp_full2[g]);
      }
      __syncwarp();
    };

    mbar_wait(kv_full, 0);
    int64_t w = next_active(0);
    if (w < n_work) {
      mbar_wait(&q_full[0], 0);
      tc_fence_after();
      issue_s(0);
      mbar_wait(do_full, 0);
      tc_fence_after();
      issue_dp_half(0);
      issue_dp_half(1);
    }
    for (uint32_t it = 0; w < n_work; ++it) {
      const int64_t wn = next_active(w + 1);
      const uint32_t qs = it & 1;
      const uint32_t q_base = smem_u32(smem + L::Q_OFF + qs * L::TILE);
      if (lane == 0) BB_PROBE(4);
      mbar_wait(p_full, it & 1);
      if (lane == 0) BB_PROBE(8);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {  // K = 128 query rows; P^T packed 2 per TMEM column
          const uint32_t a_tmem = tmem + COL_S + (ks >> 1) * 32 + (ks & 1) * 8;  // P of q chunk c in its own S columns
          umma_ts(tmem + COL_DV, a_tmem, sw128_desc(do_base + ks * 2048, 16384, 1024), idesc_acc, (it | ks) != 0);
        }
        if (MC)
          umma_commit_mc(do_empty, 3);  // dP(t) and dV(t) have read dO(t) (both CTAs count)
        else
          umma_commit(do_empty);
      }
      __syncwarp();
      if (wn < n_work) {
        mbar_wait(&q_full[qs ^ 1], ((it + 1) >> 1) & 1);
        tc_fence_after();
        issue_s(qs ^ 1);
      }
      if (lane == 0) BB_PROBE(5);
      mbar_wait(ds_full, it & 1);
      if (lane == 0) BB_PROBE(9);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const uint64_t ad = sw128_desc(ds_base + (ks >> 2) * 16384 + (ks & 3) * 32, 16, 1024);
          umma_ss(tmem + COL_DK, ad, sw128_desc(q_base + ks * 2048, 16384, 1024), idesc_acc, (it | ks) != 0);
        }
        if (MC)
          umma_commit_mc(&q_empty[qs], 3);
        else
          umma_commit(&q_empty[qs]);
#if BB_BWD_DQ128
        // one N=D MMA group (N=64 instructions are issue-bound at ~48 clk vs 32 nominal,
        // tools/ubench_mma_rate.cu); both halves become ready together
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)  // K = 128 keys
          umma_ss(tmem + COL_DP, sw128_desc(ds_base + ks * 2048, 16384, 1024),
                  sw128_desc(k_base + ks * 2048, 16384, 1024), idesc_dq, ks > 0);
#pragma unroll
        for (int h = 0; h < D / 64; ++h) umma_commit(dq_full2[h]);
#else
#pragma unroll
        for (int h = 0; h < D / 64; ++h) {
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)  // K = 128 keys; N = head dims [64h, 64h+64)
            umma_ss(tmem + COL_DP + 64 * h, sw128_desc(ds_base + ks * 2048, 16384, 1024),
                    sw128_desc(k_base + ks * 2048 + 16384 * h, 16384, 1024), idesc_dq64, ks > 0);
          umma_commit(dq_full2[h]);
        }
#endif
      }
      __syncwarp();
      if (wn < n_work) {
        mbar_wait(do_full, (it + 1) & 1);
        if (lane == 0) BB_PROBE(6);
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          if (64 * g < D) {  // these dP^T columns held dQ half g of tile t
            mbar_wait(dq_free2[g], it & 1);
            tc_fence_after();
          }
          if (lane == 0 && g == 0) BB_PROBE(7);
          issue_dp_half(g);
        }
      }
      w = wn;
    }
    if (elect_one()) umma_commit(acc_full);
    __syncwarp();
  } else if (warp >= 4 && warp < 4 + 4 * NG) {
    // ------------------------------------------------ P / dS (two column groups) + epilogue
    const int g = (warp - 4) >> 2;             // column group: query columns [CPG*g, CPG*(g+1))
    const uint32_t quad = warp & 3;
    const int row = quad * 32 + lane;          // key row of S^T / dP^T
    const int ct = threadIdx.x - 128;          // 0..NCOMP-1
    const uint32_t t_lane = (quad * 32) << 16;
    const int64_t krow = c0 + row;
    const bool key_ok = krow < p.n_k;
    const bool ragged_k = c0 + 128 > p.n_k;  // CTA-uniform: the last key tile of a ragged shard
    const int64_t k_id = key_ok ? token_id(p.layout, p.k_device, krow) : 0;
    uint8_t* ds_tile = smem + L::DS_OFF;

    // Raw global value only: the transform is applied at the smem store so the load's
    // latency hides under the tile instead of stalling the loop top.
    auto load_vec = [&](int64_t w) {  // threads 0..127: lse of query ct; 128..255: delta
      const int64_t r = item_qt(w) * 128 + (ct & 127);
      if (r >= p.n_q) return ct < 128 ? -INFINITY : 0.f;
      const int64_t at = static_cast<int64_t>(item_head(w)) * p.n_q + r;
      return __ldg((ct < 128 ? p.lse : p.delta) + at);
    };
    auto vec_val = [&](float raw) {  // stored negated for the packed FFMA2 / FADD2 forms:
      if (ct >= 128) return -raw;       //   -D,  and -lse*log2e (-inf row -> -inf, so P = 0)
      return raw == -INFINITY ? -INFINITY : -raw * 1.4426950408889634f;
    };

    int64_t w = next_active(0);
    if (w < n_work && ct < 256) vec_s[ct] = vec_val(load_vec(w));
    named_bar_sync(3, NCOMP);
    uint32_t it = 0;
    while (w < n_work) {
      if (ct == 0) BB_PROBE(24);
      const int32_t cls = tile_cls(item_qt(w));
      const int64_t r0 = static_cast<int64_t>(item_qt(w)) * 128;
      const int64_t w_next = next_active(w + 1);
      const float v_next = (w_next < n_work && ct < 256) ? load_vec(w_next) : 0.f;  // prefetch under this tile
      const float* lse2 = vec_s;
      const float* dlt = lse2 + 128;
      uint4 bits = make_uint4(~0u, ~0u, ~0u, ~0u);
      if (cls == TILE_PARTIAL) bits = row_mask_bits(p.layout, p.mask, k_id, key_ok, p.q_device, r0, p.n_q, false);
      else if (!key_ok) bits = make_uint4(0u, 0u, 0u, 0u);
      if (ct == 0) BB_PROBE(16);
      mbar_wait(s_full, it & 1);
      if (ct == 0) BB_PROBE(17);
      tc_fence_after();

      // ---- P^T = exp2(S^T * scale*log2e - lse2[q]) -> TMEM (bf16 pairs, over S^T); kept packed.
      // lse2 of a 32-query chunk is read from smem before the TMEM load so the LDS latency
      // hides under it (tcgen05.wait::ld is a compiler memory barrier).  Only partial tiles
      // (and a ragged last key tile) pay for the per-element mask.
      uint32_t pk[CH][16];
      auto p_pass = [&](auto masked_tag) {
        constexpr bool MASKED = decltype(masked_tag)::value;
#pragma unroll
        for (int c2 = 0; c2 < CH; ++c2) {
          const int c = g * CH + c2;
          float l2[32];
#pragma unroll
          for (int i = 0; i < 32; i += 4) *reinterpret_cast<float4*>(&l2[i]) = *reinterpret_cast<const float4*>(&lse2[c * 32 + i]);
          float s[32];
          tmem_ld32(tmem + t_lane + COL_S + c * 32, s);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const int qc = c * 32 + i;
            const float2 x = __ffma2_rn(make_float2(s[i], s[i + 1]), make_float2(p.scale_log2, p.scale_log2),
                                        make_float2(l2[i], l2[i + 1]));  // l2 = -lse*log2e
            float e0 = ex2_approx(x.x);
            float e1 = ex2_approx(x.y);
            if (MASKED) {
              e0 = mask_bit(bits, qc) ? e0 : 0.f;
              e1 = mask_bit(bits, qc + 1) ? e1 : 0.f;
            }
            pk[c2][i / 2] = pack_bf16(e0, e1);
          }
          tmem_st16(tmem + t_lane + COL_S + c * 32, pk[c2]);
        }
      };
      if (cls == TILE_PARTIAL || ragged_k)
        p_pass(std::true_type{});
      else
        p_pass(std::false_type{});
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(p_full);
      if (ct == 0) BB_PROBE(18);

      // ---- dS^T = P^T o (dP^T - D[q]) -> smem (K-major rows = keys); the dK/dQ MMAs of the
      // previous tile must have finished reading the buffer: dP_g(t) is issued after dK(t-1)
      // and dQ(t-1), so its commit covers them.
      mbar_wait(dp_full2[NG == 2 ? g : 1], it & 1);
      if (NG != 2) mbar_wait(dp_full2[0], it & 1);
      if (ct == 0) BB_PROBE(19);
      tc_fence_after();
#pragma unroll
      for (int c2 = 0; c2 < CH; ++c2) {
        const int c = g * CH + c2;
        float dl[32];
#pragma unroll
        for (int i = 0; i < 32; i += 4) *reinterpret_cast<float4*>(&dl[i]) = *reinterpret_cast<const float4*>(&dlt[c * 32 + i]);
        float dp[32];
        tmem_ld32(tmem + t_lane + COL_DP + c * 32, dp);
        tmem_ld_wait();
#pragma unroll
        for (int a = 0; a < 32; a += 2) {  // dS^T packed in place of P^T
          const __nv_bfloat162 pb = *reinterpret_cast<const __nv_bfloat162*>(&pk[c2][a / 2]);
          const float2 ds = __fmul2_rn(__fadd2_rn(make_float2(dp[a], dp[a + 1]), make_float2(dl[a], dl[a + 1])),
                                       make_float2(__low2float(pb), __high2float(pb)));  // dl = -D
          pk[c2][a / 2] = pack_bf16(ds.x, ds.y);
        }
      }
#pragma unroll
      for (int c2 = 0; c2 < CH; ++c2)
#pragma unroll
        for (int i = 0; i < 32; i += 8)
          *reinterpret_cast<uint4*>(ds_tile + sw128_offset(row, (g * CH + c2) * 32 + i, 16384)) =
              make_uint4(pk[c2][i / 2], pk[c2][i / 2 + 1], pk[c2][i / 2 + 2], pk[c2][i / 2 + 3]);
      fence_async_smem();
      tc_fence_before();
      mbar_arrive(ds_full);
      if (ct == 0) BB_PROBE(20);

      named_bar_sync(3, NCOMP);  // everyone is done with this tile's lse / D
      if (w_next < n_work && ct < 256) vec_s[ct] = vec_val(v_next);
      named_bar_sync(3, NCOMP);
      if (ct == 0) BB_PROBE(23);
      w = w_next;
      ++it;
    }
    // ---- dK (scaled) and dV accumulate into the resident fp32 buffers
    if (it > 0) {
      mbar_wait(acc_full, 0);
      tc_fence_after();
      float* dk_row = p.dk + (krow * p.hkv + kv_head) * static_cast<int64_t>(D);
      float* dv_row = p.dv + (krow * p.hkv + kv_head) * static_cast<int64_t>(D);
#pragma unroll 1
      for (int ce = g; ce < D / 32; ce += NG) {
        const int dcol = ce * 32;
        float a[32], b[32];
        tmem_ld32(tmem + t_lane + COL_DK + dcol, a);
        tmem_ld32(tmem + t_lane + COL_DV + dcol, b);
        tmem_ld_wait();
        if (key_ok) {
          float4* k4 = reinterpret_cast<float4*>(dk_row + dcol);
          float4* v4 = reinterpret_cast<float4*>(dv_row + dcol);
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
  } else if (warp >= 4 + 4 * NG) {
    // ------------------------------------------------ dQ drain (TMEM lane = query row)
    // dQ(t) -> swizzled smem staging (two 32-column chunks at a time) -> TMA bulk reduce-add
    // (fp32) into the circulating dQ; each TMEM half is released (dq_free) as soon as it has
    // been read.
    const uint32_t quad = warp & 3;
    const int row = quad * 32 + lane;
    const uint32_t t_lane = (quad * 32) << 16;
    const bool issuer = (quad == 0 && lane == 0);
    uint8_t* stg = smem + L::STG_OFF;
    constexpr int CHUNKS = D / 32;
    auto stage = [&](const float (&v)[32], int slot) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 x = make_float4(v[4 * i] * p.scale, v[4 * i + 1] * p.scale, v[4 * i + 2] * p.scale,
                                     v[4 * i + 3] * p.scale);
        *reinterpret_cast<float4*>(stg + slot * 16384 + row * 128 + ((i ^ (row & 7)) << 4)) = x;
      }
    };
    uint32_t it = 0;
    for (int64_t w = next_active(0); w < n_work; w = next_active(w + 1), ++it) {
      const int32_t qrow0 = static_cast<int32_t>(item_qt(w) * 128);
      const int hcol = item_head(w) * D;
      if (row == 0) BB_PROBE(21);
#pragma unroll
      for (int half = 0; half < CHUNKS / 2; ++half) {
        mbar_wait(dq_full2[half], it & 1);
        tc_fence_after();
        float a[32], b[32];
        tmem_ld32(tmem + t_lane + COL_DP + half * 64, a);
        tmem_ld32(tmem + t_lane + COL_DP + half * 64 + 32, b);
        tmem_ld_wait();
        tc_fence_before();  // this half of dQ(t) is read: release its TMEM columns
        mbar_arrive(dq_free2[half]);
        if (issuer) bulk_wait_read<0>();  // previous reduce finished reading the staging
        named_bar_sync(4, 128);
        stage(a, 0);
        stage(b, 1);
        fence_async_smem();
        named_bar_sync(4, 128);
        if (issuer) {
          tma_reduce_add_2d(&tdq, stg, hcol + half * 64, qrow0);
          tma_reduce_add_2d(&tdq, stg + 16384, hcol + half * 64 + 32, qrow0);
          bulk_commit();
        }
      }
      if (row == 0) BB_PROBE(22);
    }
    if (issuer) bulk_wait<0>();
  }

  tc_fence_before();
  if (MC)
    cluster_sync();  // no CTA leaves while its partner may still multicast into it
  else
    __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

template <int D>
int launch_bwd_d(const bb_attn_bwd_args& a, cudaStream_t st) {
  if ((a.n_q + 127) / 128 > MAX_QT)
    return set_error(BB_ERR_UNSUPPORTED, "attn_bwd: query shard of %lld rows exceeds %d (raise MAX_QT)", (long long)a.n_q, MAX_QT * 128);
  CUtensorMap tq, tk, tv, tdo, tdq;
  const uint64_t qrow = static_cast<uint64_t>(a.hq) * D * 2, krow = static_cast<uint64_t>(a.hkv) * D * 2;
  if (!make_tmap_bf16_2d(&tq, a.q, static_cast<uint64_t>(a.hq) * D, a.n_q, qrow, 64, 128) ||
      !make_tmap_bf16_2d(&tdo, a.dout, static_cast<uint64_t>(a.hq) * D, a.n_q, qrow, 64, 128) ||
      !make_tmap_bf16_2d(&tk, a.k, static_cast<uint64_t>(a.hkv) * D, a.n_k, krow, 64, 128) ||
      !make_tmap_bf16_2d(&tv, a.v, static_cast<uint64_t>(a.hkv) * D, a.n_k, krow, 64, 128) ||
      !make_tmap_2d(&tdq, a.dq, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, static_cast<uint64_t>(a.hq) * D, a.n_q, qrow * 2, 32, 128))
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
  p.kv_head0 = a.kv_head_begin;
  const unsigned n_heads = static_cast<unsigned>((a.kv_head_end ? a.kv_head_end : a.hkv) - a.kv_head_begin);
  p.scale = a.softmax_scale;
  p.scale_log2 = a.softmax_scale * 1.4426950408889634f;
  p.q_device = a.q_device;
  p.k_device = a.k_device;
  p.layout = make_layoutd(a.layout);
  p.mask = make_maskd(a.mask);
  p.probe = debug_probe_buffer();
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
  const unsigned n_kt = static_cast<unsigned>((a.n_k + 127) / 128);
  if (MC) {  // clusters of two adjacent key tiles (an odd count gets an empty partner)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((n_kt + 1) & ~1u, n_heads);
    cfg.blockDim = dim3(BWD_THREADS);
    cfg.dynamicSmemBytes = BwdSmem<D>::BYTES;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (check_cuda(cudaLaunchKernelEx(&cfg, kern, tq, tk, tv, tdo, tdq, p), "attn_bwd cluster launch"))
      return BB_ERR_CUDA;
  } else {
    dim3 grid(n_kt, n_heads);
    kern<<<grid, BWD_THREADS, BwdSmem<D>::BYTES, st>>>(tq, tk, tv, tdo, tdq, p);
  }
  return check_launch("attn_bwd_kernel");
}

}  // namespace

int launch_attn_bwd(const bb_attn_bwd_args& a, cudaStream_t st) {
  if (a.head_dim == 128) return launch_bwd_d<128>(a, st);
  if (a.head_dim == 64) return launch_bwd_d<64>(a, st);
  return set_error(BB_ERR_UNSUPPORTED, "attn_bwd: head_dim %d (kernels take 64 or 128)", a.head_dim);
}

}  // namespace bb
