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
//   warp 0      TMA: K, V once; Q (2 stages) and dO per query tile
//   warp 1      MMA: S^T = K Q^T, dP^T = V dO^T          (SS, M = keys, N = 128 queries)
//                    dV += P^T dO   with P^T read from TMEM (TS, no smem round trip)
//                    dK += dS^T Q   with dS^T read from TMEM (TS, over its own dP^T columns)
//                    dQ = dS K                          (SS; dS^T read MN-major from smem)
//   warp 2      TMEM allocator
//   warps 4-11  two groups of 4 warps, each owning half of the 128 query columns
//               (group g: TMEM columns of its half, all 128 lanes):
//               P^T -> TMEM (bf16, in place over S^T), dS^T -> TMEM (over dP^T) and
//               SWIZZLE_128B smem,
//               final dK / dV read-modify-write.
//   warps 12-15 dQ drain: the whole dQ tile TMEM -> registers at once (releasing its
//               columns for the next dP^T), then 32-column chunks through two 16 KB smem
//               staging slots into TMA bulk reduce-adds (fp32) on the circulating dQ.
// TMEM: S^T / P^T [0,128), dP^T then dQ [128,256), dV [256,256+D), dK [256+D,256+2D).
//
// Throughput bound (tools/ubench_reduce.cu): a TMA reduce-add moves ~22.6 B/clk per SM
// with every SM busy (L2-bound chip-wide), so the 64 KB dQ tile of D = 128 needs ~2.9k
// cycles against 2.56k of tensor work: the drain must never idle, and the MMA chain must
// never wait on the drain.  Registers are rebalanced with setmaxnreg so the drain warps can
// hold a full dQ row (128 fp32) and hand its TMEM columns back in one go.
#include <cuda_runtime.h>

#include <type_traits>

#include "bb_host.h"
#include "bb_mask.cuh"
#include "bb_ptx.cuh"

namespace bb {
namespace {

constexpr int NG = 2;                      // compute column groups (4 warps each)
constexpr int CPG = 128 / NG;              // query columns per group
constexpr int CH = CPG / 32;               // 32-column chunks per group
constexpr int NCOMP = NG * 128;            // compute threads
constexpr int BWD_THREADS = 128 + NCOMP + 128;  // control warps + compute + dQ drain
constexpr int MAX_QT = 4096;  // query tiles per shard the class table holds (n_q <= 524288)
// setmaxnreg budget (65536 registers for 512 threads): control 72, compute 144, drain 152
// (no spills at D = 128; a spill here reads local memory through an L1 that the 226 KB of
// shared memory leaves at ~2 KB, i.e. from L2).
constexpr uint32_t REGS_CTRL = 72, REGS_COMP = 144, REGS_DRAIN = 152;
static_assert(REGS_CTRL * 128 + REGS_COMP * NCOMP + REGS_DRAIN * 128 <= 65536, "register budget");

template <int D>
struct BwdSmem {
  static constexpr uint32_t TILE = 128 * D * 2;
  static constexpr uint32_t K_OFF = 0;
  static constexpr uint32_t V_OFF = K_OFF + TILE;
  static constexpr uint32_t Q_OFF = V_OFF + TILE;    // 2 stages
  static constexpr uint32_t DO_OFF = Q_OFF + 2 * TILE;
  static constexpr uint32_t DS_OFF = DO_OFF + TILE;  // dS^T, 128 keys x 128 queries bf16
  static constexpr uint32_t STG_OFF = DS_OFF + 128 * 128 * 2;  // 2 slots x [128 x 32] fp32 dQ staging
  static constexpr uint32_t VEC_OFF = STG_OFF + 2 * 16384;     // per column group: [lse2 64 | -D 64]
  static constexpr uint32_t BAR_OFF = VEC_OFF + NG * 512;
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
  int64_t lse_ld;  // row length of the caller's lse / delta arrays (>= n_q: a sub-shard launch)
  int32_t hq, hkv;
  int32_t kv_head0;  // first kv head of this launch (grid.y covers the range)
  float scale, scale_log2;
  int32_t q_device, k_device;
  LayoutD layout;
  MaskD mask;
  long long* probe;  // diagnostics: per-phase clock64() of CTA (0,0), see bb_debug_probe
};

#ifndef BB_WITH_PROBES  // per-phase clock64 probes: diagnostic builds only (tools/variant.py probes BB_WITH_PROBES)
#define BB_PROBE(slot) \
  do {                 \
  } while (0)
#define BWD_CTA_MARK(k) \
  do {                  \
  } while (0)
#else
// per-CTA timeline (tools/cta_timeline.py --kernel bwd): SM id, globaltimer at entry / prologue
// done / compute loop done / dK-dV stored / exit
#define BWD_CTA_MARK(k)                                                                                   \
  do {                                                                                                    \
    const int64_t cta_ = static_cast<int64_t>(blockIdx.y) * gridDim.x + blockIdx.x;                        \
    if (p.probe && 4096 + cta_ * 8 + 7 < kProbeEntries) {                                                  \
      unsigned long long t_;                                                                              \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                              \
      unsigned smid_;                                                                                     \
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid_));                                                  \
      p.probe[4096 + cta_ * 8 + 1 + (k)] = static_cast<long long>(t_);                                     \
      if ((k) == 0) p.probe[4096 + cta_ * 8] = smid_;                                                      \
    }                                                                                                     \
  } while (0)
#define BB_PROBE(slot)                                                                 \
  do {                                                                                 \
    if (p.probe && blockIdx.x == 0 && blockIdx.y == 0 && it < 16) p.probe[it * 32 + (slot)] = clock64(); \
  } while (0)
#endif

__device__ __forceinline__ int32_t bwd_class(const BwdParams& p, int64_t qt, int64_t c0) {
  const int64_t r0 = qt * 128, r1 = min(r0 + 128, p.n_q);
  const int64_t c1 = min(c0 + 128, p.n_k);
  return classify_tile(p.layout, p.mask, p.q_device, r0, r1, p.k_device, c0, c1, c1 - c0 == 128);
}

template <int D>
__global__ void __launch_bounds__(BWD_THREADS, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                    const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo,
                    const __grid_constant__ CUtensorMap tdq, const __grid_constant__ CUtensorMap tdk,
                    const __grid_constant__ CUtensorMap tdv, const __grid_constant__ BwdParams p) {
  using L = BwdSmem<D>;
  constexpr int PANELS = D / 64;
  constexpr uint32_t COL_S = 0, COL_DP = 128, COL_DV = 256, COL_DK = 256 + D;
  extern __shared__ __align__(1024) uint8_t smem[];
  if (threadIdx.x == 0) BWD_CTA_MARK(0);
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
  uint64_t* dq_free = bars + 12;  // the drain has read the whole dQ tile: its columns take dP^T
  uint64_t* acc_full = bars + 13;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);

  const int kv_head = p.kv_head0 + static_cast<int>(blockIdx.y);
  const int group = p.hq / p.hkv;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 128;  // low key tiles carry the most work
  // Query tiles that can touch this key tile (two binary searches, every thread), then the
  // work items (query head of the GQA group, query tile in [q_lo, q_hi)).
  int64_t q_lo = 0, q_hi = 0;
  if (c0 < p.n_k)
    active_runs(p.layout, p.mask, token_id(p.layout, p.k_device, c0),
                token_id(p.layout, p.k_device, min(c0 + 128, p.n_k) - 1), p.q_device, p.n_q, false, q_lo, q_hi);
  const uint32_t nr = static_cast<uint32_t>(q_hi - q_lo);
  // Each CTA walks its query tiles starting at a different one (rotation by its key tile): in a
  // fully visible block every CTA's range is the same, and in lockstep the ~148 resident CTAs
  // reduce-added into the same dQ tile at once (a 1M-token 2-GPU remote step ran at 795 TF/s
  // against 1015 for the causal own step, whose CTAs start at their own diagonal).
  const uint32_t rot = nr ? static_cast<uint32_t>(blockIdx.x) % nr : 0u;
  auto phys = [&](uint32_t li) {  // logical item index -> position in [q_lo, q_hi)
    const uint32_t x = li + rot;
    return x >= nr ? x - nr : x;
  };
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
    tma_prefetch(&tdk);
    tma_prefetch(&tdv);
    mbar_init(kv_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
    }
    mbar_init(do_full, 1);
    mbar_init(do_empty, 1);
    mbar_init(s_full, 1);
    mbar_init(p_full, NCOMP);
    mbar_init(dp_full, 1);
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
      if (4 * b + k < nr) byte |= static_cast<uint32_t>(bwd_class(p, q_lo + 4 * b + k, c0)) << (2 * k);
    cls_tab[b] = static_cast<uint8_t>(byte);
  }
  auto tile_cls = [&](uint32_t qt) {
    const uint32_t x = qt - static_cast<uint32_t>(q_lo);
    return static_cast<int32_t>((cls_tab[x >> 2] >> ((x & 3) * 2)) & 3);
  };
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) BWD_CTA_MARK(1);
  const uint32_t tmem = *tmem_slot;

  // Work items: (query head of the GQA group, query tile) in order, skipping masked tiles.
  // (nr == 0 must end at once: the class table is empty, and a head step must re-check the
  // range before reading a table entry)
  auto next_active = [&](int64_t w) {
    if (nr == 0) return n_work;
    for (;;) {
      if ((w & 0xFFFF) >= nr) w = ((w >> 16) + 1) << 16;
      if (w >= n_work) return n_work;
      if (tile_cls(static_cast<uint32_t>(q_lo) + phys(static_cast<uint32_t>(w & 0xFFFF))) != TILE_SKIP) return w;
      ++w;
    }
  };
  auto item_qt = [&](int64_t w) { return static_cast<uint32_t>(q_lo) + phys(static_cast<uint32_t>(w & 0xFFFF)); };
  auto item_head = [&](int64_t w) { return kv_head * group + static_cast<int>(w >> 16); };

  if (warp < 4) {
    setmaxnreg_dec<REGS_CTRL>();
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
          for (int pn = 0; pn < PANELS; ++pn)
            tma_load_2d(smem + L::Q_OFF + qs * L::TILE + pn * 16384, &tq, &q_full[qs], h * D + pn * 64, qrow0);
          mbar_wait(do_empty, (it & 1) ^ 1);
          BB_PROBE(2);
          mbar_expect_tx(do_full, L::TILE);
          for (int pn = 0; pn < PANELS; ++pn)
            tma_load_2d(smem + L::DO_OFF + pn * 16384, &tdo, do_full, h * D + pn * 64, qrow0);
          // dO is single-buffered: dO(t+1) can only be loaded once dV(t) has read dO(t), which
          // puts its HBM latency (~2k cycles under load) between dV(t) and dP(t+1).  Warm L2
          // with the next item's dO and Q now, a whole tile ahead, so that load hits L2.
          const int64_t wn = next_active(w + 1);
          if (wn < n_work) {
            const int32_t nrow0 = static_cast<int32_t>(item_qt(wn) * 128);
            const int nh = item_head(wn);
            for (int pn = 0; pn < PANELS; ++pn) {
              tma_prefetch_l2_2d(&tdo, nh * D + pn * 64, nrow0);
              tma_prefetch_l2_2d(&tq, nh * D + pn * 64, nrow0);
            }
          }
        }
      }
    } else if (warp == 1) {
      // ------------------------------------------------ MMA issuer
      // Per tile t:  dV(t) [P(t) ready], S(t+1), dK(t) dQ(t) [dS(t) ready], dP(t+1) [dQ(t) read].
      // S(t+1) goes out as soon as dV(t) has been issued (the tensor pipe is in order, so dV(t)
      // reads P(t) from the S columns before S(t+1) overwrites them); the compute warps then
      // start P(t+1) while dK(t)/dQ(t) run, and dP(t+1) follows dQ(t) as soon as the drain has
      // pulled dQ(t) into registers, as one N=128 group.
      constexpr uint32_t idesc_st = idesc_bf16(128, 128, false, false);  // S^T, dP^T
      constexpr uint32_t idesc_acc = idesc_bf16(128, D, false, true);    // dV (TS), dK: B MN-major
      constexpr uint32_t idesc_dq = idesc_bf16(128, D, true, true);      // dQ: A = dS (MN), B = K (MN)
      const uint32_t k_base = smem_u32(smem + L::K_OFF), v_base = smem_u32(smem + L::V_OFF);
      const uint32_t do_base = smem_u32(smem + L::DO_OFF), ds_base = smem_u32(smem + L::DS_OFF);
      auto issue_s = [&](uint32_t qs) {
        const uint32_t q_base = smem_u32(smem + L::Q_OFF + qs * L::TILE);
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks) {
            const uint32_t off = (ks >> 2) * 16384 + (ks & 3) * 32;
            umma_ss(tmem + COL_S, sw128_desc(k_base + off, 16, 1024), sw128_desc(q_base + off, 16, 1024), idesc_st,
                    ks > 0);
          }
          umma_commit(s_full);
        }
        __syncwarp();
      };
      auto issue_dp = [&]() {  // dP^T = V . dO^T
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks) {
            const uint32_t off = (ks >> 2) * 16384 + (ks & 3) * 32;
            umma_ss(tmem + COL_DP, sw128_desc(v_base + off, 16, 1024), sw128_desc(do_base + off, 16, 1024), idesc_st,
                    ks > 0);
          }
          umma_commit(dp_full);
        }
        __syncwarp();
      };

      mbar_wait(kv_full, 0);
      int64_t w = next_active(0);
      // The item after next is looked up while the issuer waits on do_full / dq_free (the
      // class-table walk is shared loads, which queue behind the SS MMAs' operand reads), not
      // at the loop top between dP(t+1) and dV(t+1).
      int64_t wn = w < n_work ? next_active(w + 1) : n_work;
      if (w < n_work) {
        mbar_wait(&q_full[0], 0);
        tc_fence_after();
        issue_s(0);
        mbar_wait(do_full, 0);
        tc_fence_after();
        issue_dp();
      }
      for (uint32_t it = 0; w < n_work; ++it) {
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
          for (int ks = 0; ks < 8; ++ks) {  // dS^T of q chunk c packed over its own dP^T columns (TS)
            const uint32_t a_tmem = tmem + COL_DP + (ks >> 1) * 32 + (ks & 1) * 8;
            umma_ts(tmem + COL_DK, a_tmem, sw128_desc(q_base + ks * 2048, 16384, 1024), idesc_acc, (it | ks) != 0);
          }
          umma_commit(&q_empty[qs]);
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)  // K = 128 keys
            umma_ss(tmem + COL_DP, sw128_desc(ds_base + ks * 2048, 16384, 1024),
                    sw128_desc(k_base + ks * 2048, 16384, 1024), idesc_dq, ks > 0);
          umma_commit(dq_full);
        }
        __syncwarp();
        if (lane == 0) BB_PROBE(10);
        const int64_t wnn = wn < n_work ? next_active(wn + 1) : n_work;
        if (wn < n_work) {
          mbar_wait(do_full, (it + 1) & 1);
          if (lane == 0) BB_PROBE(6);
          mbar_wait(dq_free, it & 1);  // these dP^T columns held dQ(t)
          if (lane == 0) BB_PROBE(7);
          tc_fence_after();
          issue_dp();
          if (lane == 0) BB_PROBE(11);
        }
        w = wn;
        wn = wnn;
      }
      if (elect_one()) umma_commit(acc_full);
      __syncwarp();
    }
  } else if (warp < 4 + 4 * NG) {
    // ------------------------------------------------ P / dS (two column groups) + epilogue
    setmaxnreg_inc<REGS_COMP>();
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

    // lse / D of the group's 64 query columns live in a per-group smem copy, so only the 128
    // threads of a group synchronise on it (named barrier 5 + g), never the two groups with
    // each other.  Thread gt of the group fetches one value for the next item during the dS
    // pass (gt < 64: lse of column 64g + gt; else D of column 64g + gt - 64); the transform is
    // applied at the store so the load's latency hides there.
    const int gt = ct & 127;
    float* vec_g = reinterpret_cast<float*>(smem + L::VEC_OFF + g * 512);  // [lse2 64 | -D 64]
    const float* lse2 = vec_g - CPG * g;  // indexed by the tile's query column (group g: [64g, 64g+64))
    const float* dlt = vec_g + 64 - CPG * g;
    auto load_vec = [&](int64_t w) {
      const int64_t r = static_cast<int64_t>(item_qt(w)) * 128 + CPG * g + (gt & 63);
      if (r >= p.n_q) return gt < 64 ? -INFINITY : 0.f;
      return __ldg((gt < 64 ? p.lse : p.delta) + static_cast<int64_t>(item_head(w)) * p.lse_ld + r);
    };
    auto store_vec = [&](float raw) {  // stored negated for the packed FFMA2 / FADD2 forms:
      vec_g[gt] = gt >= 64 ? -raw : raw == -INFINITY ? -INFINITY : -raw * 1.4426950408889634f;  // -D, -lse*log2e
    };
    auto group_sync = [&]() { named_bar_sync(5 + g, 128); };

    // The next item, its class and its lse / D are looked up while this tile's dP^T is still
    // in flight (between the P and dS passes), so the loop top is just the S^T wait: the
    // class-table walk is a chain of dependent shared loads.
    int64_t w = next_active(0);
    int32_t cls = w < n_work ? tile_cls(item_qt(w)) : TILE_SKIP;
    if (w < n_work) store_vec(load_vec(w));
    uint32_t it = 0;
    while (w < n_work) {
      if (ct == 0) BB_PROBE(24);
      if (ct == 128) BB_PROBE(25);
      uint4 bits = make_uint4(~0u, ~0u, ~0u, ~0u);
      if (cls == TILE_PARTIAL)
        bits = row_mask_bits(p.layout, p.mask, k_id, key_ok, p.q_device, static_cast<int64_t>(item_qt(w)) * 128,
                             p.n_q, false);
      else if (!key_ok)
        bits = make_uint4(0u, 0u, 0u, 0u);
      if (ct == 0) BB_PROBE(16);
      mbar_wait(s_full, it & 1);
      if (ct == 0) BB_PROBE(17);
      if (ct == 128) BB_PROBE(26);
      tc_fence_after();
      group_sync();  // this tile's lse / D (stored at the end of the last one) are visible

      // ---- P^T = exp2(S^T * scale*log2e - lse2[q]) -> TMEM (bf16 pairs, over S^T); kept packed.
      // lse2 of a 32-query chunk is read from smem before the TMEM load so the LDS latency
      // hides under it (tcgen05.wait::ld is a compiler memory barrier).  Only partial tiles
      // (and a ragged last key tile) pay for the per-element mask.
      // Every shared-memory load this tile needs is issued well ahead of its first use: under the
      // SS MMAs' operand fetch (128 B/clk, the whole port) an LDS waits hundreds of cycles, and
      // the warp issues in order.  lse of both chunks now; the class byte of the next query
      // tile now (read after the P pass); -D of both chunks under the last S chunk's TMEM load.
      float l2[CH][32];
#pragma unroll
      for (int c2 = 0; c2 < CH; ++c2)
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *reinterpret_cast<float4*>(&l2[c2][i]) = *reinterpret_cast<const float4*>(&lse2[(g * CH + c2) * 32 + i]);
      const bool same_head = (static_cast<uint32_t>(w & 0xFFFF) + 1) < nr;  // next item: same head, next tile
      const uint32_t nxt = phys(static_cast<uint32_t>(w & 0xFFFF) + 1);      // its class-table index
      const uint32_t cls_byte = same_head ? cls_tab[nxt >> 2] : 0u;
      uint32_t pk[CH][16];
      float dl[CH][32];
      auto load_dl = [&]() {
#pragma unroll
        for (int c2 = 0; c2 < CH; ++c2)
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4*>(&dl[c2][i]) = *reinterpret_cast<const float4*>(&dlt[(g * CH + c2) * 32 + i]);
      };
      auto p_pass = [&](auto masked_tag) {
        constexpr bool MASKED = decltype(masked_tag)::value;
#pragma unroll
        for (int c2 = 0; c2 < CH; ++c2) {
          const int c = g * CH + c2;
          float s[32];
          tmem_ld32(tmem + t_lane + COL_S + c * 32, s);
          if (c2 == CH - 1) load_dl();  // -D of both chunks: issued under the last chunk's TMEM load
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const int qc = c * 32 + i;
            const float2 x = __ffma2_rn(make_float2(s[i], s[i + 1]), make_float2(p.scale_log2, p.scale_log2),
                                        make_float2(l2[c2][i], l2[c2][i + 1]));  // l2 = -lse*log2e
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
      if (ct == 128) BB_PROBE(27);
      // Next item: the following query tile of the same head unless the prefetched class says
      // it is masked out (or the range ends); the general walk only then.
      int64_t w_next;
      int32_t cls_next;
      const int32_t c_adj = static_cast<int32_t>((cls_byte >> ((nxt & 3) * 2)) & 3);
      if (same_head && c_adj != TILE_SKIP) {
        w_next = w + 1;
        cls_next = c_adj;
      } else {
        w_next = next_active(w + 1);
        cls_next = w_next < n_work ? tile_cls(item_qt(w_next)) : TILE_SKIP;
      }
      const float v_next = w_next < n_work ? load_vec(w_next) : 0.f;  // lands during the dS pass

      // ---- dS^T = P^T o (dP^T - D[q]) -> smem (K-major rows = keys); the dK/dQ MMAs of the
      // previous tile must have finished reading the buffer: dP(t) is issued after dK(t-1)
      // and dQ(t-1), so its commit covers them.
      if (ct == 0) BB_PROBE(30);
      if (ct == 128) BB_PROBE(31);
      mbar_wait(dp_full, it & 1);
      if (ct == 0) BB_PROBE(19);
      if (ct == 128) BB_PROBE(28);
      tc_fence_after();
#pragma unroll
      for (int c2 = 0; c2 < CH; ++c2) {
        const int c = g * CH + c2;
        float dp[32];
        tmem_ld32(tmem + t_lane + COL_DP + c * 32, dp);
        tmem_ld_wait();
#pragma unroll
        for (int a = 0; a < 32; a += 2) {  // dS^T packed in place of P^T
          const __nv_bfloat162 pb = *reinterpret_cast<const __nv_bfloat162*>(&pk[c2][a / 2]);
          const float2 ds = __fmul2_rn(__fadd2_rn(make_float2(dp[a], dp[a + 1]), make_float2(dl[c2][a], dl[c2][a + 1])),
                                       make_float2(__low2float(pb), __high2float(pb)));  // dl = -D
          pk[c2][a / 2] = pack_bf16(ds.x, ds.y);
        }
        tmem_st16(tmem + t_lane + COL_DP + c * 32, pk[c2]);  // dK's A operand (TS)
      }
#pragma unroll
      for (int c2 = 0; c2 < CH; ++c2)
#pragma unroll
        for (int i = 0; i < 32; i += 8)
          *reinterpret_cast<uint4*>(ds_tile + sw128_offset(row, (g * CH + c2) * 32 + i, 16384)) =
              make_uint4(pk[c2][i / 2], pk[c2][i / 2 + 1], pk[c2][i / 2 + 2], pk[c2][i / 2 + 3]);
      fence_async_smem();
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(ds_full);
      if (ct == 0) BB_PROBE(20);
      if (ct == 128) BB_PROBE(29);

      group_sync();  // the group is done with this tile's lse / D
      if (w_next < n_work) store_vec(v_next);
      if (ct == 0) BB_PROBE(23);
      w = w_next;
      cls = cls_next;
      ++it;
    }
    // ---- dK (scaled) and dV accumulate into the resident fp32 buffers: staged in shared memory
    // (Q / dO / dS buffers, free once the last MMA retired) and added by TMA bulk reduce-add, so
    // the CTA never waits on global loads (a register read-modify-write took ~20-25 us per CTA:
    // its loads queue behind the other SMs' dQ reduce traffic in L2)
    if (ct == 0) BWD_CTA_MARK(2);
    if (it > 0) {
      mbar_wait(acc_full, 0);
      if (ct == 0) BWD_CTA_MARK(5);
      tc_fence_after();
      uint8_t* stage_k = smem + L::Q_OFF;   // D/32 chunks of [128 keys x 32] fp32, SWIZZLE_128B
      uint8_t* stage_v = smem + L::DO_OFF;  // (dO + dS buffers)
#pragma unroll 1
      for (int ce = g; ce < D / 32; ce += NG) {
        const int dcol = ce * 32;
        float a[32], b[32];
        tmem_ld32(tmem + t_lane + COL_DK + dcol, a);
        tmem_ld32(tmem + t_lane + COL_DV + dcol, b);
        tmem_ld_wait();
        uint8_t* kd = stage_k + ce * 16384 + row * 128;
        uint8_t* vd = stage_v + ce * 16384 + row * 128;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          *reinterpret_cast<float4*>(kd + ((i ^ (row & 7)) << 4)) =
              make_float4(a[4 * i] * p.scale, a[4 * i + 1] * p.scale, a[4 * i + 2] * p.scale, a[4 * i + 3] * p.scale);
          *reinterpret_cast<float4*>(vd + ((i ^ (row & 7)) << 4)) = make_float4(b[4 * i], b[4 * i + 1], b[4 * i + 2], b[4 * i + 3]);
        }
      }
      fence_async_smem();
      named_bar_sync(7, NCOMP);
      if (ct == 0) {  // rows past n_k (a ragged last key tile) fall outside the maps and are dropped
        for (int ce = 0; ce < D / 32; ++ce) {
          tma_reduce_add_2d(&tdk, stage_k + ce * 16384, kv_head * D + ce * 32, static_cast<int32_t>(c0));
          tma_reduce_add_2d(&tdv, stage_v + ce * 16384, kv_head * D + ce * 32, static_cast<int32_t>(c0));
        }
        bulk_commit();
        bulk_wait<0>();
      }
    }
  } else {
    // ------------------------------------------------ dQ drain (TMEM lane = query row)
    // The whole dQ(t) row comes out of TMEM at once (D fp32 registers per thread) and its
    // columns are released (dq_free) before any staging, so dP(t+1) never waits on the
    // reduce; then D/32 chunks of 32 columns alternate between the two 16 KB staging slots,
    // each a TMA bulk reduce-add (fp32) into the circulating dQ.  A slot is restaged once the
    // reduce issued from it two chunks earlier has finished reading it (bulk_wait_read<1>).
    setmaxnreg_inc<REGS_DRAIN>();
    constexpr int CHUNKS = D / 32;
    // (16-column chunks through 8 KB SWIZZLE_64B slots measured 10 % slower: twice the
    // barriers per tile, and half-line reduce rows.
    // (An FMA-pipe exp2 share in the P pass, 1/8 .. 1/2 of the pairs: no change, 989-996 vs
    // 1000 TF/s -- the P pass is not MUFU-bound here.)
    // Coalesced red.global.add.v4.f32 (4 rows x 128 B per warp instruction, read back from the
    // staging slot) for every other chunk, TMA reduce for the rest: 903 vs 1014 TF/s.
    // red.global.add.v4.f32 from registers for half the columns measured 20 % slower overall:
    // the one-row-per-lane pattern floods the LSU / MIO queue the compute warps' tcgen05.ld/st
    // go through, doubling their P pass.)
    const uint32_t quad = warp & 3;
    const int row = quad * 32 + lane;
    const uint32_t t_lane = (quad * 32) << 16;
    const bool issuer = (quad == 0 && lane == 0);
    uint8_t* stg = smem + L::STG_OFF;
    uint32_t it = 0, chunk = 0;
    for (int64_t w = next_active(0); w < n_work; w = next_active(w + 1), ++it) {
      const int32_t qrow0 = static_cast<int32_t>(item_qt(w) * 128);
      const int hcol = item_head(w) * D;
      if (row == 0) BB_PROBE(21);
      mbar_wait(dq_full, it & 1);
      tc_fence_after();
      float v[CHUNKS][32];
#pragma unroll
      for (int c = 0; c < CHUNKS; ++c) tmem_ld32(tmem + t_lane + COL_DP + c * 32, v[c]);
      tmem_ld_wait();
      tc_fence_before();  // dQ(t) is in registers: its TMEM columns go back to dP(t+1)
      mbar_arrive(dq_free);
#pragma unroll
      for (int c = 0; c < CHUNKS; ++c, ++chunk) {
        const uint32_t slot = chunk & 1;
        if (issuer) bulk_wait_read<1>();  // the reduce issued from this slot has read it
        named_bar_sync(4, 128);
        uint8_t* dst = stg + slot * 16384 + row * 128;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          *reinterpret_cast<float4*>(dst + ((i ^ (row & 7)) << 4)) =
              make_float4(v[c][4 * i] * p.scale, v[c][4 * i + 1] * p.scale, v[c][4 * i + 2] * p.scale,
                          v[c][4 * i + 3] * p.scale);
        fence_async_smem();
        named_bar_sync(4, 128);
        if (issuer) {
          tma_reduce_add_2d(&tdq, stg + slot * 16384, hcol + c * 32, qrow0);
          bulk_commit();
        }
      }
      if (row == 0) BB_PROBE(22);
    }
    if (issuer) bulk_wait<0>();
  }

  tc_fence_before();
  if (warp == 4 && lane == 0) BWD_CTA_MARK(3);  // this compute warp's dK / dV rows stored
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
  if (threadIdx.x == 0) BWD_CTA_MARK(4);
}

template <int D>
int launch_bwd_d(const bb_attn_bwd_args& a, cudaStream_t st, int64_t lse_ld) {
  if ((a.n_q + 127) / 128 > MAX_QT)  // bb_api.cu splits larger shards before they get here
    return set_error(BB_ERR_UNSUPPORTED, "attn_bwd: query shard of %lld rows exceeds %d (raise MAX_QT)", (long long)a.n_q, MAX_QT * 128);
  CUtensorMap tq, tk, tv, tdo, tdq, tdk, tdv;
  const uint64_t qrow = static_cast<uint64_t>(a.hq) * D * 2, krow = static_cast<uint64_t>(a.hkv) * D * 2;
  if (!make_tmap_bf16_2d(&tq, a.q, static_cast<uint64_t>(a.hq) * D, a.n_q, qrow, 64, 128) ||
      !make_tmap_bf16_2d(&tdo, a.dout, static_cast<uint64_t>(a.hq) * D, a.n_q, qrow, 64, 128) ||
      !make_tmap_bf16_2d(&tk, a.k, static_cast<uint64_t>(a.hkv) * D, a.n_k, krow, 64, 128) ||
      !make_tmap_bf16_2d(&tv, a.v, static_cast<uint64_t>(a.hkv) * D, a.n_k, krow, 64, 128) ||
      !make_tmap_2d(&tdq, a.dq, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, static_cast<uint64_t>(a.hq) * D, a.n_q, qrow * 2, 32, 128) ||
      !make_tmap_2d(&tdk, a.dk, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, static_cast<uint64_t>(a.hkv) * D, a.n_k, krow * 2, 32, 128) ||
      !make_tmap_2d(&tdv, a.dv, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, static_cast<uint64_t>(a.hkv) * D, a.n_k, krow * 2, 32, 128))
    return BB_ERR_CUDA;
  BwdParams p{};
  p.lse = a.lse;
  p.delta = a.delta;
  p.dq = a.dq;
  p.dk = a.dk;
  p.dv = a.dv;
  p.n_q = a.n_q;
  p.lse_ld = lse_ld;
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
  dim3 grid(n_kt, n_heads);
  kern<<<grid, BWD_THREADS, BwdSmem<D>::BYTES, st>>>(tq, tk, tv, tdo, tdq, tdk, tdv, p);
  return check_launch("attn_bwd_kernel");
}

}  // namespace

int launch_attn_bwd(const bb_attn_bwd_args& a, cudaStream_t st, int64_t lse_ld) {
  if (a.head_dim == 128) return launch_bwd_d<128>(a, st, lse_ld);
  if (a.head_dim == 64) return launch_bwd_d<64>(a, st, lse_ld);
  return set_error(BB_ERR_UNSUPPORTED, "attn_bwd: head_dim %d (kernels take 64 or 128)", a.head_dim);
}

}  // namespace bb
