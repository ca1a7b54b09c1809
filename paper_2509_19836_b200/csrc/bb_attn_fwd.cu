// One forward ring step of BurstAttention on sm_100a (distributed.py:174-188).
//
// For query shard i (resident) and visiting key shard j it computes, per head,
//   S = Q K^T * scale  masked on global token ids (masks.py:89-104),
//   lse_step = row_logsumexp(S),  O_step = softmax(S) V,
// and folds them into the running (O, lse) with the exact lse_merge /
// exp_gap weights of distributed.py:184-188 -- the merge is the epilogue.
//
// CTA = 2 query tiles of 128 rows x one head; K/V tiles of 128 keys stream
// through a 5-slot TMA ring and are shared by both query tiles.
//   warp 0      TMA producer (Q once, then K_j, V_j)
//   warp 1      MMA issuer: S_k = Q_k K_j^T (SS, M=128,N=128) and
//               O_k += P_k V_j (TS: P read from TMEM, V MN-major from smem) into TMEM
//   warp 2      TMEM allocator
//   warps 4-7   softmax for query tile 0, warps 8-11 for query tile 1:
//               one thread per row, online softmax in the log2 domain with a
//               lazy (threshold 8) rescale of the TMEM O accumulator, P (bf16)
//               written back over its own S columns in TMEM (tcgen05.st), where the
//               P.V MMA reads it as the A operand -- no shared-memory round trip.
// Registers: setmaxnreg gives the softmax warpgroups 216 (S row in registers, no spills;
// a spill here goes to L2, the 226 KB of shared memory leaves L1 ~2 KB) and the control
// warpgroup 64.  Tiles are classified from the closed-form id bounds (bb_mask.cuh): fully
// masked tiles are never loaded or multiplied, fully visible tiles skip the per-element
// predicate.
#include <cuda_runtime.h>

#include <type_traits>

#include "bb_host.h"
#include "bb_mask.cuh"
#include "bb_ptx.cuh"

namespace bb {
namespace {

constexpr int FWD_THREADS = 384;
constexpr int MAX_KT = 4096;  // key tiles per shard the class table holds (n_k <= 524288)
constexpr int KV_SLOTS = 5;
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 units: P may reach 2^8 before O is rescaled
constexpr uint32_t REGS_CTRL = 64, REGS_SOFTMAX = 216;
// setmaxnreg.inc blocks until the CTA's pool has the registers: the pool is what the launch
// allocated (168 per thread at 384 threads), not the 64K register file.
static_assert(REGS_CTRL * 128 + REGS_SOFTMAX * 256 <= 168 * FWD_THREADS, "register budget");
#ifndef BB_FWD_POLY
// Every BB_FWD_POLY-th exponential pair of an unmasked tile goes to a cubic on the FMA pipe
// (ex2_poly2) instead of MUFU (16 lanes/clk/SM: a 128x128 tile's exps need as many cycles as
// its two MMAs).  0 = MUFU only.
#define BB_FWD_POLY 0
#endif

template <int D>
struct FwdSmem {
  static constexpr uint32_t TILE = 128 * D * 2;  // one Q / K / V tile, D/64 panels of 16 KB
  static constexpr uint32_t Q_OFF = 0;
  static constexpr uint32_t KV_OFF = Q_OFF + 2 * TILE;
  static constexpr uint32_t BAR_OFF = KV_OFF + KV_SLOTS * TILE;
  static constexpr uint32_t CLS_OFF = BAR_OFF + 256;  // per key tile: class(q tile 0) | class(q tile 1) << 2
  static constexpr uint32_t BYTES = CLS_OFF + MAX_KT / 2;
};

struct FwdParams {
  float* o;
  float* lse;
  int64_t n_q, n_k;
  int64_t lse_ld;  // row length of the caller's lse array (>= n_q: a sub-shard launch, bb_api.cu)
  int32_t hq, hkv;
  float scale_log2;
  int32_t q_device, k_device;
  LayoutD layout;
  MaskD mask;
  int32_t q_pairs;  // number of 256-row query blocks
  uint2* o16;       // optional bf16 copy of O after the merge (4 columns per uint2)
  long long* probe;  // diagnostics (BB_PROBE=1): clock64() per phase of CTA (0,0)
};

#ifndef BB_WITH_PROBES  // per-phase clock64 probes: diagnostic builds only (tools/variant.py probes BB_WITH_PROBES)
#define FWD_PROBE(idx, slot) \
  do {                 \
  } while (0)
#define FWD_CTA_MARK(k) \
  do {                  \
  } while (0)
#else
// per-CTA timeline: SM id and globaltimer (ns) at entry / prologue done / epilogue / exit
#define FWD_CTA_MARK(k)                                                                                   \
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
#ifndef BB_PROBE_TAIL
#define BB_PROBE_TAIL 0  // 1: softmax probes index the last 16 key tiles (j_hi - 1 - j) instead of the first
#endif
#define FWD_PROBE(idx, slot)                                                                         \
  do {                                                                                               \
    if (p.probe && blockIdx.x == 0 && blockIdx.y == 0 && (idx) < 16) p.probe[512 + (idx) * 32 + (slot)] = clock64(); \
  } while (0)
#endif

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
                    const __grid_constant__ CUtensorMap tv, const __grid_constant__ FwdParams p) {
  using L = FwdSmem<D>;
  constexpr int PANELS = D / 64;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023) != 0) __trap();

  if (threadIdx.x == 0) FWD_CTA_MARK(0);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;                      // [KV_SLOTS]
  uint64_t* kv_empty = bars + 1 + KV_SLOTS;          // [KV_SLOTS]
  uint64_t* s_full = bars + 1 + 2 * KV_SLOTS;        // [2]
  uint64_t* p_full = bars + 3 + 2 * KV_SLOTS;        // [2]
  uint64_t* pv_done = bars + 5 + 2 * KV_SLOTS;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 7 + 2 * KV_SLOTS);

  const int head = blockIdx.y;
  const int kv_head = head / (p.hq / p.hkv);
  const int64_t m0 = static_cast<int64_t>(p.q_pairs - 1 - blockIdx.x) * 256;  // heavy rows first
  int64_t j_lo, j_hi;  // key tiles that can touch this CTA's queries (two binary searches, every thread)
  active_runs(p.layout, p.mask, token_id(p.layout, p.q_device, m0),
              token_id(p.layout, p.q_device, min(m0 + 256, p.n_q) - 1), p.k_device, p.n_k, true, j_lo, j_hi);
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
  // Classify both query tiles against every key tile once; the warp roles look classes up
  // (re-deriving them per tile put the id arithmetic on every role's critical path).
  uint8_t* cls_tab = smem + L::CLS_OFF;
  for (int64_t b = threadIdx.x; b < (j_hi - j_lo + 1) / 2; b += FWD_THREADS) {
    uint32_t byte = 0;
    for (int k = 0; k < 2; ++k) {
      const int64_t jj = j_lo + 2 * b + k;
      if (jj < j_hi) byte |= static_cast<uint32_t>(fwd_class(p, 0, m0, jj) | (fwd_class(p, 1, m0, jj) << 2)) << (4 * k);
    }
    cls_tab[b] = static_cast<uint8_t>(byte);
  }
  auto tile_nib = [&](int64_t jj) {  // class(q tile 0) | class(q tile 1) << 2 of key tile jj
    const int64_t x = jj - j_lo;
    return static_cast<uint32_t>(cls_tab[x >> 1] >> (4 * (x & 1))) & 15u;
  };
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) FWD_CTA_MARK(1);

  if (warp < 4) {
    setmaxnreg_dec<REGS_CTRL>();
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
        for (int64_t j = j_lo; j < j_hi; ++j) {
          if (tile_nib(j) == 0) continue;  // both query tiles skip
          for (int which = 0; which < 2; ++which, ++use) {
            const uint32_t s = use % KV_SLOTS, ph = (use / KV_SLOTS) & 1;
            FWD_PROBE(use >> 1, 0 + which * 2);
            mbar_wait(&kv_empty[s], ph ^ 1);
            FWD_PROBE(use >> 1, 1 + which * 2);
            mbar_expect_tx(&kv_full[s], L::TILE);
            for (int pn = 0; pn < PANELS; ++pn)
              tma_load_2d(smem + L::KV_OFF + s * L::TILE + pn * 16384, which ? &tv : &tk, &kv_full[s],
                          kv_head * D + pn * 64, static_cast<int32_t>(j * 128));
          }
        }
      }
    } else if (warp == 1) {
      // ------------------------------------------------ MMA issuer
      // Order per active kv tile j (jn = next active tile):  PV0(j), S0(jn), PV1(j), S1(jn).
      // S0(jn) only needs softmax 0 to have consumed S0(j) (it has: P0(j) is ready), so
      // query tile 0's softmax of jn overlaps PV1(j) and S1(jn) overlaps softmax 1 -- the
      // tensor pipe never waits on both softmax groups at once.
      constexpr uint32_t idesc_s = idesc_bf16(128, 128, false, false);
      constexpr uint32_t idesc_o = idesc_bf16(128, D, false, true);
      uint32_t issued0 = 0, issued1 = 0;
      auto kv_slot = [](uint32_t use) { return use % KV_SLOTS; };
      auto kv_par = [](uint32_t use) { return (use / KV_SLOTS) & 1; };
      auto issue_s = [&](int q, uint32_t k_base) {
        if (elect_one()) {
          const uint32_t q_base = smem_u32(smem + L::Q_OFF + q * L::TILE);
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks) {
            const uint32_t off = (ks >> 2) * 16384 + (ks & 3) * 32;
            umma_ss(tmem + (q * 128u), sw128_desc(q_base + off, 16, 1024), sw128_desc(k_base + off, 16, 1024),
                    idesc_s, ks > 0);
          }
          umma_commit(&s_full[q]);
        }
        __syncwarp();
      };
      auto issue_pv = [&](int q, uint32_t v_base, uint32_t& issued) {
        mbar_wait(&p_full[q], issued & 1);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)  // A = P: 16 keys (8 packed columns) per k-step
            umma_ts(tmem + (256u + q * D), tmem + q * 128u + ks * 8u, sw128_desc(v_base + ks * 2048, 16384, 1024),
                    idesc_o, (issued | ks) != 0);
          umma_commit(&pv_done[q]);
        }
        __syncwarp();
        ++issued;
      };
      // next key tile either query tile uses, and its class nibble (no arrays: an array written
      // through a pointer lives in local memory, i.e. behind an L2 round trip every tile)
      auto next_active = [&](int64_t from, uint32_t& nib) {
        for (int64_t jj = from; jj < j_hi; ++jj) {
          nib = tile_nib(jj);
          if (nib != 0) return jj;
        }
        nib = 0;
        return j_hi;
      };
      mbar_wait(q_full, 0);
      uint32_t nib, nib_n;
      int64_t j = next_active(j_lo, nib);
      if (j < j_hi) {  // prologue: S of the first active tile
        mbar_wait(&kv_full[kv_slot(0)], kv_par(0));
        tc_fence_after();
        const uint32_t k_base = smem_u32(smem + L::KV_OFF + kv_slot(0) * L::TILE);
        if (nib & 3u) issue_s(0, k_base);
        if (nib >> 2) issue_s(1, k_base);
        if (elect_one()) umma_commit(&kv_empty[kv_slot(0)]);
        __syncwarp();
      }
      for (uint32_t t = 0; j < j_hi; ++t) {
        const int64_t jn = next_active(j + 1, nib_n);
        const uint32_t uv = 2 * t + 1, uk = 2 * t + 2;
        if (lane == 0) FWD_PROBE(t, 4);
        mbar_wait(&kv_full[kv_slot(uv)], kv_par(uv));
        if (lane == 0) FWD_PROBE(t, 5);
        tc_fence_after();
        const uint32_t v_base = smem_u32(smem + L::KV_OFF + kv_slot(uv) * L::TILE);
        const uint32_t kn_base = smem_u32(smem + L::KV_OFF + kv_slot(uk) * L::TILE);
        if (nib & 3u) issue_pv(0, v_base, issued0);
        if (lane == 0) FWD_PROBE(t, 7);
        if (jn < j_hi) {
          mbar_wait(&kv_full[kv_slot(uk)], kv_par(uk));
          tc_fence_after();
          if (nib_n & 3u) issue_s(0, kn_base);
        }
        if (nib >> 2) issue_pv(1, v_base, issued1);
        if (lane == 0) FWD_PROBE(t, 9);
        if (jn < j_hi) {
          if (nib_n >> 2) issue_s(1, kn_base);
          if (elect_one()) umma_commit(&kv_empty[kv_slot(uk)]);
          __syncwarp();
        }
        if (elect_one()) umma_commit(&kv_empty[kv_slot(uv)]);
        __syncwarp();
        j = jn;
        nib = nib_n;
      }
    }
  } else {
    // ------------------------------------------------ softmax / correction / epilogue
    setmaxnreg_inc<REGS_SOFTMAX>();
    const int q = (warp - 4) >> 2;  // query tile of this warpgroup
    const uint32_t quad = warp & 3;
    const int row = quad * 32 + lane;
    const int64_t qrow = m0 + 128 * q + row;
    const bool row_ok = qrow < p.n_q;
    const int64_t q_id = row_ok ? token_id(p.layout, p.q_device, qrow) : 0;
    const uint32_t t_lane = (quad * 32) << 16;
    const float sl2 = p.scale_log2;

    float m_run = -INFINITY, l_run = 0.f;
    uint32_t t = 0;
    // The class of the next key tile is read one tile ahead (a shared load behind the MMAs'
    // operand fetch waits hundreds of cycles; the warp issues in order).
    int64_t j = j_lo;
    int32_t cls = j < j_hi ? static_cast<int32_t>((tile_nib(j) >> (2 * q)) & 3u) : TILE_SKIP;
    for (; j < j_hi; ++j) {
      const int32_t cls_next = j + 1 < j_hi ? static_cast<int32_t>((tile_nib(j + 1) >> (2 * q)) & 3u) : TILE_SKIP;
      if (cls == TILE_SKIP) {
        cls = cls_next;
        continue;
      }
      if (row == 0) FWD_PROBE(BB_PROBE_TAIL ? static_cast<uint32_t>(j_hi - 1 - j) : t, 16 + 8 * q);
      mbar_wait(&s_full[q], t & 1);
      if (row == 0) FWD_PROBE(BB_PROBE_TAIL ? static_cast<uint32_t>(j_hi - 1 - j) : t, 17 + 8 * q);
      tc_fence_after();
      uint4 bits = make_uint4(~0u, ~0u, ~0u, ~0u);
      if (cls == TILE_PARTIAL)
        bits = row_mask_bits(p.layout, p.mask, q_id, row_ok, p.k_device, j * 128, p.n_k, true);
      if (row == 0) FWD_PROBE(BB_PROBE_TAIL ? static_cast<uint32_t>(j_hi - 1 - j) : t, 22 + 8 * q);
      float s[128];
#pragma unroll
      for (int c = 0; c < 4; ++c)
        tmem_ld32(tmem + t_lane + (q * 128u) + c * 32, *reinterpret_cast<float(*)[32]>(&s[c * 32]));
      tmem_ld_wait();
      if (cls == TILE_PARTIAL) {
#pragma unroll
        for (int c = 0; c < 128; ++c)
          if (!mask_bit(bits, c)) s[c] = -INFINITY;
      }
      if (row == 0) FWD_PROBE(BB_PROBE_TAIL ? static_cast<uint32_t>(j_hi - 1 - j) : t, 23 + 8 * q);
      // Row max as an 8-way tree of 3-input maxes (a 128-long dependent chain is ~512+ cycles).
      float mx8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mx8[i] = fmax3(s[i], s[i + 8], s[i + 16]);
#pragma unroll
      for (int c = 24; c < 120; c += 16)
#pragma unroll
        for (int i = 0; i < 8; ++i) mx8[i] = fmax3(mx8[i], s[c + i], s[c + 8 + i]);
#pragma unroll
      for (int i = 0; i < 8; ++i) mx8[i] = fmaxf(mx8[i], s[120 + i]);
      const float mx = fmax3(fmax3(mx8[0], mx8[1], mx8[2]), fmax3(mx8[3], mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]));
      const float m_tile = mx * sl2;
      const bool need = m_tile > m_run + RESCALE_THRESHOLD;
      float alpha = 1.f;
      if (need) {
        alpha = (m_run == -INFINITY) ? 0.f : ex2_approx(m_run - m_tile);
        m_run = m_tile;
        l_run *= alpha;
      }
      const float neg_m = (m_run == -INFINITY) ? 0.f : -m_run;
      // The P buffer and the O accumulator are free once the previous P.V retired (with the
      // MMA order PV(j-1) .. S(j) this has already happened by the time S(j) is ready).
      if (t > 0) {
        mbar_wait(&pv_done[q], (t - 1) & 1);
        if (row == 0) FWD_PROBE(BB_PROBE_TAIL ? static_cast<uint32_t>(j_hi - 1 - j) : t, 18 + 8 * q);
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
      // P = 2^(S*scale*log2e - m) with packed fp32x2 arithmetic (FFMA2 for the scale, FADD2 for
      // the row sums), packed to bf16x2 and stored over the S columns it came from, 32 keys at a
      // time.  Masked tiles stay on MUFU (its ex2(-inf) = 0 is exact).
      float2 acc4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      const float2 sl2x2 = make_float2(sl2, sl2), negm2 = make_float2(neg_m, neg_m);
      auto exp_pass = [&](auto masked_tag) {
        constexpr bool MASKED = decltype(masked_tag)::value;
#pragma unroll
        for (int c = 0; c < 128; c += 32) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float2 x = __ffma2_rn(make_float2(s[c + 2 * i], s[c + 2 * i + 1]), sl2x2, negm2);
            const float2 e = (!MASKED && BB_FWD_POLY > 0 && (i % (BB_FWD_POLY > 0 ? BB_FWD_POLY : 1)) == 0)
                                 ? ex2_poly2(x)
                                 : make_float2(ex2_approx(x.x), ex2_approx(x.y));
            acc4[i & 3] = __fadd2_rn(acc4[i & 3], e);
            pk[i] = pack_bf16(e.x, e.y);
          }
          tmem_st16(tmem + t_lane + q * 128u + c / 2, pk);
        }
      };
      if (cls == TILE_PARTIAL)
        exp_pass(std::true_type{});
      else
        exp_pass(std::false_type{});
      l_run += ((acc4[0].x + acc4[0].y) + (acc4[1].x + acc4[1].y)) + ((acc4[2].x + acc4[2].y) + (acc4[3].x + acc4[3].y));
      if (row == 0) FWD_PROBE(BB_PROBE_TAIL ? static_cast<uint32_t>(j_hi - 1 - j) : t, 20 + 8 * q);
      tmem_st_wait();
      if (row == 0) FWD_PROBE(BB_PROBE_TAIL ? static_cast<uint32_t>(j_hi - 1 - j) : t, 21 + 8 * q);
      tc_fence_before();
      mbar_arrive(&p_full[q]);
      if (row == 0) FWD_PROBE(BB_PROBE_TAIL ? static_cast<uint32_t>(j_hi - 1 - j) : t, 19 + 8 * q);
      ++t;
      cls = cls_next;
    }

    float* o_row = p.o + (qrow * p.hq + head) * static_cast<int64_t>(D);
    uint2* o16_row = (p.o16 && row_ok) ? p.o16 + (qrow * p.hq + head) * static_cast<int64_t>(D / 4) : nullptr;
    bool written = false;
    if (row == 0) {
      if (q == 0) FWD_CTA_MARK(2);
      else FWD_CTA_MARK(4);
    }
    if (t > 0) {
      mbar_wait(&pv_done[q], (t - 1) & 1);
      tc_fence_after();
      // lse_step in natural log: sum exp(S) = 2^m_run * l_run.
      const float lse_step = (l_run > 0.f) ? (m_run * 0.69314718055994531f + logf(l_run)) : -INFINITY;
      float w_step = 0.f, w_old = 0.f, lse_new = -INFINITY;
      const bool write = row_ok && lse_step != -INFINITY;
      written = write;
      float* lse_ptr = p.lse + static_cast<int64_t>(head) * p.lse_ld + qrow;
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
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        float o[32];
        tmem_ld32(tmem + t_lane + (256u + q * D) + c * 32, o);
        tmem_ld_wait();
        if (write) {
          float4* __restrict__ dst = reinterpret_cast<float4*>(o_row + c * 32);
          // the previous O (ring merge) is loaded whole before any store: interleaved, each load
          // waited a memory round trip behind the previous (possibly aliasing) store
          float4 prev[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) prev[i] = w_old != 0.f ? dst[i] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float4 r = make_float4(o[4 * i] * w_step, o[4 * i + 1] * w_step, o[4 * i + 2] * w_step,
                                   o[4 * i + 3] * w_step);
            if (w_old != 0.f) {
              r.x += w_old * prev[i].x;
              r.y += w_old * prev[i].y;
              r.z += w_old * prev[i].z;
              r.w += w_old * prev[i].w;
            }
            dst[i] = r;
            if (o16_row) o16_row[c * 8 + i] = make_uint2(pack_bf16(r.x, r.y), pack_bf16(r.z, r.w));
          }
        }
      }
    }
    // Rows this step leaves untouched still need their bf16 copy (the running O as it is).
    if (o16_row && !written) {
      const float4* src = reinterpret_cast<const float4*>(o_row);
#pragma unroll 4
      for (int i = 0; i < D / 4; ++i) {
        const float4 r = src[i];
        o16_row[i] = make_uint2(pack_bf16(r.x, r.y), pack_bf16(r.z, r.w));
      }
    }
  }

  if (warp >= 4 && (warp & 3) == 0 && lane == 0) FWD_CTA_MARK((warp == 4) ? 5 : 6);  // softmax WG done
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
  if (threadIdx.x == 0) FWD_CTA_MARK(3);
}

template <int D>
int launch_fwd_d(const bb_attn_fwd_args& a, cudaStream_t st, int64_t lse_ld) {
  if ((a.n_k + 127) / 128 > MAX_KT)  // bb_api.cu splits larger shards before they get here
    return set_error(BB_ERR_UNSUPPORTED, "attn_fwd: key shard of %lld rows exceeds %d (raise MAX_KT)", (long long)a.n_k, MAX_KT * 128);
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
  p.lse_ld = lse_ld;
  p.hq = a.hq;
  p.hkv = a.hkv;
  p.scale_log2 = a.softmax_scale * 1.4426950408889634f;
  p.q_device = a.q_device;
  p.k_device = a.k_device;
  p.layout = make_layoutd(a.layout);
  p.mask = make_maskd(a.mask);
  p.q_pairs = static_cast<int32_t>((a.n_q + 255) / 256);
  p.probe = debug_probe_buffer();
  p.o16 = static_cast<uint2*>(a.o_bf16);
  using L = FwdSmem<D>;
  auto kern = attn_fwd_kernel<D>;
  static uint64_t attr_done = 0;  // per device: the attribute is per-context
  int dev = 0;
  cudaGetDevice(&dev);
  if (!((attr_done >> dev) & 1)) {
    if (check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::BYTES),
                   "attn_fwd smem attribute"))
      return BB_ERR_CUDA;
    attr_done |= uint64_t(1) << dev;
  }
  dim3 grid(p.q_pairs, a.hq);
  kern<<<grid, FWD_THREADS, L::BYTES, st>>>(tq, tk, tv, p);
  return check_launch("attn_fwd_kernel");
}

}  // namespace

int launch_attn_fwd(const bb_attn_fwd_args& a, cudaStream_t st, int64_t lse_ld) {
  if (a.head_dim == 128) return launch_fwd_d<128>(a, st, lse_ld);
  if (a.head_dim == 64) return launch_fwd_d<64>(a, st, lse_ld);
  return set_error(BB_ERR_UNSUPPORTED, "attn_fwd: head_dim %d (kernels take 64 or 128)", a.head_dim);
}

}  // namespace bb
