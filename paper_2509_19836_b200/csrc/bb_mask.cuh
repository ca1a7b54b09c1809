// Token-id layouts and mask predicates evaluated inside the attention kernels.
//
// Restates burstsim's host-side integer logic so the kernels never need the
// dense G^2 n x n boolean pair masks the reference builds:
//   layouts  -> partitioning.py:85-112  (contiguous / zigzag / striped / block_striped)
//   masks    -> masks.py:89-104         (full / causal / sliding_window / block_sparse)
// Ids are 1-based global token positions, as in the reference.
//
// Every divisor is resolved on the host (LayoutD / MaskD): the warp roles classify
// tiles on their critical path, and device-side int64 division (a long MUFU.RCP
// based subroutine) was measured at several thousand cycles per tile.
#pragma once
#include <cstdint>

#include "../../include/burst_b200.h"

namespace bb {

enum : int32_t { LAYOUT_CONTIGUOUS = 0, LAYOUT_ZIGZAG = 1, LAYOUT_STRIPED = 2, LAYOUT_BLOCK_STRIPED = 3 };
enum : int32_t { MASK_FULL = 0, MASK_CAUSAL = 1, MASK_WINDOW = 2, MASK_BLOCK = 3 };
enum : int32_t { TILE_SKIP = 0, TILE_FULL = 1, TILE_PARTIAL = 2 };

struct LayoutD {
  int32_t kind;
  int32_t g;      // devices
  int64_t n;      // seq_len
  int64_t p;      // contiguous: N/G rows per device; zigzag: N/(2G) rows per half
  int64_t bl;     // block_striped block length
  uint32_t per;   // block_striped: tokens per device per block (bl / G)
};

struct MaskD {
  int32_t kind;
  uint32_t block_len;
  int64_t window;
  int64_t num_blocks;
  const uint8_t* block_mask;
  const int32_t* row_span;  // [num_blocks][2] first / last nonzero column per block row (or null)
  const int32_t* col_span;  // [num_blocks][2] first / last nonzero row per block column (or null)
};

inline LayoutD make_layoutd(const bb_layout& L) {
  LayoutD d{};
  d.kind = L.kind;
  d.g = L.devices;
  d.n = L.seq_len;
  d.p = L.kind == LAYOUT_ZIGZAG ? L.seq_len / (2 * L.devices) : L.seq_len / L.devices;
  d.bl = L.block_len;
  d.per = L.kind == LAYOUT_BLOCK_STRIPED ? static_cast<uint32_t>(L.block_len / L.devices) : 1u;
  return d;
}

inline MaskD make_maskd(const bb_mask& M) {
  MaskD d{};
  d.kind = M.kind;
  d.block_len = static_cast<uint32_t>(M.block_len > 0 ? M.block_len : 1);
  d.window = M.window;
  d.num_blocks = M.num_blocks;
  d.block_mask = M.block_mask;
  d.row_span = M.row_span;
  d.col_span = M.col_span;
  return d;
}

// Global 1-based id of local row `r` (0-based) on 1-based device `dev`.
__host__ __device__ __forceinline__ int64_t token_id(const LayoutD& L, int32_t dev, int64_t r) {
  switch (L.kind) {
    case LAYOUT_ZIGZAG:
      return r < L.p ? (dev - 1) * L.p + r + 1 : L.n - dev * L.p + (r - L.p) + 1;
    case LAYOUT_STRIPED:
      return dev + static_cast<int64_t>(L.g) * r;
    case LAYOUT_BLOCK_STRIPED: {
      const uint32_t ru = static_cast<uint32_t>(r);  // shard rows < 2^31
      const uint32_t blk = ru / L.per;
      return static_cast<int64_t>(blk) * L.bl + static_cast<int64_t>(ru - blk * L.per) * L.g + dev;
    }
    default:  // contiguous
      return (dev - 1) * L.p + r + 1;
  }
}

__device__ __forceinline__ bool pair_allowed(const MaskD& M, int64_t q, int64_t k) {
  switch (M.kind) {
    case MASK_CAUSAL:
      return k <= q;
    case MASK_WINDOW: {
      const int64_t gap = q - k;
      return gap >= 0 && gap < M.window;
    }
    case MASK_BLOCK: {
      const uint32_t qb = static_cast<uint32_t>(q - 1) / M.block_len;
      const uint32_t kb = static_cast<uint32_t>(k - 1) / M.block_len;
      return M.block_mask[static_cast<int64_t>(qb) * M.num_blocks + kb] != 0;
    }
    default:
      return true;
  }
}

// Classify the (query rows [r0,r1) of device qdev) x (key rows [c0,c1) of kdev) tile.
// Shard-local ids are strictly increasing (partitioning.py:96-111), so the
// first/last id of a run bound every id inside it.  `full_width` is false when
// the key tile is ragged (columns past n_k must still be masked per element).
static __device__ __forceinline__ int32_t classify_tile(const LayoutD& L, const MaskD& M, int32_t qdev, int64_t r0,
                                                     int64_t r1, int32_t kdev, int64_t c0, int64_t c1,
                                                     bool full_width) {
  if (r1 <= r0 || c1 <= c0) return TILE_SKIP;
  const int64_t qa = token_id(L, qdev, r0), qb = token_id(L, qdev, r1 - 1);
  const int64_t ka = token_id(L, kdev, c0), kb = token_id(L, kdev, c1 - 1);
  int32_t cls = TILE_PARTIAL;
  switch (M.kind) {
    case MASK_FULL:
      cls = TILE_FULL;
      break;
    case MASK_CAUSAL:
      if (ka > qb) return TILE_SKIP;
      if (kb <= qa) cls = TILE_FULL;
      break;
    case MASK_WINDOW:
      if (ka > qb || qa - kb >= M.window) return TILE_SKIP;
      if (kb <= qa && qb - ka < M.window) cls = TILE_FULL;
      break;
    case MASK_BLOCK: {
      const uint32_t qb0 = static_cast<uint32_t>(qa - 1) / M.block_len, qb1 = static_cast<uint32_t>(qb - 1) / M.block_len;
      const uint32_t kb0 = static_cast<uint32_t>(ka - 1) / M.block_len, kb1 = static_cast<uint32_t>(kb - 1) / M.block_len;
      if ((qb1 - qb0 + 1) * (kb1 - kb0 + 1) <= 256) {
        bool any = false, all = true;
        for (uint32_t x = qb0; x <= qb1; ++x)
          for (uint32_t y = kb0; y <= kb1; ++y) {
            const bool on = M.block_mask[static_cast<int64_t>(x) * M.num_blocks + y] != 0;
            any |= on;
            all &= on;
          }
        if (!any) return TILE_SKIP;
        if (all) cls = TILE_FULL;
      }
      break;
    }
    default:
      break;
  }
  if (cls == TILE_FULL && !full_width) cls = TILE_PARTIAL;
  return cls;
}

// First index in [lo, hi) where a monotone (false..false true..true) predicate holds; hi if none.
template <class F>
__device__ __forceinline__ int64_t first_true(int64_t lo, int64_t hi, F pred) {
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (pred(mid))
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

// Candidate range [lo, hi) of 128-runs on the "other" side that can touch a fixed run of
// tokens with ids in [fa, fb]: everything outside is fully masked.  Ids grow with the run
// index, so for causal / sliding-window masks the range comes from two binary searches;
// full and block-sparse masks keep the whole range (the class table still skips blocks).
//   fixed_is_query: the fixed run holds queries and the runs are keys (forward); else the
//   fixed run holds keys and the runs are queries (backward).
__device__ __forceinline__ void active_runs(const LayoutD& L, const MaskD& M, int64_t fa, int64_t fb,
                                            int32_t dev, int64_t n_rows, bool fixed_is_query, int64_t& lo,
                                            int64_t& hi) {
  const int64_t n_runs = (n_rows + 127) / 128;
  lo = 0;
  hi = n_runs;
  auto first_id = [&](int64_t j) { return token_id(L, dev, j * 128); };
  auto last_id = [&](int64_t j) { return token_id(L, dev, min(j * 128 + 128, n_rows) - 1); };
  if (M.kind == MASK_BLOCK && M.row_span && M.col_span) {
    // union of the nonzero spans of the fixed run's block rows (columns), then the runs
    // whose ids fall inside it
    const int64_t b0 = static_cast<uint32_t>(fa - 1) / M.block_len, b1 = static_cast<uint32_t>(fb - 1) / M.block_len;
    if (b1 - b0 > 64) return;
    const int32_t* span = fixed_is_query ? M.row_span : M.col_span;
    int64_t blo = INT64_MAX, bhi = -1;
    for (int64_t b = b0; b <= b1; ++b) {
      const int32_t s0 = span[2 * b], s1 = span[2 * b + 1];
      if (s0 >= 0) {
        blo = min(blo, static_cast<int64_t>(s0));
        bhi = max(bhi, static_cast<int64_t>(s1));
      }
    }
    if (bhi < 0) {
      lo = hi = 0;
      return;
    }
    const int64_t id_lo = blo * M.block_len + 1, id_hi = (bhi + 1) * M.block_len;
    lo = first_true(0, n_runs, [&](int64_t j) { return last_id(j) >= id_lo; });
    hi = first_true(lo, n_runs, [&](int64_t j) { return first_id(j) > id_hi; });
    return;
  }
  if (M.kind != MASK_CAUSAL && M.kind != MASK_WINDOW) return;
  if (fixed_is_query) {
    // keys: live iff first key <= last query (causal), and last query - ... window lower edge
    hi = first_true(0, n_runs, [&](int64_t j) { return first_id(j) > fb; });
    if (M.kind == MASK_WINDOW) lo = first_true(0, hi, [&](int64_t j) { return fa - last_id(j) < M.window; });
  } else {
    // queries: live iff last query >= first key, and (window) first query - last key < w
    lo = first_true(0, n_runs, [&](int64_t j) { return last_id(j) >= fa; });
    if (M.kind == MASK_WINDOW) hi = first_true(lo, n_runs, [&](int64_t j) { return first_id(j) - fb >= M.window; });
  }
}

// Bits [lo, hi) of a 128-bit row mask (0 <= lo, hi <= 128).
__device__ __forceinline__ uint4 range_bits(int32_t lo, int32_t hi) {
  uint32_t w[4];
#pragma unroll
  for (int wd = 0; wd < 4; ++wd) {
    const int32_t a = max(lo - 32 * wd, 0), b = min(hi - 32 * wd, 32);
    w[wd] = a >= b ? 0u : ((b == 32 ? 0xFFFFFFFFu : ((1u << b) - 1u)) & ~((1u << a) - 1u));
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

__device__ __forceinline__ int64_t floor_div(int64_t a, int64_t b) {  // b > 0
  const int64_t q = a / b;
  return (a % b != 0 && a < 0) ? q - 1 : q;
}

// 128-bit row mask of a PARTIAL tile: bit c set iff (this thread's token, the c-th token of
// the other side's 128-run) is allowed.  fixed_is_query: the thread owns a query row and the
// run is keys (forward); otherwise the thread owns a key and the run is queries (backward).
// Entries past other_n (ragged shard end) are masked.
//
// Causal / sliding-window / full masks allow a contiguous interval of the other side's ids,
// and within a 128-run those ids form at most a few arithmetic runs (consecutive for
// contiguous / zigzag rows, step G for striped and inside a block_striped block), so the mask
// is the union of at most a few bit ranges -- no per-element work.  Block-sparse masks (and
// runs that split into more pieces) take the per-element predicate.
static __device__ __noinline__ uint4 row_mask_bits(const LayoutD& Lref, const MaskD& Mref, int64_t fixed_id,
                                                   bool fixed_ok, int32_t other_dev, int64_t other0,
                                                   int64_t other_n, bool fixed_is_query) {
  // The callers pass references into __grid_constant__ kernel parameters, which this
  // out-of-line function can only read through generic loads: copy them once.
  const LayoutD L = Lref;
  const MaskD M = Mref;
  if (!fixed_ok || other0 >= other_n) return make_uint4(0u, 0u, 0u, 0u);
  const int32_t n = static_cast<int32_t>(other_n - other0 < 128 ? other_n - other0 : 128);
  if (M.kind != MASK_BLOCK) {
    // interval [vlo, vhi] of the other side's ids that the fixed token may pair with
    int64_t vlo = INT64_MIN / 4, vhi = INT64_MAX / 4;
    if (M.kind == MASK_CAUSAL || M.kind == MASK_WINDOW) {
      const int64_t w = M.kind == MASK_WINDOW ? M.window : INT64_MAX / 4;
      if (fixed_is_query) {  // keys k with q - w < k <= q
        vhi = fixed_id;
        vlo = fixed_id - w + 1;
      } else {  // queries q with k <= q < k + w
        vlo = fixed_id;
        vhi = fixed_id + w - 1;
      }
    }
    // walk the run's arithmetic segments [c0, c1): id = id0 + step * (c - c0); a zigzag run
    // splits at the shard's half (row p), a block_striped run at every block (per rows)
    const int64_t step = (L.kind == LAYOUT_STRIPED || L.kind == LAYOUT_BLOCK_STRIPED) ? L.g : 1;
    if (L.kind != LAYOUT_BLOCK_STRIPED || L.per >= 32) {
      uint4 bits = make_uint4(0u, 0u, 0u, 0u);
      for (int32_t c0 = 0; c0 < n;) {
        int64_t c1 = n;
        if (L.kind == LAYOUT_ZIGZAG && other0 + c0 < L.p && other0 + n > L.p) c1 = L.p - other0;
        if (L.kind == LAYOUT_BLOCK_STRIPED) {
          const int64_t nxt = ((other0 + c0) / L.per + 1) * L.per - other0;
          if (nxt < c1) c1 = nxt;
        }
        const int64_t id0 = token_id(L, other_dev, other0 + c0);
        // c in [c0, c1) with vlo <= id0 + step (c - c0) <= vhi
        const int64_t skip = -floor_div(id0 - vlo, step);  // first c - c0 with id >= vlo
        const int64_t lo = c0 + (skip > 0 ? skip : 0);
        const int64_t hi = c0 + floor_div(vhi - id0, step) + 1;
        const int32_t ra = static_cast<int32_t>(lo < c1 ? lo : c1), rb = static_cast<int32_t>(hi < c1 ? hi : c1);
        if (ra < rb) {
          const uint4 r = range_bits(ra, rb);
          bits.x |= r.x;
          bits.y |= r.y;
          bits.z |= r.z;
          bits.w |= r.w;
        }
        c0 = static_cast<int32_t>(c1);
      }
      return bits;
    }
  }
  uint32_t w[4];
#pragma unroll
  for (int wd = 0; wd < 4; ++wd) {
    uint32_t bits = 0;
#pragma unroll 1
    for (int b = 0; b < 32; ++b) {
      const int64_t r = other0 + wd * 32 + b;
      if (r >= other_n) break;
      const int64_t id = token_id(L, other_dev, r);
      const bool ok = fixed_is_query ? pair_allowed(M, fixed_id, id) : pair_allowed(M, id, fixed_id);
      bits |= static_cast<uint32_t>(ok) << b;
    }
    w[wd] = bits;
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

__device__ __forceinline__ bool mask_bit(const uint4& b, int c) {
  const uint32_t word = c < 32 ? b.x : c < 64 ? b.y : c < 96 ? b.z : b.w;
  return (word >> (c & 31)) & 1u;
}

}  // namespace bb
