// Token-id layouts and mask predicates evaluated inside the attention kernels.
//
// Restates burstsim's host-side integer logic so the kernels never need the
// dense G^2 n x n boolean pair masks the reference builds:
//   layouts  -> partitioning.py:85-112  (contiguous / zigzag / striped / block_striped)
//   masks    -> masks.py:89-104         (full / causal / sliding_window / block_sparse)
// Ids are 1-based global token positions, as in the reference.
#pragma once
#include <cstdint>

#include "../../include/burst_b200.h"

namespace bb {

enum : int32_t { LAYOUT_CONTIGUOUS = 0, LAYOUT_ZIGZAG = 1, LAYOUT_STRIPED = 2, LAYOUT_BLOCK_STRIPED = 3 };
enum : int32_t { MASK_FULL = 0, MASK_CAUSAL = 1, MASK_WINDOW = 2, MASK_BLOCK = 3 };
enum : int32_t { TILE_SKIP = 0, TILE_FULL = 1, TILE_PARTIAL = 2 };

// Global 1-based id of local row `r` (0-based) on 1-based device `dev`.
__host__ __device__ __forceinline__ int64_t token_id(const bb_layout& L, int32_t dev, int64_t r) {
  const int64_t g = L.devices;
  switch (L.kind) {
    case LAYOUT_ZIGZAG: {
      const int64_t p = L.seq_len / (2 * g);
      return r < p ? (dev - 1) * p + r + 1 : L.seq_len - dev * p + (r - p) + 1;
    }
    case LAYOUT_STRIPED:
      return dev + g * r;
    case LAYOUT_BLOCK_STRIPED: {
      const int64_t per = L.block_len / g;  // tokens a device owns inside one block
      return (r / per) * L.block_len + (r % per) * g + dev;
    }
    default: {  // contiguous
      const int64_t p = L.seq_len / g;
      return (dev - 1) * p + r + 1;
    }
  }
}

__device__ __forceinline__ bool pair_allowed(const bb_mask& M, int64_t q, int64_t k) {
  switch (M.kind) {
    case MASK_CAUSAL:
      return k <= q;
    case MASK_WINDOW: {
      const int64_t gap = q - k;
      return gap >= 0 && gap < M.window;
    }
    case MASK_BLOCK:
      return M.block_mask[((q - 1) / M.block_len) * M.num_blocks + (k - 1) / M.block_len] != 0;
    default:
      return true;
  }
}

// Classify the (query rows [r0,r1) of device qdev) x (key rows [c0,c1) of kdev) tile.
// Shard-local ids are strictly increasing (partitioning.py:96-111), so the
// first/last id of a run bound every id inside it.  `full_width` is false when
// the key tile is ragged (columns past n_k must still be masked per element).
__device__ __forceinline__ int32_t classify_tile(const bb_layout& L, const bb_mask& M, int32_t qdev,
                                                 int64_t r0, int64_t r1, int32_t kdev, int64_t c0,
                                                 int64_t c1, bool full_width) {
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
      const int64_t qb0 = (qa - 1) / M.block_len, qb1 = (qb - 1) / M.block_len;
      const int64_t kb0 = (ka - 1) / M.block_len, kb1 = (kb - 1) / M.block_len;
      if ((qb1 - qb0 + 1) * (kb1 - kb0 + 1) <= 256) {
        bool any = false, all = true;
        for (int64_t x = qb0; x <= qb1; ++x)
          for (int64_t y = kb0; y <= kb1; ++y) {
            const bool on = M.block_mask[x * M.num_blocks + y] != 0;
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

}  // namespace bb
