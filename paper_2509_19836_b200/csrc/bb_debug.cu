// Mask realisation dump (bb_debug_mask_tiles): the tile classes and per-element allowed bits
// exactly as attn_fwd_kernel / attn_bwd_kernel derive them on the device -- the same
// active_runs range search, classify_tile and row_mask_bits (bb_mask.cuh) with the same
// arguments -- so tests can compare the kernels' mask against the reference's
// local_pair_mask (partitioning.py:120-169) bit for bit.  Not on the hot path.
#include <cuda_runtime.h>

#include "bb_host.h"
#include "bb_mask.cuh"

namespace bb {
namespace {

struct DbgArgs {
  LayoutD layout;
  MaskD mask;
  int32_t q_device, k_device;
  int64_t n_q, n_k;
  int32_t view;  // 0: forward (CTA = 256 query rows), 1: backward (CTA = 128 key rows)
};

// One thread per (query tile, key tile): the class the kernel uses, SKIP outside the CTA's
// active_runs range.
__global__ void classes_kernel(const __grid_constant__ DbgArgs a, int8_t* cls, int64_t n_qt, int64_t n_kt) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= n_qt * n_kt) return;
  const int64_t qt = idx / n_kt, kt = idx % n_kt;
  const int64_t r0 = qt * 128, r1 = min(r0 + 128, a.n_q);
  const int64_t c0 = kt * 128, c1 = min(c0 + 128, a.n_k);
  int64_t lo, hi;
  bool in_range;
  if (a.view == 0) {  // attn_fwd_kernel: query pair m0 = 256 * (qt / 2), key tiles [lo, hi)
    const int64_t m0 = (qt / 2) * 256;
    active_runs(a.layout, a.mask, token_id(a.layout, a.q_device, m0),
                token_id(a.layout, a.q_device, min(m0 + 256, a.n_q) - 1), a.k_device, a.n_k, true, lo, hi);
    in_range = kt >= lo && kt < hi;
  } else {  // attn_bwd_kernel: key tile c0, query tiles [lo, hi)
    active_runs(a.layout, a.mask, token_id(a.layout, a.k_device, c0), token_id(a.layout, a.k_device, c1 - 1),
                a.q_device, a.n_q, false, lo, hi);
    in_range = qt >= lo && qt < hi;
  }
  cls[idx] = in_range ? static_cast<int8_t>(
                            classify_tile(a.layout, a.mask, a.q_device, r0, r1, a.k_device, c0, c1, c1 - c0 == 128))
                      : static_cast<int8_t>(TILE_SKIP);
}

// One thread per fixed row (a query row in the forward view, a key row in the backward view)
// and other-side tile: the allowed bits the kernel applies, written densely as allowed[q][k].
__global__ void bits_kernel(const __grid_constant__ DbgArgs a, const int8_t* cls, uint8_t* allowed, int64_t n_kt) {
  const int64_t n_fixed = a.view == 0 ? a.n_q : a.n_k;
  const int64_t n_other_t = a.view == 0 ? n_kt : (a.n_q + 127) / 128;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= n_fixed * n_other_t) return;
  const int64_t f = idx / n_other_t, ot = idx % n_other_t;
  const int64_t qt = a.view == 0 ? f / 128 : ot, kt = a.view == 0 ? ot : f / 128;
  const int32_t c = cls[qt * n_kt + kt];
  const int64_t o0 = ot * 128, o_n = a.view == 0 ? a.n_k : a.n_q;
  uint4 bits;
  if (c == TILE_SKIP) {
    bits = make_uint4(0u, 0u, 0u, 0u);
  } else if (c == TILE_PARTIAL) {
    const int32_t fdev = a.view == 0 ? a.q_device : a.k_device, odev = a.view == 0 ? a.k_device : a.q_device;
    bits = row_mask_bits(a.layout, a.mask, token_id(a.layout, fdev, f), true, odev, o0, o_n, a.view == 0);
  } else {  // FULL: every in-range element (rows past the shard end never reach the output)
    bits = make_uint4(~0u, ~0u, ~0u, ~0u);
  }
  for (int b = 0; b < 128 && o0 + b < o_n; ++b) {
    const int64_t q = a.view == 0 ? f : o0 + b, k = a.view == 0 ? o0 + b : f;
    allowed[q * a.n_k + k] = mask_bit(bits, b) ? 1 : 0;
  }
}

}  // namespace
}  // namespace bb

using namespace bb;

extern "C" int bb_debug_mask_tiles(const bb_layout* layout, const bb_mask* mask, int32_t q_device, int32_t k_device,
                                   int64_t n_q, int64_t n_k, int32_t view, int8_t* classes, uint8_t* allowed,
                                   void* stream) {
  if (!layout || !mask || !classes) return set_error(BB_ERR_INVALID, "bb_debug_mask_tiles: null argument");
  if (n_q < 1 || n_k < 1 || (view != 0 && view != 1))
    return set_error(BB_ERR_INVALID, "bb_debug_mask_tiles: bad extent or view");
  if (q_device < 1 || q_device > layout->devices || k_device < 1 || k_device > layout->devices)
    return set_error(BB_ERR_INVALID, "bb_debug_mask_tiles: device indices must lie in [1, %d]", layout->devices);
  DbgArgs a{};
  a.layout = make_layoutd(*layout);
  a.mask = make_maskd(*mask);
  a.q_device = q_device;
  a.k_device = k_device;
  a.n_q = n_q;
  a.n_k = n_k;
  a.view = view;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n_qt = (n_q + 127) / 128, n_kt = (n_k + 127) / 128;
  classes_kernel<<<static_cast<unsigned>((n_qt * n_kt + 127) / 128), 128, 0, st>>>(a, classes, n_qt, n_kt);
  if (int rc = check_launch("mask classes_kernel")) return rc;
  if (!allowed) return BB_OK;
  const int64_t work = (view == 0 ? n_q * n_kt : n_k * n_qt);
  bits_kernel<<<static_cast<unsigned>((work + 127) / 128), 128, 0, st>>>(a, classes, allowed, n_kt);
  return check_launch("mask bits_kernel");
}
