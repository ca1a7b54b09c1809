// extern "C" boundary (include/burst_b200.h): argument validation, error
// reporting, TMA descriptor construction and the LM-head orchestration.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "bb_host.h"

namespace bb {

std::atomic<int64_t> g_launches{0};
static thread_local char g_err[512] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_cuda(cudaError_t err, const char* what) {
  if (err == cudaSuccess) return BB_OK;
  return set_error(BB_ERR_CUDA, "%s: %s", what, cudaGetErrorString(err));
}

int check_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return check_cuda(cudaGetLastError(), what);
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool make_tmap_bf16_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                       uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer) {
  return make_tmap_2d(map, base, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, inner, outer, row_stride_bytes, box_inner,
                      box_outer);
}

bool make_tmap_2d(CUtensorMap* map, const void* base, CUtensorMapDataType dtype, uint64_t inner, uint64_t outer,
                  uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swizzle) {
  auto fn = encode_fn();
  if (!fn) {
    set_error(BB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
    return false;
  }
  if (reinterpret_cast<uintptr_t>(base) % 16 || row_stride_bytes % 16) {
    set_error(BB_ERR_INVALID, "TMA operand must be 16-byte aligned (base %p, row stride %llu B)", base,
              (unsigned long long)row_stride_bytes);
    return false;
  }
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estride[2] = {1, 1};
  CUresult r = fn(map, dtype, 2, const_cast<void*>(base), dims, strides, box,
                  estride, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error(BB_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d): dims %llu x %llu, stride %llu, box %u x %u",
              (int)r, (unsigned long long)inner, (unsigned long long)outer,
              (unsigned long long)row_stride_bytes, box_inner, box_outer);
    return false;
  }
  return true;
}

long long* debug_probe_buffer() {
  static long long* buf = nullptr;
  static bool checked = false;
  if (!checked) {
    checked = true;
    const char* e = getenv("BB_PROBE");
    if (e && *e == '1' && cudaMalloc(&buf, kProbeEntries * sizeof(long long)) == cudaSuccess)
      cudaMemset(buf, 0, kProbeEntries * sizeof(long long));
  }
  return buf;
}

int num_sms() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

int launch_preprocess(const void*, const float*, float*, int64_t, int32_t, int32_t, cudaStream_t);
int launch_permute(void*, const void*, const int64_t*, int64_t, int64_t, int, cudaStream_t);
int launch_cast_pad(void*, const float*, int64_t, int32_t, int32_t, cudaStream_t);
int launch_fill_u32(void*, uint32_t, int64_t, cudaStream_t);
int launch_add_rows(float*, const float*, int64_t, int64_t, int64_t, int64_t, cudaStream_t);
int launch_lmhead_reduce(const float*, const float*, const float*, int64_t, int32_t, float*, float*,
                         cudaStream_t);
int launch_lmhead_dlogits(const float*, const float*, const int64_t*, int64_t, int64_t, int64_t, void*,
                          cudaStream_t);

static int validate_ring_step(const bb_layout& L, const bb_mask& M, int64_t n_q, int64_t n_k, int32_t hq,
                              int32_t hkv, int32_t d, int32_t qdev, int32_t kdev, const char* who) {
  if (n_q <= 0 || n_k <= 0) return set_error(BB_ERR_INVALID, "%s: empty shard (n_q=%lld, n_k=%lld)", who, (long long)n_q, (long long)n_k);
  if (hq <= 0 || hkv <= 0 || hq % hkv) return set_error(BB_ERR_INVALID, "%s: hq=%d must be a multiple of hkv=%d", who, hq, hkv);
  if (d != 64 && d != 128) return set_error(BB_ERR_UNSUPPORTED, "%s: head_dim %d (64 or 128)", who, d);
  if (L.devices < 1 || qdev < 1 || qdev > L.devices || kdev < 1 || kdev > L.devices)
    return set_error(BB_ERR_INVALID, "%s: device indices must lie in [1, %d], got i=%d, j=%d", who, L.devices, qdev, kdev);
  if (L.kind < 0 || L.kind > 3) return set_error(BB_ERR_INVALID, "%s: unknown layout kind %d", who, L.kind);
  if (M.kind < 0 || M.kind > 3) return set_error(BB_ERR_INVALID, "%s: unknown mask kind %d", who, M.kind);
  // ShardLayout's divisibility rules (partitioning.py:53-72): every device id the kernels
  // evaluate (token_id) must come from a valid layout, or the closed forms divide by zero.
  if (L.seq_len < 1 || L.seq_len % L.devices)
    return set_error(BB_ERR_INVALID, "%s: sequence length %lld must be divisible by %d devices", who,
                     (long long)L.seq_len, L.devices);
  if (L.kind == BB_LAYOUT_ZIGZAG && L.seq_len % (2 * static_cast<int64_t>(L.devices)))
    return set_error(BB_ERR_INVALID, "%s: zigzag layout needs seq_len divisible by 2*devices", who);
  if (L.kind == BB_LAYOUT_BLOCK_STRIPED &&
      (L.block_len < 1 || L.block_len % L.devices || L.seq_len % L.block_len))
    return set_error(BB_ERR_INVALID,
                     "%s: block_striped layout needs block_len (%lld) > 0, divisible by %d devices, dividing seq_len %lld",
                     who, (long long)L.block_len, L.devices, (long long)L.seq_len);
  if (M.kind == BB_MASK_BLOCK_SPARSE && (!M.block_mask || M.block_len < 1))
    return set_error(BB_ERR_INVALID, "%s: block_sparse mask needs block_mask and block_len", who);
  // masks.py:78-86: the block mask must tile the whole sequence (the kernels index it by the
  // block of every global id in [1, N]).
  if (M.kind == BB_MASK_BLOCK_SPARSE && M.num_blocks * M.block_len != L.seq_len)
    return set_error(BB_ERR_INVALID, "%s: block mask of %lld blocks x %lld does not cover seq_len %lld", who,
                     (long long)M.num_blocks, (long long)M.block_len, (long long)L.seq_len);
  if (M.kind == BB_MASK_SLIDING_WINDOW && M.window < 1)
    return set_error(BB_ERR_INVALID, "%s: sliding_window width must be >= 1", who);
  // Query rows are local rows [0, n_q) of device q_device, key rows [0, n_k) of k_device.
  // n_q < N/G is how the sequence-selective recompute runs only the front rows
  // (checkpointing.py:149-157); n_q, n_k < N/G together are how a single-device layer call
  // with nq != nk (oracle.py:80-119) runs on one shard of max(nq, nk) ids.
  if (n_q > L.seq_len / L.devices || n_k > L.seq_len / L.devices)
    return set_error(BB_ERR_INVALID, "%s: shard sizes (%lld, %lld) exceed N/G = %lld/%d", who,
                     (long long)n_q, (long long)n_k, (long long)L.seq_len, L.devices);
  return BB_OK;
}

// ---- shards larger than one launch takes (MAX_SHARD_ROWS) --------------------------------
// A zigzag shard is two runs of consecutive token ids (chunks i and 2G+1-i of the sequence in
// 2G chunks) and a contiguous shard one run, so both are exactly sub-shards of a contiguous
// layout with more devices: chunk c of contiguous(N, G') is device c.  The masks read global
// ids only, so a step over such a shard is the same math as the steps over every pair of its
// sub-shards (the forward merges them like ring steps; the backward accumulates).  Striped
// layouts have no such runs; they keep the per-launch limit.
std::atomic<int64_t> g_split_rows{0};  // test hook (bb_debug_set_split_rows); 0 = MAX_SHARD_ROWS

struct SubShard {
  int32_t dev;
  int64_t row0, rows;
};

// Sub-shards of rows [0, n) of device `dev`, as devices of contiguous(N, g_out); false when the
// layout cannot be split this way.
bool split_shard(const bb_layout& L, int32_t dev, int64_t n, int64_t limit, int32_t& g_out, std::vector<SubShard>& out) {
  int64_t g0;
  std::vector<int32_t> chunks;  // this device's chunks of contiguous(N, g0), in row order
  if (L.kind == BB_LAYOUT_ZIGZAG) {
    g0 = 2 * static_cast<int64_t>(L.devices);
    chunks = {dev, static_cast<int32_t>(g0 + 1 - dev)};
  } else if (L.kind == BB_LAYOUT_CONTIGUOUS) {
    g0 = L.devices;
    chunks = {dev};
  } else {
    return false;
  }
  int64_t f = 1;
  while (L.seq_len / (g0 * f) > limit) f *= 2;
  if (L.seq_len % (g0 * f) || g0 * f > INT32_MAX) return false;
  const int64_t rows = L.seq_len / (g0 * f);
  g_out = static_cast<int32_t>(g0 * f);
  out.clear();
  int64_t row0 = 0;
  for (int32_t c : chunks)
    for (int64_t k = 0; k < f && row0 < n; ++k, row0 += rows)
      out.push_back({static_cast<int32_t>((c - 1) * f + k + 1), row0, std::min(rows, n - row0)});
  return true;
}

int64_t split_limit() {
  const int64_t r = g_split_rows.load();
  return r > 0 ? r : MAX_SHARD_ROWS;
}

bool needs_split(int64_t n, int64_t limit) { return n > limit; }

}  // namespace bb

using namespace bb;

extern "C" {

const char* bb_last_error(void) { return g_err; }

int bb_debug_probe(int64_t* host_out, int32_t n) {
  long long* buf = debug_probe_buffer();
  if (!buf) return set_error(BB_ERR_UNSUPPORTED, "set BB_PROBE=1 before the first launch");
  if (n > kProbeEntries) n = kProbeEntries;
  return check_cuda(cudaMemcpy(host_out, buf, n * sizeof(long long), cudaMemcpyDeviceToHost), "probe copy");
}
int32_t bb_abi_version(void) { return 1; }
int64_t bb_launch_count(void) { return g_launches.load(); }

int bb_attn_fwd_step(const bb_attn_fwd_args* a, void* stream) {
  if (!a) return set_error(BB_ERR_INVALID, "bb_attn_fwd_step: null args");
  if (int rc = validate_ring_step(a->layout, a->mask, a->n_q, a->n_k, a->hq, a->hkv, a->head_dim, a->q_device,
                                  a->k_device, "bb_attn_fwd_step"))
    return rc;
  if (a->o_bf16 && (reinterpret_cast<uintptr_t>(a->o_bf16) & 15))
    return set_error(BB_ERR_INVALID, "bb_attn_fwd_step: o_bf16 must be 16-byte aligned");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t limit = split_limit();
  if (!needs_split(a->n_k, limit)) return launch_attn_fwd(*a, st, a->n_q);
  int32_t gq = 0, gk = 0;
  std::vector<SubShard> qs, ks;
  if (!split_shard(a->layout, a->q_device, a->n_q, limit, gq, qs) || !split_shard(a->layout, a->k_device, a->n_k, limit, gk, ks))
    return set_error(BB_ERR_UNSUPPORTED, "bb_attn_fwd_step: a key shard of %lld rows (> %lld) needs a zigzag or contiguous layout",
                     (long long)a->n_k, (long long)limit);
  const int64_t qrow = static_cast<int64_t>(a->hq) * a->head_dim, krow = static_cast<int64_t>(a->hkv) * a->head_dim;
  for (const SubShard& q : qs) {
    for (size_t i = 0; i < ks.size(); ++i) {
      const SubShard& k = ks[i];
      bb_attn_fwd_args b = *a;
      b.layout = bb_layout{BB_LAYOUT_CONTIGUOUS, gq, a->layout.seq_len, 0};
      b.q_device = q.dev;
      b.k_device = k.dev;
      b.n_q = q.rows;
      b.n_k = k.rows;
      b.q = static_cast<const char*>(a->q) + q.row0 * qrow * 2;
      b.o = a->o + q.row0 * qrow;
      b.lse = a->lse + q.row0;
      b.k = static_cast<const char*>(a->k) + k.row0 * krow * 2;
      b.v = static_cast<const char*>(a->v) + k.row0 * krow * 2;
      b.o_bf16 = (a->o_bf16 && i + 1 == ks.size()) ? static_cast<char*>(a->o_bf16) + q.row0 * qrow * 2 : nullptr;
      if (int rc = launch_attn_fwd(b, st, a->n_q)) return rc;
    }
  }
  return BB_OK;
}

int bb_attn_bwd_step(const bb_attn_bwd_args* a, void* stream) {
  if (!a) return set_error(BB_ERR_INVALID, "bb_attn_bwd_step: null args");
  if (int rc = validate_ring_step(a->layout, a->mask, a->n_q, a->n_k, a->hq, a->hkv, a->head_dim, a->q_device,
                                  a->k_device, "bb_attn_bwd_step"))
    return rc;
  if (a->kv_head_end != 0 && (a->kv_head_begin < 0 || a->kv_head_end > a->hkv || a->kv_head_begin >= a->kv_head_end))
    return set_error(BB_ERR_INVALID, "bb_attn_bwd_step: kv head range [%d, %d) outside [0, %d)", a->kv_head_begin,
                     a->kv_head_end, a->hkv);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t limit = split_limit();
  if (!needs_split(a->n_q, limit)) return launch_attn_bwd(*a, st, a->n_q);
  int32_t gq = 0, gk = 0;
  std::vector<SubShard> qs, ks;
  if (!split_shard(a->layout, a->q_device, a->n_q, limit, gq, qs) || !split_shard(a->layout, a->k_device, a->n_k, limit, gk, ks))
    return set_error(BB_ERR_UNSUPPORTED, "bb_attn_bwd_step: a query shard of %lld rows (> %lld) needs a zigzag or contiguous layout",
                     (long long)a->n_q, (long long)limit);
  const int64_t qrow = static_cast<int64_t>(a->hq) * a->head_dim, krow = static_cast<int64_t>(a->hkv) * a->head_dim;
  for (const SubShard& k : ks) {
    for (const SubShard& q : qs) {
      bb_attn_bwd_args b = *a;
      b.layout = bb_layout{BB_LAYOUT_CONTIGUOUS, gq, a->layout.seq_len, 0};
      b.q_device = q.dev;
      b.k_device = k.dev;
      b.n_q = q.rows;
      b.n_k = k.rows;
      b.q = static_cast<const char*>(a->q) + q.row0 * qrow * 2;
      b.dout = static_cast<const char*>(a->dout) + q.row0 * qrow * 2;
      b.lse = a->lse + q.row0;
      b.delta = a->delta + q.row0;
      b.dq = a->dq + q.row0 * qrow;
      b.k = static_cast<const char*>(a->k) + k.row0 * krow * 2;
      b.v = static_cast<const char*>(a->v) + k.row0 * krow * 2;
      b.dk = a->dk + k.row0 * krow;
      b.dv = a->dv + k.row0 * krow;
      if (int rc = launch_attn_bwd(b, st, a->n_q)) return rc;
    }
  }
  return BB_OK;
}

int bb_debug_set_split_rows(int64_t rows) {
  if (rows < 0 || rows % 128) return set_error(BB_ERR_INVALID, "bb_debug_set_split_rows: %lld is not a multiple of 128", (long long)rows);
  g_split_rows.store(rows);
  return BB_OK;
}

int bb_attn_bwd_preprocess(const void* dout, const float* o, float* delta, int64_t n, int32_t heads,
                           int32_t head_dim, void* stream) {
  if (n <= 0 || heads <= 0) return set_error(BB_ERR_INVALID, "bb_attn_bwd_preprocess: empty input");
  return launch_preprocess(dout, o, delta, n, heads, head_dim, static_cast<cudaStream_t>(stream));
}

int bb_permute_rows(void* dst, const void* src, const int64_t* index, int64_t n_rows, int64_t row_bytes,
                    int32_t scatter, void* stream) {
  return launch_permute(dst, src, index, n_rows, row_bytes, scatter, static_cast<cudaStream_t>(stream));
}

int bb_fill_u32(void* dst, uint32_t value, int64_t count, void* stream) {
  return launch_fill_u32(dst, value, count, static_cast<cudaStream_t>(stream));
}

int bb_add_rows_f32(float* dst, const float* src, int64_t rows, int64_t cols, int64_t dst_ld, int64_t src_ld,
                    void* stream) {
  return launch_add_rows(dst, src, rows, cols, dst_ld, src_ld, static_cast<cudaStream_t>(stream));
}

int bb_cast_pad_bf16(void* dst, const float* src, int64_t rows, int32_t cols_in, int32_t cols_out,
                     void* stream) {
  if (cols_out < cols_in) return set_error(BB_ERR_INVALID, "bb_cast_pad_bf16: cols_out < cols_in");
  return launch_cast_pad(dst, src, rows, cols_in, cols_out, static_cast<cudaStream_t>(stream));
}

int bb_gemm_bf16(const void* a, const void* b, float* c, int64_t m, int64_t n, int64_t k, int32_t a_mn,
                 int32_t b_mn, int32_t accumulate, void* stream) {
  return launch_gemm(a, b, c, m, n, k, a_mn ? m : k, b_mn ? n : k, n, a_mn != 0, b_mn != 0,
                     accumulate ? GEMM_ACCUM : GEMM_STORE, nullptr, false, static_cast<cudaStream_t>(stream));
}

int bb_gemm_bf16_rows(const void* a, const void* b, void* c, const int64_t* row_map, int64_t m, int64_t n, int64_t k,
                      int32_t b_mn, void* stream) {
  return launch_gemm_bf16(a, b, c, row_map, m, n, k, k, b_mn ? n : k, n, b_mn != 0, static_cast<cudaStream_t>(stream));
}

static int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

struct LmWorkspace {
  float* logits;
  void* g;
  float* pmax;
  float* psum;
  float* tgt;
  float* lse;
  int64_t bytes;
};

static LmWorkspace carve(void* base, int64_t rows, int64_t vocab, int64_t tiles) {
  const int64_t ldv = align_up(vocab, 8);
  int64_t off = 0;
  auto take = [&](int64_t bytes) {
    const int64_t at = off;
    off = align_up(off + bytes, 256);
    return static_cast<char*>(base) + at;
  };
  LmWorkspace w{};
  w.logits = reinterpret_cast<float*>(take(rows * ldv * 4));
  w.g = take(rows * ldv * 2);
  w.pmax = reinterpret_cast<float*>(take(rows * tiles * 4));
  w.psum = reinterpret_cast<float*>(take(rows * tiles * 4));
  w.tgt = reinterpret_cast<float*>(take(rows * 4));
  w.lse = reinterpret_cast<float*>(take(rows * 4));
  w.bytes = off;
  return w;
}

int64_t bb_lmhead_workspace_bytes(int64_t n, int64_t vocab, int64_t dim, int64_t rows_per_tile) {
  (void)dim;
  const int64_t rows = rows_per_tile < n ? rows_per_tile : n;
  const int64_t tiles = (vocab + gemm_n_tile() - 1) / gemm_n_tile();
  static char dummy[1];
  return carve(dummy, rows, vocab, tiles).bytes;
}

int bb_lmhead_fused(const bb_lmhead_args* a, void* stream) {
  if (!a) return set_error(BB_ERR_INVALID, "bb_lmhead_fused: null args");
  if (a->n < 1 || a->vocab < 1 || a->dim < 1) return set_error(BB_ERR_INVALID, "n, vocab, dim must all be >= 1");
  if (a->rows_per_tile < 1 || a->vocab_per_tile < 1)
    return set_error(BB_ERR_INVALID, "tile sizes must be >= 1, got rows=%lld, vocab=%lld",
                     (long long)a->rows_per_tile, (long long)a->vocab_per_tile);
  if (a->dim % 8) return set_error(BB_ERR_UNSUPPORTED, "bb_lmhead_fused: dim %lld must be a multiple of 8", (long long)a->dim);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t rows_tile = a->rows_per_tile < a->n ? a->rows_per_tile : a->n;
  const int64_t tiles = (a->vocab + gemm_n_tile() - 1) / gemm_n_tile();
  const int64_t ldv = align_up(a->vocab, 8);
  LmWorkspace w = carve(a->workspace, rows_tile, a->vocab, tiles);
  if (!a->workspace || a->workspace_bytes < w.bytes)
    return set_error(BB_ERR_INVALID, "bb_lmhead_fused: workspace %lld B < required %lld B",
                     (long long)a->workspace_bytes, (long long)w.bytes);
  const char* h = static_cast<const char*>(a->h);
  for (int64_t r0 = 0; r0 < a->n; r0 += rows_tile) {  // row tiles reduced in fixed order (lmhead.py:67)
    const int64_t rows = (a->n - r0) < rows_tile ? (a->n - r0) : rows_tile;
    const void* h_tile = h + r0 * a->dim * 2;
    LogitsEpilogue le{a->targets + r0, w.pmax, w.psum, w.tgt};
    int rc = launch_gemm(h_tile, a->w, w.logits, rows, a->vocab, a->dim, a->dim, a->dim, ldv, false, false,
                         GEMM_LOGITS, &le, true, st);
    if (rc) return rc;
    rc = launch_lmhead_reduce(w.pmax, w.psum, w.tgt, rows, static_cast<int32_t>(tiles), w.lse, a->loss + r0, st);
    if (rc) return rc;
    rc = launch_lmhead_dlogits(w.logits, w.lse, a->targets + r0, rows, a->vocab, ldv, w.g, st);
    if (rc) return rc;
    // dH[r0:r1] = G . W        (A = G K-major over vocab, B = W MN-major)
    rc = launch_gemm(w.g, a->w, a->dh + r0 * a->dim, rows, a->dim, a->vocab, ldv, a->dim, a->dim, false, true,
                     GEMM_STORE, nullptr, true, st);
    if (rc) return rc;
    // dW += G^T . H[r0:r1]     (A = G MN-major, B = H MN-major)
    rc = launch_gemm(w.g, h_tile, a->dw, a->vocab, a->dim, rows, ldv, a->dim, a->dim, true, true, GEMM_ACCUM,
                     nullptr, false, st);
    if (rc) return rc;
  }
  return BB_OK;
}

// ---- float64 tile math (numerics.py:35-116, oracle.py:129-154) ----
#define BB_ST static_cast<cudaStream_t>(stream)
int bb_matmul_f64(const double* a, int64_t sa0, int64_t sa1, const double* b, int64_t sb0, int64_t sb1,
                  double* c, int64_t m, int64_t n, int64_t k, void* stream) {
  if ((m * k && !a) || (k * n && !b) || (m * n && !c)) return set_error(BB_ERR_INVALID, "bb_matmul_f64: null operand");
  return launch_matmul_f64(a, sa0, sa1, b, sb0, sb1, c, m, n, k, BB_ST);
}
int bb_scale_mask_f64(double* s, const uint8_t* allowed, double scale, int64_t n, void* stream) {
  if (n < 0) return set_error(BB_ERR_INVALID, "bb_scale_mask_f64: negative length");
  return launch_scale_mask_f64(s, allowed, scale, n, BB_ST);
}
int bb_row_logsumexp_f64(const double* s, int64_t rows, int64_t cols, int64_t lds, double* out, void* stream) {
  if (rows < 0 || cols <= 0 || lds < cols)
    return set_error(BB_ERR_INVALID, "row_logsumexp requires a nonempty matrix (rows %lld, cols %lld, lds %lld)",
                     (long long)rows, (long long)cols, (long long)lds);
  return launch_row_lse_f64(s, rows, cols, lds, out, BB_ST);
}
int bb_lse_merge_f64(const double* a, const double* b, double* out, int64_t n, void* stream) {
  if (n < 0) return set_error(BB_ERR_INVALID, "bb_lse_merge_f64: negative length");
  return launch_lse_merge_f64(a, b, out, n, BB_ST);
}
int bb_exp_shifted_f64(const double* s, const double* lse, double* out, int64_t rows, int64_t cols, void* stream) {
  if (rows < 0 || cols < 0) return set_error(BB_ERR_INVALID, "bb_exp_shifted_f64: negative extent");
  return launch_exp_shifted_f64(s, lse, out, rows, cols, BB_ST);
}
int bb_exp_gap_f64(const double* a, const double* b, double* out, int64_t n, void* stream) {
  if (n < 0) return set_error(BB_ERR_INVALID, "bb_exp_gap_f64: negative length");
  return launch_exp_gap_f64(a, b, out, n, BB_ST);
}
int bb_rowsum_hadamard_f64(const double* a, const double* b, double* out, int64_t rows, int64_t cols, void* stream) {
  if (rows < 0 || cols < 0) return set_error(BB_ERR_INVALID, "bb_rowsum_hadamard_f64: negative extent");
  return launch_rowsum_hadamard_f64(a, b, out, rows, cols, BB_ST);
}
int bb_xent_f64(const double* logits, const double* lse, const int64_t* targets, int64_t rows, int64_t vocab,
                double* loss, double* g, void* stream) {
  if (rows < 0 || vocab <= 0) return set_error(BB_ERR_INVALID, "bb_xent_f64: bad extent");
  return launch_xent_f64(logits, lse, targets, rows, vocab, loss, g, BB_ST);
}
#undef BB_ST

}  // extern "C"
