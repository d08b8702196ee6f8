// sts_sparse_decode.cu — gathered-KV sparse flash-decode for the gamma+1
// verification rows (x GQA group) on sm_100a.
//
// BF16 path (the product path).  Per CTA: one (unit, split) — a contiguous
// slice of the unit's selected-key list.  Each warp owns a private
// cp.async ring of STAGES tiles of 16 gathered keys (K and V rows, 16-byte
// copies, XOR-swizzled so ldmatrix is conflict-free) and its own online
// softmax state, so the steady state needs no CTA barrier.  The math runs on
// the tensor cores "transposed": S^T = K.Q^T and O^T += V^T.P^T with
// mma.sync m16n8k16 (keys / head-dim as M, the stacked query rows as N in
// steps of 8), so M = 20 (gamma+1 = 5 rows x GQA 4) costs 3 n-tiles instead
// of padding rows to 32; P^T is re-laid out for the second MMA with
// movmatrix.trans.  At the end the warps are merged through shared memory and
// either the final rows (splits == 1) or fp32 partials + LSE (merged by
// sts_lse_merge) are written.
//
// F32 path (parity): CUDA-core fp32, one warp per query row, lanes over keys.
#include "sts_decode.cuh"

namespace sts {
namespace {

__device__ __forceinline__ int unit_count(const DecodeParams& p, int64_t u) {
  return p.idx ? p.cnt[u] : p.n_dense;
}

// ---------------------------------------------------------------------------
// F32 parity path: one warp per query row; lanes stride over keys.
// ---------------------------------------------------------------------------
constexpr int F32_WARPS = 4;

__global__ void __launch_bounds__(F32_WARPS * 32) sparse_decode_f32_kernel(DecodeParams p) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t u = blockIdx.y;
  const int split = blockIdx.x;
  const int D = p.d;
  const int M = p.M;
  const int cnt = unit_count(p, u);
  const int c0 = (int)((int64_t)split * cnt / p.splits);
  const int c1 = (int)((int64_t)(split + 1) * cnt / p.splits);
  const int64_t ukv = p.kv_div > 1 ? u / p.kv_div : u;
  const float* kg = static_cast<const float*>(p.k) + ukv * p.kv_stride;
  const float* vg = static_cast<const float*>(p.v) + ukv * p.kv_stride;
  const int32_t* idxg = p.idx ? p.idx + u * p.idx_ld : nullptr;
  const uint32_t* memg = p.member ? p.member + u * p.idx_ld : nullptr;

  for (int r = warp; r < M; r += F32_WARPS) {
    const float* q = static_cast<const float*>(p.q) + (u * M + r) * (int64_t)D;
    float m = -INFINITY, l = 0.f;
    float acc[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) acc[t] = 0.f;
    const int rm = r % p.rows_per_head;
    for (int base = c0; base < c1; base += 32) {
      const int j = base + lane;
      bool ok = j < c1;
      int pos = 0;
      float s = -INFINITY;
      if (ok) {
        pos = idxg ? idxg[j] : j;
        if (p.causal_base >= 0) ok = ok && (pos + p.pos_offset - p.causal_base <= rm);
        if (memg) ok = ok && ((memg[j] >> (r & 31)) & 1u);
      }
      if (ok) {
        const float* kr = kg + (int64_t)pos * p.row_stride;
        float dot = 0.f;
        for (int e = 0; e < D; ++e) dot = fmaf(q[e], kr[e], dot);
        s = dot * p.scale;
      }
      float tmax = s;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
      const float m_new = fmaxf(m, tmax);
      if (m_new == -INFINITY) continue;
      const float alpha = expf(m - m_new);
      const float pj = ok ? expf(s - m_new) : 0.f;
      float psum = pj;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) psum += __shfl_xor_sync(0xffffffffu, psum, o);
      l = l * alpha + psum;
      m = m_new;
#pragma unroll
      for (int t = 0; t < 8; ++t) acc[t] *= alpha;
      for (int src = 0; src < 32; ++src) {
        const float pk = __shfl_sync(0xffffffffu, pj, src);
        const int posk = __shfl_sync(0xffffffffu, pos, src);
        if (pk == 0.f) continue;
        const float* vr = vg + (int64_t)posk * p.row_stride;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const int e = lane + 32 * t;
          if (e < D) acc[t] = fmaf(pk, vr[e], acc[t]);
        }
      }
    }
    const float lse = l > 0.f ? m + logf(l) : -INFINITY;
    if (p.splits == 1) {
      float* og = static_cast<float*>(p.out) + (u * M + r) * (int64_t)D;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int e = lane + 32 * t;
        if (e < D) og[e] = l > 0.f ? acc[t] / l : 0.f;
      }
      if (lane == 0) {
        if (p.lse) p.lse[u * M + r] = lse;
        if (!(l > 0.f)) set_status(p.status, STS_DEV_EMPTY_ROW);
      }
    } else {
      const int64_t base = ((int64_t)split * p.units + u) * M + r;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int e = lane + 32 * t;
        if (e < D) p.o_part[base * D + e] = l > 0.f ? acc[t] / l : 0.f;
      }
      if (lane == 0) p.l_part[base] = lse;
    }
  }
}

}  // namespace

// splits so that units*splits CTAs fill the chip in whole waves of 2 CTAs/SM
int auto_splits(int64_t units, int64_t keys_per_unit) {
  const int64_t slots = 2LL * num_sms();
  int64_t tiles = (keys_per_unit + KEY_TILE * 8 - 1) / (KEY_TILE * 8);  // >= 8 tiles per CTA
  int64_t best = 1;
  double best_eff = 0.0;
  for (int64_t s = 1; s <= 64 && s <= (tiles > 0 ? tiles : 1); ++s) {
    const int64_t ctas = units * s;
    const int64_t waves = (ctas + slots - 1) / slots;
    const double eff = (double)ctas / (double)(waves * slots);
    // prefer fuller last waves, then more parallelism up to ~8 waves
    const double score = eff - 0.002 * (double)s;
    if (waves <= 16 && score > best_eff) {
      best_eff = score;
      best = s;
    }
  }
  return (int)best;
}

}  // namespace sts

using namespace sts;

extern "C" size_t sts_sparse_decode_workspace_bytes(int64_t units, int32_t M, int32_t d, int32_t splits) {
  // bf16: persistent stream-K partials; f32: split-K partials (splits > 1)
  const size_t f32 = splits <= 1 ? 0 : (size_t)splits * units * M * ((size_t)d + 1) * sizeof(float) + 256;
  const size_t bf16 = stream_workspace_bytes(MODE_DECODE, units, M, d);
  return f32 > bf16 ? f32 : bf16;
}

static int sparse_decode_impl(int32_t dtype, int32_t out_dtype, const void* q_dev, const void* k_cache_dev,
                                 const void* v_cache_dev, int64_t kv_unit_stride, int64_t kv_row_stride,
                                 int64_t units,
                                 int32_t M, int32_t d, const int32_t* idx_dev, int64_t idx_ld,
                                 const int32_t* cnt_dev, int32_t n_dense,
                                 const uint32_t* member_dev, int32_t causal_base,
                                 int32_t rows_per_head, int32_t pos_offset, float scale,
                                 void* out_dev, float* lse_dev, int32_t splits,
                                 int32_t* status_dev, void* workspace_dev,
                                 size_t workspace_bytes, void* stream, int64_t kv_div) {
  STS_REQUIRE(units >= 0, STS_ERR_CONTRACT, "units must be >= 0");
  if (units == 0) return STS_OK;
  STS_REQUIRE(q_dev && k_cache_dev && v_cache_dev && out_dev, STS_ERR_CONTRACT, "null buffer");
  STS_REQUIRE(M >= 1, STS_ERR_CONTRACT, "M must be >= 1");
  STS_REQUIRE(!member_dev || M <= 32, STS_ERR_CONTRACT, "row membership bits need M <= 32");
  STS_REQUIRE(rows_per_head >= 1, STS_ERR_CONTRACT, "rows_per_head must be >= 1");
  STS_REQUIRE(idx_dev ? (cnt_dev != nullptr) : (n_dense >= 0), STS_ERR_CONTRACT,
              "index list needs counts / dense needs n_dense");
  STS_REQUIRE(dtype == STS_DTYPE_BF16 || (splits >= 1 && splits <= 4096), STS_ERR_CONTRACT,
              "splits must be in [1, 4096]");
  STS_REQUIRE(dtype != STS_DTYPE_F32 || units <= 65535, STS_ERR_CONTRACT, "f32 path: units must be <= 65535 (grid.y)");
  cudaStream_t st = static_cast<cudaStream_t>(stream);

  DecodeParams p;
  memset(&p, 0, sizeof(p));
  p.q = q_dev;
  p.k = k_cache_dev;
  p.v = v_cache_dev;
  p.kv_stride = kv_unit_stride;
  p.kv_div = kv_div;
  p.row_stride = kv_row_stride > 0 ? kv_row_stride : d;
  STS_REQUIRE(p.row_stride >= d, STS_ERR_CONTRACT, "kv_row_stride must be >= d");
  p.units = units;
  p.M = M;
  p.d = d;
  p.idx = idx_dev;
  p.idx_ld = idx_ld;
  p.cnt = cnt_dev;
  p.n_dense = n_dense;
  p.member = member_dev;
  p.causal_base = causal_base;
  p.rows_per_head = rows_per_head;
  p.pos_offset = pos_offset;
  p.scale = scale;
  p.out = out_dev;
  STS_REQUIRE(out_dtype == dtype || out_dtype == STS_DTYPE_F32, STS_ERR_CONTRACT,
              "out_dtype must equal dtype or be F32 (partials for a later LSE merge)");
  p.out_f32 = out_dtype == STS_DTYPE_F32 ? 1 : 0;
  p.lse = lse_dev;
  p.splits = splits;
  p.status = status_dev;
  p.o_part = nullptr;
  p.l_part = nullptr;
  p.lse_in = nullptr;
  p.probs_out = nullptr;
  p.out_ld = 0;
  p.probs_mode = 0;
  p.pieces = nullptr;
  p.schedule = 0;
  if (dtype == STS_DTYPE_BF16) {
    // bf16: `splits` picks the work schedule (0 auto, 1 persistent stream-K,
    // 2/3/4/6/8 thread-block clusters of that many CTAs per unit)
    STS_REQUIRE(splits == 0 || splits == 1 || splits == 2 || splits == 3 || splits == 4 || splits == 6 ||
                    splits == 8,
                STS_ERR_CONTRACT, "bf16 schedule must be 0 (auto), 1 (stream-K) or a cluster size in {2,3,4,6,8}, got %d",
                splits);
    p.schedule = splits;
    return stream_launch(MODE_DECODE, p, workspace_dev, workspace_bytes, st);
  }
  if (splits > 1) {
    size_t need = (size_t)splits * units * M * ((size_t)d + 1) * sizeof(float);
    STS_REQUIRE(workspace_dev && workspace_bytes >= need, STS_ERR_CONTRACT,
                "sparse decode workspace too small: need %zu, got %zu", need, workspace_bytes);
    p.o_part = static_cast<float*>(workspace_dev);
    p.l_part = p.o_part + (size_t)splits * units * M * d;
  }

  int rc;
  if (dtype == STS_DTYPE_F32) {
    STS_REQUIRE(d >= 1 && d <= 256, STS_ERR_CONTRACT, "f32 sparse decode supports d <= 256");
    dim3 grid(splits, (unsigned)units);
    sparse_decode_f32_kernel<<<grid, F32_WARPS * 32, 0, st>>>(p);
    STS_LAUNCH_CHECK();
    rc = STS_OK;
  } else {
    set_error("unknown dtype %d", dtype);
    return STS_ERR_CONTRACT;
  }
  if (rc != STS_OK || splits == 1) return rc;
  return lse_merge_launch(p.o_part, p.l_part, splits, units * M, d, dtype, out_dev, lse_dev, st);
}

extern "C" int sts_sparse_decode(int32_t dtype, int32_t out_dtype, const void* q_dev, const void* k_cache_dev,
                                 const void* v_cache_dev, int64_t kv_unit_stride, int64_t kv_row_stride,
                                 int64_t units, int32_t M, int32_t d, const int32_t* idx_dev, int64_t idx_ld,
                                 const int32_t* cnt_dev, int32_t n_dense, const uint32_t* member_dev,
                                 int32_t causal_base, int32_t rows_per_head, int32_t pos_offset, float scale,
                                 void* out_dev, float* lse_dev, int32_t splits, int32_t* status_dev,
                                 void* workspace_dev, size_t workspace_bytes, void* stream) {
  return sparse_decode_impl(dtype, out_dtype, q_dev, k_cache_dev, v_cache_dev, kv_unit_stride, kv_row_stride, units,
                            M, d, idx_dev, idx_ld, cnt_dev, n_dense, member_dev, causal_base, rows_per_head,
                            pos_offset, scale, out_dev, lse_dev, splits, status_dev, workspace_dev, workspace_bytes,
                            stream, 1);
}

extern "C" int sts_sparse_prefill(int32_t dtype, int32_t out_dtype, const void* q_dev, const void* k_cache_dev,
                                  const void* v_cache_dev, int64_t kv_unit_stride, int64_t kv_row_stride,
                                  int64_t kv_units, int32_t rows, int32_t M, int32_t d, const int32_t* idx_dev,
                                  int64_t idx_ld, const int32_t* cnt_dev, float scale, void* out_dev, float* lse_dev,
                                  int32_t* status_dev, void* workspace_dev, size_t workspace_bytes, void* stream) {
  STS_REQUIRE(kv_units >= 0 && rows >= 0, STS_ERR_CONTRACT, "kv_units and rows must be >= 0");
  STS_REQUIRE(idx_dev && cnt_dev, STS_ERR_CONTRACT, "sparse prefill needs per-row index lists");
  // unit (g, t) = g*rows + t attends exactly its list (already causal); its
  // K/V block is g's: kv_div = rows
  return sparse_decode_impl(dtype, out_dtype, q_dev, k_cache_dev, v_cache_dev, kv_unit_stride, kv_row_stride,
                            kv_units * rows, M, d, idx_dev, idx_ld, cnt_dev, 0, nullptr, -1, 1, 0, scale, out_dev,
                            lse_dev, 1, status_dev, workspace_dev, workspace_bytes, stream, rows > 1 ? rows : 1);
}

extern "C" int32_t sts_sparse_decode_schedule(int64_t units, int32_t M, int32_t d, int64_t keys_per_unit,
                                              int32_t schedule) {
  if (units <= 0 || M < 1 || M > 48 || (d != 64 && d != 128)) return 0;
  if (schedule != 0) return schedule;
  DecodeParams p;
  memset(&p, 0, sizeof(p));
  p.units = units;
  p.M = M;
  p.d = d;
  p.n_dense = keys_per_unit > 0x7fffffff ? 0x7fffffff : (int)keys_per_unit;
  p.plan_only = 1;
  const int r = verify_decode_launch(MODE_DECODE, p, nullptr);
  return r >= 1 && r <= 8 ? r : 0;
}

extern "C" int32_t sts_auto_splits(int64_t units, int64_t keys_per_unit) {
  return auto_splits(units, keys_per_unit);
}

// ---------------------------------------------------------------------------
// draft-score capture
// ---------------------------------------------------------------------------
extern "C" size_t sts_draft_workspace_bytes(int64_t units, int32_t GR, int32_t n_keys) {
  (void)n_keys;
  return capture_workspace_bytes(units, GR);
}

extern "C" int sts_draft_lse(int32_t dtype, const void* q_dev, const void* k_cache_dev,
                             int64_t kv_unit_stride, int64_t units, int32_t G, int32_t R,
                             int32_t d, int32_t n_keys, int32_t pos_offset, int32_t base,
                             float scale, float* lse_dev, void* workspace_dev,
                             size_t workspace_bytes, void* stream) {
  STS_REQUIRE(dtype == STS_DTYPE_BF16, STS_ERR_CONTRACT, "draft scores run in bf16");
  STS_REQUIRE(units >= 0 && G >= 1 && R >= 1 && n_keys >= 0, STS_ERR_CONTRACT, "bad draft shape");
  STS_REQUIRE(units <= 65535, STS_ERR_CONTRACT, "units must be <= 65535");
  STS_REQUIRE(q_dev && k_cache_dev && lse_dev, STS_ERR_CONTRACT, "null buffer");
  if (units == 0) return STS_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return capture_launch(0, q_dev, k_cache_dev, kv_unit_stride, units, G, R, d, n_keys, pos_offset, base, scale,
                        lse_dev, nullptr, 0, nullptr, 0, workspace_dev, workspace_bytes, st);
}

extern "C" int sts_draft_probs(int32_t dtype, const void* q_dev, const void* k_cache_dev,
                               int64_t kv_unit_stride, int64_t units, int32_t G, int32_t R,
                               int32_t d, int32_t n_keys, int32_t pos_offset, int32_t base,
                               float scale, const float* lse_dev, int32_t mode, float* out_dev,
                               int64_t out_ld, void* stream) {
  STS_REQUIRE(dtype == STS_DTYPE_BF16, STS_ERR_CONTRACT, "draft scores run in bf16");
  STS_REQUIRE(units >= 0 && G >= 1 && R >= 1 && n_keys >= 0, STS_ERR_CONTRACT, "bad draft shape");
  STS_REQUIRE(units <= 65535, STS_ERR_CONTRACT, "units must be <= 65535");
  STS_REQUIRE(q_dev && k_cache_dev && lse_dev && out_dev, STS_ERR_CONTRACT, "null buffer");
  STS_REQUIRE(mode == 0 || mode == 1, STS_ERR_CONTRACT, "mode must be 0 (S) or 1 (R)");
  STS_REQUIRE(out_ld >= n_keys, STS_ERR_CONTRACT, "out_ld must be >= n_keys");
  if (units == 0) return STS_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return capture_launch(1, q_dev, k_cache_dev, kv_unit_stride, units, G, R, d, n_keys, pos_offset, base, scale,
                        nullptr, lse_dev, mode, out_dev, out_ld, nullptr, 0, st);
}

extern "C" int sts_draft_scores(int32_t dtype, const void* q_dev, const void* k_cache_dev,
                                int64_t kv_unit_stride, int64_t units, int32_t G, int32_t R,
                                int32_t d, int32_t n_keys, int32_t pos_offset, int32_t base,
                                float scale, float* out_dev, int64_t out_ld, void* stream) {
  STS_REQUIRE(dtype == STS_DTYPE_BF16, STS_ERR_CONTRACT, "draft scores run in bf16");
  STS_REQUIRE(units >= 0 && G >= 1 && R >= 1 && n_keys >= 0, STS_ERR_CONTRACT, "bad draft shape");
  STS_REQUIRE(units <= 65535, STS_ERR_CONTRACT, "units must be <= 65535");
  STS_REQUIRE(q_dev && k_cache_dev && out_dev, STS_ERR_CONTRACT, "null buffer");
  STS_REQUIRE(out_ld >= n_keys, STS_ERR_CONTRACT, "out_ld must be >= n_keys");
  if (units == 0) return STS_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return capture_launch(1, q_dev, k_cache_dev, kv_unit_stride, units, G, R, d, n_keys, pos_offset, base, scale,
                        nullptr, nullptr, 2, out_dev, out_ld, nullptr, 0, st);
}
