// sts_select_dist.cu — sequence-sharded top-k selection (context-parallel
// decode).
//
// A logical row of n committed positions is split over P ranks; this rank
// holds the positions [lo, lo + n_local) of it (page-aligned).  The global
// top-k under the reference rule (score descending, ties to the lowest global
// index, src/numkit.py:84) is found without moving any score across ranks:
//
//   begin    keys of the local positions (fp32 order keys, or fp64 page-sum
//            keys in numpy reduceat order) + local histogram of digit 0
//   round r  (host: hist_global = allreduce_sum(hist_local))
//            advance: every rank walks the SAME global histogram, so every
//            rank derives the same digit / prefix / remaining k; the local
//            count of the chosen bin is kept (this rank's ties)
//            hist:    local histogram of digit r+1 under the new prefix
//   finish   (host: ties_all = allgather(ties_local))
//            emit: keys strictly above the threshold, plus this rank's share
//            of the threshold ties — the first (need - ties on lower ranks)
//            of them in index order — plus the extras and the in-block tail,
//            as ascending LOCAL offsets.
//
// Digits are 8 bits from the top (4 rounds for token keys, 8 for page keys);
// a row whose chosen bin is taken whole (remaining k == bin count) is resolved
// early and skips the remaining rounds' work.  Collectives stay O(rounds + 1)
// for all rows of all layers at once (one histogram buffer per round).
#include "sts_common.cuh"

namespace sts {
namespace {

constexpr int DD_BITS = 8;
constexpr int DD_BINS = 1 << DD_BITS;
constexpr int DIST_THREADS = 512;
constexpr int DIST_CHUNK = 8192;      // keys per CTA in the key / histogram passes
constexpr int EMIT_THREADS = 1024;
constexpr int EMIT_WARPS = EMIT_THREADS / 32;

struct DistState {
  uint64_t prefix;  // chosen digits so far (in key space)
  uint64_t pmask;   // bits of the key the prefix covers
  int krem;         // keys still to take at / below the prefix
  int done;         // 1: resolved (threshold = prefix under pmask)
  int dense;        // 1: budget >= n, every position selected
  int ties_global;  // keys matching the final prefix, all ranks
  int ties_local;   // ... on this rank
  int pad[3];
};

struct DistParams {
  const float* scores;
  int64_t ld;
  const int32_t* row_src;
  int nsrc;
  int64_t rows;
  int n_global;   // committed positions of the logical row
  int lo;         // first global position held here
  int n_local;    // positions held here (lo + n_local <= n_global not required)
  int k_top;      // tokens (page_size 1) or pages to select
  int page_size;
  DistState* state;
  uint8_t* keys;  // [rows][nkeys_pad] of K
  int64_t keys_ld;
};

__device__ __forceinline__ int local_committed(const DistParams& p) {
  const int hi = p.n_global - p.lo;  // positions < n_global held here
  return hi < 0 ? 0 : (hi < p.n_local ? hi : p.n_local);
}

__device__ __forceinline__ float dist_value(const DistParams& p, const int32_t* srcs, int j) {
  float acc = p.scores[(int64_t)srcs[0] * p.ld + j];
  for (int s = 1; s < p.nsrc; ++s) acc = __fadd_rn(acc, p.scores[(int64_t)srcs[s] * p.ld + j]);
  return acc;
}

// numpy pairwise_sum (float64) over row values [start, start+n) — the same
// order as sts_select.cu / oracle numpy_pairwise_sum
__device__ double dist_pairwise(const DistParams& p, const int32_t* srcs, int start, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, (double)dist_value(p, srcs, start + i));
    return r;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = (double)dist_value(p, srcs, start + j);
    int i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], (double)dist_value(p, srcs, start + i + j));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, (double)dist_value(p, srcs, start + i));
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(dist_pairwise(p, srcs, start, n2), dist_pairwise(p, srcs, start + n2, n - n2));
}

__device__ __forceinline__ void load_srcs(const DistParams& p, int64_t r, int32_t (&srcs)[8]) {
  if (p.row_src) {
    for (int s = 0; s < p.nsrc; ++s) srcs[s] = p.row_src[r * p.nsrc + s];
  } else {
    srcs[0] = (int32_t)r;
  }
}

// number of local keys of a row: tokens, or pages (lo is page-aligned)
__device__ __forceinline__ int local_keys(const DistParams& p) {
  const int nc = local_committed(p);
  return p.page_size == 1 ? nc : (nc + p.page_size - 1) / p.page_size;
}

template <typename K>
__device__ __forceinline__ int digit_of(K key, int round) {
  constexpr int KB = sizeof(K) * 8;
  return (int)((key >> (KB - DD_BITS * (round + 1))) & (K)(DD_BINS - 1));
}

// keys of the local positions + round-0 histogram; grid (chunks, rows)
template <typename K>
__global__ void __launch_bounds__(DIST_THREADS) dist_keys_kernel(DistParams p, int32_t* hist) {
  __shared__ uint32_t sh[DD_BINS];
  const int64_t r = blockIdx.y;
  for (int i = threadIdx.x; i < DD_BINS; i += DIST_THREADS) sh[i] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    DistState s;
    s.prefix = 0;
    s.pmask = 0;
    s.krem = p.k_top;
    const int n_units = p.page_size == 1 ? p.n_global : (p.n_global + p.page_size - 1) / p.page_size;
    s.dense = p.k_top >= n_units ? 1 : 0;
    s.done = s.dense;
    s.ties_global = 0;
    s.ties_local = 0;
    s.pad[0] = s.pad[1] = s.pad[2] = 0;
    p.state[r] = s;
  }
  __syncthreads();
  const int nk = local_keys(p);
  const int nc = local_committed(p);
  int32_t srcs[8];
  load_srcs(p, r, srcs);
  K* keys = reinterpret_cast<K*>(p.keys + r * p.keys_ld * sizeof(K));
  const int j_end = min(nk, (int)(blockIdx.x + 1) * DIST_CHUNK);
  for (int j = blockIdx.x * DIST_CHUNK + threadIdx.x; j < j_end; j += DIST_THREADS) {
    K key;
    if constexpr (sizeof(K) == 4) {
      key = f32_key(dist_value(p, srcs, j));
    } else {
      const int start = j * p.page_size;
      const int len = min(p.page_size, nc - start);
      const double x0 = (double)dist_value(p, srcs, start);
      key = f64_key(len == 1 ? x0 : __dadd_rn(x0, dist_pairwise(p, srcs, start + 1, len - 1)));
    }
    keys[j] = key;
    atomicAdd(&sh[digit_of<K>(key, 0)], 1u);
  }
  __syncthreads();
  int32_t* h = hist + r * DD_BINS;
  for (int i = threadIdx.x; i < DD_BINS; i += DIST_THREADS)
    if (sh[i]) atomicAdd(h + i, (int)sh[i]);
}

// local histogram of digit `round` among keys matching the row's prefix
template <typename K>
__global__ void __launch_bounds__(DIST_THREADS) dist_hist_kernel(DistParams p, int round, int32_t* hist) {
  __shared__ uint32_t sh[DD_BINS];
  const int64_t r = blockIdx.y;
  const DistState st = p.state[r];
  if (st.done) return;
  for (int i = threadIdx.x; i < DD_BINS; i += DIST_THREADS) sh[i] = 0;
  __syncthreads();
  const int nk = local_keys(p);
  const K* keys = reinterpret_cast<const K*>(p.keys + r * p.keys_ld * sizeof(K));
  const K pm = (K)st.pmask, pf = (K)st.prefix;
  const int j_end = min(nk, (int)(blockIdx.x + 1) * DIST_CHUNK);
  for (int j = blockIdx.x * DIST_CHUNK + threadIdx.x; j < j_end; j += DIST_THREADS) {
    const K key = keys[j];
    if ((key & pm) == pf) atomicAdd(&sh[digit_of<K>(key, round)], 1u);
  }
  __syncthreads();
  int32_t* h = hist + r * DD_BINS;
  for (int i = threadIdx.x; i < DD_BINS; i += DIST_THREADS)
    if (sh[i]) atomicAdd(h + i, (int)sh[i]);
}

// advance every row by one digit from the GLOBAL histogram; one warp per row
template <typename K>
__global__ void dist_advance_kernel(DistParams p, int round, const int32_t* hist_global,
                                    const int32_t* hist_local) {
  constexpr int KB = sizeof(K) * 8;
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= p.rows) return;
  DistState st = p.state[r];
  if (st.done) return;
  const int32_t* hg = hist_global + r * DD_BINS;
  // lane owns bins 255-8*lane .. 248-8*lane (descending)
  int cnt[8];
  int lsum = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    cnt[q] = hg[DD_BINS - 1 - 8 * lane - q];
    lsum += cnt[q];
  }
  int incl = lsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const int excl = incl - lsum;
  const bool mine = excl < st.krem && st.krem <= incl;
  const uint32_t who = __ballot_sync(0xffffffffu, mine);
  if (who == 0) return;  // inconsistent histogram (cannot happen): leave the row unresolved
  if (lane != __ffs(who) - 1) return;
  int acc = excl, digit = 0, inbin = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    if (acc < st.krem && st.krem <= acc + cnt[q]) {
      digit = DD_BINS - 1 - 8 * lane - q;
      inbin = cnt[q];
      break;
    }
    acc += cnt[q];
  }
  const int shift = KB - DD_BITS * (round + 1);
  st.prefix |= (uint64_t)digit << shift;
  st.pmask |= (uint64_t)(DD_BINS - 1) << shift;
  st.krem -= acc;
  if (shift == 0 || st.krem == inbin) {
    st.done = 1;
    st.ties_global = inbin;
    st.ties_local = hist_local[r * DD_BINS + digit];
  }
  p.state[r] = st;
}

__device__ __forceinline__ int emit_block_scan(int v, int* warp_tot, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int x = warp_tot[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    warp_tot[lane] = x;
  }
  __syncthreads();
  const int before = warp > 0 ? warp_tot[warp - 1] : 0;
  total = warp_tot[EMIT_WARPS - 1];
  __syncthreads();
  return before + incl - v;
}

struct EmitParams {
  int rank;
  int nranks;
  const int32_t* ties_all;  // [nranks][rows]
  uint32_t flags;
  int recent_window;
  int tail_len;
  int n_kv_local;           // positions held here (committed + tail)
  int32_t* idx_out;
  int64_t idx_ld;
  int32_t* cnt_out;
  int32_t* status;
  uint32_t* page_bits;      // [rows][page_bits_ld] scratch (page mode)
  int64_t page_bits_ld;
};

// one CTA per row: ascending local offsets of the selected positions.
// Phase 1 decides the local keys (tokens, or pages) in index order: above the
// threshold, or a threshold tie whose global tie rank (ties on lower ranks +
// local rank) is below the remaining k.  Token mode writes indices directly;
// page mode records a page bitmap and phase 2 expands it to tokens.  Extras
// (sink, recent window, current — global positions) and the in-block tail
// are added in the token pass.
template <typename K>
__global__ void __launch_bounds__(EMIT_THREADS) dist_emit_kernel(DistParams p, EmitParams e) {
  __shared__ int warp_tot[EMIT_WARPS];
  const int64_t r = blockIdx.x;
  const DistState st = p.state[r];
  const int nc = local_committed(p);
  const int nk = local_keys(p);
  const int ps = p.page_size;
  const K* keys = reinterpret_cast<const K*>(p.keys + r * p.keys_ld * sizeof(K));
  int32_t* out = e.idx_out + r * e.idx_ld;
  uint32_t* pbits = e.page_bits ? e.page_bits + r * e.page_bits_ld : nullptr;
  int before = 0;
  for (int q = 0; q < e.rank; ++q) before += e.ties_all[(int64_t)q * p.rows + r];
  int need = st.krem - before;
  need = need < 0 ? 0 : need;
  const bool all_ties = need >= st.ties_local;
  const int lo_extra = e.recent_window > 0 ? p.n_global - e.recent_window : p.n_global;
  const bool cur = (e.flags & STS_SEL_CURRENT) != 0, sink = (e.flags & STS_SEL_SINK) != 0;
  const K pm = (K)st.pmask, pf = (K)st.prefix;
  const int lane = threadIdx.x & 31;

  auto is_extra = [&](int j) {
    const int g = p.lo + j;
    return g >= lo_extra || (sink && g == 0) || (cur && g == p.n_global - 1);
  };

  int run_sel = 0, run_tie = 0;
  for (int base = 0; base < nk; base += 4 * EMIT_THREADS) {
    const int j0 = base + 4 * threadIdx.x;
    uint32_t sel = 0, eq = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = j0 + q;
      if (j >= nk) break;
      if (st.dense) {
        sel |= 1u << q;
        continue;
      }
      const K mk = keys[j] & pm;
      sel |= mk > pf ? (1u << q) : 0u;
      eq |= mk == pf ? (1u << q) : 0u;
    }
    if (all_ties) {
      sel |= eq;
    } else {
      int tie_tot;
      int rank = run_tie + emit_block_scan(__popc(eq), warp_tot, tie_tot);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if ((eq >> q) & 1u) {
          if (rank < need) sel |= 1u << q;
          ++rank;
        }
      run_tie += tie_tot;
    }
    if (ps == 1) {
      if (j0 + 3 >= lo_extra - p.lo || (sink && p.lo == 0 && j0 == 0) || (cur && j0 + 3 >= p.n_global - 1 - p.lo)) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (j0 + q < nk && is_extra(j0 + q)) sel |= 1u << q;
      }
      int sel_tot;
      int pos = run_sel + emit_block_scan(__popc(sel), warp_tot, sel_tot);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if ((sel >> q) & 1u) {
          if (pos < e.idx_ld) out[pos] = j0 + q;
          else set_status(e.status, STS_DEV_IDX_CAPACITY);
          ++pos;
        }
      run_sel += sel_tot;
    } else {
      // 8 lanes x 4 pages = one 32-bit word of the page bitmap
      uint32_t w = (sel & 0xfu) << ((lane & 7) * 4);
      w |= __shfl_xor_sync(0xffffffffu, w, 1);
      w |= __shfl_xor_sync(0xffffffffu, w, 2);
      w |= __shfl_xor_sync(0xffffffffu, w, 4);
      if ((lane & 7) == 0 && j0 < nk) pbits[j0 >> 5] = w;
    }
  }
  if (ps > 1) {
    __syncthreads();  // page bitmap (global, this CTA's own writes) visible block-wide
    for (int base = 0; base < nc; base += 4 * EMIT_THREADS) {
      const int j0 = base + 4 * threadIdx.x;
      uint32_t sel = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = j0 + q;
        if (j >= nc) break;
        const int pg = j / ps;
        if (((pbits[pg >> 5] >> (pg & 31)) & 1u) || is_extra(j)) sel |= 1u << q;
      }
      int sel_tot;
      int pos = run_sel + emit_block_scan(__popc(sel), warp_tot, sel_tot);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if ((sel >> q) & 1u) {
          if (pos < e.idx_ld) out[pos] = j0 + q;
          else set_status(e.status, STS_DEV_IDX_CAPACITY);
          ++pos;
        }
      run_sel += sel_tot;
    }
  }
  // in-block tail: global [n_global, n_global + tail_len) held here
  const int t_lo = max(p.n_global - p.lo, 0);
  const int t_hi = min(p.n_global + e.tail_len - p.lo, e.n_kv_local);
  for (int j = t_lo + threadIdx.x; j < t_hi; j += EMIT_THREADS) {
    const int pos = run_sel + (j - t_lo);
    if (pos < e.idx_ld) out[pos] = j;
    else set_status(e.status, STS_DEV_IDX_CAPACITY);
  }
  if (threadIdx.x == 0) e.cnt_out[r] = run_sel + max(t_hi - t_lo, 0);
}

}  // namespace
}  // namespace sts

namespace sts {
namespace {

int64_t dist_keys_ld(int32_t n_local, int32_t page_size) {
  const int64_t nk = page_size == 1 ? n_local : ((int64_t)n_local + page_size - 1) / page_size;
  return (nk + 3) & ~int64_t(3);
}

int64_t dist_bits_ld(int32_t n_local, int32_t page_size) {
  if (page_size == 1) return 0;
  return (dist_keys_ld(n_local, page_size) + 31) / 32 + 1;
}

size_t dist_ws_bytes(int64_t rows, int32_t n_local, int32_t page_size) {
  const size_t state = ((size_t)rows * sizeof(DistState) + 255) & ~size_t(255);
  const size_t ksz = page_size == 1 ? 4 : 8;
  const size_t keys = ((size_t)rows * dist_keys_ld(n_local, page_size) * ksz + 255) & ~size_t(255);
  const size_t bits = (size_t)rows * dist_bits_ld(n_local, page_size) * 4;
  return state + keys + bits + 256;
}

int dist_params(const sts_dist_rows* g, void* ws, size_t ws_bytes, DistParams& p, uint32_t** bits) {
  STS_REQUIRE(g != nullptr, STS_ERR_CONTRACT, "null geometry");
  STS_REQUIRE(g->rows >= 0 && g->rows <= 65535, STS_ERR_CONTRACT, "rows must be in [0, 65535]");
  STS_REQUIRE(g->nsrc >= 1 && g->nsrc <= 8, STS_ERR_CONTRACT, "nsrc must be in [1, 8], got %d", g->nsrc);
  STS_REQUIRE(g->row_src_dev || g->nsrc == 1, STS_ERR_CONTRACT, "nsrc > 1 needs a row_src table");
  STS_REQUIRE(g->page_size >= 1, STS_ERR_INPUT, "page_size must be >= 1");
  STS_REQUIRE(g->n_global >= 0 && g->n_local >= 0 && g->lo >= 0, STS_ERR_CONTRACT, "bad shard geometry");
  STS_REQUIRE(g->lo % g->page_size == 0 || g->n_local == 0, STS_ERR_CONTRACT, "shard start %d is not page-aligned (page %d)", g->lo,
              g->page_size);
  STS_REQUIRE(g->k_top >= 1, STS_ERR_INPUT, "k must be >= 1");
  STS_REQUIRE(g->ld >= 1 && (g->n_local == 0 || g->scores_dev), STS_ERR_CONTRACT, "bad score rows");
  const size_t need = dist_ws_bytes(g->rows, g->n_local, g->page_size);
  STS_REQUIRE(ws && ws_bytes >= need, STS_ERR_CONTRACT, "dist select workspace too small: need %zu, got %zu", need,
              ws_bytes);
  p.scores = g->scores_dev;
  p.ld = g->ld;
  p.row_src = g->row_src_dev;
  p.nsrc = g->nsrc;
  p.rows = g->rows;
  p.n_global = g->n_global;
  p.lo = g->lo;
  p.n_local = g->n_local;
  p.k_top = g->k_top;
  p.page_size = g->page_size;
  uint8_t* base = static_cast<uint8_t*>(ws);
  const size_t state = ((size_t)g->rows * sizeof(DistState) + 255) & ~size_t(255);
  const size_t ksz = g->page_size == 1 ? 4 : 8;
  const size_t keys = ((size_t)g->rows * dist_keys_ld(g->n_local, g->page_size) * ksz + 255) & ~size_t(255);
  p.state = reinterpret_cast<DistState*>(base);
  p.keys = base + state;
  p.keys_ld = dist_keys_ld(g->n_local, g->page_size);
  *bits = reinterpret_cast<uint32_t*>(base + state + keys);
  return STS_OK;
}

dim3 dist_grid(const DistParams& p) {
  const int64_t nk = p.page_size == 1 ? p.n_local : ((int64_t)p.n_local + p.page_size - 1) / p.page_size;
  const int64_t chunks = nk > 0 ? (nk + DIST_CHUNK - 1) / DIST_CHUNK : 1;
  return dim3((unsigned)chunks, (unsigned)p.rows);
}

__global__ void dist_ties_kernel(const DistState* state, int64_t rows, int32_t* ties_local) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < rows) ties_local[r] = state[r].ties_local;
}

}  // namespace
}  // namespace sts

using namespace sts;

extern "C" int32_t sts_dist_select_rounds(int32_t page_size) { return page_size == 1 ? 4 : 8; }

extern "C" size_t sts_dist_select_workspace_bytes(int64_t rows, int32_t n_local, int32_t page_size) {
  return dist_ws_bytes(rows, n_local, page_size < 1 ? 1 : page_size);
}

extern "C" int sts_dist_select_begin(const sts_dist_rows* g, int32_t* hist_local_dev, void* workspace_dev,
                                     size_t workspace_bytes, void* stream) {
  DistParams p;
  uint32_t* bits;
  int rc = dist_params(g, workspace_dev, workspace_bytes, p, &bits);
  if (rc != STS_OK) return rc;
  if (p.rows == 0) return STS_OK;
  STS_REQUIRE(hist_local_dev, STS_ERR_CONTRACT, "null histogram");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  STS_CUDA_CHECK(cudaMemsetAsync(hist_local_dev, 0, (size_t)p.rows * DD_BINS * 4, st));
  if (p.page_size == 1) dist_keys_kernel<uint32_t><<<dist_grid(p), DIST_THREADS, 0, st>>>(p, hist_local_dev);
  else dist_keys_kernel<uint64_t><<<dist_grid(p), DIST_THREADS, 0, st>>>(p, hist_local_dev);
  STS_LAUNCH_CHECK();
  return STS_OK;
}

extern "C" int sts_dist_select_round(const sts_dist_rows* g, int32_t round, const int32_t* hist_global_dev,
                                     int32_t* hist_local_dev, int32_t* ties_local_dev, void* workspace_dev,
                                     size_t workspace_bytes, void* stream) {
  DistParams p;
  uint32_t* bits;
  int rc = dist_params(g, workspace_dev, workspace_bytes, p, &bits);
  if (rc != STS_OK) return rc;
  const int rounds = sts_dist_select_rounds(p.page_size);
  STS_REQUIRE(round >= 0 && round < rounds, STS_ERR_CONTRACT, "round %d out of [0, %d)", round, rounds);
  if (p.rows == 0) return STS_OK;
  STS_REQUIRE(hist_global_dev && hist_local_dev, STS_ERR_CONTRACT, "null histogram");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int wpb = 8;
  const unsigned grid = (unsigned)((p.rows + wpb - 1) / wpb);
  if (p.page_size == 1) dist_advance_kernel<uint32_t><<<grid, wpb * 32, 0, st>>>(p, round, hist_global_dev, hist_local_dev);
  else dist_advance_kernel<uint64_t><<<grid, wpb * 32, 0, st>>>(p, round, hist_global_dev, hist_local_dev);
  STS_LAUNCH_CHECK();
  if (round + 1 < rounds) {
    STS_CUDA_CHECK(cudaMemsetAsync(hist_local_dev, 0, (size_t)p.rows * DD_BINS * 4, st));
    if (p.page_size == 1) dist_hist_kernel<uint32_t><<<dist_grid(p), DIST_THREADS, 0, st>>>(p, round + 1, hist_local_dev);
    else dist_hist_kernel<uint64_t><<<dist_grid(p), DIST_THREADS, 0, st>>>(p, round + 1, hist_local_dev);
    STS_LAUNCH_CHECK();
  }
  if (ties_local_dev) {
    dist_ties_kernel<<<(unsigned)((p.rows + 255) / 256), 256, 0, st>>>(p.state, p.rows, ties_local_dev);
    STS_LAUNCH_CHECK();
  }
  return STS_OK;
}

extern "C" int sts_dist_select_finish(const sts_dist_rows* g, int32_t rank, int32_t nranks,
                                      const int32_t* ties_all_dev, uint32_t flags, int32_t recent_window,
                                      int32_t tail_len, int32_t n_kv_local, int32_t* idx_out_dev, int64_t idx_ld,
                                      int32_t* cnt_out_dev, int32_t* status_dev, void* workspace_dev,
                                      size_t workspace_bytes, void* stream) {
  DistParams p;
  uint32_t* bits;
  int rc = dist_params(g, workspace_dev, workspace_bytes, p, &bits);
  if (rc != STS_OK) return rc;
  STS_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, STS_ERR_CONTRACT, "bad rank %d of %d", rank, nranks);
  STS_REQUIRE(recent_window >= 0 && tail_len >= 0, STS_ERR_INPUT, "recent_window / tail_len must be >= 0");
  STS_REQUIRE(n_kv_local >= 0, STS_ERR_CONTRACT, "n_kv_local must be >= 0");
  if (p.rows == 0) return STS_OK;
  STS_REQUIRE(ties_all_dev && idx_out_dev && cnt_out_dev, STS_ERR_CONTRACT, "null buffer");
  EmitParams e;
  e.rank = rank;
  e.nranks = nranks;
  e.ties_all = ties_all_dev;
  e.flags = flags;
  e.recent_window = recent_window;
  e.tail_len = tail_len;
  e.n_kv_local = n_kv_local;
  e.idx_out = idx_out_dev;
  e.idx_ld = idx_ld;
  e.cnt_out = cnt_out_dev;
  e.status = status_dev;
  e.page_bits = p.page_size == 1 ? nullptr : bits;
  e.page_bits_ld = dist_bits_ld(p.n_local, p.page_size);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (p.page_size == 1) dist_emit_kernel<uint32_t><<<(unsigned)p.rows, EMIT_THREADS, 0, st>>>(p, e);
  else dist_emit_kernel<uint64_t><<<(unsigned)p.rows, EMIT_THREADS, 0, st>>>(p, e);
  STS_LAUNCH_CHECK();
  return STS_OK;
}
