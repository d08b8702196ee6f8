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
// Digits are 11 bits from the top (3 rounds for token keys, 6 for page keys);
// a row whose chosen bin is taken whole (remaining k == bin count) is resolved
// early and skips the remaining rounds' work.  Collectives stay O(rounds + 1)
// for all rows of all layers at once (one histogram buffer per round).
#include "sts_common.cuh"

namespace sts {
namespace {

// digits of DD_BITS from the top; the last digit takes the remaining bits
// (32-bit keys: 11 + 11 + 10, 64-bit page keys: 5 x 11 + 9)
constexpr int DD_BITS = 11;
constexpr int DD_BINS = 1 << DD_BITS;  // histogram row stride (bins of the widest digit)

__host__ __device__ constexpr int dd_rounds(int kbits) { return (kbits + DD_BITS - 1) / DD_BITS; }
__host__ __device__ constexpr int dd_shift(int kbits, int round) {
  return kbits - DD_BITS * (round + 1) > 0 ? kbits - DD_BITS * (round + 1) : 0;
}
__host__ __device__ constexpr int dd_width(int kbits, int round) {
  return kbits - DD_BITS * round < DD_BITS ? kbits - DD_BITS * round : DD_BITS;
}
constexpr int DIST_THREADS = 512;
#ifndef STS_DIST_CHUNK
#define STS_DIST_CHUNK 32768
#endif
constexpr int DIST_CHUNK = STS_DIST_CHUNK;  // keys per CTA in the key / histogram passes

struct DistState {
  uint64_t prefix;  // chosen digits so far (in key space)
  uint64_t pmask;   // bits of the key the prefix covers
  int krem;         // keys still to take at / below the prefix
  int done;         // 1: resolved (threshold = prefix under pmask)
  int dense;        // 1: budget >= n, every position selected
  int ties_global;  // keys matching the final prefix, all ranks
  int ties_local;   // ... on this rank
  int bad;          // 1: the global histogram could not place the remaining k (inconsistent ranks)
  int pad[2];
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
  int vec4;       // score rows 16-byte aligned with ld % 4 == 0 (token keys load float4)
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
  return (int)((key >> dd_shift(KB, round)) & (K)((1 << dd_width(KB, round)) - 1));
}

// fp64 key of a FULL page of PS tokens held in registers: 16-byte loads of
// every source (summed in fp32, source order), then the numpy reduceat
// segment order x0 + pairwise(x[1:PS]) of dist_pairwise, unrolled
template <int PS>
__device__ __forceinline__ double page_sum_regs(const DistParams& p, const int32_t* srcs, int start) {
  float x[PS];
#pragma unroll
  for (int t = 0; t < PS / 4; ++t) {
    float4 a = *reinterpret_cast<const float4*>(p.scores + (int64_t)srcs[0] * p.ld + start + 4 * t);
#pragma unroll
    for (int q = 1; q < 8; ++q)
      if (q < p.nsrc) {
        const float4 v = *reinterpret_cast<const float4*>(p.scores + (int64_t)srcs[q] * p.ld + start + 4 * t);
        a.x = __fadd_rn(a.x, v.x);
        a.y = __fadd_rn(a.y, v.y);
        a.z = __fadd_rn(a.z, v.z);
        a.w = __fadd_rn(a.w, v.w);
      }
    x[4 * t] = a.x;
    x[4 * t + 1] = a.y;
    x[4 * t + 2] = a.z;
    x[4 * t + 3] = a.w;
  }
  constexpr int n = PS - 1;  // pairwise over x[1 .. PS)
  double res;
  if constexpr (n < 8) {
    res = 0.0;
#pragma unroll
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, (double)x[1 + i]);
  } else {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = (double)x[1 + j];
    constexpr int body = n - n % 8;
#pragma unroll
    for (int i = 8; i < body; i += 8)
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], (double)x[1 + i + j]);
    res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                    __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
#pragma unroll
    for (int i = body; i < n; ++i) res = __dadd_rn(res, (double)x[1 + i]);
  }
  return __dadd_rn((double)x[0], res);
}

// keys of the local positions + round-0 histogram; a linear grid of
// rows x chunks, ROW-fastest: the CTAs resident together cover the same
// position chunk of every row, so a draft row mapped into several target rows
// (mode S sums each target row's mapped draft rows) is read from HBM once and
// from L2 for its other targets
// token keys of 4 consecutive positions j..j+3: one 16-byte load per source
// row (NS sources; NS = 0: p.nsrc at run time), summed in source order
template <int NS>
__device__ __forceinline__ float4 dist_sum4(const DistParams& p, const int32_t* srcs, int j) {
  constexpr int MAXS = NS > 0 ? NS : 8;
  float4 v[MAXS];
#pragma unroll
  for (int q = 0; q < MAXS; ++q)
    if (NS > 0 || q < p.nsrc) v[q] = __ldg(reinterpret_cast<const float4*>(p.scores + (int64_t)srcs[q] * p.ld + j));
  float4 a = v[0];
#pragma unroll
  for (int q = 1; q < MAXS; ++q)
    if (NS > 0 || q < p.nsrc) {
      a.x = __fadd_rn(a.x, v[q].x);
      a.y = __fadd_rn(a.y, v[q].y);
      a.z = __fadd_rn(a.z, v[q].z);
      a.w = __fadd_rn(a.w, v[q].w);
    }
  return a;
}

template <typename K, int NS = 0>
__global__ void __launch_bounds__(DIST_THREADS) dist_keys_kernel(DistParams p, int32_t* hist) {
  __shared__ uint32_t sh[DD_BINS];
  const int64_t r = (int64_t)blockIdx.x % p.rows;
  const int chunk = (int)((int64_t)blockIdx.x / p.rows);
  for (int i = threadIdx.x; i < DD_BINS; i += DIST_THREADS) sh[i] = 0;
  if (chunk == 0 && threadIdx.x == 0) {
    DistState s;
    s.prefix = 0;
    s.pmask = 0;
    s.krem = p.k_top;
    const int n_units = p.page_size == 1 ? p.n_global : (p.n_global + p.page_size - 1) / p.page_size;
    s.dense = p.k_top >= n_units ? 1 : 0;
    s.done = s.dense;
    s.ties_global = 0;
    s.ties_local = 0;
    s.bad = s.pad[0] = s.pad[1] = 0;
    p.state[r] = s;
  }
  __syncthreads();
  const int nk = local_keys(p);
  const int nc = local_committed(p);
  int32_t srcs[8];
  load_srcs(p, r, srcs);
  K* keys = reinterpret_cast<K*>(p.keys + r * p.keys_ld * sizeof(K));
  const int j_end = min(nk, (chunk + 1) * DIST_CHUNK);
  if constexpr (sizeof(K) == 4) {
    if (p.vec4) {
      // 4 consecutive positions per thread: one 16-byte load per source row
      // (rows are padded to a multiple of 4), sources summed in order
      // two 4-position groups per iteration: both groups' loads in flight together
      auto put = [&](int j, const float4& a) {
        const uint4 k4 = make_uint4(f32_key(a.x), f32_key(a.y), f32_key(a.z), f32_key(a.w));
        *reinterpret_cast<uint4*>(keys + j) = k4;
        atomicAdd(&sh[digit_of<K>(k4.x, 0)], 1u);
        if (j + 1 < j_end) atomicAdd(&sh[digit_of<K>(k4.y, 0)], 1u);
        if (j + 2 < j_end) atomicAdd(&sh[digit_of<K>(k4.z, 0)], 1u);
        if (j + 3 < j_end) atomicAdd(&sh[digit_of<K>(k4.w, 0)], 1u);
      };
      constexpr int STEP = 4 * DIST_THREADS;
      int j = chunk * DIST_CHUNK + 4 * threadIdx.x;
      if constexpr (NS > 0) {
        for (; j + STEP < j_end; j += 2 * STEP) {
          const float4 a = dist_sum4<NS>(p, srcs, j), b = dist_sum4<NS>(p, srcs, j + STEP);
          put(j, a);
          put(j + STEP, b);
        }
      }
      for (; j < j_end; j += STEP) put(j, dist_sum4<NS>(p, srcs, j));
      __syncthreads();
      int32_t* h = hist + r * DD_BINS;
      for (int i = threadIdx.x; i < DD_BINS; i += DIST_THREADS)
        if (sh[i]) atomicAdd(h + i, (int)sh[i]);
      return;
    }
  }
  for (int j = chunk * DIST_CHUNK + threadIdx.x; j < j_end; j += DIST_THREADS) {
    K key;
    if constexpr (sizeof(K) == 4) {
      key = f32_key(dist_value(p, srcs, j));
    } else {
      const int start = j * p.page_size;
      const int len = min(p.page_size, nc - start);
      if (p.vec4 && len == p.page_size && (p.page_size == 8 || p.page_size == 16 || p.page_size == 32)) {
        key = f64_key(p.page_size == 16   ? page_sum_regs<16>(p, srcs, start)
                      : p.page_size == 8  ? page_sum_regs<8>(p, srcs, start)
                                          : page_sum_regs<32>(p, srcs, start));
      } else {
        const double x0 = (double)dist_value(p, srcs, start);
        key = f64_key(len == 1 ? x0 : __dadd_rn(x0, dist_pairwise(p, srcs, start + 1, len - 1)));
      }
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
  if constexpr (sizeof(K) == 4) {
    // keys rows are padded to a multiple of 4 and 16-byte aligned
    for (int j = blockIdx.x * DIST_CHUNK + 4 * threadIdx.x; j < j_end; j += 4 * DIST_THREADS) {
      const uint4 k4 = *reinterpret_cast<const uint4*>(keys + j);
      const K kk[4] = {k4.x, k4.y, k4.z, k4.w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (j + q < j_end && (kk[q] & pm) == pf) atomicAdd(&sh[digit_of<K>(kk[q], round)], 1u);
    }
  } else {
    for (int j = blockIdx.x * DIST_CHUNK + threadIdx.x; j < j_end; j += DIST_THREADS) {
      const K key = keys[j];
      if ((key & pm) == pf) atomicAdd(&sh[digit_of<K>(key, round)], 1u);
    }
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
  // lane owns PER consecutive bins, descending: nb-1-PER*lane .. nb-PER-PER*lane
  const int nb = 1 << dd_width(KB, round);
  const int per = nb / 32;  // widths >= 9 bits: >= 16 bins per lane
  int lsum = 0;
  for (int q = 0; q < per; ++q) lsum += hg[nb - 1 - per * lane - q];
  int incl = lsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const int excl = incl - lsum;
  const bool mine = excl < st.krem && st.krem <= incl;
  const uint32_t who = __ballot_sync(0xffffffffu, mine);
  if (who == 0) {  // inconsistent histogram (ranks disagree on k / shards): flag it, finish reports it
    if (lane == 0) p.state[r].bad = 1;
    return;
  }
  if (lane != __ffs(who) - 1) return;
  int acc = excl, digit = 0, inbin = 0;
  for (int q = 0; q < per; ++q) {
    const int c = hg[nb - 1 - per * lane - q];
    if (acc < st.krem && st.krem <= acc + c) {
      digit = nb - 1 - per * lane - q;
      inbin = c;
      break;
    }
    acc += c;
  }
  const int shift = dd_shift(KB, round);
  st.prefix |= (uint64_t)digit << shift;
  st.pmask |= (uint64_t)(nb - 1) << shift;
  st.krem -= acc;
  if (shift == 0 || st.krem == inbin) {
    st.done = 1;
    st.ties_global = inbin;
    st.ties_local = hist_local[r * DD_BINS + digit];
  }
  p.state[r] = st;
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
  uint32_t* bits;           // [rows][bits_ld] selected-key bitmap (tokens, or pages)
  int64_t bits_ld;
  int32_t* key_cnt;         // [rows][key_chunks] threshold ties per key chunk
  int32_t* tok_cnt;         // [rows][tok_chunks] selected tokens per token chunk
  int key_chunks;
  int tok_chunks;
};

// The emit is split over (chunk, row) CTAs of EMIT_CHUNK keys / tokens:
//   ties   count the threshold ties of each key chunk
//   bits   selected-key bitmap: keys above the threshold, plus the ties whose
//          global rank (ties on lower ranks + earlier chunks + in-chunk rank)
//          is below the remaining k
//   count  selected tokens per token chunk (bitmap of the token's key, or an
//          extra: sink / recent window / current)
//   emit   ascending local offsets at the chunk's prefix; chunk 0 adds the
//          in-block tail and the row count
// Each warp owns 1024 consecutive keys as 32 ballot words (lane w keeps word w).
constexpr int EMIT_THREADS = 512;
constexpr int EMIT_WARPS = EMIT_THREADS / 32;
constexpr int EMIT_CHUNK = EMIT_WARPS * 1024;

struct EmitRow {
  int need;      // ties this rank takes
  bool all_ties; // every local tie is taken
};

__device__ __forceinline__ EmitRow emit_row(const DistState& st, const EmitParams& e, int64_t r, int64_t rows) {
  int before = 0;
  for (int q = 0; q < e.rank; ++q) before += e.ties_all[(int64_t)q * rows + r];
  EmitRow er;
  er.need = max(st.krem - before, 0);
  er.all_ties = er.need >= st.ties_local;
  return er;
}

// exclusive prefix of counts[0 .. c) (one row's chunk counts), block-wide
__device__ __forceinline__ int chunk_prefix(const int32_t* counts, int c, int* red) {
  int s = 0;
  for (int i = threadIdx.x; i < c; i += EMIT_THREADS) s += counts[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  int t = 0;
#pragma unroll
  for (int w = 0; w < EMIT_WARPS; ++w) t += red[w];
  __syncthreads();
  return t;
}

// exclusive scan of one value per warp (lane 0's), block-wide
__device__ __forceinline__ int warp_offsets(int v, int* red, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  int before = 0;
  total = 0;
#pragma unroll
  for (int w = 0; w < EMIT_WARPS; ++w) {
    const int x = red[w];
    before += w < warp ? x : 0;
    total += x;
  }
  __syncthreads();
  return before;
}

__device__ __forceinline__ int lane_excl_scan(int v, int& warp_total) {
  const int lane = threadIdx.x & 31;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  warp_total = __shfl_sync(0xffffffffu, incl, 31);
  return incl - v;
}

// gt / eq ballot words of this warp's 1024 keys; lane w returns word w
template <typename K>
__device__ __forceinline__ void key_words(const K* keys, int nk, int64_t j0, K pm, K pf, uint32_t& gt, uint32_t& eq) {
  const int lane = threadIdx.x & 31;
  gt = eq = 0;
#pragma unroll 8
  for (int w = 0; w < 32; ++w) {
    const int64_t j = j0 + 32 * w + lane;
    bool g = false, q = false;
    if (j < nk) {
      const K mk = keys[j] & pm;
      g = mk > pf;
      q = mk == pf;
    }
    const uint32_t bg = __ballot_sync(0xffffffffu, g), bq = __ballot_sync(0xffffffffu, q);
    if (lane == w) {
      gt = bg;
      eq = bq;
    }
  }
}

// 32-bit keys: 16-byte loads, 4 keys per lane per 128-key block; the 8 lanes
// of a block quarter OR their nibbles into one word, then lane w takes word w
__device__ __forceinline__ void key_words(const uint32_t* keys, int nk, int64_t j0, uint32_t pm, uint32_t pf,
                                          uint32_t& gt, uint32_t& eq) {
  const int lane = threadIdx.x & 31;
  gt = eq = 0;
  uint4 k4[8];
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int64_t j = j0 + 128 * it + 4 * lane;
    k4[it] = j < nk ? *reinterpret_cast<const uint4*>(keys + j) : make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int64_t j = j0 + 128 * it + 4 * lane;
    const uint32_t kk[4] = {k4[it].x, k4[it].y, k4[it].z, k4[it].w};
    uint32_t g = 0, q = 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const uint32_t mk = kk[t] & pm;
      const bool in = j + t < nk;
      g |= (in && mk > pf) ? (1u << t) : 0u;
      q |= (in && mk == pf) ? (1u << t) : 0u;
    }
    g <<= 4 * (lane & 7);
    q <<= 4 * (lane & 7);
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      g |= __shfl_xor_sync(0xffffffffu, g, o);
      q |= __shfl_xor_sync(0xffffffffu, q, o);
    }
    // words 4*it .. 4*it+3 now sit in lanes 0, 8, 16, 24
    const uint32_t gw = __shfl_sync(0xffffffffu, g, 8 * (lane & 3));
    const uint32_t qw = __shfl_sync(0xffffffffu, q, 8 * (lane & 3));
    if ((lane >> 2) == it) {
      gt = gw;
      eq = qw;
    }
  }
}

// selected bit of local token j (its key's bitmap bit, or an extra)
struct TokenSel {
  const uint32_t* bits;
  int ps, nc, lo, n_global, lo_extra;
  bool sink, cur;
  __device__ __forceinline__ bool operator()(int64_t j) const {
    if (j >= nc) return false;
    const int64_t k = ps == 1 ? j : j / ps;
    const int g = lo + (int)j;
    return ((bits[k >> 5] >> (k & 31)) & 1u) || g >= lo_extra || (sink && g == 0) || (cur && g == n_global - 1);
  }
};

// bits of [a, b) inside the 32-token word starting at w0
__device__ __forceinline__ uint32_t range_bits(int64_t a, int64_t b, int64_t w0) {
  const int64_t l = max(a - w0, (int64_t)0), h = min(b - w0, (int64_t)32);
  if (h <= l) return 0u;
  return (h - l == 32 ? 0xffffffffu : ((1u << (h - l)) - 1u)) << l;
}

// token mode: the selected tokens of word w (bitmap word | extras), committed only
__device__ __forceinline__ uint32_t token_word_from(const TokenSel& t, int64_t w, uint32_t key_word) {
  const int64_t w0 = 32 * w;
  if (w0 >= t.nc) return 0u;
  uint32_t m = key_word | range_bits((int64_t)t.lo_extra - t.lo, t.nc, w0);
  if (t.sink && t.lo == 0 && w == 0) m |= 1u;
  if (t.cur) m |= range_bits((int64_t)t.n_global - 1 - t.lo, (int64_t)t.n_global - t.lo, w0);
  return m & range_bits(0, t.nc, w0);
}

__device__ __forceinline__ uint32_t token_word(const TokenSel& t, int64_t w) {
  return 32 * w >= t.nc ? 0u : token_word_from(t, w, t.bits[w]);
}

__device__ __forceinline__ TokenSel token_sel(const DistParams& p, const EmitParams& e, int64_t r) {
  TokenSel t;
  t.bits = e.bits + r * e.bits_ld;
  t.ps = p.page_size;
  t.nc = local_committed(p);
  t.lo = p.lo;
  t.n_global = p.n_global;
  t.lo_extra = e.recent_window > 0 ? p.n_global - e.recent_window : p.n_global;
  t.sink = (e.flags & STS_SEL_SINK) != 0;
  t.cur = (e.flags & STS_SEL_CURRENT) != 0;
  return t;
}

template <typename K>
__global__ void __launch_bounds__(EMIT_THREADS) dist_emit_ties_kernel(DistParams p, EmitParams e) {
  __shared__ int red[EMIT_WARPS];
  const int64_t r = blockIdx.y;
  const DistState st = p.state[r];
  const EmitRow er = emit_row(st, e, r, p.rows);
  int cnt = 0;
  if (!st.dense && !er.all_ties) {
    const K* keys = reinterpret_cast<const K*>(p.keys + r * p.keys_ld * sizeof(K));
    uint32_t gt, eq;
    key_words(keys, local_keys(p), (int64_t)blockIdx.x * EMIT_CHUNK + (threadIdx.x >> 5) * 1024, (K)st.pmask,
                 (K)st.prefix, gt, eq);
    int c = __popc(eq);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    int total;
    warp_offsets(c, red, total);
    cnt = total;
  }
  if (threadIdx.x == 0) e.key_cnt[r * e.key_chunks + blockIdx.x] = cnt;
}

template <typename K>
__global__ void __launch_bounds__(EMIT_THREADS) dist_emit_bits_kernel(DistParams p, EmitParams e) {
  __shared__ int red[EMIT_WARPS];
  const int64_t r = blockIdx.y;
  const DistState st = p.state[r];
  const EmitRow er = emit_row(st, e, r, p.rows);
  const int nk = local_keys(p);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t j0 = (int64_t)blockIdx.x * EMIT_CHUNK + warp * 1024;
  uint32_t* bits = e.bits + r * e.bits_ld;
  const int64_t word = j0 / 32 + lane;
  const bool valid = 32 * word < nk;
  uint32_t sel;
  if (st.dense) {
    const int64_t left = nk - 32 * word;
    sel = left >= 32 ? 0xffffffffu : (left > 0 ? (1u << left) - 1u : 0u);
  } else {
    const K* keys = reinterpret_cast<const K*>(p.keys + r * p.keys_ld * sizeof(K));
    uint32_t gt, eq;
    if constexpr (sizeof(K) == 4) {
      // the CTA's 64 KB key chunk arrives by one bulk copy into shared memory
      // (no registers held while in flight; ~3 CTAs' chunks per SM at once)
      extern __shared__ __align__(16) uint8_t kbuf[];
      __shared__ __align__(8) uint64_t kbar;
      const int64_t c0 = (int64_t)blockIdx.x * EMIT_CHUNK;
      const int64_t padded = ((int64_t)nk + 3) & ~int64_t(3);
      const int cn = (int)min((int64_t)EMIT_CHUNK, max((int64_t)0, padded - c0));
      if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&kbar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      }
      __syncthreads();
      if (cn > 0) {
        if (threadIdx.x == 0) {
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&kbar)),
                       "r"((uint32_t)cn * 4u) : "memory");
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                  smem_u32(kbuf)),
              "l"(reinterpret_cast<uint64_t>(keys + c0)), "r"((uint32_t)cn * 4u), "r"(smem_u32(&kbar))
              : "memory");
        }
        uint32_t done = 0;
        while (!done)
          asm volatile(
              "{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0;\n selp.u32 %0, 1, 0, q;\n}\n"
              : "=r"(done)
              : "r"(smem_u32(&kbar))
              : "memory");
      }
      key_words(reinterpret_cast<const uint32_t*>(kbuf), (int)(nk - c0), (int64_t)warp * 1024, (uint32_t)st.pmask,
                (uint32_t)st.prefix, gt, eq);
    } else {
      key_words(keys, nk, j0, (K)st.pmask, (K)st.prefix, gt, eq);
    }
    sel = gt;
    if (er.all_ties) {
      sel |= eq;
    } else {
      const int base = chunk_prefix(e.key_cnt + r * e.key_chunks, blockIdx.x, red);
      int wt;
      const int lx = lane_excl_scan(__popc(eq), wt);
      int total;
      const int rank0 = base + warp_offsets(wt, red, total) + lx;
      int take = min(max(er.need - rank0, 0), __popc(eq));
      uint32_t x = eq;
      while (take-- > 0) {
        const uint32_t low = x & (0u - x);
        sel |= low;
        x ^= low;
      }
    }
  }
  if (valid) bits[word] = sel;
  if (p.page_size == 1) {
    // token mode: key chunk == token chunk, so the selected-token count of the
    // chunk (keys | extras) is known here and the count pass is skipped
    const TokenSel ts = token_sel(p, e, r);
    int c = __popc(token_word_from(ts, word, valid ? sel : 0u));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    int total;
    warp_offsets(c, red, total);
    if (threadIdx.x == 0) e.tok_cnt[r * e.tok_chunks + blockIdx.x] = total;
  }
}

__global__ void __launch_bounds__(EMIT_THREADS) dist_emit_count_kernel(DistParams p, EmitParams e) {
  __shared__ int red[EMIT_WARPS];
  const int64_t r = blockIdx.y;
  const TokenSel sel = token_sel(p, e, r);
  const int lane = threadIdx.x & 31;
  const int64_t j0 = (int64_t)blockIdx.x * EMIT_CHUNK + (threadIdx.x >> 5) * 1024;
  int c = 0;
  if (sel.ps == 1) {
    c = __popc(token_word(sel, (int64_t)blockIdx.x * (EMIT_CHUNK / 32) + threadIdx.x));
  } else if (j0 < sel.nc) {
#pragma unroll 4
    for (int w = 0; w < 32; ++w) c += sel(j0 + 32 * w + lane) ? 1 : 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  int total;
  warp_offsets(c, red, total);
  if (threadIdx.x == 0) e.tok_cnt[r * e.tok_chunks + blockIdx.x] = total;
}

__global__ void __launch_bounds__(EMIT_THREADS) dist_emit_write_kernel(DistParams p, EmitParams e) {
  __shared__ int red[EMIT_WARPS];
  const int64_t r = blockIdx.y;
  const TokenSel sel = token_sel(p, e, r);
  const int lane = threadIdx.x & 31;
  const int64_t j0 = (int64_t)blockIdx.x * EMIT_CHUNK + (threadIdx.x >> 5) * 1024;
  int32_t* out = e.idx_out + r * e.idx_ld;
  const int32_t* tc = e.tok_cnt + r * e.tok_chunks;
  const int64_t w = (int64_t)blockIdx.x * (EMIT_CHUNK / 32) + threadIdx.x;
  uint32_t m = sel.ps == 1 ? token_word(sel, w) : 0u;  // issued before the prefix sum
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const DistState st = p.state[r];
    if (!st.done || st.bad) set_status(e.status, STS_DEV_SELECT_INCONSISTENT);
  }
  const int base = chunk_prefix(tc, blockIdx.x, red);
  if (sel.ps == 1) {
    // one token word per thread
    int wt;
    const int lx = lane_excl_scan(__popc(m), wt);
    int total;
    int at = base + warp_offsets(wt, red, total) + lx;
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1u;
      if (at < e.idx_ld) out[at] = (int32_t)(32 * w + b);
      else set_status(e.status, STS_DEV_IDX_CAPACITY);
      ++at;
    }
  } else {
    uint32_t mine = 0;
    if (j0 < sel.nc) {
#pragma unroll 4
      for (int ww = 0; ww < 32; ++ww) {
        const uint32_t b = __ballot_sync(0xffffffffu, sel(j0 + 32 * ww + lane));
        if (lane == ww) mine = b;
      }
    }
    int wt;
    lane_excl_scan(__popc(mine), wt);
    int total;
    int pos = base + warp_offsets(wt, red, total);
    if (j0 < sel.nc) {
      const uint32_t lt = (1u << lane) - 1u;
      for (int ww = 0; ww < 32; ++ww) {
        const uint32_t b = __shfl_sync(0xffffffffu, mine, ww);
        if ((b >> lane) & 1u) {
          const int at = pos + __popc(b & lt);
          if (at < e.idx_ld) out[at] = (int32_t)(j0 + 32 * ww + lane);
          else set_status(e.status, STS_DEV_IDX_CAPACITY);
        }
        pos += __popc(b);
      }
    }
  }
  if (blockIdx.x == 0) {
    // in-block tail: global [n_global, n_global + tail_len) held here
    const int all = chunk_prefix(tc, e.tok_chunks, red);
    const int t_lo = max(p.n_global - p.lo, 0);
    const int t_hi = min(p.n_global + e.tail_len - p.lo, e.n_kv_local);
    for (int j = t_lo + threadIdx.x; j < t_hi; j += EMIT_THREADS) {
      const int at = all + (j - t_lo);
      if (at < e.idx_ld) out[at] = j;
      else set_status(e.status, STS_DEV_IDX_CAPACITY);
    }
    if (threadIdx.x == 0) e.cnt_out[r] = all + max(t_hi - t_lo, 0);
  }
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
  return (dist_keys_ld(n_local, page_size) + 31) / 32 + 1;
}

int64_t dist_key_chunks(int32_t n_local, int32_t page_size) {
  const int64_t nk = page_size == 1 ? n_local : ((int64_t)n_local + page_size - 1) / page_size;
  return nk > 0 ? (nk + EMIT_CHUNK - 1) / EMIT_CHUNK : 1;
}

int64_t dist_tok_chunks(int32_t n_local) { return n_local > 0 ? ((int64_t)n_local + EMIT_CHUNK - 1) / EMIT_CHUNK : 1; }

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// workspace: [state][keys][selected-key bitmap][tie counts per key chunk][token counts per token chunk]
struct DistWs {
  size_t state, keys, bits, key_cnt, tok_cnt;
};

DistWs dist_ws_layout(int64_t rows, int32_t n_local, int32_t page_size) {
  DistWs w;
  const size_t ksz = page_size == 1 ? 4 : 8;
  w.state = align256((size_t)rows * sizeof(DistState));
  w.keys = align256((size_t)rows * dist_keys_ld(n_local, page_size) * ksz);
  w.bits = align256((size_t)rows * dist_bits_ld(n_local, page_size) * 4);
  w.key_cnt = align256((size_t)rows * dist_key_chunks(n_local, page_size) * 4);
  w.tok_cnt = align256((size_t)rows * dist_tok_chunks(n_local) * 4);
  return w;
}

size_t dist_ws_bytes(int64_t rows, int32_t n_local, int32_t page_size) {
  const DistWs w = dist_ws_layout(rows, n_local, page_size);
  return w.state + w.keys + w.bits + w.key_cnt + w.tok_cnt + 256;
}

int dist_params(const sts_dist_rows* g, void* ws, size_t ws_bytes, DistParams& p, EmitParams* e = nullptr) {
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
  p.vec4 = (g->ld % 4 == 0 && (reinterpret_cast<uintptr_t>(g->scores_dev) & 15) == 0) ? 1 : 0;
  const DistWs w = dist_ws_layout(g->rows, g->n_local, g->page_size);
  uint8_t* base = static_cast<uint8_t*>(ws);
  p.state = reinterpret_cast<DistState*>(base);
  p.keys = base + w.state;
  p.keys_ld = dist_keys_ld(g->n_local, g->page_size);
  if (e) {
    e->bits = reinterpret_cast<uint32_t*>(base + w.state + w.keys);
    e->bits_ld = dist_bits_ld(g->n_local, g->page_size);
    e->key_cnt = reinterpret_cast<int32_t*>(base + w.state + w.keys + w.bits);
    e->tok_cnt = reinterpret_cast<int32_t*>(base + w.state + w.keys + w.bits + w.key_cnt);
    e->key_chunks = (int)dist_key_chunks(g->n_local, g->page_size);
    e->tok_chunks = (int)dist_tok_chunks(g->n_local);
  }
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

extern "C" int32_t sts_dist_select_rounds(int32_t page_size) { return page_size == 1 ? dd_rounds(32) : dd_rounds(64); }

extern "C" int32_t sts_dist_select_bins(void) { return DD_BINS; }

extern "C" size_t sts_dist_select_workspace_bytes(int64_t rows, int32_t n_local, int32_t page_size) {
  return dist_ws_bytes(rows, n_local, page_size < 1 ? 1 : page_size);
}

extern "C" int sts_dist_select_begin(const sts_dist_rows* g, int32_t* hist_local_dev, void* workspace_dev,
                                     size_t workspace_bytes, void* stream) {
  DistParams p;
  int rc = dist_params(g, workspace_dev, workspace_bytes, p);
  if (rc != STS_OK) return rc;
  if (p.rows == 0) return STS_OK;
  STS_REQUIRE(hist_local_dev, STS_ERR_CONTRACT, "null histogram");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  STS_CUDA_CHECK(cudaMemsetAsync(hist_local_dev, 0, (size_t)p.rows * DD_BINS * 4, st));
  const dim3 g2 = dist_grid(p);
  STS_REQUIRE((int64_t)g2.x * g2.y < (int64_t(1) << 31), STS_ERR_CONTRACT, "rows x position chunks too large");
  const unsigned lin = (unsigned)((int64_t)g2.x * g2.y);  // rows x chunks, row-fastest
  if (p.page_size == 1 && p.nsrc == 4 && p.vec4) dist_keys_kernel<uint32_t, 4><<<lin, DIST_THREADS, 0, st>>>(p, hist_local_dev);
  else if (p.page_size == 1 && p.nsrc == 7 && p.vec4) dist_keys_kernel<uint32_t, 7><<<lin, DIST_THREADS, 0, st>>>(p, hist_local_dev);
  else if (p.page_size == 1) dist_keys_kernel<uint32_t><<<lin, DIST_THREADS, 0, st>>>(p, hist_local_dev);
  else dist_keys_kernel<uint64_t><<<lin, DIST_THREADS, 0, st>>>(p, hist_local_dev);
  STS_LAUNCH_CHECK();
  return STS_OK;
}

extern "C" int sts_dist_select_round(const sts_dist_rows* g, int32_t round, const int32_t* hist_global_dev,
                                     int32_t* hist_local_dev, int32_t* ties_local_dev, void* workspace_dev,
                                     size_t workspace_bytes, void* stream) {
  DistParams p;
  int rc = dist_params(g, workspace_dev, workspace_bytes, p);
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
  EmitParams e;
  int rc = dist_params(g, workspace_dev, workspace_bytes, p, &e);
  if (rc != STS_OK) return rc;
  STS_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, STS_ERR_CONTRACT, "bad rank %d of %d", rank, nranks);
  STS_REQUIRE(recent_window >= 0 && tail_len >= 0, STS_ERR_INPUT, "recent_window / tail_len must be >= 0");
  STS_REQUIRE(n_kv_local >= 0, STS_ERR_CONTRACT, "n_kv_local must be >= 0");
  if (p.rows == 0) return STS_OK;
  STS_REQUIRE(ties_all_dev && idx_out_dev && cnt_out_dev, STS_ERR_CONTRACT, "null buffer");
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
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const dim3 kgrid((unsigned)e.key_chunks, (unsigned)p.rows), tgrid((unsigned)e.tok_chunks, (unsigned)p.rows);
  if (p.page_size == 1) {
    dist_emit_ties_kernel<uint32_t><<<kgrid, EMIT_THREADS, 0, st>>>(p, e);
    STS_LAUNCH_CHECK();
    constexpr int kbytes = EMIT_CHUNK * 4;
    static const cudaError_t attr =
        cudaFuncSetAttribute(dist_emit_bits_kernel<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, kbytes);
    STS_CUDA_CHECK(attr);
    dist_emit_bits_kernel<uint32_t><<<kgrid, EMIT_THREADS, kbytes, st>>>(p, e);
  } else {
    dist_emit_ties_kernel<uint64_t><<<kgrid, EMIT_THREADS, 0, st>>>(p, e);
    STS_LAUNCH_CHECK();
    dist_emit_bits_kernel<uint64_t><<<kgrid, EMIT_THREADS, 0, st>>>(p, e);
  }
  STS_LAUNCH_CHECK();
  if (p.page_size > 1) {  // token mode: counted by the bits pass
    dist_emit_count_kernel<<<tgrid, EMIT_THREADS, 0, st>>>(p, e);
    STS_LAUNCH_CHECK();
  }
  dist_emit_write_kernel<<<tgrid, EMIT_THREADS, 0, st>>>(p, e);
  STS_LAUNCH_CHECK();
  return STS_OK;
}
