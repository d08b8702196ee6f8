// sts_select.cu — sparsity-mask construction on sm_100a.
//
// Two kernels, one CTA (1024 threads) per logical row:
//   select_reg_kernel  token mode, rows <= 36K keys: the row lives in
//                      registers (up to 36 keys per thread), see below;
//   select_kernel      page mode and longer rows: keys in shared memory or a
//                      global slot.
// Both give identical results (same keys, same radix rule, same emit order).
//
// select_kernel: the row's values are formed on the
// fly (fp32 sum of nsrc source rows: identity for mode R, head-group sum for
// mode S), turned into order-preserving integer keys, and the k-th largest
// key is found by an MSB-first radix select with 12-bit digits and 4096-bin
// shared-memory histograms.  The emit pass walks indices in ascending order
// with ballot-based block scans, so ties at the threshold go to the lowest
// indices (the stable-argsort rule of src/numkit.py:84) and the output comes
// out sorted without a sort.
//
// Page mode (page_size > 1) reproduces src/sparsity.py:94-101: fp64 page sums
// in numpy add.reduceat order (x0 + pairwise(x[1:]), see pairwise_sum; by
// lane octets for 9-129-token pages, page_key_lanes), all-pairs ranks for rows
// of <= 256 pages or a 64-bit-key radix select over pages, then expansion by
// selected page (or a scan over positions when extras are requested).
//
// select_kernel's keys live in shared memory when the row fits, else in a
// per-CTA slot of the global workspace (persistent grid over rows).
#include <stdlib.h>

#include <type_traits>

#include "sts_common.cuh"

namespace sts {
namespace {

constexpr int SEL_THREADS = 1024;
constexpr int SEL_WARPS = SEL_THREADS / 32;
constexpr int DIGIT_BITS = 12;
constexpr int NBINS = 1 << DIGIT_BITS;

struct SelectParams {
  const float* scores;
  int64_t ld;
  const int32_t* row_src;
  int nsrc;
  int64_t rows;
  const int32_t* row_len;
  int n_common;
  double budget;
  int budget_is_fraction;
  int page_size;
  uint32_t flags;
  int recent_window;
  int tail_len;
  int32_t* idx_out;
  int64_t idx_ld;
  int32_t* cnt_out;
  int32_t* status;
  uint8_t* gbuf;          // global key buffers (nullptr => shared memory)
  int64_t gbuf_stride;    // bytes per CTA slot
  int64_t buf_bytes;      // bytes of one key buffer (smem or global)
};

constexpr int CAND_BYTES = 16384;  // candidate keys after the first digit

struct SelShared {
  uint32_t hist[NBINS];
  int warp_tot[SEL_WARPS];
  int bcast[8];
  uint8_t cand[CAND_BYTES];
};

// value of logical-row element j: fp32 sum over sources in order
__device__ __forceinline__ float row_value(const SelectParams& p, const int32_t* srcs, int j) {
  const float* base = p.scores;
  float acc = base[(int64_t)srcs[0] * p.ld + j];
  for (int s = 1; s < p.nsrc; ++s) acc = __fadd_rn(acc, base[(int64_t)srcs[s] * p.ld + j]);
  return acc;
}

// numpy pairwise_sum (float64) over row values [start, start+n)
__device__ double pairwise_sum(const SelectParams& p, const int32_t* srcs, int start, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, (double)row_value(p, srcs, start + i));
    return r;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = (double)row_value(p, srcs, start + j);
    int i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], (double)row_value(p, srcs, start + i + j));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, (double)row_value(p, srcs, start + i));
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pairwise_sum(p, srcs, start, n2), pairwise_sum(p, srcs, start + n2, n - n2));
}

__device__ __forceinline__ double page_sum(const SelectParams& p, const int32_t* srcs, int start, int len) {
  // np.add.reduceat segment: x[start] + pairwise(x[start+1 : start+len])
  double x0 = (double)row_value(p, srcs, start);
  if (len == 1) return x0;
  return __dadd_rn(x0, pairwise_sum(p, srcs, start + 1, len - 1));
}

// Block-wide exclusive scan of an int in thread order (3 barriers).
__device__ __forceinline__ int block_scan_int(int v, int* warp_tot, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int x = warp_tot[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    warp_tot[lane] = x;  // inclusive prefix over warps
  }
  __syncthreads();
  const int before = warp > 0 ? warp_tot[warp - 1] : 0;
  total = warp_tot[SEL_WARPS - 1];
  __syncthreads();
  return before + incl - v;
}

// Radix select: k-th largest key (1-based k <= n) among keys[0..n).
// On return T is that key, need = how many keys equal to T belong to the
// top-k (the rest are strictly greater), ties = how many keys equal T.
// After the first digit the surviving keys are compacted into `cand` (when
// they fit) so later digits only touch the candidates.
template <typename K>
__device__ void radix_select(const K* keys, int n, int k, K key_or, K key_and, SelShared& sh, K* cand, int cand_cap,
                             K& T, int& need, int& ties) {
  constexpr int KBITS = sizeof(K) * 8;
  const K diff = key_or ^ key_and;  // bits that vary across the row
  if (diff == 0) {                  // every key identical: all ties
    T = key_and;
    need = k;
    ties = n;
    return;
  }
  const int h = KBITS - 1 - (sizeof(K) == 8 ? __clzll((long long)diff) : __clz((int)diff));
  // bits above h are common to all keys: start the first digit at bit h so the
  // histogram spreads over the bits that actually discriminate (probability
  // rows share sign + most exponent bits; a fixed top digit piles them into a
  // handful of bins and serialises the shared-memory atomics)
  K pmask = h + 1 >= KBITS ? (K)0 : ~(((K)1 << (h + 1)) - 1);
  K prefix = key_and & pmask;
  int krem = k;
  const K* src = keys;
  int len = n;
  bool compacted = false;
  for (int top = h;; top -= DIGIT_BITS) {
    const int s = top - DIGIT_BITS + 1 < 0 ? 0 : top - DIGIT_BITS + 1;
    const int width = top - s + 1;
    const int nb = 1 << width;
    for (int i = threadIdx.x; i < nb; i += SEL_THREADS) sh.hist[i] = 0;
    __syncthreads();
    if constexpr (sizeof(K) == 4) {
      // 4 keys per thread per step (128-bit shared loads)
      const int n4 = ((reinterpret_cast<uintptr_t>(src) & 15) == 0) ? len / 4 : 0;
      for (int v = threadIdx.x; v < n4; v += SEL_THREADS) {
        const uint4 q = reinterpret_cast<const uint4*>(src)[v];
        const uint32_t kk[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (((K)kk[e] & pmask) == prefix) atomicAdd(&sh.hist[(uint32_t)(((K)kk[e] >> s) & (K)(nb - 1))], 1u);
      }
      for (int j = 4 * n4 + threadIdx.x; j < len; j += SEL_THREADS) {
        const K key = src[j];
        if ((key & pmask) == prefix) atomicAdd(&sh.hist[(uint32_t)((key >> s) & (K)(nb - 1))], 1u);
      }
    } else {
      for (int j = threadIdx.x; j < len; j += SEL_THREADS) {
        const K key = src[j];
        if ((key & pmask) == prefix) atomicAdd(&sh.hist[(uint32_t)((key >> s) & (K)(nb - 1))], 1u);
      }
    }
    __syncthreads();
    // descending scan over bins: thread t owns bins nb-1-4t .. nb-4-4t
    int local[4];
    int lsum = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int b = nb - 1 - 4 * (int)threadIdx.x - q;
      local[q] = (b >= 0) ? (int)sh.hist[b] : 0;
      lsum += local[q];
    }
    int total;
    int excl = block_scan_int(lsum, sh.warp_tot, total);
    if (excl < krem && krem <= excl + lsum) {
      int acc = excl;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (acc < krem && krem <= acc + local[q]) {
          sh.bcast[0] = nb - 1 - 4 * (int)threadIdx.x - q;
          sh.bcast[1] = acc;
          sh.bcast[2] = local[q];
        }
        acc += local[q];
      }
    }
    __syncthreads();
    const int digit = sh.bcast[0];
    const int above = sh.bcast[1];
    const int inbin = sh.bcast[2];
    __syncthreads();
    prefix |= (K)digit << s;
    pmask |= (K)(nb - 1) << s;
    krem -= above;
    if (s == 0) {
      ties = inbin;
      break;
    }
    if (sizeof(K) == 8 && !compacted && inbin <= cand_cap && inbin < len) {
      if (threadIdx.x == 0) sh.bcast[3] = 0;
      __syncthreads();
      const int lane = threadIdx.x & 31;
      for (int j0 = 0; j0 < len; j0 += SEL_THREADS) {
        const int j = j0 + threadIdx.x;
        const K key = j < len ? src[j] : (K)0;
        const bool m = j < len && (key & pmask) == prefix;
        const uint32_t bal = __ballot_sync(0xffffffffu, m);
        int base = 0;
        if (lane == 0 && bal) base = atomicAdd(&sh.bcast[3], __popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (m) cand[base + __popc(bal & ((1u << lane) - 1u))] = key;
      }
      __syncthreads();
      src = cand;
      len = inbin;
      compacted = true;
    }
  }
  T = prefix;
  need = krem;
}

// block-wide OR / AND of per-thread partials (used to locate varying key bits)
template <typename K>
__device__ __forceinline__ void block_or_and(K& v_or, K& v_and, SelShared& sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v_or |= __shfl_xor_sync(0xffffffffu, v_or, o);
    v_and &= __shfl_xor_sync(0xffffffffu, v_and, o);
  }
  K* red = reinterpret_cast<K*>(sh.cand);  // scratch (cand is free at this point)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    red[warp] = v_or;
    red[SEL_WARPS + warp] = v_and;
  }
  __syncthreads();
  K a = (K)0, b = ~(K)0;
#pragma unroll 8
  for (int w = 0; w < SEL_WARPS; ++w) {
    a |= red[w];
    b &= red[SEL_WARPS + w];
  }
  __syncthreads();
  v_or = a;
  v_and = b;
}

__device__ __forceinline__ bool is_extra(const SelectParams& p, int j, int n) {
  if ((p.flags & STS_SEL_CURRENT) && j == n - 1) return true;
  if ((p.flags & STS_SEL_SINK) && j == 0) return true;
  if (p.recent_window > 0 && j >= n - p.recent_window) return true;
  return false;
}

__device__ __forceinline__ void write_idx(const SelectParams& p, int32_t* out, int pos, int val) {
  if (pos < p.idx_ld) out[pos] = val;
  else set_status(p.status, STS_DEV_IDX_CAPACITY);
}

// Form the logical row's fp32 values (sum of sources, in source order) for
// j in [0, n) and hand each to `sink(j, value)`; 4 elements per thread per
// step with 128-bit loads when rows are 16-byte aligned, two steps in flight.
template <typename Sink>
__device__ __forceinline__ void for_row_values(const SelectParams& p, const int32_t* srcs, int n, Sink sink) {
  const bool vec = (p.ld % 4) == 0 && (reinterpret_cast<uintptr_t>(p.scores) % 16) == 0;
  int j0 = 0;
  if (vec) {
    const int n4 = n / 4;
    for (int v = threadIdx.x; v < n4; v += 2 * SEL_THREADS) {
      const int v2 = v + SEL_THREADS;
      const bool has2 = v2 < n4;
      float4 a = *reinterpret_cast<const float4*>(p.scores + (int64_t)srcs[0] * p.ld + 4 * v);
      float4 b = has2 ? *reinterpret_cast<const float4*>(p.scores + (int64_t)srcs[0] * p.ld + 4 * v2)
                      : make_float4(0.f, 0.f, 0.f, 0.f);
      for (int s = 1; s < p.nsrc; ++s) {
        const float* base = p.scores + (int64_t)srcs[s] * p.ld;
        const float4 x = *reinterpret_cast<const float4*>(base + 4 * v);
        a.x = __fadd_rn(a.x, x.x); a.y = __fadd_rn(a.y, x.y); a.z = __fadd_rn(a.z, x.z); a.w = __fadd_rn(a.w, x.w);
        if (has2) {
          const float4 y = *reinterpret_cast<const float4*>(base + 4 * v2);
          b.x = __fadd_rn(b.x, y.x); b.y = __fadd_rn(b.y, y.y); b.z = __fadd_rn(b.z, y.z); b.w = __fadd_rn(b.w, y.w);
        }
      }
      sink(4 * v, a.x); sink(4 * v + 1, a.y); sink(4 * v + 2, a.z); sink(4 * v + 3, a.w);
      if (has2) { sink(4 * v2, b.x); sink(4 * v2 + 1, b.y); sink(4 * v2 + 2, b.z); sink(4 * v2 + 3, b.w); }
    }
    j0 = 4 * n4;
  }
  for (int j = j0 + threadIdx.x; j < n; j += SEL_THREADS) sink(j, row_value(p, srcs, j));
}

// numpy pairwise_sum over values already staged in `vals` (see pairwise_sum)
__device__ double pairwise_vals(const float* vals, int start, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, (double)vals[start + i]);
    return r;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = (double)vals[start + j];
    int i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], (double)vals[start + i + j]);
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, (double)vals[start + i]);
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pairwise_vals(vals, start, n2), pairwise_vals(vals, start + n2, n - n2));
}

// np.add.reduceat segment of page pg, x[start] + pairwise(x[start+1 : start+len]),
// computed by the 8 lanes (lane & 7) of an aligned octet for pages whose
// pairwise part has 8..128 elements: lane j accumulates chain r[j] (elements
// j, j+8, ... of the 8-aligned body), the octet combines
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) by shuffles, lane 0 adds the tail and
// x[start] — the same operations in the same order as pairwise_vals.  Every
// lane of the warp must call it (shuffles); pages >= P return 0.
__device__ __forceinline__ uint64_t page_key_lanes(const float* vals, int pg, int P, int n_row, int ps) {
  const int j = threadIdx.x & 7;
  const bool live = pg < P;
  const int start = live ? pg * ps : 0;
  const int len = live ? min(ps, n_row - start) : 1;
  const int m = len - 1;  // pairwise part
  const bool chains = m >= 8;  // (m <= 128 by the caller's page size)
  const int body = m - m % 8;
  double r = 0.0;
  if (chains) {
    r = (double)vals[start + 1 + j];
    for (int i = 8; i < body; i += 8) r = __dadd_rn(r, (double)vals[start + 1 + i + j]);
  }
  double o = __shfl_xor_sync(0xffffffffu, r, 1);
  r = __dadd_rn(r, o);  // lanes 0,2,4,6: (r0+r1), (r2+r3), ...
  o = __shfl_xor_sync(0xffffffffu, r, 2);
  r = __dadd_rn(r, o);  // lanes 0,4
  o = __shfl_xor_sync(0xffffffffu, r, 4);
  r = __dadd_rn(r, o);  // lane 0: the tree
  uint64_t key = 0ull;
  if (j == 0 && live) {
    double res;
    if (chains) {
      res = r;
      for (int i = body; i < m; ++i) res = __dadd_rn(res, (double)vals[start + 1 + i]);
    } else {
      res = 0.0;
      for (int i = 0; i < m; ++i) res = __dadd_rn(res, (double)vals[start + 1 + i]);
    }
    const double x0 = (double)vals[start];
    key = f64_key(len == 1 ? x0 : __dadd_rn(x0, res));
  }
  return key;
}

// Emit pass over `len` candidates in index order, 4 per thread per chunk.
// sel(j, tie_rank_before_j_is_lt_need) decides membership; writes ascending.
template <typename KeyAt, typename Extra>
__device__ __forceinline__ int emit_sorted(const SelectParams& p, SelShared& sh, int32_t* out, int len,
                                           KeyAt key_at, uint64_t T, int need, Extra extra, int out_base,
                                           bool write_bits, uint32_t* bits, bool all_ties = false) {
  int run_sel = 0, run_tie = 0;
  for (int base = 0; base < len; base += 4 * SEL_THREADS) {
    const int j0 = base + 4 * threadIdx.x;
    uint64_t k4[4];
    int nt = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = j0 + q;
      k4[q] = j < len ? key_at(j) : 0ull;
      nt += (j < len && k4[q] == T) ? 1 : 0;
    }
    int tie_tot = 0, tie_ex = 0;
    if (!all_ties && need > 0) tie_ex = block_scan_int(nt, sh.warp_tot, tie_tot);
    bool f[4];
    int ns = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = j0 + q;
      bool sel = false;
      if (j < len) {
        const bool tie = k4[q] == T;
        sel = k4[q] > T || (tie && need > 0 && (all_ties || run_tie + tie_ex < need)) || extra(j);
        tie_ex += tie ? 1 : 0;
      }
      f[q] = sel;
      ns += sel ? 1 : 0;
    }
    if (write_bits) {
      // page mode: record selected pages as a bitmap (4 bits per thread)
      const uint32_t nib = (f[0] ? 1u : 0u) | (f[1] ? 2u : 0u) | (f[2] ? 4u : 0u) | (f[3] ? 8u : 0u);
      const int lane = threadIdx.x & 31;
      uint32_t w = nib << ((lane & 7) * 4);
      w |= __shfl_xor_sync(0xffffffffu, w, 1);
      w |= __shfl_xor_sync(0xffffffffu, w, 2);
      w |= __shfl_xor_sync(0xffffffffu, w, 4);
      if ((lane & 7) == 0 && j0 < len) bits[j0 >> 5] = w;
      run_tie += tie_tot;
      continue;
    }
    int sel_tot;
    int sel_ex = block_scan_int(ns, sh.warp_tot, sel_tot);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (f[q]) write_idx(p, out, out_base + run_sel + sel_ex++, j0 + q);
    run_sel += sel_tot;
    run_tie += tie_tot;
  }
  return run_sel;
}

// Token-mode emit: 8 keys per thread per step (two 128-bit shared loads),
// one block scan per 8192 keys when every tie at T is taken, two otherwise.
__device__ int emit_tokens(const SelectParams& p, SelShared& sh, int32_t* out, const uint32_t* keys, int n,
                           uint32_t T, int need, bool all_ties) {
  const int lo_extra = p.recent_window > 0 ? n - p.recent_window : n;  // [lo_extra, n) always kept
  const bool cur = (p.flags & STS_SEL_CURRENT) != 0, sink = (p.flags & STS_SEL_SINK) != 0;
  int run_sel = 0, run_tie = 0;
  for (int base = 0; base < n; base += 8 * SEL_THREADS) {
    const int j0 = base + 8 * threadIdx.x;
    uint32_t k8[8];
    if (j0 + 8 <= n) {
      const uint4 a = reinterpret_cast<const uint4*>(keys + j0)[0];
      const uint4 b = reinterpret_cast<const uint4*>(keys + j0)[1];
      k8[0] = a.x; k8[1] = a.y; k8[2] = a.z; k8[3] = a.w;
      k8[4] = b.x; k8[5] = b.y; k8[6] = b.z; k8[7] = b.w;
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) k8[q] = j0 + q < n ? keys[j0 + q] : 0u;
    }
    uint32_t gt = 0, eq = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const bool valid = j0 + q < n;
      gt |= (valid && k8[q] > T) ? (1u << q) : 0u;
      eq |= (valid && k8[q] == T) ? (1u << q) : 0u;
    }
    uint32_t sel = gt;
    if (all_ties) {
      sel |= eq;
    } else {
      int tie_tot;
      const int tie_ex = block_scan_int(__popc(eq), sh.warp_tot, tie_tot);
      int rank = run_tie + tie_ex;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if ((eq >> q) & 1u) {
          if (rank < need) sel |= 1u << q;
          ++rank;
        }
      run_tie += tie_tot;
    }
    // always-include extras (current, sink, recent window): only near the ends
    if (j0 + 7 >= lo_extra || (sink && j0 == 0) || (cur && j0 + 7 >= n - 1)) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int j = j0 + q;
        if (j < n && (j >= lo_extra || (sink && j == 0) || (cur && j == n - 1))) sel |= 1u << q;
      }
    }
    int sel_tot;
    int pos = run_sel + block_scan_int(__popc(sel), sh.warp_tot, sel_tot);
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if ((sel >> q) & 1u) write_idx(p, out, pos++, j0 + q);
    run_sel += sel_tot;
  }
  return run_sel;
}

constexpr int RANK_PAGES = SEL_THREADS / 4;  // page rows up to this many pages use all-pairs ranks

// Tokens of the selected pages (pbits) in ascending order: a block scan over
// the pages gives each selected page its output slot; the page's positions
// are written by a quarter-warp (8 lanes x 16 B).  Returns the token count.
__device__ int expand_pages(const SelectParams& p, SelShared& sh, int32_t* out, const uint32_t* pbits, int P, int n,
                            int ps) {
  const int lane = threadIdx.x & 31;
  int run = 0;
  for (int base = 0; base < P; base += SEL_THREADS) {
    const int pg = base + threadIdx.x;
    const bool sel = pg < P && ((pbits[pg >> 5] >> (pg & 31)) & 1u);
    int tot;
    const int rank = run + block_scan_int(sel ? 1 : 0, sh.warp_tot, tot);
    // every selected page but the row's last is whole: slot = rank * ps
    uint32_t m = __ballot_sync(0xffffffffu, sel);
    while (m) {  // the warp's selected pages, one at a time, 32 lanes per page
      const int src = __ffs(m) - 1;
      m &= m - 1;
      const int g = __shfl_sync(0xffffffffu, pg, src), rk = __shfl_sync(0xffffffffu, rank, src);
      const int len = min(ps, n - g * ps);
      for (int e = lane; e < len; e += 32) write_idx(p, out, rk * ps + e, g * ps + e);
    }
    run += tot;
  }
  // the row's last page may be partial: it is the last selected page if selected
  const int last_len = n - (P - 1) * ps;
  const bool last_sel = P > 0 && ((pbits[(P - 1) >> 5] >> ((P - 1) & 31)) & 1u);
  return run * ps - (last_sel ? ps - last_len : 0);
}

__global__ void __launch_bounds__(SEL_THREADS, 1) select_kernel(SelectParams p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  SelShared& sh = *reinterpret_cast<SelShared*>(smem_raw);
  uint8_t* buf = p.gbuf ? (p.gbuf + (int64_t)blockIdx.x * p.gbuf_stride)
                        : (smem_raw + ((sizeof(SelShared) + 15) & ~size_t(15)));

  for (int64_t r = blockIdx.x; r < p.rows; r += gridDim.x) {
    const int n = p.row_len ? p.row_len[r] : p.n_common;
    int32_t* out = p.idx_out + r * p.idx_ld;
    int32_t srcs_local[8];
    const int32_t* srcs;
    int32_t ident = (int32_t)r;
    if (p.row_src) {
      for (int s = 0; s < p.nsrc && s < 8; ++s) srcs_local[s] = p.row_src[r * p.nsrc + s];
      srcs = srcs_local;
    } else {
      srcs = &ident;
    }
    int b;
    if (p.budget_is_fraction) {
      double c = ceil(p.budget * (double)n);
      b = c < 1.0 ? 1 : (int)c;
    } else {
      b = (int)p.budget;
    }
    auto extra = [&](int j) { return is_extra(p, j, n); };

    int count = 0;
    if (n <= 0) {
      // empty committed range: only the tail
    } else if (b >= n) {
      // dense fallback (src/sparsity.py:90-91)
      for (int j = threadIdx.x; j < n; j += SEL_THREADS) write_idx(p, out, j, j);
      count = n;
    } else if (p.page_size == 1) {
      uint32_t* keys = reinterpret_cast<uint32_t*>(buf);
      uint32_t k_or = 0u, k_and = 0xffffffffu;
      for_row_values(p, srcs, n, [&](int j, float v) {
        const uint32_t key = f32_key(v);
        keys[j] = key;
        k_or |= key;
        k_and &= key;
      });
      block_or_and(k_or, k_and, sh);  // (its barrier also publishes keys[])
      uint32_t T;
      int need, ties;
      radix_select<uint32_t>(keys, n, b, k_or, k_and, sh, reinterpret_cast<uint32_t*>(sh.cand), CAND_BYTES / 4, T,
                             need, ties);
      count = emit_tokens(p, sh, out, keys, n, T, need, need == ties);    } else {
      const int ps = p.page_size;
      const int P = (n + ps - 1) / ps;
      const int kp = (b + ps - 1) / ps;
      float* vals = reinterpret_cast<float*>(buf);
      uint64_t* pkeys = reinterpret_cast<uint64_t*>(buf + (((int64_t)n * 4 + 15) & ~int64_t(15)));
      uint32_t* pbits = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(pkeys) + (((int64_t)P * 8 + 15) & ~int64_t(15)));
      if (kp >= P) {
        for (int w = threadIdx.x; w < (P + 31) / 32; w += SEL_THREADS) pbits[w] = 0xffffffffu;
      } else {
        for_row_values(p, srcs, n, [&](int j, float v) { vals[j] = v; });
        __syncthreads();
        uint64_t p_or = 0ull, p_and = ~0ull;
        if (ps >= 9 && ps <= 129) {
          // 8 lanes per page: lane j sums pairwise chain j, the chains meet in
          // numpy's fixed tree order through shuffles (see page_key_lanes)
          for (int base = 0; base < P; base += SEL_THREADS / 8) {
            const int pg = base + (int)(threadIdx.x >> 3);
            const uint64_t key = page_key_lanes(vals, pg, P, n, ps);
            if ((threadIdx.x & 7) == 0 && pg < P) {
              pkeys[pg] = key;
              p_or |= key;
              p_and &= key;
            }
          }
        } else {
          for (int pg = threadIdx.x; pg < P; pg += SEL_THREADS) {
            const int start = pg * ps;
            const int len = min(ps, n - start);
            // np.add.reduceat segment: x[start] + pairwise(x[start+1 : start+len])
            const double x0 = (double)vals[start];
            const uint64_t key = f64_key(len == 1 ? x0 : __dadd_rn(x0, pairwise_vals(vals, start + 1, len - 1)));
            pkeys[pg] = key;
            p_or |= key;
            p_and &= key;
          }
        }
        block_or_and(p_or, p_and, sh);  // (its barriers also publish pkeys[])
        if (P <= RANK_PAGES) {
          // few pages: exact ranks by all-pairs comparison (4 threads per page,
          // a quarter of the keys each) instead of 64-bit radix passes; rank =
          // #greater + #equal at a lower index (the stable tie rule)
          int* part = reinterpret_cast<int*>(sh.cand);  // [4][RANK_PAGES]
          const int t = threadIdx.x % RANK_PAGES, q = threadIdx.x / RANK_PAGES;
          if (t < P) {
            const uint64_t kt = pkeys[t];
            const int i0 = q * P / 4, i1 = (q + 1) * P / 4;
            int c = 0;
            for (int i = i0; i < i1; ++i) {
              const uint64_t ki = pkeys[i];
              c += (ki > kt || (ki == kt && i < t)) ? 1 : 0;
            }
            part[q * RANK_PAGES + t] = c;
          }
          __syncthreads();
          if (q == 0) {
            const bool sel = t < P && part[t] + part[RANK_PAGES + t] + part[2 * RANK_PAGES + t] +
                                              part[3 * RANK_PAGES + t] < kp;
            const uint32_t bal = __ballot_sync(0xffffffffu, sel);
            if ((threadIdx.x & 31) == 0 && threadIdx.x < ((P + 31) & ~31)) pbits[threadIdx.x >> 5] = bal;
          }
        } else {
          uint64_t T;
          int need, ties;
          radix_select<uint64_t>(pkeys, P, kp, p_or, p_and, sh, reinterpret_cast<uint64_t*>(sh.cand), CAND_BYTES / 8,
                                 T, need, ties);
          emit_sorted(p, sh, out, P, [&](int j) { return pkeys[j]; }, T, need, [](int) { return false; }, 0, true,
                      pbits, need == ties);
        }
      }
      __syncthreads();
      if (p.flags == 0 && p.recent_window == 0) {
        // no extras: the tokens are the selected pages, expanded in page order
        count = expand_pages(p, sh, out, pbits, P, n, ps);
      } else {
        count = emit_sorted(p, sh, out, n,
                            [&](int j) { return (uint64_t)((pbits[(j / ps) >> 5] >> ((j / ps) & 31)) & 1u); },
                            0ull, 0, extra, 0, false, nullptr);  // selected iff page bit (key) > 0
      }
    }
    // in-block tail (mode S: the verify block's own positions)
    for (int t = threadIdx.x; t < p.tail_len; t += SEL_THREADS) write_idx(p, out, count + t, max(n, 0) + t);
    count += p.tail_len;
    if (threadIdx.x == 0) p.cnt_out[r] = count;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Token mode with the row in registers (rows <= 32 * KPT * 32 keys, KPT <= 36).
//
// One 1024-thread CTA per row.  Warp w owns the contiguous slice
// [w*32*KPT, (w+1)*32*KPT) of the row; lane l holds positions
// w*32*KPT + 128*g + 4*l + e (g < KPT/4, e < 4), so each source is read with
// KPT/4 coalesced 16-byte loads per thread.  The radix passes read the keys
// from registers (no key buffer, no candidate compaction); a pass stops early
// when the threshold bin is taken whole.  Emit: per-g lane prefixes by a
// packed warp scan (8-bit fields), warp totals -> one cross-warp scan, so
// indices come out ascending and ties at the threshold go to the lowest
// positions (src/numkit.py:84), exactly as select_kernel.  (A row split over
// a 2-CTA cluster with DSMEM histograms measured slower: 51 vs 44 us at c2.)
// ---------------------------------------------------------------------------
// exclusive prefix over the CTA's NW warps of a warp-uniform value (1 barrier;
// the caller syncs before scratch is reused)
template <int NW>
__device__ __forceinline__ int warp_excl_scan_of_warps(int v, int* scratch, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  int x = lane < NW ? scratch[lane] : 0;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += t;
  }
  total = __shfl_sync(0xffffffffu, x, 31);
  return __shfl_sync(0xffffffffu, x, warp) - v;
}

// block-wide exclusive scan in thread order for NW warps (3 barriers)
template <int NW>
__device__ __forceinline__ int block_scan_nw(int v, int* warp_tot, int& total) {
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
    int x = lane < NW ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    if (lane < NW) warp_tot[lane] = x;  // inclusive prefix over warps
  }
  __syncthreads();
  const int before = warp > 0 ? warp_tot[warp - 1] : 0;
  total = warp_tot[NW - 1];
  __syncthreads();
  return before + incl - v;
}

// Lane-exclusive prefixes and warp totals of per-g nibble popcounts, packed
// 4 groups per word in 8-bit fields (a lane count is <= 4, a warp's <= 128).
template <int G, typename M>
struct NibbleScan {
  static constexpr int W = (G + 3) / 4;
  uint32_t excl[W], tot[W];
  __device__ __forceinline__ NibbleScan(M bits) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      uint32_t v = 0u;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (4 * w + q < G) v |= (uint32_t)__popc((uint32_t)(bits >> (4 * (4 * w + q))) & 15u) << (8 * q);
      uint32_t x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += t;
      }
      excl[w] = x - v;
      tot[w] = __shfl_sync(0xffffffffu, x, 31);
    }
  }
  __device__ __forceinline__ int before(int g) const { return (int)((excl[g >> 2] >> (8 * (g & 3))) & 255u); }
  __device__ __forceinline__ int total(int g) const { return (int)((tot[g >> 2] >> (8 * (g & 3))) & 255u); }
};

__device__ __forceinline__ int popc_m(uint32_t x) { return __popc(x); }
__device__ __forceinline__ int popc_m(unsigned long long x) { return __popcll(x); }

// one histogram pass over the register keys; FULL: every key of the thread is
// in the row, FIRST: every valid key matches the prefix (common bits)
template <int KPT, bool FULL, bool FIRST, typename M>
__device__ __forceinline__ void hist_pass(const uint32_t (&key)[KPT], M valid, uint32_t pmask,
                                          uint32_t prefix, int s, uint32_t bmask, uint32_t* hist) {
#pragma unroll
  for (int i = 0; i < KPT; ++i) {
    bool m = FIRST ? true : (key[i] & pmask) == prefix;
    if (!FULL) m = m && ((valid >> i) & 1);
    if (m) atomicAdd(&hist[(key[i] >> s) & bmask], 1u);
  }
}

template <int KPT, int NSRC>
__global__ void __launch_bounds__(SEL_THREADS, 1) select_reg_kernel(SelectParams p) {
  constexpr int NT = SEL_THREADS, NW = SEL_WARPS, G = KPT / 4;
  constexpr int BPT = NBINS / NT;  // histogram bins per thread in the scan
  static_assert(KPT % 4 == 0 && KPT <= 64 && NW == 32 && BPT * NT == NBINS, "layout");
  using M = typename std::conditional<(KPT > 32), unsigned long long, uint32_t>::type;  // one bit per key slot
  constexpr M ONE = 1;
  __shared__ uint32_t hist[NBINS];
  __shared__ int scan_a[NW], scan_b[NW];
  __shared__ int bc[3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool vec = (p.ld % 4) == 0 && (reinterpret_cast<uintptr_t>(p.scores) % 16) == 0;
  const int nsrc = NSRC > 0 ? NSRC : p.nsrc;

  for (int64_t r = blockIdx.x; r < p.rows; r += gridDim.x) {
    const int n = p.row_len ? p.row_len[r] : p.n_common;
    int32_t* out = p.idx_out + r * p.idx_ld;
    int b;
    if (p.budget_is_fraction) {
      const double c = ceil(p.budget * (double)n);
      b = c < 1.0 ? 1 : (int)c;
    } else {
      b = (int)p.budget;
    }
    int count = 0;
    if (n <= 0) {
    } else if (b >= n) {  // dense fallback (src/sparsity.py:90-91)
      for (int j = threadIdx.x; j < n; j += SEL_THREADS) write_idx(p, out, j, j);
      count = n;
    } else {
      const int wbase = warp * 32 * KPT;
      const int jl = wbase + 4 * lane;  // position of (g, e) = jl + 128 g + e
      const bool full = wbase + 32 * KPT <= n;  // warp-uniform
      const float* srcp[NSRC > 0 ? NSRC : 8];
#pragma unroll
      for (int s = 0; s < (NSRC > 0 ? NSRC : 8); ++s)
        if (s < nsrc) srcp[s] = p.scores + (int64_t)(p.row_src ? p.row_src[r * nsrc + s] : (int32_t)r) * p.ld;
      // row values: fp32 sum over the sources in order (mode-S group reduction)
      uint32_t key[KPT];
      if (full && vec) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
          float4 a = __ldg(reinterpret_cast<const float4*>(srcp[0] + jl + 128 * g));
#pragma unroll
          for (int s = 1; s < (NSRC > 0 ? NSRC : 8); ++s)
            if (s < nsrc) {
              const float4 x = __ldg(reinterpret_cast<const float4*>(srcp[s] + jl + 128 * g));
              a.x = __fadd_rn(a.x, x.x);
              a.y = __fadd_rn(a.y, x.y);
              a.z = __fadd_rn(a.z, x.z);
              a.w = __fadd_rn(a.w, x.w);
            }
          key[4 * g] = f32_key(a.x);
          key[4 * g + 1] = f32_key(a.y);
          key[4 * g + 2] = f32_key(a.z);
          key[4 * g + 3] = f32_key(a.w);
        }
      } else {
#pragma unroll
        for (int i = 0; i < KPT; ++i) {
          const int j = jl + 128 * (i >> 2) + (i & 3);
          float a = 0.f;
          if (j < n) {
            a = __ldg(srcp[0] + j);
            for (int s = 1; s < nsrc; ++s) a = __fadd_rn(a, __ldg(srcp[s] + j));
          }
          key[i] = f32_key(a);
        }
      }
      M valid = ~(M)0;
      if (!full) {
        valid = 0;
#pragma unroll
        for (int i = 0; i < KPT; ++i) valid |= (jl + 128 * (i >> 2) + (i & 3) < n ? ONE : (M)0) << i;
      }
      uint32_t k_or = 0u, k_and = 0xffffffffu;
      if (full) {
#pragma unroll
        for (int i = 0; i < KPT; ++i) {
          k_or |= key[i];
          k_and &= key[i];
        }
      } else {
#pragma unroll
        for (int i = 0; i < KPT; ++i)
          if ((valid >> i) & 1) {
            k_or |= key[i];
            k_and &= key[i];
          }
      }
      k_or = __reduce_or_sync(0xffffffffu, k_or);
      k_and = __reduce_and_sync(0xffffffffu, k_and);
      if (lane == 0) {
        scan_a[warp] = (int)k_or;
        scan_b[warp] = (int)k_and;
      }
      __syncthreads();
      k_or = __reduce_or_sync(0xffffffffu, lane < NW ? (uint32_t)scan_a[lane] : 0u);
      k_and = __reduce_and_sync(0xffffffffu, lane < NW ? (uint32_t)scan_b[lane] : 0xffffffffu);
      __syncthreads();  // scan scratch is rewritten below

      // MSB-first radix select over the bits that vary across the row;
      // afterwards the threshold class is {key : (key & pmask) == prefix}
      uint32_t pmask = 0xffffffffu, prefix = k_and;
      int need = b, ties = n;
      const uint32_t diff = k_or ^ k_and;
      if (diff != 0u) {
        int top = 31 - __clz((int)diff);
        pmask = top >= 31 ? 0u : ~((2u << top) - 1u);
        prefix = k_and & pmask;
        int krem = b;
        for (bool first = true;; top -= DIGIT_BITS, first = false) {
          const int s = top - DIGIT_BITS + 1 < 0 ? 0 : top - DIGIT_BITS + 1;
          const int nb = 1 << (top - s + 1);
          uint32_t* h = hist;
          if (!first) __syncthreads();  // previous pass's readers of hist are done
          for (int q = threadIdx.x; q < nb; q += NT) h[q] = 0u;
          __syncthreads();
          const uint32_t bmask = (uint32_t)(nb - 1);
          if (first) {
            if (full) hist_pass<KPT, true, true, M>(key, valid, pmask, prefix, s, bmask, h);
            else hist_pass<KPT, false, true, M>(key, valid, pmask, prefix, s, bmask, h);
          } else {
            if (full) hist_pass<KPT, true, false, M>(key, valid, pmask, prefix, s, bmask, h);
            else hist_pass<KPT, false, false, M>(key, valid, pmask, prefix, s, bmask, h);
          }
          __syncthreads();
          int local[BPT], lsum = 0;
#pragma unroll
          for (int q = 0; q < BPT; ++q) {
            const int bin = nb - 1 - BPT * (int)threadIdx.x - q;
            local[q] = bin >= 0 ? (int)h[bin] : 0;
            lsum += local[q];
          }
          int total;
          const int excl = block_scan_nw<NW>(lsum, scan_a, total);
          if (excl < krem && krem <= excl + lsum) {
            int a = excl;
#pragma unroll
            for (int q = 0; q < BPT; ++q) {
              if (a < krem && krem <= a + local[q]) {
                bc[0] = nb - 1 - BPT * (int)threadIdx.x - q;
                bc[1] = a;
                bc[2] = local[q];
              }
              a += local[q];
            }
          }
          __syncthreads();
          const int digit = bc[0], above = bc[1], inbin = bc[2];
          prefix |= (uint32_t)digit << s;
          pmask |= bmask << s;
          krem -= above;
          if (s == 0 || inbin == krem) {  // exact key, or the whole bin is taken
            need = krem;
            ties = inbin;
            break;
          }
        }
      }

      // emit ascending: above-threshold keys, the first `need` of the class, extras
      M gt = 0, eq = 0;
#pragma unroll
      for (int i = 0; i < KPT; ++i) {
        const uint32_t hk = key[i] & pmask;
        gt |= (hk > prefix ? ONE : (M)0) << i;
        eq |= (hk == prefix ? ONE : (M)0) << i;
      }
      gt &= valid;
      eq &= valid;
      M sel = gt;
      const int lo_extra = p.recent_window > 0 ? n - p.recent_window : n;
      const bool cur = (p.flags & STS_SEL_CURRENT) != 0, sink = (p.flags & STS_SEL_SINK) != 0;
      const int whi = wbase + 32 * KPT - 1;
      if (whi >= lo_extra || (sink && wbase == 0) || (cur && whi >= n - 1 && wbase <= n - 1)) {
#pragma unroll
        for (int i = 0; i < KPT; ++i) {
          const int j = jl + 128 * (i >> 2) + (i & 3);
          if (j < n && (j >= lo_extra || (sink && j == 0) || (cur && j == n - 1))) sel |= ONE << i;
        }
      }
      if (need == ties) {
        sel |= eq;
      } else {
        int tot;
        int rank = warp_excl_scan_of_warps<NW>(__reduce_add_sync(0xffffffffu, (uint32_t)popc_m(eq)), scan_b, tot);
        const NibbleScan<G, M> ns(eq);
#pragma unroll
        for (int g = 0; g < G; ++g) {
          int rr = rank + ns.before(g);
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if ((eq >> (4 * g + e)) & 1) {
              if (rr < need) sel |= ONE << (4 * g + e);
              ++rr;
            }
          rank += ns.total(g);
        }
      }
      int pos = warp_excl_scan_of_warps<NW>(__reduce_add_sync(0xffffffffu, (uint32_t)popc_m(sel)), scan_a, count);
      const NibbleScan<G, M> ns(sel);
      const bool fits = count <= p.idx_ld;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        int q = pos + ns.before(g);
        uint32_t nib = (uint32_t)(sel >> (4 * g)) & 15u;
        while (nib) {  // set bits only (a tenth of the keys at 90% sparsity)
          const int e = __ffs(nib) - 1;
          if (fits) out[q] = jl + 128 * g + e;
          else write_idx(p, out, q, jl + 128 * g + e);
          ++q;
          nib &= nib - 1u;
        }
        pos += ns.total(g);
      }
    }
    // in-block tail (mode S: the verify block's own positions)
    for (int t = threadIdx.x; t < p.tail_len; t += NT) write_idx(p, out, count + t, max(n, 0) + t);
    if (threadIdx.x == 0) p.cnt_out[r] = count + p.tail_len;
    __syncthreads();
  }
}

// page_aggregate as a standalone op (src/sparsity.py:72-83): one thread per page
__global__ void page_aggregate_kernel(SelectParams p, double* out, int64_t out_ld) {
  const int64_t r = blockIdx.y;
  const int n = p.row_len ? p.row_len[r] : p.n_common;
  const int ps = p.page_size;
  const int P = (n + ps - 1) / ps;
  const int32_t ident = (int32_t)r;
  for (int pg = blockIdx.x * blockDim.x + threadIdx.x; pg < P; pg += gridDim.x * blockDim.x) {
    const int start = pg * ps;
    out[r * out_ld + pg] = ps == 1 ? (double)row_value(p, &ident, start)
                                   : page_sum(p, &ident, start, min(ps, n - start));
  }
}

int64_t key_buf_bytes(int32_t max_len, int32_t page_size) {
  int64_t tok = ((int64_t)max_len * 4 + 15) & ~int64_t(15);
  if (page_size == 1) return (tok + 127) & ~int64_t(127);
  int64_t pages = ((int64_t)max_len + page_size - 1) / page_size;
  int64_t b = tok + ((pages * 8 + 15) & ~int64_t(15)) + ((pages + 31) / 32 + 32) * 4;
  return (b + 127) & ~int64_t(127);
}

constexpr int64_t SEL_SMEM_BUDGET = 227 * 1024 - (int64_t)sizeof(SelShared) - 256;

// one CTA per row (grid-stride over rows beyond 2^30)
template <int KPT, int NSRC>
int launch_reg(const SelectParams& p, int64_t rows, cudaStream_t st) {
  select_reg_kernel<KPT, NSRC><<<(unsigned)rows, SEL_THREADS, 0, st>>>(p);
  STS_LAUNCH_CHECK();
  return STS_OK;
}

}  // namespace
}  // namespace sts

using namespace sts;

extern "C" size_t sts_select_workspace_bytes(int64_t rows, int32_t max_len, int32_t page_size) {
  if (key_buf_bytes(max_len, page_size) <= SEL_SMEM_BUDGET) return 0;
  int64_t slots = rows < 4 * num_sms() ? rows : 4 * num_sms();
  return (size_t)(slots * key_buf_bytes(max_len, page_size));
}

extern "C" int sts_select_topk(const float* scores_dev, int64_t ld, const int32_t* row_src_dev,
                               int32_t nsrc, int64_t rows, const int32_t* row_len_dev,
                               int32_t n_common, double budget, int32_t budget_is_fraction,
                               int32_t page_size, uint32_t flags, int32_t recent_window,
                               int32_t tail_len, int32_t* idx_out_dev, int64_t idx_ld,
                               int32_t* cnt_out_dev, int32_t* status_dev, void* workspace_dev,
                               size_t workspace_bytes, void* stream) {
  STS_REQUIRE(rows >= 0, STS_ERR_CONTRACT, "rows must be >= 0");
  if (rows == 0) return STS_OK;
  STS_REQUIRE(scores_dev && idx_out_dev && cnt_out_dev, STS_ERR_CONTRACT, "null buffer");
  STS_REQUIRE(nsrc >= 1 && nsrc <= 8, STS_ERR_CONTRACT, "nsrc must be in [1, 8], got %d", nsrc);
  STS_REQUIRE(row_src_dev || nsrc == 1, STS_ERR_CONTRACT, "nsrc > 1 needs a row_src table");
  STS_REQUIRE(page_size >= 1, STS_ERR_INPUT, "page_size must be >= 1");
  STS_REQUIRE(recent_window >= 0, STS_ERR_INPUT, "recent_window must be >= 0");
  STS_REQUIRE(tail_len >= 0, STS_ERR_CONTRACT, "tail_len must be >= 0");
  if (budget_is_fraction) {
    STS_REQUIRE(budget > 0.0 && budget <= 1.0, STS_ERR_INPUT,
                "fractional budget must be in (0, 1], got %g", budget);
  } else {
    STS_REQUIRE(budget >= 1.0, STS_ERR_INPUT, "token budget must be >= 1, got %g", budget);
  }
  STS_REQUIRE(row_len_dev || n_common >= 0, STS_ERR_CONTRACT, "n_common must be >= 0");
  STS_REQUIRE(ld >= 1, STS_ERR_CONTRACT, "ld must be >= 1");
  const int32_t max_len = row_len_dev ? (int32_t)ld : n_common;

  SelectParams p;
  p.scores = scores_dev;
  p.ld = ld;
  p.row_src = row_src_dev;
  p.nsrc = nsrc;
  p.rows = rows;
  p.row_len = row_len_dev;
  p.n_common = n_common;
  p.budget = budget;
  p.budget_is_fraction = budget_is_fraction;
  p.page_size = page_size;
  p.flags = flags;
  p.recent_window = recent_window;
  p.tail_len = tail_len;
  p.idx_out = idx_out_dev;
  p.idx_ld = idx_ld;
  p.cnt_out = cnt_out_dev;
  p.status = status_dev;
  p.buf_bytes = key_buf_bytes(max_len, page_size);

  // token rows that fit in registers (<= 36K keys): select_reg_kernel
  // (c2: 44 us vs 63 us for select_kernel, profiles/r02/select/)
  if (page_size == 1 && max_len <= 36 * 32 * SEL_WARPS) {
    const int64_t grid = rows < ((int64_t)1 << 30) ? rows : ((int64_t)1 << 30);
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (max_len <= 8 * 32 * SEL_WARPS) return launch_reg<8, 0>(p, grid, st);
    if (max_len <= 16 * 32 * SEL_WARPS) return launch_reg<16, 0>(p, grid, st);
    if (max_len <= 32 * 32 * SEL_WARPS) {
      if (nsrc == 1) return launch_reg<32, 1>(p, grid, st);
      if (nsrc == 4) return launch_reg<32, 4>(p, grid, st);
      return launch_reg<32, 0>(p, grid, st);
    }
    // just past 32K (mode-R rows: the committed context plus their in-block prefix)
    if (nsrc == 1) return launch_reg<36, 1>(p, grid, st);
    return launch_reg<36, 0>(p, grid, st);
  }
  const size_t sh_bytes = (sizeof(SelShared) + 15) & ~size_t(15);
  size_t smem = sh_bytes;
  int grid;
  if (p.buf_bytes <= SEL_SMEM_BUDGET) {
    p.gbuf = nullptr;
    p.gbuf_stride = 0;
    smem += (size_t)p.buf_bytes;
    grid = (int)(rows < (int64_t)1 << 30 ? rows : (1 << 30));
  } else {
    int64_t slots = rows < 4 * num_sms() ? rows : 4 * num_sms();
    size_t need = (size_t)(slots * p.buf_bytes);
    STS_REQUIRE(workspace_dev && workspace_bytes >= need, STS_ERR_CONTRACT,
                "select workspace too small: need %zu bytes, got %zu", need, workspace_bytes);
    p.gbuf = static_cast<uint8_t*>(workspace_dev);
    p.gbuf_stride = p.buf_bytes;
    grid = (int)slots;
  }
  static const cudaError_t attr = cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                       (int)(sh_bytes + SEL_SMEM_BUDGET));
  STS_CUDA_CHECK(attr);
  select_kernel<<<grid, SEL_THREADS, smem, static_cast<cudaStream_t>(stream)>>>(p);
  STS_LAUNCH_CHECK();
  return STS_OK;
}

extern "C" int sts_page_aggregate(const float* scores_dev, int64_t ld, int64_t rows,
                                  const int32_t* row_len_dev, int32_t n_common, int32_t page_size,
                                  double* out_dev, int64_t out_ld, void* stream) {
  STS_REQUIRE(page_size >= 1, STS_ERR_CONTRACT, "page_size must be >= 1");
  STS_REQUIRE(rows >= 0 && rows <= 65535, STS_ERR_CONTRACT, "rows must be in [0, 65535]");
  if (rows == 0) return STS_OK;
  STS_REQUIRE(scores_dev && out_dev, STS_ERR_CONTRACT, "null buffer");
  SelectParams p;
  memset(&p, 0, sizeof(p));
  p.scores = scores_dev;
  p.ld = ld;
  p.nsrc = 1;
  p.rows = rows;
  p.row_len = row_len_dev;
  p.n_common = n_common;
  p.page_size = page_size;
  const int32_t max_len = row_len_dev ? (int32_t)ld : n_common;
  const int pages = (max_len + page_size - 1) / page_size;
  dim3 grid((pages + 255) / 256 > 0 ? (pages + 255) / 256 : 1, (unsigned)rows);
  page_aggregate_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(p, out_dev, out_ld);
  STS_LAUNCH_CHECK();
  return STS_OK;
}
