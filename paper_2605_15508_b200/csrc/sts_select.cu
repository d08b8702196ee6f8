// sts_select.cu — sparsity-mask construction on sm_100a.
//
// One CTA (1024 threads) per logical row.  The row's values are formed on the
// fly (fp32 sum of nsrc source rows: identity for mode R, head-group sum for
// mode S), turned into order-preserving integer keys, and the k-th largest
// key is found by an MSB-first radix select with 12-bit digits and 4096-bin
// shared-memory histograms.  The emit pass walks indices in ascending order
// with ballot-based block scans, so ties at the threshold go to the lowest
// indices (the stable-argsort rule of src/numkit.py:84) and the output comes
// out sorted without a sort.
//
// Page mode (page_size > 1) reproduces src/sparsity.py:94-101: fp64 page sums
// in numpy add.reduceat order (x0 + pairwise(x[1:]), see pairwise_sum), a
// 64-bit-key radix select over pages, then page expansion.
//
// Keys live in shared memory when the row fits (<= SEL_SMEM_MAX_LEN), else in
// a per-CTA slot of the global workspace (persistent grid over rows).
#include <stdlib.h>

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
        block_or_and(p_or, p_and, sh);
        uint64_t T;
        int need, ties;
        radix_select<uint64_t>(pkeys, P, kp, p_or, p_and, sh, reinterpret_cast<uint64_t*>(sh.cand), CAND_BYTES / 8, T,
                               need, ties);
        emit_sorted(p, sh, out, P, [&](int j) { return pkeys[j]; }, T, need, [](int) { return false; }, 0, true,
                    pbits, need == ties);
      }
      __syncthreads();
      count = emit_sorted(p, sh, out, n,
                          [&](int j) { return (uint64_t)((pbits[(j / ps) >> 5] >> ((j / ps) & 31)) & 1u); },
                          0ull, 0, extra, 0, false, nullptr);  // selected iff page bit (key) > 0
    }
    // in-block tail (mode S: the verify block's own positions)
    for (int t = threadIdx.x; t < p.tail_len; t += SEL_THREADS) write_idx(p, out, count + t, max(n, 0) + t);
    count += p.tail_len;
    if (threadIdx.x == 0) p.cnt_out[r] = count;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Select v2 (token mode, rows <= 48K): 16-bit key prefixes in shared memory.
// Only the top 16 bits of each order key (sign, exponent, 7 mantissa bits)
// are kept on chip (2 bytes per position: three rows fit on one SM, 256 rows
// run in one wave on 148 SMs).  Two 8-bit radix passes find the 16-bit
// threshold prefix (the first one fused into row formation); the low 16 bits
// are resolved only for the positions in the threshold bin, recomputing their
// full keys from the score rows (typically a few hundred per row).  Emit walks
// positions in order: prefix above -> selected, prefix equal -> full-key
// compare + tie rank (ties to the lowest index), extras always.
// ---------------------------------------------------------------------------
constexpr int SV2_THREADS = 512;
constexpr int SV2_WARPS = SV2_THREADS / 32;
constexpr int SV2_MAX = 49152;

struct SV2Shared {
  uint32_t hist[256];
  int warp_tot[SV2_WARPS];
  int bcast[4];
};

__device__ __forceinline__ int sv2_scan(int v, int* warp_tot, int& total) {
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
    int x = lane < SV2_WARPS ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    if (lane < SV2_WARPS) warp_tot[lane] = x;
  }
  __syncthreads();
  const int before = warp > 0 ? warp_tot[warp - 1] : 0;
  total = warp_tot[SV2_WARPS - 1];
  __syncthreads();
  return before + incl - v;
}

// warp-aggregated shared-memory histogram increment (hot bins: one atomic per
// distinct bin per warp instead of one per lane)
__device__ __forceinline__ void sv2_hist_add(uint32_t* hist, int bin, bool active) {
  const unsigned mask = __ballot_sync(0xffffffffu, active);
  if (!active) return;
  const unsigned peers = __match_any_sync(mask, bin);
  const int leader = __ffs(peers) - 1;
  if ((int)(threadIdx.x & 31) == leader) atomicAdd(&hist[bin], (unsigned)__popc(peers));
}

// pick the digit whose descending cumulative count reaches krem (256 bins)
__device__ __forceinline__ void sv2_pick(SV2Shared& sh, int krem, int& digit, int& above, int& inbin) {
  const int tid = threadIdx.x;
  const int v = tid < 256 ? (int)sh.hist[255 - tid] : 0;
  int tot;
  const int excl = sv2_scan(v, sh.warp_tot, tot);
  if (tid < 256 && v > 0 && excl < krem && krem <= excl + v) {
    sh.bcast[0] = 255 - tid;
    sh.bcast[1] = excl;
    sh.bcast[2] = v;
  }
  __syncthreads();
  digit = sh.bcast[0];
  above = sh.bcast[1];
  inbin = sh.bcast[2];
  __syncthreads();
}

__global__ void __launch_bounds__(SV2_THREADS) select_v2_kernel(SelectParams p) {
  __shared__ SV2Shared sh;
  extern __shared__ __align__(16) uint16_t k16[];  // [n] key prefixes
  const int tid = threadIdx.x;
  const int64_t r = blockIdx.x;
  const int n = p.row_len ? p.row_len[r] : p.n_common;
  int32_t* out = p.idx_out + r * p.idx_ld;
  int32_t srcs[8];
  if (p.row_src) {
    for (int q = 0; q < p.nsrc && q < 8; ++q) srcs[q] = p.row_src[r * p.nsrc + q];
  } else {
    srcs[0] = (int32_t)r;
  }
  int b;
  if (p.budget_is_fraction) {
    const double cc = ceil(p.budget * (double)n);
    b = cc < 1.0 ? 1 : (int)cc;
  } else {
    b = (int)p.budget;
  }
  const bool cur = (p.flags & STS_SEL_CURRENT) != 0, sink = (p.flags & STS_SEL_SINK) != 0;
  const int lo_extra = p.recent_window > 0 ? n - p.recent_window : n;
  auto extra = [&](int j) { return j >= lo_extra || (sink && j == 0) || (cur && j == n - 1); };
  auto full_key = [&](int j) { return f32_key(row_value(p, srcs, j)); };

  int count = 0;
  if (n <= 0) {
  } else if (b >= n) {
    for (int j = tid; j < n; j += SV2_THREADS) write_idx(p, out, j, j);
    count = n;
  } else {
    // 1. formation: 16-bit prefixes + histogram of their top 8 bits
    if (tid < 256) sh.hist[tid] = 0;
    __syncthreads();
    const bool vec = (p.ld % 4) == 0 && (reinterpret_cast<uintptr_t>(p.scores) % 16) == 0;
    const int n4 = vec ? n / 4 : 0;
    for (int v0 = 0; v0 < n4; v0 += SV2_THREADS) {
      const int v = v0 + tid;
      const bool ok = v < n4;
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      if (ok) {
        a = *reinterpret_cast<const float4*>(p.scores + (int64_t)srcs[0] * p.ld + 4 * v);
        for (int q = 1; q < p.nsrc; ++q) {
          const float4 x = *reinterpret_cast<const float4*>(p.scores + (int64_t)srcs[q] * p.ld + 4 * v);
          a.x = __fadd_rn(a.x, x.x); a.y = __fadd_rn(a.y, x.y); a.z = __fadd_rn(a.z, x.z); a.w = __fadd_rn(a.w, x.w);
        }
      }
      const uint32_t k0 = f32_key(a.x) >> 16, k1 = f32_key(a.y) >> 16, k2 = f32_key(a.z) >> 16, k3 = f32_key(a.w) >> 16;
      if (ok) {
        uint2 packed;
        packed.x = k0 | (k1 << 16);
        packed.y = k2 | (k3 << 16);
        *reinterpret_cast<uint2*>(k16 + 4 * v) = packed;
      }
      sv2_hist_add(sh.hist, (int)(k0 >> 8), ok);
      sv2_hist_add(sh.hist, (int)(k1 >> 8), ok);
      sv2_hist_add(sh.hist, (int)(k2 >> 8), ok);
      sv2_hist_add(sh.hist, (int)(k3 >> 8), ok);
    }
    for (int j0 = 4 * n4; j0 < n; j0 += SV2_THREADS) {
      const int j = j0 + tid;
      const bool ok = j < n;
      const uint32_t k = ok ? full_key(j) >> 16 : 0u;
      if (ok) k16[j] = (uint16_t)k;
      sv2_hist_add(sh.hist, (int)(k >> 8), ok);
    }
    __syncthreads();
    int d1, above, inbin;
    sv2_pick(sh, b, d1, above, inbin);
    int krem = b - above;
    // 2. second 8 bits of the prefix
    uint32_t t16 = (uint32_t)d1 << 8;
    uint32_t pm16 = 0xff00u;
    if (krem != inbin) {
      if (tid < 256) sh.hist[tid] = 0;
      __syncthreads();
      for (int j0 = 0; j0 < n; j0 += SV2_THREADS) {
        const int j = j0 + tid;
        const uint32_t k = j < n ? k16[j] : 0u;
        const bool m = j < n && (k >> 8) == (uint32_t)d1;
        sv2_hist_add(sh.hist, (int)(k & 0xffu), m);
      }
      __syncthreads();
      int d2;
      sv2_pick(sh, krem, d2, above, inbin);
      krem -= above;
      t16 |= (uint32_t)d2;
      pm16 = 0xffffu;
    }
    // 3. low 16 bits among the positions whose prefix equals t16 (full keys
    //    recomputed from the score rows)
    uint32_t T = t16 << 16, pmask = pm16 << 16;
    bool all_bin = krem == inbin;
    for (int shift = 8; shift >= 0 && !all_bin && pm16 == 0xffffu; shift -= 8) {
      if (tid < 256) sh.hist[tid] = 0;
      __syncthreads();
      for (int j0 = 0; j0 < n; j0 += SV2_THREADS) {
        const int j = j0 + tid;
        const bool cand = j < n && k16[j] == t16;
        uint32_t key = 0;
        if (cand) key = full_key(j);
        const bool m = cand && (key & pmask) == T;
        sv2_hist_add(sh.hist, (int)((key >> shift) & 0xffu), m);
      }
      __syncthreads();
      int d;
      sv2_pick(sh, krem, d, above, inbin);
      krem -= above;
      T |= (uint32_t)d << shift;
      pmask |= 0xffu << shift;
      all_bin = krem == inbin;
    }
    // here: keys with (key & pmask) > T (prefix-wise) are above; == T are the
    // threshold ties of which the first krem (index order) are taken
    // (all of them when all_bin)
    // 4. emit in index order
    int run_sel = 0, run_tie = 0;
    for (int base = 0; base < n; base += 4 * SV2_THREADS) {
      const int j0 = base + 4 * tid;
      uint32_t sel = 0, eq = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = j0 + q;
        if (j >= n) break;
        const uint32_t k = k16[j];
        if ((k & pm16) > (t16 & pm16)) {
          sel |= 1u << q;
        } else if ((k & pm16) == (t16 & pm16)) {
          if (pm16 != 0xffffu || pmask == 0xffff0000u) {
            eq |= 1u << q;  // resolved at the prefix level
          } else {
            const uint32_t mk = full_key(j) & pmask;
            if (mk > T) sel |= 1u << q;
            else if (mk == T) eq |= 1u << q;
          }
        }
      }
      int tie_tot = 0;
      if (all_bin) {
        sel |= eq;
      } else {
        int rank = run_tie + sv2_scan(__popc(eq), sh.warp_tot, tie_tot);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if ((eq >> q) & 1u) {
            if (rank < krem) sel |= 1u << q;
            ++rank;
          }
        run_tie += tie_tot;
      }
      if (j0 + 3 >= lo_extra || (sink && j0 == 0) || (cur && j0 + 3 >= n - 1)) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (j0 + q < n && extra(j0 + q)) sel |= 1u << q;
      }
      int sel_tot;
      int pos = run_sel + sv2_scan(__popc(sel), sh.warp_tot, sel_tot);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if ((sel >> q) & 1u) write_idx(p, out, pos++, j0 + q);
      run_sel += sel_tot;
    }
    count = run_sel;
  }
  for (int t = tid; t < p.tail_len; t += SV2_THREADS) write_idx(p, out, count + t, max(n, 0) + t);
  if (tid == 0) p.cnt_out[r] = count + p.tail_len;
}

// ---------------------------------------------------------------------------
// Cluster select (token mode): a thread-block cluster of C CTAs per row, CTA c
// holding the keys of positions [c*n/C, (c+1)*n/C) in its shared memory.  The
// radix passes exchange 256-bin histograms through distributed shared memory
// (every CTA sums the same C histograms, so every CTA picks the same digit);
// after the threshold is known each CTA publishes its tie and selection
// counts, derives its tie share (ties go to the lowest global index) and its
// output offset, and emits its range.  Rows are spread over C SMs instead of
// one: the per-row latency of the single-CTA kernel is what bounds it.
// ---------------------------------------------------------------------------
constexpr int CSEL_THREADS = 512;
constexpr int CSEL_WARPS = CSEL_THREADS / 32;
constexpr int CSEL_BITS = 8;
constexpr int CSEL_BINS = 1 << CSEL_BITS;
constexpr int CSEL_KEYS = 16384;  // keys per CTA held in shared memory (64 KB)

struct CSelShared {
  uint32_t hist[CSEL_BINS];
  int xch[8];          // values published to the cluster
  int warp_tot[CSEL_WARPS];
  int bcast[4];
};

__device__ __forceinline__ unsigned csel_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void csel_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t csel_ld(const void* local, unsigned rank) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(local), ra, v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(ra) : "memory");
  return v;
}

__device__ __forceinline__ int csel_block_scan(int v, int* warp_tot, int& total) {
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
    int x = lane < CSEL_WARPS ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    if (lane < CSEL_WARPS) warp_tot[lane] = x;
  }
  __syncthreads();
  const int before = warp > 0 ? warp_tot[warp - 1] : 0;
  total = warp_tot[CSEL_WARPS - 1];
  __syncthreads();
  return before + incl - v;
}

template <int C>
__global__ void __launch_bounds__(CSEL_THREADS) select_cluster_kernel(SelectParams p) {
  __shared__ CSelShared sh;
  extern __shared__ __align__(16) uint32_t csel_keys[];  // CSEL_KEYS keys (dynamic shared memory)
  const unsigned c = csel_rank();
  const int64_t r = blockIdx.x / C;
  const int tid = threadIdx.x;
  const int n = p.row_len ? p.row_len[r] : p.n_common;
  int32_t* out = p.idx_out + r * p.idx_ld;
  int32_t srcs[8];
  if (p.row_src) {
    for (int q = 0; q < p.nsrc && q < 8; ++q) srcs[q] = p.row_src[r * p.nsrc + q];
  } else {
    srcs[0] = (int32_t)r;
  }
  int b;
  if (p.budget_is_fraction) {
    const double cc = ceil(p.budget * (double)n);
    b = cc < 1.0 ? 1 : (int)cc;
  } else {
    b = (int)p.budget;
  }
  const int lo = (int)((int64_t)c * (n > 0 ? n : 0) / C), hi = (int)((int64_t)(c + 1) * (n > 0 ? n : 0) / C);
  const int len = hi - lo;
  const bool dense = n > 0 && b >= n;
  const bool cur = (p.flags & STS_SEL_CURRENT) != 0, sink = (p.flags & STS_SEL_SINK) != 0;
  const int lo_extra = p.recent_window > 0 ? n - p.recent_window : n;
  auto extra = [&](int g) { return g >= lo_extra || (sink && g == 0) || (cur && g == n - 1); };

  // 1. keys of this CTA's positions (+ OR / AND of the varying bits)
  uint32_t k_or = 0u, k_and = 0xffffffffu;
  if (!dense)
    for (int j = tid; j < len; j += CSEL_THREADS) {
      const uint32_t key = f32_key(row_value(p, srcs, lo + j));
      csel_keys[j] = key;
      k_or |= key;
      k_and &= key;
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    k_or |= __shfl_xor_sync(0xffffffffu, k_or, o);
    k_and &= __shfl_xor_sync(0xffffffffu, k_and, o);
  }
  if (tid < CSEL_BINS) sh.hist[tid] = 0;
  if (tid == 0) {
    sh.bcast[0] = 0;
    sh.bcast[1] = -1;
  }
  __syncthreads();
  if ((tid & 31) == 0) {
    atomicOr(reinterpret_cast<unsigned*>(&sh.bcast[0]), k_or);
    atomicAnd(reinterpret_cast<unsigned*>(&sh.bcast[1]), k_and);
  }
  __syncthreads();
  if (tid == 0) {
    sh.xch[0] = sh.bcast[0];
    sh.xch[1] = sh.bcast[1];
  }
  csel_sync();
  uint32_t g_or = 0u, g_and = 0xffffffffu;
  for (unsigned q = 0; q < (unsigned)C; ++q) {
    g_or |= csel_ld(&sh.xch[0], q);
    g_and &= csel_ld(&sh.xch[1], q);
  }

  // 2. radix passes over the varying bits, 8 bits per pass, histograms summed
  //    over the cluster
  uint32_t prefix = 0u, pmask = 0u;
  int krem = b, ties_g = 0;
  bool resolved = dense || n <= 0;
  const uint32_t diff = g_or ^ g_and;
  if (!resolved && diff == 0u) {  // every committed key equal: all ties
    prefix = g_and;
    pmask = 0xffffffffu;
    ties_g = n;
    resolved = true;
  }
  int top = resolved ? -1 : 31 - __clz((int)diff);
  if (!resolved) {
    pmask = top >= 31 ? 0u : ~((2u << top) - 1u);
    prefix = g_and & pmask;
  }
  while (!resolved) {
    const int s0 = top - CSEL_BITS + 1 < 0 ? 0 : top - CSEL_BITS + 1;
    const int width = top - s0 + 1;
    const uint32_t dm = (1u << width) - 1u;
    csel_sync();  // every CTA is done reading the previous pass's histograms
    if (tid < CSEL_BINS) sh.hist[tid] = 0;
    __syncthreads();
    for (int j = tid; j < len; j += CSEL_THREADS) {
      const uint32_t key = csel_keys[j];
      if ((key & pmask) == prefix) atomicAdd(&sh.hist[(key >> s0) & dm], 1u);
    }
    csel_sync();
    // every CTA sums the same C histograms and finds the same digit
    int cnt = 0;
    if (tid < CSEL_BINS)
      for (unsigned q = 0; q < (unsigned)C; ++q) cnt += (int)csel_ld(&sh.hist[tid], q);
    // descending inclusive scan over bins (bin 255 first): thread tid holds bin 255 - tid
    int v = tid < CSEL_BINS ? 0 : 0;
    __shared__ int s_cnt[CSEL_BINS];
    if (tid < CSEL_BINS) s_cnt[tid] = cnt;
    __syncthreads();
    v = tid < CSEL_BINS ? s_cnt[CSEL_BINS - 1 - tid] : 0;
    int tot;
    const int excl = csel_block_scan(v, sh.warp_tot, tot);
    if (tid < CSEL_BINS && excl < krem && krem <= excl + v) {
      sh.bcast[2] = CSEL_BINS - 1 - tid;
      sh.bcast[3] = excl;
      sh.xch[7] = v;
    }
    __syncthreads();
    const int digit = sh.bcast[2], above = sh.bcast[3], inbin = sh.xch[7];
    prefix |= (uint32_t)digit << s0;
    pmask |= dm << s0;
    krem -= above;
    if (s0 == 0 || krem == inbin) {
      ties_g = inbin;
      resolved = true;
    }
    top = s0 - 1;
  }

  // 3. round A: this CTA's threshold ties -> its share of them (ties go to the
  //    lowest global index, i.e. to the lower CTAs first)
  const bool all_ties = krem >= ties_g;  // every key of the final bin is taken
  int t_loc = 0;
  if (!dense && n > 0)
    for (int j = tid; j < len; j += CSEL_THREADS) t_loc += (csel_keys[j] & pmask) == prefix ? 1 : 0;
  int tt;
  csel_block_scan(t_loc, sh.warp_tot, tt);
  if (tid == 0) sh.xch[2] = tt;
  csel_sync();
  int tie_before = 0;
  for (unsigned q = 0; q < c; ++q) tie_before += (int)csel_ld(&sh.xch[2], q);
  const int need = all_ties ? 0x7fffffff : krem - tie_before;  // ties this CTA takes, by local rank

  // selection flags of 4 consecutive local positions (block-wide tie ranks)
  auto flags4 = [&](int j0, int& run_tie) -> uint32_t {
    uint32_t sel = 0, eq = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = j0 + q;
      if (j >= len) break;
      const uint32_t mk = csel_keys[j] & pmask;
      if (mk > prefix) sel |= 1u << q;
      else if (mk == prefix) eq |= 1u << q;
    }
    int tie_tot;
    int rank = run_tie + csel_block_scan(__popc(eq), sh.warp_tot, tie_tot);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if ((eq >> q) & 1u) {
        if (rank < need) sel |= 1u << q;
        ++rank;
      }
      if (j0 + q < len && extra(lo + j0 + q)) sel |= 1u << q;
    }
    run_tie += tie_tot;
    return sel;
  };

  // round B: this CTA's selection count -> its output offset
  int sel_loc = 0;
  if (dense) {
    sel_loc = len;
  } else if (n > 0) {
    int run_tie = 0, cnt_acc = 0;
    for (int base = 0; base < len; base += 4 * CSEL_THREADS) cnt_acc += __popc(flags4(base + 4 * tid, run_tie));
    csel_block_scan(cnt_acc, sh.warp_tot, sel_loc);
  }
  if (tid == 0) sh.xch[3] = sel_loc;
  csel_sync();
  int out_off = 0, total = 0;
  for (unsigned q = 0; q < (unsigned)C; ++q) {
    const int sq = (int)csel_ld(&sh.xch[3], q);
    out_off += q < c ? sq : 0;
    total += sq;
  }
  csel_sync();  // published counts read by everyone (a CTA may now exit)

  // 4. emit this CTA's positions in ascending order
  if (dense) {
    for (int j = tid; j < len; j += CSEL_THREADS) write_idx(p, out, out_off + j, lo + j);
  } else if (n > 0) {
    int run_sel = 0, run_tie = 0;
    for (int base = 0; base < len; base += 4 * CSEL_THREADS) {
      const int j0 = base + 4 * tid;
      const uint32_t sel = flags4(j0, run_tie);
      int sel_tot;
      int pos = out_off + run_sel + csel_block_scan(__popc(sel), sh.warp_tot, sel_tot);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if ((sel >> q) & 1u) write_idx(p, out, pos++, lo + j0 + q);
      run_sel += sel_tot;
    }
  }
  // 5. in-block tail and the count (last CTA of the cluster)
  if (c == (unsigned)(C - 1)) {
    for (int t = tid; t < p.tail_len; t += CSEL_THREADS) write_idx(p, out, total + t, (n > 0 ? n : 0) + t);
    if (tid == 0) p.cnt_out[r] = total + p.tail_len;
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

  // experimental (STS_SELECT_V2=1): token-mode rows <= 48K through the 16-bit
  // prefix select.  Parity-tested, but measured slower at c2 (158 vs 63 us:
  // the threshold-bin candidates' full keys are recomputed with scattered,
  // latency-bound loads in three passes), so off by default.
  {
    static const int env = getenv("STS_SELECT_V2") ? atoi(getenv("STS_SELECT_V2")) : 0;
    if (env == 1 && page_size == 1 && max_len > 0 && max_len <= SV2_MAX && rows <= ((int64_t)1 << 31) - 1) {
      const size_t smem2 = (((size_t)max_len * 2 + 15) & ~size_t(15));
      static const cudaError_t a2 =
          cudaFuncSetAttribute(select_v2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SV2_MAX * 2);
      STS_CUDA_CHECK(a2);
      select_v2_kernel<<<(unsigned)rows, SV2_THREADS, smem2, static_cast<cudaStream_t>(stream)>>>(p);
      STS_LAUNCH_CHECK();
      return STS_OK;
    }
  }
  // experimental (STS_SELECT_CLUSTER=1): token-mode rows that fit C x 16K keys
  // through one thread-block cluster per row.  Measured slower than the
  // single-CTA kernel at c2 (150 vs 63 us: 8-bit digits without candidate
  // compaction serialise on hot shared-memory histogram bins), so off by default.
  {
    static const int env = getenv("STS_SELECT_CLUSTER") ? atoi(getenv("STS_SELECT_CLUSTER")) : 0;
    const int64_t per = CSEL_KEYS;
    if (env == 1 && page_size == 1 && max_len > 0 && max_len <= 8 * per && rows * 2 <= (int64_t)1 << 30) {
      int C = (int)((max_len + per - 1) / per);
      C = C < 2 ? 2 : (C <= 2 ? 2 : (C <= 4 ? 4 : 8));
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)(rows * C));
      cfg.blockDim = dim3(CSEL_THREADS);
      cfg.dynamicSmemBytes = CSEL_KEYS * 4;
      cfg.stream = static_cast<cudaStream_t>(stream);
      static const bool attr_ok =
          cudaFuncSetAttribute(select_cluster_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, CSEL_KEYS * 4) ==
              cudaSuccess &&
          cudaFuncSetAttribute(select_cluster_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, CSEL_KEYS * 4) ==
              cudaSuccess &&
          cudaFuncSetAttribute(select_cluster_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, CSEL_KEYS * 4) ==
              cudaSuccess;
      STS_REQUIRE(attr_ok, STS_ERR_CUDA, "cluster select setup failed");
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = C;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      p.gbuf = nullptr;
      cudaError_t e;
      if (C == 2) e = cudaLaunchKernelEx(&cfg, select_cluster_kernel<2>, p);
      else if (C == 4) e = cudaLaunchKernelEx(&cfg, select_cluster_kernel<4>, p);
      else e = cudaLaunchKernelEx(&cfg, select_cluster_kernel<8>, p);
      STS_CUDA_CHECK(e);
      count_launch();
      return STS_OK;
    }
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
