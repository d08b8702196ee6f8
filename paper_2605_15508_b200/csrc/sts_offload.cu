// sts_offload.cu — mask-driven KV prefetch from host memory into an HBM page
// pool (the strategies of the reference's offload model,
// src/offloadsim.py:153-211, the pages_touched wire format of
// src/specdec.py:236-255).
//
//   sts_page_plan  per unit (batch, layer, kv-head): the ascending unique
//                  pages its key list touches, and the key list re-expressed
//                  as rows of the unit's pool slice (rank(page)*P + offset)
//   sts_page_copy  copies the planned pages of a range of units from pinned,
//                  device-mapped host K/V into the pool: one warp per page,
//                  16-byte loads over the host link, a few CTAs so the copy
//                  runs beside the attention of earlier layers
//
// The gathered decode then runs unchanged on the pool with the re-expressed
// lists, so its results are bit-identical to the HBM-resident run.
#include "sts_common.cuh"

namespace sts {
namespace {

constexpr int PLAN_THREADS = 256;

__global__ void __launch_bounds__(PLAN_THREADS) page_plan_kernel(const int32_t* __restrict__ idx, int64_t idx_ld,
                                                                 const int32_t* __restrict__ cnt, int page_size,
                                                                 int32_t* __restrict__ pages, int64_t pages_ld,
                                                                 int32_t* __restrict__ npages,
                                                                 int32_t* __restrict__ idx_pool, int tail_page0,
                                                                 int tail_rank0, int32_t* status) {
  __shared__ int warp_sums[PLAN_THREADS / 32];
  __shared__ int carry_rank, carry_page;
  const int64_t u = blockIdx.x;
  const int n = cnt[u];
  const int32_t* il = idx + u * idx_ld;
  int32_t* ol = idx_pool + u * idx_ld;
  int32_t* pl = pages + u * pages_ld;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    carry_rank = -1;
    carry_page = -1;
  }
  __syncthreads();
  for (int base = 0; base < n; base += PLAN_THREADS) {
    const int i = base + threadIdx.x;
    const bool live = i < n;
    const int pos = live ? il[i] : 0;
    const int pg = pos / page_size;
    const bool tail = tail_page0 >= 0 && pg >= tail_page0;  // the in-block tail: fixed ranks
    const int prev = (i == base) ? carry_page : (live ? il[i - 1] / page_size : -1);
    const int flag = (live && pg != prev && !tail) ? 1 : 0;
    // block inclusive scan of flags
    int x = flag;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    int off = 0;
    for (int w = 0; w < warp; ++w) off += warp_sums[w];
    const int crank = carry_rank + off + x;  // rank among the committed pages
    const int rank = tail ? tail_rank0 + (pg - tail_page0) : crank;
    if (live) {
      if (flag) {  // committed pages fill ranks [0, tail_rank0); the tail's ranks are fixed
        if (rank < (tail_page0 >= 0 ? tail_rank0 : pages_ld)) pl[rank] = pg;
        else set_status(status, STS_DEV_IDX_CAPACITY);
      }
      ol[i] = rank * page_size + (pos - pg * page_size);
    }
    __syncthreads();
    const int last = min(base + PLAN_THREADS, n) - 1;  // the chunk's last live key carries
    if (i == last) {
      carry_rank = crank;
      carry_page = pg;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) npages[u] = carry_rank + 1;
}

// Resident page pool with least-recently-used eviction across steps (the
// reference's "prefetch" strategy, src/offloadsim.py:173-209, run per unit):
// one CTA per unit.  slot_page / slot_last persist between calls (-1: empty).
// The step's committed pages already resident stay in their slots; the
// missing ones (ascending) take the free slots in the reference's eviction
// order — empty slots first, then by (step of last use, page) ascending,
// which is the order of the reference's LRU dict for one unit — and every
// page the step uses is stamped with `step`.
constexpr int CACHE_THREADS = 256;

__global__ void __launch_bounds__(CACHE_THREADS) page_cache_plan_kernel(
    const int32_t* __restrict__ idx, int64_t idx_ld, const int32_t* __restrict__ cnt, int page_size,
    int tail_page0, int tail_rank0, int32_t* __restrict__ slot_page, int32_t* __restrict__ slot_last,
    int64_t slots_ld, int C, int step, int32_t* __restrict__ copy_pages, int32_t* __restrict__ copy_slots,
    int32_t* __restrict__ ncopy, int32_t* __restrict__ idx_pool, int32_t* status) {
  extern __shared__ int32_t cache_sm[];
  const int NP = tail_page0;                    // committed pages of the unit
  uint32_t* need = reinterpret_cast<uint32_t*>(cache_sm);     // [ceil(NP/32)]
  int32_t* page_slot = cache_sm + (NP + 31) / 32;            // [NP]
  int32_t* kept = page_slot + NP;                             // [C]
  int32_t* miss = kept + C;                                   // [C] missing pages, ascending
  const int age_off = ((NP + 31) / 32 + NP + 2 * C + 1) & ~1;  // in 4-byte words, rounded to 8 bytes
  uint64_t* age = reinterpret_cast<uint64_t*>(cache_sm + age_off);  // [C] eviction keys
  __shared__ int warp_sums[CACHE_THREADS / 32];
  __shared__ int run_s;
  const int64_t u = blockIdx.x;
  const int n = cnt[u];
  const int32_t* il = idx + u * idx_ld;
  int32_t* sp = slot_page + u * slots_ld;
  int32_t* sl = slot_last + u * slots_ld;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int w = threadIdx.x; w < (NP + 31) / 32; w += CACHE_THREADS) need[w] = 0u;
  for (int q = threadIdx.x; q < NP; q += CACHE_THREADS) page_slot[q] = -1;
  if (threadIdx.x == 0) run_s = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += CACHE_THREADS) {
    const int pg = il[i] / page_size;
    if (pg < NP) atomicOr(&need[pg >> 5], 1u << (pg & 31));
  }
  __syncthreads();
  for (int s = threadIdx.x; s < C; s += CACHE_THREADS) {
    const int q = sp[s];
    const bool k = q >= 0 && q < NP && ((need[q >> 5] >> (q & 31)) & 1u);
    kept[s] = k ? 1 : 0;
    if (k) page_slot[q] = s;
  }
  __syncthreads();
  // missing pages, ascending (block scan over the page range)
  for (int base = 0; base < NP; base += CACHE_THREADS) {
    const int pg = base + threadIdx.x;
    const int f = (pg < NP && ((need[pg >> 5] >> (pg & 31)) & 1u) && page_slot[pg] < 0) ? 1 : 0;
    int x = f;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    int off = run_s;
    for (int w = 0; w < warp; ++w) off += warp_sums[w];
    if (f) {
      const int k = off + x - 1;
      if (k < C) miss[k] = pg;
    }
    __syncthreads();
    if (threadIdx.x == CACHE_THREADS - 1) run_s = off + x;
    __syncthreads();
  }
  const int M = run_s;
  // the free slots' eviction ranks: empty first, then (last use, page) ascending
  for (int s = threadIdx.x; s < C; s += CACHE_THREADS)
    age[s] = kept[s] ? ~0ull : (((uint64_t)(uint32_t)(sl[s] + 1) << 32) | (uint32_t)(sp[s] + 1));
  __syncthreads();
  int nfree_local = 0;
  for (int s = threadIdx.x; s < C; s += CACHE_THREADS) {
    if (kept[s]) continue;
    ++nfree_local;
    const uint64_t ks = age[s];
    int rank = 0;
    for (int t = 0; t < C; ++t) {
      const uint64_t kt = age[t];  // kept slots sort last (~0), never below a free one
      rank += (kt < ks || (kt == ks && t < s)) ? 1 : 0;
    }
    if (rank < M) {
      const int pg = miss[rank];
      copy_pages[u * slots_ld + rank] = pg;
      copy_slots[u * slots_ld + rank] = s;
      sp[s] = pg;
      page_slot[pg] = s;
    }
  }
  int nfree = nfree_local;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nfree += __shfl_xor_sync(0xffffffffu, nfree, o);
  __syncthreads();
  if (lane == 0) warp_sums[warp] = nfree;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int w = 0; w < CACHE_THREADS / 32; ++w) tot += warp_sums[w];
    if (M > tot) set_status(status, STS_DEV_IDX_CAPACITY);  // the step needs more pages than the pool holds
    ncopy[u] = M < tot ? M : tot;
  }
  // stamp the step's pages, re-express the key list as pool rows
  for (int q = threadIdx.x; q < NP; q += CACHE_THREADS)
    if (((need[q >> 5] >> (q & 31)) & 1u) && page_slot[q] >= 0) sl[page_slot[q]] = step;
  int32_t* ol = idx_pool + u * idx_ld;
  for (int i = threadIdx.x; i < n; i += CACHE_THREADS) {
    const int pos = il[i];
    const int pg = pos / page_size;
    int rank;
    if (pg < NP) {
      rank = page_slot[pg];
      if (rank < 0) rank = 0;  // (capacity exceeded: flagged above)
    } else {
      rank = tail_rank0 + (pg - tail_page0);
    }
    ol[i] = rank * page_size + (pos - pg * page_size);
  }
}

// one warp per (unit, page): K and V page copies, 16-byte vectors.  The grid
// is (CTAs per unit, units): units copy side by side, and each lane issues
// all its loads of a page before its stores, so a page costs one host-link
// round trip rather than one per vector.
__global__ void __launch_bounds__(256) page_copy_kernel(const uint8_t* __restrict__ host_k,
                                                        const uint8_t* __restrict__ host_v, int64_t host_unit_bytes,
                                                        int64_t host_row_bytes, uint8_t* __restrict__ pool_k,
                                                        uint8_t* __restrict__ pool_v, int64_t pool_unit_bytes,
                                                        const int32_t* __restrict__ pages, int64_t pages_ld,
                                                        const int32_t* __restrict__ npages,
                                                        const int32_t* __restrict__ slots, int64_t unit_begin,
                                                        int page_size, int row_bytes, int n_rows_host, int tail_page0,
                                                        int tail_rank0) {
  constexpr int MAXV = 8;  // 16-byte vectors per lane held in flight (per K and per V)
  const int lane = threadIdx.x & 31;
  const int64_t u = unit_begin + blockIdx.y;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t page_bytes = (int64_t)page_size * row_bytes;
  const int vec_per_row = row_bytes / 16;
  const int np = npages[u];
  const int ntail = tail_rank0 >= 0 ? (int)pages_ld - tail_rank0 : 0;
  const uint8_t* sk = host_k + u * host_unit_bytes;
  const uint8_t* sv = host_v + u * host_unit_bytes;
  for (int64_t ww = gw; ww < np + ntail; ww += nw) {
    const int64_t w = ww < np ? (slots ? (int64_t)slots[u * pages_ld + ww] : ww) : tail_rank0 + (ww - np);
    const int pg = ww < np ? pages[u * pages_ld + ww] : tail_page0 + (int)(w - tail_rank0);
    if (pg * page_size >= n_rows_host) continue;
    const int rows = min(page_size, n_rows_host - pg * page_size);
    const int nvec = rows * vec_per_row;
    uint8_t* dk = pool_k + u * pool_unit_bytes + w * page_bytes;
    uint8_t* dv = pool_v + u * pool_unit_bytes + w * page_bytes;
    for (int e0 = 0; e0 < nvec; e0 += 32 * MAXV) {
      int4 a[MAXV], b[MAXV];
#pragma unroll
      for (int t = 0; t < MAXV; ++t) {
        const int e = e0 + t * 32 + lane;
        if (e < nvec) {
          const int r = e / vec_per_row, c = e - r * vec_per_row;
          const int64_t src = (int64_t)(pg * page_size + r) * host_row_bytes + c * 16;
          a[t] = __ldg(reinterpret_cast<const int4*>(sk + src));
          b[t] = __ldg(reinterpret_cast<const int4*>(sv + src));
        }
      }
#pragma unroll
      for (int t = 0; t < MAXV; ++t) {
        const int e = e0 + t * 32 + lane;
        if (e < nvec) {
          const int r = e / vec_per_row, c = e - r * vec_per_row;
          *reinterpret_cast<int4*>(dk + (int64_t)r * row_bytes + c * 16) = a[t];
          *reinterpret_cast<int4*>(dv + (int64_t)r * row_bytes + c * 16) = b[t];
        }
      }
    }
  }
}

}  // namespace
}  // namespace sts

using namespace sts;

extern "C" int sts_page_plan(const int32_t* idx_dev, int64_t idx_ld, const int32_t* cnt_dev, int64_t units,
                             int32_t page_size, int32_t tail_page0, int32_t tail_rank0, int32_t* pages_dev,
                             int64_t pages_ld, int32_t* npages_dev, int32_t* idx_pool_dev, int32_t* status_dev,
                             void* stream) {
  STS_REQUIRE(tail_page0 < 0 || (tail_rank0 >= 0 && tail_rank0 < pages_ld), STS_ERR_CONTRACT,
              "tail_rank0 must be in [0, pages_ld)");
  STS_REQUIRE(units >= 0 && page_size >= 1 && pages_ld >= 1, STS_ERR_CONTRACT, "bad page plan shape");
  if (units == 0) return STS_OK;
  STS_REQUIRE(idx_dev && cnt_dev && pages_dev && npages_dev && idx_pool_dev, STS_ERR_CONTRACT, "null buffer");
  STS_REQUIRE(units <= 0x7fffffffLL, STS_ERR_CONTRACT, "too many units");
  page_plan_kernel<<<(unsigned)units, PLAN_THREADS, 0, static_cast<cudaStream_t>(stream)>>>(
      idx_dev, idx_ld, cnt_dev, page_size, pages_dev, pages_ld, npages_dev, idx_pool_dev, tail_page0,
      tail_rank0, status_dev);
  STS_LAUNCH_CHECK();
  return STS_OK;
}

extern "C" int sts_page_cache_plan(const int32_t* idx_dev, int64_t idx_ld, const int32_t* cnt_dev, int64_t units,
                                   int32_t page_size, int32_t tail_page0, int32_t tail_rank0, int32_t* slot_page_dev,
                                   int32_t* slot_last_dev, int64_t slots_ld, int32_t slots, int32_t step,
                                   int32_t* copy_pages_dev, int32_t* copy_slots_dev, int32_t* ncopy_dev,
                                   int32_t* idx_pool_dev, int32_t* status_dev, void* stream) {
  STS_REQUIRE(units >= 0 && page_size >= 1 && tail_page0 >= 0, STS_ERR_CONTRACT, "bad page cache shape");
  STS_REQUIRE(slots >= 1 && slots <= tail_rank0 && slots <= slots_ld, STS_ERR_CONTRACT,
              "slots must be in [1, min(tail_rank0, slots_ld)]");
  STS_REQUIRE(tail_page0 <= 16384 && slots <= 4096, STS_ERR_CONTRACT,
              "page cache supports up to 16384 committed pages and 4096 slots per unit");
  STS_REQUIRE(step >= 0, STS_ERR_CONTRACT, "step must be >= 0");
  if (units == 0) return STS_OK;
  STS_REQUIRE(idx_dev && cnt_dev && slot_page_dev && slot_last_dev && copy_pages_dev && copy_slots_dev && ncopy_dev &&
                  idx_pool_dev,
              STS_ERR_CONTRACT, "null buffer");
  STS_REQUIRE(units <= 0x7fffffffLL, STS_ERR_CONTRACT, "too many units");
  const size_t smem = ((size_t)(tail_page0 + 31) / 32 + tail_page0 + 2 * (size_t)slots + 1) * 4 + 8 * (size_t)slots + 8;
  static const cudaError_t attr =
      cudaFuncSetAttribute(page_cache_plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  STS_CUDA_CHECK(attr);
  page_cache_plan_kernel<<<(unsigned)units, CACHE_THREADS, smem, static_cast<cudaStream_t>(stream)>>>(
      idx_dev, idx_ld, cnt_dev, page_size, tail_page0, tail_rank0, slot_page_dev, slot_last_dev, slots_ld, slots, step,
      copy_pages_dev, copy_slots_dev, ncopy_dev, idx_pool_dev, status_dev);
  STS_LAUNCH_CHECK();
  return STS_OK;
}

extern "C" int sts_page_copy(const void* host_k, const void* host_v, int64_t host_unit_stride,
                             int64_t host_row_stride, int32_t n_rows_host, void* pool_k, void* pool_v,
                             int64_t pool_unit_stride, int32_t d, int32_t elem_bytes, const int32_t* pages_dev,
                             int64_t pages_ld, const int32_t* npages_dev, const int32_t* slots_dev,
                             int64_t unit_begin, int64_t unit_end, int32_t page_size, int32_t tail_page0,
                             int32_t tail_rank0, int32_t ctas, void* stream) {
  STS_REQUIRE(unit_begin >= 0 && unit_end >= unit_begin && page_size >= 1 && d >= 1, STS_ERR_CONTRACT,
              "bad page copy shape");
  if (unit_end == unit_begin) return STS_OK;
  STS_REQUIRE(host_k && host_v && pool_k && pool_v && pages_dev && npages_dev, STS_ERR_CONTRACT, "null buffer");
  const int row_bytes = d * elem_bytes;
  STS_REQUIRE(row_bytes % 16 == 0 && (host_row_stride * elem_bytes) % 16 == 0 &&
                  (host_unit_stride * elem_bytes) % 16 == 0 && (pool_unit_stride * elem_bytes) % 16 == 0,
              STS_ERR_CONTRACT, "page copy needs 16-byte aligned rows and strides");
  STS_REQUIRE(ctas >= 1 && ctas <= 4096, STS_ERR_CONTRACT, "ctas must be in [1, 4096]");
  STS_REQUIRE(unit_end - unit_begin <= 65535, STS_ERR_CONTRACT, "at most 65535 units per page copy");
  const int64_t nu = unit_end - unit_begin;
  const unsigned per_unit = (unsigned)(ctas / nu > 1 ? ctas / nu : 1);  // `ctas` in total, split over the units
  page_copy_kernel<<<dim3(per_unit, (unsigned)nu), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(host_k), static_cast<const uint8_t*>(host_v), host_unit_stride * elem_bytes,
      host_row_stride * elem_bytes, static_cast<uint8_t*>(pool_k), static_cast<uint8_t*>(pool_v),
      pool_unit_stride * elem_bytes, pages_dev, pages_ld, npages_dev, slots_dev, unit_begin, page_size, row_bytes,
      n_rows_host, tail_page0, tail_page0 >= 0 ? tail_rank0 : -1);
  STS_LAUNCH_CHECK();
  return STS_OK;
}
