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

// one warp per (unit, page): K and V page copies, 16-byte vectors
__global__ void __launch_bounds__(256) page_copy_kernel(const uint8_t* __restrict__ host_k,
                                                        const uint8_t* __restrict__ host_v, int64_t host_unit_bytes,
                                                        int64_t host_row_bytes, uint8_t* __restrict__ pool_k,
                                                        uint8_t* __restrict__ pool_v, int64_t pool_unit_bytes,
                                                        const int32_t* __restrict__ pages, int64_t pages_ld,
                                                        const int32_t* __restrict__ npages, int64_t unit_begin,
                                                        int64_t unit_end, int page_size, int row_bytes,
                                                        int n_rows_host, int tail_page0, int tail_rank0) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t page_bytes = (int64_t)page_size * row_bytes;
  const int vec_per_row = row_bytes / 16;
  for (int64_t u = unit_begin; u < unit_end; ++u) {
    const int np = npages[u];
    const int ntail = tail_rank0 >= 0 ? (int)pages_ld - tail_rank0 : 0;
    for (int64_t ww = gw; ww < np + ntail; ww += nw) {
      const int64_t w = ww < np ? ww : tail_rank0 + (ww - np);
      const int pg = ww < np ? pages[u * pages_ld + w] : tail_page0 + (int)(w - tail_rank0);
      if (pg * page_size >= n_rows_host) continue;
      const int rows = min(page_size, n_rows_host - pg * page_size);
      const int nvec = rows * vec_per_row;
      const uint8_t* sk = host_k + u * host_unit_bytes;
      const uint8_t* sv = host_v + u * host_unit_bytes;
      uint8_t* dk = pool_k + u * pool_unit_bytes + w * page_bytes;
      uint8_t* dv = pool_v + u * pool_unit_bytes + w * page_bytes;
      for (int e = lane; e < nvec; e += 32) {
        const int r = e / vec_per_row, c = e - r * vec_per_row;
        const int64_t src = (int64_t)(pg * page_size + r) * host_row_bytes + c * 16;
        const int4 a = __ldg(reinterpret_cast<const int4*>(sk + src));
        const int4 b = __ldg(reinterpret_cast<const int4*>(sv + src));
        *reinterpret_cast<int4*>(dk + (int64_t)r * row_bytes + c * 16) = a;
        *reinterpret_cast<int4*>(dv + (int64_t)r * row_bytes + c * 16) = b;
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

extern "C" int sts_page_copy(const void* host_k, const void* host_v, int64_t host_unit_stride,
                             int64_t host_row_stride, int32_t n_rows_host, void* pool_k, void* pool_v,
                             int64_t pool_unit_stride, int32_t d, int32_t elem_bytes, const int32_t* pages_dev,
                             int64_t pages_ld, const int32_t* npages_dev, int64_t unit_begin, int64_t unit_end,
                             int32_t page_size, int32_t tail_page0, int32_t tail_rank0, int32_t ctas,
                             void* stream) {
  STS_REQUIRE(unit_begin >= 0 && unit_end >= unit_begin && page_size >= 1 && d >= 1, STS_ERR_CONTRACT,
              "bad page copy shape");
  if (unit_end == unit_begin) return STS_OK;
  STS_REQUIRE(host_k && host_v && pool_k && pool_v && pages_dev && npages_dev, STS_ERR_CONTRACT, "null buffer");
  const int row_bytes = d * elem_bytes;
  STS_REQUIRE(row_bytes % 16 == 0 && (host_row_stride * elem_bytes) % 16 == 0 &&
                  (host_unit_stride * elem_bytes) % 16 == 0 && (pool_unit_stride * elem_bytes) % 16 == 0,
              STS_ERR_CONTRACT, "page copy needs 16-byte aligned rows and strides");
  STS_REQUIRE(ctas >= 1 && ctas <= 4096, STS_ERR_CONTRACT, "ctas must be in [1, 4096]");
  page_copy_kernel<<<ctas, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(host_k), static_cast<const uint8_t*>(host_v), host_unit_stride * elem_bytes,
      host_row_stride * elem_bytes, static_cast<uint8_t*>(pool_k), static_cast<uint8_t*>(pool_v),
      pool_unit_stride * elem_bytes, pages_dev, pages_ld, npages_dev, unit_begin, unit_end, page_size, row_bytes,
      n_rows_host, tail_page0, tail_page0 >= 0 ? tail_rank0 : -1);
  STS_LAUNCH_CHECK();
  return STS_OK;
}
