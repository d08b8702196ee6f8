// sts_merge.cu — log-sum-exp merge of partial attention results (split-K
// partials inside one GPU, or per-rank partials of the sequence-sharded path),
// and the mode-R row-union builder.
#include "sts_common.cuh"

namespace sts {
namespace {

constexpr int MERGE_WARPS = 8;

__global__ void __launch_bounds__(MERGE_WARPS * 32) lse_merge_kernel(
    const float* __restrict__ o_part, const float* __restrict__ lse_part, int nparts, int64_t rows,
    int d, int out_dtype, void* out, float* lse_out) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * MERGE_WARPS + (threadIdx.x >> 5);
  if (row >= rows) return;
  float m = -INFINITY;
  for (int q = 0; q < nparts; ++q) m = fmaxf(m, lse_part[(int64_t)q * rows + row]);
  float tot = 0.f;
  if (m != -INFINITY)
    for (int q = 0; q < nparts; ++q) tot += expf(lse_part[(int64_t)q * rows + row] - m);
  if (lane == 0 && lse_out) lse_out[row] = tot > 0.f ? m + logf(tot) : -INFINITY;
  if (!out || !o_part) return;
  for (int e = lane; e < d; e += 32) {
    float acc = 0.f;
    if (tot > 0.f) {
      for (int q = 0; q < nparts; ++q) {
        const float l = lse_part[(int64_t)q * rows + row];
        if (l == -INFINITY) continue;
        acc += expf(l - m) * o_part[((int64_t)q * rows + row) * d + e];
      }
      acc /= tot;
    }
    if (out_dtype == STS_DTYPE_BF16)
      static_cast<__nv_bfloat16*>(out)[row * d + e] = __float2bfloat16_rn(acc);
    else
      static_cast<float*>(out)[row * d + e] = acc;
  }
}

// ---- mode-R union ----------------------------------------------------------
__global__ void union_scatter_kernel(const int32_t* __restrict__ idx_in, int64_t in_ld,
                                     const int32_t* __restrict__ cnt_in, const int32_t* __restrict__ src,
                                     int M, int n_max, uint32_t* bitmap, int32_t* status) {
  const int64_t u = blockIdx.y;
  const int m = blockIdx.z;
  const int list = src[u * M + m];
  const int c = cnt_in[list];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < c; i += gridDim.x * blockDim.x) {
    const int j = idx_in[(int64_t)list * in_ld + i];
    if (j < 0 || j >= n_max) {
      set_status(status, STS_DEV_BAD_INDEX);
      continue;
    }
    atomicOr(&bitmap[u * n_max + j], 1u << m);
  }
}

constexpr int UNION_THREADS = 1024;

__global__ void __launch_bounds__(UNION_THREADS) union_compact_kernel(
    const uint32_t* __restrict__ bitmap, int n_max, int32_t* idx_out, uint32_t* member_out,
    int64_t out_ld, int32_t* cnt_out, int32_t* status) {
  __shared__ int warp_tot[UNION_THREADS / 32];
  const int64_t u = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int run = 0;
  for (int base = 0; base < n_max; base += UNION_THREADS) {
    const int j = base + threadIdx.x;
    const uint32_t bits = j < n_max ? bitmap[u * n_max + j] : 0u;
    const bool f = bits != 0u;
    const uint32_t bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0) warp_tot[warp] = __popc(bal);
    __syncthreads();
    int before = 0, tot = 0;
    for (int w = 0; w < UNION_THREADS / 32; ++w) {
      before += w < warp ? warp_tot[w] : 0;
      tot += warp_tot[w];
    }
    __syncthreads();
    if (f) {
      const int pos = run + before + __popc(bal & ((1u << lane) - 1u));
      if (pos < out_ld) {
        idx_out[u * out_ld + pos] = j;
        member_out[u * out_ld + pos] = bits;
      } else {
        set_status(status, STS_DEV_IDX_CAPACITY);
      }
    }
    run += tot;
  }
  if (threadIdx.x == 0) cnt_out[u] = run < out_ld ? run : (int)out_ld;
}

// Same merge, parts addressed through a device array of pointers — one per
// rank's symmetric-memory buffer (peer addresses over NVLink): a one-shot
// all-gather + merge with no staging copy.  Arithmetic order = lse_merge_kernel.
__global__ void __launch_bounds__(MERGE_WARPS * 32) lse_merge_ptrs_kernel(
    const float* const* __restrict__ parts, int nparts, int64_t rows, int d, int64_t o_off, int64_t l_off,
    int out_dtype, void* out, float* lse_out) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * MERGE_WARPS + (threadIdx.x >> 5);
  if (row >= rows) return;
  float m = -INFINITY;
  for (int q = 0; q < nparts; ++q) m = fmaxf(m, __ldcg(parts[q] + l_off + row));
  float tot = 0.f;
  if (m != -INFINITY)
    for (int q = 0; q < nparts; ++q) tot += expf(__ldcg(parts[q] + l_off + row) - m);
  if (lane == 0 && lse_out) lse_out[row] = tot > 0.f ? m + logf(tot) : -INFINITY;
  if (!out) return;
  for (int e = lane; e < d; e += 32) {
    float acc = 0.f;
    if (tot > 0.f) {
      for (int q = 0; q < nparts; ++q) {
        const float l = __ldcg(parts[q] + l_off + row);
        if (l == -INFINITY) continue;
        acc += expf(l - m) * __ldcg(parts[q] + o_off + row * d + e);
      }
      acc /= tot;
    }
    if (out_dtype == STS_DTYPE_BF16)
      static_cast<__nv_bfloat16*>(out)[row * d + e] = __float2bfloat16_rn(acc);
    else
      static_cast<float*>(out)[row * d + e] = acc;
  }
}

}  // namespace

int lse_merge_launch(const float* o_part, const float* lse_part, int nparts, int64_t rows, int d,
                     int out_dtype, void* out, float* lse_out, cudaStream_t st) {
  if (rows == 0) return STS_OK;
  const int64_t blocks = (rows + MERGE_WARPS - 1) / MERGE_WARPS;
  lse_merge_kernel<<<(unsigned)blocks, MERGE_WARPS * 32, 0, st>>>(o_part, lse_part, nparts, rows, d,
                                                                  out_dtype, out, lse_out);
  STS_LAUNCH_CHECK();
  return STS_OK;
}

}  // namespace sts

using namespace sts;

extern "C" int sts_lse_merge(const float* o_part_dev, const float* lse_part_dev, int32_t nparts,
                             int64_t rows, int32_t d, int32_t out_dtype, void* out_dev,
                             float* lse_out_dev, void* stream) {
  STS_REQUIRE(nparts >= 1 && rows >= 0 && d >= 1, STS_ERR_CONTRACT, "bad merge shape");
  STS_REQUIRE(lse_part_dev, STS_ERR_CONTRACT, "null lse_part");
  STS_REQUIRE(out_dtype == STS_DTYPE_F32 || out_dtype == STS_DTYPE_BF16, STS_ERR_CONTRACT, "bad dtype");
  return lse_merge_launch(o_part_dev, lse_part_dev, nparts, rows, d, out_dtype, out_dev, lse_out_dev,
                          static_cast<cudaStream_t>(stream));
}

extern "C" int sts_row_union(const int32_t* idx_in_dev, int64_t in_ld, const int32_t* cnt_in_dev,
                             const int32_t* src_dev, int64_t units, int32_t M, int32_t n_max,
                             uint32_t* bitmap_ws_dev, int32_t* idx_out_dev, uint32_t* member_out_dev,
                             int64_t out_ld, int32_t* cnt_out_dev, int32_t* status_dev, void* stream) {
  STS_REQUIRE(units >= 0 && M >= 1 && M <= 32 && n_max >= 1, STS_ERR_CONTRACT, "bad union shape");
  STS_REQUIRE(units <= 65535, STS_ERR_CONTRACT, "units must be <= 65535");
  STS_REQUIRE(idx_in_dev && cnt_in_dev && src_dev && bitmap_ws_dev && idx_out_dev && member_out_dev &&
                  cnt_out_dev,
              STS_ERR_CONTRACT, "null buffer");
  if (units == 0) return STS_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  STS_CUDA_CHECK(cudaMemsetAsync(bitmap_ws_dev, 0, (size_t)units * n_max * sizeof(uint32_t), st));
  dim3 g1(8, (unsigned)units, (unsigned)M);
  union_scatter_kernel<<<g1, 256, 0, st>>>(idx_in_dev, in_ld, cnt_in_dev, src_dev, M, n_max,
                                           bitmap_ws_dev, status_dev);
  STS_LAUNCH_CHECK();
  union_compact_kernel<<<(unsigned)units, UNION_THREADS, 0, st>>>(bitmap_ws_dev, n_max, idx_out_dev,
                                                                  member_out_dev, out_ld, cnt_out_dev,
                                                                  status_dev);
  STS_LAUNCH_CHECK();
  return STS_OK;
}

// ---------------------------------------------------------------------------
// Algorithm 1 (headmap.find_head_mapping, src/headmap.py:83-125) on the GPU:
// per-row top-k index lists -> bitsets, then for every (a-head, b-head) pair
// the total popcount of the AND of their bitsets (integer: deterministic).
// ---------------------------------------------------------------------------
namespace sts {
namespace {

__global__ void bitset_scatter_kernel(const int32_t* __restrict__ idx, int64_t idx_ld, const int32_t* __restrict__ cnt,
                                      int32_t words, uint32_t* bits) {
  const int64_t r = blockIdx.x;
  const int c = cnt[r];
  uint32_t* row = bits + r * words;
  for (int j = threadIdx.x; j < c; j += blockDim.x) {
    const int i = idx[r * idx_ld + j];
    if (i >= 0 && i < words * 32) atomicOr(row + (i >> 5), 1u << (i & 31));
  }
}

constexpr int OVL_THREADS = 256;

__global__ void __launch_bounds__(OVL_THREADS) bitset_overlap_kernel(const uint32_t* __restrict__ a,
                                                                     const uint32_t* __restrict__ b,
                                                                     int64_t W, int32_t Tb,
                                                                     unsigned long long* scores) {
  const int64_t ia = blockIdx.y, ib = blockIdx.x;
  const uint4* pa = reinterpret_cast<const uint4*>(a + ia * W);
  const uint4* pb = reinterpret_cast<const uint4*>(b + ib * W);
  unsigned long long acc = 0;
  const int64_t W4 = W / 4;
  for (int64_t w = threadIdx.x; w < W4; w += OVL_THREADS) {
    const uint4 x = __ldg(pa + w), y = __ldg(pb + w);
    acc += __popc(x.x & y.x) + __popc(x.y & y.y) + __popc(x.z & y.z) + __popc(x.w & y.w);
  }
  for (int64_t w = 4 * W4 + threadIdx.x; w < W; w += OVL_THREADS) acc += __popc(a[ia * W + w] & b[ib * W + w]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ unsigned long long s_acc[OVL_THREADS / 32];
  if ((threadIdx.x & 31) == 0) s_acc[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int i = 0; i < OVL_THREADS / 32; ++i) t += s_acc[i];
    scores[ia * Tb + ib] += t;  // one block per pair: no race
  }
}

}  // namespace
}  // namespace sts

extern "C" int sts_topk_bitsets(const int32_t* idx_dev, int64_t idx_ld, const int32_t* cnt_dev, int64_t rows,
                                int32_t words, uint32_t* bits_out_dev, void* stream) {
  STS_REQUIRE(rows >= 0 && words >= 1, STS_ERR_CONTRACT, "rows must be >= 0 and words >= 1");
  if (rows == 0) return STS_OK;
  STS_REQUIRE(idx_dev && cnt_dev && bits_out_dev, STS_ERR_CONTRACT, "null buffer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  STS_CUDA_CHECK(cudaMemsetAsync(bits_out_dev, 0, (size_t)rows * words * 4, st));
  sts::bitset_scatter_kernel<<<(unsigned)rows, 128, 0, st>>>(idx_dev, idx_ld, cnt_dev, words, bits_out_dev);
  STS_LAUNCH_CHECK();
  return STS_OK;
}

extern "C" int sts_bitset_overlap(const uint32_t* a_dev, int32_t Ta, const uint32_t* b_dev, int32_t Tb, int64_t W,
                                  unsigned long long* scores_dev, void* stream) {
  STS_REQUIRE(Ta >= 0 && Tb >= 0 && W >= 0, STS_ERR_CONTRACT, "bad overlap shape");
  STS_REQUIRE(Ta <= 65535, STS_ERR_CONTRACT, "Ta must be <= 65535");
  if (Ta == 0 || Tb == 0 || W == 0) return STS_OK;
  STS_REQUIRE(a_dev && b_dev && scores_dev, STS_ERR_CONTRACT, "null buffer");
  STS_REQUIRE((reinterpret_cast<uintptr_t>(a_dev) | reinterpret_cast<uintptr_t>(b_dev)) % 16 == 0 && W % 4 == 0,
              STS_ERR_CONTRACT, "bitsets must be 16-byte aligned with W % 4 == 0");
  dim3 grid((unsigned)Tb, (unsigned)Ta);
  sts::bitset_overlap_kernel<<<grid, sts::OVL_THREADS, 0, static_cast<cudaStream_t>(stream)>>>(a_dev, b_dev, W, Tb,
                                                                                               scores_dev);
  STS_LAUNCH_CHECK();
  return STS_OK;
}

extern "C" int sts_lse_merge_ptrs(const void* part_ptrs_dev, int32_t nparts, int64_t rows, int32_t d,
                                  int64_t o_offset, int64_t l_offset, int32_t out_dtype, void* out_dev,
                                  float* lse_out_dev, void* stream) {
  STS_REQUIRE(nparts >= 1 && rows >= 0 && d >= 1, STS_ERR_CONTRACT, "bad merge shape");
  STS_REQUIRE(out_dtype == STS_DTYPE_F32 || out_dtype == STS_DTYPE_BF16, STS_ERR_CONTRACT, "bad out dtype");
  if (rows == 0) return STS_OK;
  STS_REQUIRE(part_ptrs_dev, STS_ERR_CONTRACT, "null part pointer array");
  const int64_t blocks = (rows + MERGE_WARPS - 1) / MERGE_WARPS;
  lse_merge_ptrs_kernel<<<(unsigned)blocks, MERGE_WARPS * 32, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const float* const*>(part_ptrs_dev), nparts, rows, d, o_offset, l_offset, out_dtype, out_dev,
      lse_out_dev);
  STS_LAUNCH_CHECK();
  return STS_OK;
}
