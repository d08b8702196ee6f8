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

// |A ∩ B| of two bitsets is the dot product of their 0/1 bit vectors, so the
// all-pairs overlap is an integer GEMM: scores[Ta][Tb] += A[Ta][K] · B[Tb][K]ᵀ
// with K = 32·W bits.  It runs on the int8 tensor cores (mma.sync m16n8k32
// u8·u8 → s32, exact): each 4-bit nibble of a bitset word expands to four
// 0/1 bytes with one multiply — (x·0x204081) & 0x01010101 puts bit i at byte
// i — straight into the MMA fragment registers, so the bitsets stay 1 bit per
// element in memory.  CTA tile 128 a-rows × 64 b-rows, four warps of 64 × 32
// (4 × 4 MMAs per 32-bit word), words staged through shared memory in chunks
// of OVL_KC with padded rows (the 8 row groups of a warp hit distinct banks).
constexpr int OVL_THREADS = 128;
constexpr int OVL_TA = 128, OVL_TB = 64;
constexpr int OVL_KC = 32;  // words per chunk
constexpr int OVL_PITCH = OVL_KC + 1;

__device__ __forceinline__ uint32_t nibble_bytes(uint32_t x, int shift) {
  return (((x >> shift) & 15u) * 0x204081u) & 0x01010101u;
}

__device__ __forceinline__ void mma_u8_16832(int (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

__global__ void __launch_bounds__(OVL_THREADS) bitset_overlap_kernel(const uint32_t* __restrict__ a, int32_t Ta,
                                                                     const uint32_t* __restrict__ b, int32_t Tb,
                                                                     int64_t ld, int64_t W, int64_t kspan,
                                                                     unsigned long long* scores) {
  __shared__ uint32_t As[OVL_TA * OVL_PITCH];
  __shared__ uint32_t Bs[OVL_TB * OVL_PITCH];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int wa = (warp >> 1) * 64, wb = (warp & 1) * 32;  // warp tile origin inside the CTA tile
  const int64_t a0 = (int64_t)blockIdx.y * OVL_TA, b0 = (int64_t)blockIdx.x * OVL_TB;
  // loader: 8 threads per row, one uint4 each (a: 16 rows per pass x 8 passes, b: x 4)
  const int lr = tid >> 3, lc = tid & 7;
  int acc[4][4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][j][e] = 0;
  const int64_t W4 = W / 4;  // W % 4 == 0 (checked on the host)
  // split-K: this CTA takes words [kspan * z, kspan * (z + 1)) (kspan % OVL_KC == 0)
  const int64_t k_lo = kspan * blockIdx.z, k_hi = k_lo + kspan < W ? k_lo + kspan : W;
  for (int64_t c0 = k_lo; c0 < k_hi; c0 += OVL_KC) {
    const int64_t v = c0 / 4 + lc;
    uint4 xa[OVL_TA / 16], xb[OVL_TB / 16];
#pragma unroll
    for (int i = 0; i < OVL_TA / 16; ++i) {
      const int64_t r = a0 + lr + 16 * i;
      xa[i] = r < Ta && v < W4 ? __ldg(reinterpret_cast<const uint4*>(a + r * ld) + v) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int i = 0; i < OVL_TB / 16; ++i) {
      const int64_t r = b0 + lr + 16 * i;
      xb[i] = r < Tb && v < W4 ? __ldg(reinterpret_cast<const uint4*>(b + r * ld) + v) : make_uint4(0, 0, 0, 0);
    }
    __syncthreads();  // previous chunk consumed
#pragma unroll
    for (int i = 0; i < OVL_TA / 16; ++i) {
      uint32_t* d = As + (lr + 16 * i) * OVL_PITCH + 4 * lc;
      d[0] = xa[i].x; d[1] = xa[i].y; d[2] = xa[i].z; d[3] = xa[i].w;
    }
#pragma unroll
    for (int i = 0; i < OVL_TB / 16; ++i) {
      uint32_t* d = Bs + (lr + 16 * i) * OVL_PITCH + 4 * lc;
      d[0] = xb[i].x; d[1] = xb[i].y; d[2] = xb[i].z; d[3] = xb[i].w;
    }
    __syncthreads();
#pragma unroll 2
    for (int w = 0; w < OVL_KC; ++w) {
      uint32_t bf[4][2];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const uint32_t y = Bs[(wb + nt * 8 + g) * OVL_PITCH + w];
        bf[nt][0] = nibble_bytes(y, 4 * q);
        bf[nt][1] = nibble_bytes(y, 16 + 4 * q);
      }
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const uint32_t x0 = As[(wa + mt * 16 + g) * OVL_PITCH + w];
        const uint32_t x1 = As[(wa + mt * 16 + 8 + g) * OVL_PITCH + w];
        const uint32_t af[4] = {nibble_bytes(x0, 4 * q), nibble_bytes(x1, 4 * q), nibble_bytes(x0, 16 + 4 * q),
                                nibble_bytes(x1, 16 + 4 * q)};
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) mma_u8_16832(acc[mt][nt], af, bf[nt]);
      }
    }
  }
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t ia = a0 + wa + mt * 16 + g + 8 * h;
      if (ia >= Ta) continue;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t ib = b0 + wb + nt * 8 + 2 * q + e;
          // integer adds commute: the split-K partials land in any order, same result
          if (ib < Tb) atomicAdd(scores + ia * Tb + ib, (unsigned long long)acc[mt][nt][2 * h + e]);
        }
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
  // per-CTA counts are signed 32-bit: at most 2^25 words (2^30 bits) per split
  const int64_t gx = (Tb + sts::OVL_TB - 1) / sts::OVL_TB, gy = (Ta + sts::OVL_TA - 1) / sts::OVL_TA;
  const int64_t chunks = (W + sts::OVL_KC - 1) / sts::OVL_KC;
  int64_t ksplit = (3 * (int64_t)sts::num_sms() + gx * gy - 1) / (gx * gy);  // ~3 CTAs per SM
  const int64_t min_split = (W + (int64_t(1) << 25) - 1) >> 25;
  ksplit = ksplit < min_split ? min_split : ksplit;
  ksplit = ksplit > chunks ? chunks : ksplit;
  STS_REQUIRE(ksplit <= 65535, STS_ERR_CONTRACT, "bitsets too long (W = %lld words)", (long long)W);
  const int64_t kspan = (chunks + ksplit - 1) / ksplit * sts::OVL_KC;
  ksplit = (W + kspan - 1) / kspan;
  const dim3 grid((unsigned)gx, (unsigned)gy, (unsigned)ksplit);
  sts::bitset_overlap_kernel<<<grid, sts::OVL_THREADS, 0, static_cast<cudaStream_t>(stream)>>>(
      a_dev, Ta, b_dev, Tb, W, W, kspan, scores_dev);
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
