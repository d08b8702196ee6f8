// sts_block_f64.cu — reference-exact masked block attention with attention /
// score recording: the per-head body of the reference's toy-model forward
// (src/toymodel.py:315-352, `_run_block`), used by the model-level drop-in
// (forward_prefill / forward_decode / forward_block, paper_2605_15508_b200/
// model.py) so that recorded draft rows, selected masks and greedy tokens are
// the reference's own.
//
// Math in fp64 exactly as the reference states it: s = (q . k) * inv_sqrt_d
// over the causal prefix, allowed set = the row's mask (or the causal prefix),
// w = exp(s - max) zeroed outside the set, w /= sum, out = w @ V cast to fp32;
// recordings are w (fp32, zeros outside the set) and the raw causal scores
// (fp32, dense even for masked heads, zeros beyond the row's position).
//
// One CTA per (head, query row); the row's scores live in shared memory
// (fp64, n_end entries).  This is the parity path of the drop-in, not the
// bandwidth path (that is the bf16 gather kernel of sts_verify_decode.cu).
#include "sts_common.cuh"

namespace sts {
namespace {

constexpr int BF_THREADS = 256;

__device__ __forceinline__ double block_reduce(double v, double* red, bool is_max) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double x = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmax(v, x) : v + x;
  }
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double r = red[0];
  for (int w = 1; w < BF_THREADS / 32; ++w) r = is_max ? fmax(r, red[w]) : r + red[w];
  return r;
}

struct BlockF64Params {
  const float* q;
  const float* k;
  const float* v;
  int64_t kv_head_stride;
  int64_t kv_row_stride;
  int heads, m, d, start_pos;
  double scale;
  const int32_t* idx;
  int64_t idx_ld;
  const int32_t* cnt;
  const int32_t* list_of_row;
  int flags;
  float* out;
  int64_t out_ld;
  float* probs;
  float* scores;
  int64_t rec_ld;
  int32_t* status;
};

__global__ void __launch_bounds__(BF_THREADS) block_attention_f64_kernel(BlockF64Params p) {
  extern __shared__ double smem[];
  const int hr = blockIdx.x;
  const int h = hr / p.m, r = hr % p.m;
  const int pos = p.start_pos + r;
  const int n_end = p.start_pos + p.m;
  const int D = p.d;
  double* w = smem;                  // [n_end]
  double* qs = smem + n_end;         // [D]
  double* red = qs + D;              // [BF_THREADS / 32]
  double* part = red + BF_THREADS / 32;  // [slices][D]
  const float* kg = p.k + (int64_t)h * p.kv_head_stride;
  const float* vg = p.v + (int64_t)h * p.kv_head_stride;
  const float* qg = p.q + ((int64_t)h * p.m + r) * D;
  for (int e = threadIdx.x; e < D; e += BF_THREADS) qs[e] = (double)qg[e];
  for (int j = threadIdx.x; j < n_end; j += BF_THREADS) w[j] = -INFINITY;
  __syncthreads();

  const int list = p.list_of_row ? p.list_of_row[hr] : (p.idx ? hr : -1);
  auto score = [&](int j) {
    const float* kr = kg + (int64_t)j * p.kv_row_stride;
    double acc = 0.0;
    for (int e = 0; e < D; ++e) acc = fma(qs[e], (double)kr[e], acc);
    return acc * p.scale;
  };
  float* srow = p.scores ? p.scores + (int64_t)hr * p.rec_ld : nullptr;
  if (list < 0 || srow) {
    for (int j = threadIdx.x; j < n_end; j += BF_THREADS) {
      const double s = j <= pos ? score(j) : 0.0;
      if (srow) srow[j] = (float)s;
      if (list < 0 && j <= pos) w[j] = s;
    }
  }
  __syncthreads();
  if (list >= 0) {
    const int c = p.cnt[list];
    const int32_t* il = p.idx + (int64_t)list * p.idx_ld;
    if (c <= 0 && threadIdx.x == 0) set_status(p.status, STS_DEV_EMPTY_ROW);
    for (int t = threadIdx.x; t < c; t += BF_THREADS) {
      const int j = il[t];
      if (j < 0 || j > pos) {
        set_status(p.status, STS_DEV_BAD_INDEX);
        continue;
      }
      w[j] = score(j);
    }
    // rows always see their own position (forward_decode's mask ∪ {current},
    // specdec._clamp_current): src/toymodel.py:467-475, src/specdec.py:212-216
    if ((p.flags & STS_BLOCK_INCLUDE_SELF) && threadIdx.x == 0) w[pos] = score(pos);
  }
  __syncthreads();

  double mx = -INFINITY;
  for (int j = threadIdx.x; j < n_end; j += BF_THREADS) mx = fmax(mx, w[j]);
  mx = block_reduce(mx, red, true);
  double sum = 0.0;
  if (mx != -INFINITY) {
    for (int j = threadIdx.x; j < n_end; j += BF_THREADS) {
      const double e = w[j] == -INFINITY ? 0.0 : exp(w[j] - mx);
      w[j] = e;
      sum += e;
    }
  } else {
    for (int j = threadIdx.x; j < n_end; j += BF_THREADS) w[j] = 0.0;
  }
  sum = block_reduce(sum, red, false);
  float* prow = p.probs ? p.probs + (int64_t)hr * p.rec_ld : nullptr;
  for (int j = threadIdx.x; j < n_end; j += BF_THREADS) {
    w[j] = sum > 0.0 ? w[j] / sum : 0.0;  // the reference divides: w /= w.sum()
    if (prow) prow[j] = (float)w[j];
  }
  __syncthreads();

  // out[e] = sum_j w[j] * V[j][e]: the CTA splits into BF_THREADS / D key slices of D lanes
  const int slices = BF_THREADS / D;
  const int sl = threadIdx.x / D, e = threadIdx.x % D;
  if (sl < slices) {
    double acc = 0.0;
    for (int j = sl; j <= pos; j += slices) {
      const double wj = w[j];
      if (wj != 0.0) acc = fma(wj, (double)vg[(int64_t)j * p.kv_row_stride + e], acc);
    }
    part[sl * D + e] = acc;
  }
  __syncthreads();
  if (threadIdx.x < D) {
    double t = 0.0;
    for (int s2 = 0; s2 < slices; ++s2) t += part[s2 * D + threadIdx.x];
    p.out[(int64_t)r * p.out_ld + (int64_t)h * D + threadIdx.x] = (float)t;
  }
  if (threadIdx.x == 0 && !(sum > 0.0)) set_status(p.status, STS_DEV_EMPTY_ROW);
}

}  // namespace
}  // namespace sts

using namespace sts;

extern "C" int sts_block_attention_f64(const float* q_dev, const float* k_cache_dev, const float* v_cache_dev,
                                       int64_t kv_head_stride, int64_t kv_row_stride, int32_t heads, int32_t m,
                                       int32_t d, int32_t start_pos, double scale, const int32_t* idx_dev,
                                       int64_t idx_ld, const int32_t* cnt_dev, const int32_t* list_of_row_dev,
                                       int32_t flags, float* out_dev, int64_t out_ld, float* probs_dev, float* scores_dev,
                                       int64_t rec_ld, int32_t* status_dev, void* stream) {
  STS_REQUIRE(heads >= 0 && m >= 0 && d >= 1 && d <= BF_THREADS && start_pos >= 0, STS_ERR_CONTRACT,
              "bad block shape (head_dim must be in [1, %d])", BF_THREADS);
  if (heads == 0 || m == 0) return STS_OK;
  STS_REQUIRE(q_dev && k_cache_dev && v_cache_dev && out_dev, STS_ERR_CONTRACT, "null buffer");
  STS_REQUIRE(!idx_dev || cnt_dev, STS_ERR_CONTRACT, "index lists need counts");
  STS_REQUIRE(!list_of_row_dev || idx_dev, STS_ERR_CONTRACT, "list_of_row needs index lists");
  STS_REQUIRE(kv_row_stride >= d, STS_ERR_CONTRACT, "kv_row_stride must be >= d");
  STS_REQUIRE(out_ld >= (int64_t)heads * d, STS_ERR_CONTRACT, "out_ld must be >= heads * d");
  const int64_t n_end = (int64_t)start_pos + m;
  STS_REQUIRE(!(probs_dev || scores_dev) || rec_ld >= n_end, STS_ERR_CONTRACT, "rec_ld must be >= start_pos + m");
  STS_REQUIRE((int64_t)heads * m <= 0x7fffffffLL, STS_ERR_CONTRACT, "too many (head, row) pairs");
  const size_t smem = ((size_t)n_end + d + BF_THREADS / 32 + (size_t)(BF_THREADS / d) * d) * sizeof(double);
  STS_REQUIRE(smem <= 227 * 1024, STS_ERR_CONTRACT,
              "reference-exact block attention keeps a row's fp64 scores in shared memory: n = %lld too long",
              (long long)n_end);
  STS_CUDA_CHECK(cudaFuncSetAttribute(block_attention_f64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      227 * 1024));
  BlockF64Params p;
  p.q = q_dev;
  p.k = k_cache_dev;
  p.v = v_cache_dev;
  p.kv_head_stride = kv_head_stride;
  p.kv_row_stride = kv_row_stride;
  p.heads = heads;
  p.m = m;
  p.d = d;
  p.start_pos = start_pos;
  p.scale = scale;
  p.idx = idx_dev;
  p.idx_ld = idx_ld;
  p.cnt = cnt_dev;
  p.list_of_row = list_of_row_dev;
  p.flags = flags;
  p.out = out_dev;
  p.out_ld = out_ld;
  p.probs = probs_dev;
  p.scores = scores_dev;
  p.rec_ld = rec_ld;
  p.status = status_dev;
  block_attention_f64_kernel<<<(unsigned)(heads * m), BF_THREADS, smem, static_cast<cudaStream_t>(stream)>>>(p);
  STS_LAUNCH_CHECK();
  return STS_OK;
}
