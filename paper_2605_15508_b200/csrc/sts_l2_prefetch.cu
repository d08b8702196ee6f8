// sts_l2_prefetch.cu — pull the first keys of every unit's selected K/V rows
// into L2 while the step's queries are still crossing the host link.
//
// attend_host (the host-buffer entry of the verify step) must copy the target
// Q over the link (~40 us for 1.3 MB at c2) before the attention can start:
// the gathered decode needs Q for its first tile. The K/V rows do not, so this
// kernel runs beside the copy and prefetches, for each unit, the rows of the
// first `keys_per_part` keys of each of the `parts` contiguous shares the
// decode's CTAs of a unit start from (clusters of `parts` CTAs split a unit's
// tiles in order). Sized to the L2, those lines are the first the attention
// reads, so they are still resident when it does. Prefetch only: no result
// depends on it.
#include "sts_common.cuh"

namespace sts {
namespace {

constexpr int PF_L2_THREADS = 256;

__global__ void __launch_bounds__(PF_L2_THREADS) kv_prefetch_l2_kernel(
    const uint8_t* __restrict__ k, const uint8_t* __restrict__ v, int64_t unit_bytes, int64_t row_bytes_stride,
    int row_bytes, const int32_t* __restrict__ idx, int64_t idx_ld, const int32_t* __restrict__ cnt, int parts,
    int keys_per_part) {
  const int64_t u = blockIdx.x;
  const int n = cnt[u];
  const int lines = (row_bytes + 127) / 128;
  const int64_t total = (int64_t)parts * keys_per_part * lines * 2;
  for (int64_t i = threadIdx.x; i < total; i += PF_L2_THREADS) {
    const int kv = (int)(i & 1);
    const int64_t rest = i >> 1;
    const int line = (int)(rest % lines);
    const int64_t kk = rest / lines;
    const int part = (int)(kk / keys_per_part);
    const int j = (int)((int64_t)part * n / parts + kk % keys_per_part);
    if (j >= (int)((int64_t)(part + 1) * n / parts)) continue;
    const int key = idx ? __ldg(idx + u * idx_ld + j) : j;
    const uint8_t* a = (kv ? v : k) + u * unit_bytes + (int64_t)key * row_bytes_stride + line * 128;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
  }
}

}  // namespace
}  // namespace sts

using namespace sts;

extern "C" int sts_kv_prefetch_l2(const void* k_cache_dev, const void* v_cache_dev, int64_t kv_unit_stride,
                                  int64_t kv_row_stride, int64_t units, int32_t d, int32_t elem_bytes,
                                  const int32_t* idx_dev, int64_t idx_ld, const int32_t* cnt_dev, int32_t parts,
                                  int32_t keys_per_part, void* stream) {
  STS_REQUIRE(units >= 0 && d >= 1 && (elem_bytes == 2 || elem_bytes == 4) && parts >= 1 && keys_per_part >= 0,
              STS_ERR_CONTRACT, "bad prefetch shape");
  if (units == 0 || keys_per_part == 0) return STS_OK;
  STS_REQUIRE(k_cache_dev && v_cache_dev && cnt_dev, STS_ERR_CONTRACT, "null buffer");
  STS_REQUIRE(units <= 0x7fffffff, STS_ERR_CONTRACT, "too many units");
  kv_prefetch_l2_kernel<<<(unsigned)units, PF_L2_THREADS, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(k_cache_dev), static_cast<const uint8_t*>(v_cache_dev), kv_unit_stride * elem_bytes,
      kv_row_stride * elem_bytes, d * elem_bytes, idx_dev, idx_ld, cnt_dev, parts, keys_per_part);
  STS_LAUNCH_CHECK();
  return STS_OK;
}
