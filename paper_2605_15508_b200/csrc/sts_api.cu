// sts_api.cu — host-side pieces of the C-ABI: thread-local error message,
// ABI version, SM count cache.
#include <atomic>

#include "sts_common.cuh"

namespace sts {

static thread_local char g_last_error[512] = "";
static std::atomic<unsigned long long> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

int num_sms() {
  static int cached = 0;
  if (cached == 0) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0)
      cached = n;
    else
      return 148;  // B200 default when no device is visible
  }
  return cached;
}

}  // namespace sts

extern "C" const char* sts_last_error(void) { return sts::g_last_error; }

extern "C" int sts_abi_version(void) { return STS_ABI_VERSION; }

extern "C" unsigned long long sts_launch_count(void) { return sts::g_launches.load(std::memory_order_relaxed); }
