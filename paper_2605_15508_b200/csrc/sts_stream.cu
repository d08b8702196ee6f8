// sts_stream.cu — workspace plan and launch glue of the persistent stream-K
// gather kernels (sts_gather.cu): per-unit arrival counters (zeroed per
// launch) followed by the fp32 partial (O, LSE) slots, one per (CTA, unit)
// pair a CTA can touch.
#include <stdlib.h>

#include "sts_decode.cuh"

namespace sts {
namespace {


// largest grid any gather configuration can use (bounds the partial slots)
int max_grid() { return num_sms() * 16; }
// dynamic chunks per launch (their partial slots follow the static ones)
int nch_max() { return num_sms() * 8; }

constexpr size_t SCHED_BYTES = 256;

size_t counters_bytes(int64_t units) { return (((size_t)units * 4 + 255) & ~size_t(255)) + SCHED_BYTES; }

// dynamic share of the tiles (STS_DYN_FRAC; default 0 = fully static: the
// measured c2 / c4 optimum so far) and minimum chunk
float dyn_frac() {
  static float f = -1.f;
  if (f < 0.f) {
    const char* e = getenv("STS_DYN_FRAC");
    f = e ? (float)atof(e) : 0.f;
    if (f < 0.f || f > 1.f) f = 0.f;
  }
  return f;
}
int dyn_chunk() {
  static int c = -1;
  if (c < 0) {
    const char* e = getenv("STS_DYN_CHUNK");
    c = e ? atoi(e) : 6;
    if (c < 1) c = 6;
  }
  return c;
}

}  // namespace

size_t stream_workspace_bytes(int mode, int64_t units, int M, int d) {
  if (mode == MODE_PROBS) return 0;
  const int64_t slots = (int64_t)max_grid() + nch_max() + units;
  const size_t pieces = ((size_t)units * 8 + 255) & ~size_t(255);
  const size_t per_slot = (size_t)M * ((mode == MODE_DECODE ? d : 0) + 1) * sizeof(float);
  return counters_bytes(units) + pieces + (size_t)slots * per_slot + 256;
}

int stream_launch(int mode, DecodeParams& p, void* ws, size_t ws_bytes, cudaStream_t st) {
  // the gather kernels address rows with 32-bit byte offsets inside a unit
  STS_REQUIRE(p.kv_stride >= 0 && p.kv_stride * 2 <= (int64_t(1) << 32) &&
                  (int64_t)p.n_dense * p.row_stride * 2 <= (int64_t(1) << 32),
              STS_ERR_CONTRACT, "one (batch, layer, head) unit of the cache must span < 4 GiB");
  const size_t need = stream_workspace_bytes(mode, p.units, p.M, p.d);
  if (mode != MODE_PROBS) {
    STS_REQUIRE(ws && ws_bytes >= need, STS_ERR_CONTRACT, "gather workspace too small: need %zu, got %zu", need,
                ws_bytes);
    uint8_t* base = static_cast<uint8_t*>(ws);
    const size_t cbytes = counters_bytes(p.units);
    const size_t pieces = ((size_t)p.units * 8 + 255) & ~size_t(255);
    p.counters = reinterpret_cast<int*>(base);
    p.sched = reinterpret_cast<int*>(base + cbytes - SCHED_BYTES);
    p.pieces = reinterpret_cast<int2*>(base + cbytes);
    p.nch_max = nch_max();
    p.dyn_chunk = dyn_chunk();
    p.dyn_frac = dyn_frac();
    p.pref_units = p.units <= VERIFY_PREF_MAX_UNITS ? (int)p.units : 0;
    const int64_t slots = (int64_t)max_grid() + nch_max() + p.units;
    p.l_part = reinterpret_cast<float*>(base + cbytes + pieces);
    p.o_part = p.l_part + slots * p.M;
    // float4 merge loads need 16-byte aligned slots
    p.o_part = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(p.o_part) + 15) & ~uintptr_t(15));
    STS_CUDA_CHECK(cudaMemsetAsync(p.counters, 0, cbytes, st));
  } else {
    p.sched = nullptr;
    p.pieces = nullptr;
    p.pref_units = 0;
    p.dyn_frac = 0.f;
  }
  return gather_launch(mode, p, st);
}

}  // namespace sts
