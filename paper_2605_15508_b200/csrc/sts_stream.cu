// sts_stream.cu — workspace plan and launch glue of the persistent gather
// kernels (sts_verify_decode.cu): the per-unit piece table (first and last
// schedule range holding the unit's tiles) followed by the fp32 partial
// (O, LSE) slots, one per (CTA range, unit) pair a CTA can touch.  Nothing in
// the workspace needs zeroing between launches.
#include "sts_decode.cuh"

namespace sts {
namespace {

// largest grid any gather configuration can use (bounds the partial slots)
int max_grid() { return num_sms() * 16; }

size_t pieces_bytes(int64_t units) { return ((size_t)units * 8 + 255) & ~size_t(255); }

}  // namespace

size_t stream_workspace_bytes(int mode, int64_t units, int M, int d) {
  if (mode == MODE_PROBS) return 0;
  const int64_t slots = (int64_t)max_grid() + units;
  const size_t per_slot = (size_t)M * ((mode == MODE_DECODE ? d : 0) + 1) * sizeof(float);
  return pieces_bytes(units) + (size_t)slots * per_slot + 256;
}

int stream_launch(int mode, DecodeParams& p, void* ws, size_t ws_bytes, cudaStream_t st) {
  // the gather kernels address rows with 32-bit byte offsets inside a unit
  STS_REQUIRE(p.kv_stride >= 0 && p.kv_stride * 2 <= (int64_t(1) << 32) &&
                  (int64_t)p.n_dense * p.row_stride * 2 <= (int64_t(1) << 32),
              STS_ERR_CONTRACT, "one (batch, layer, head) unit of the cache must span < 4 GiB");
  if (mode != MODE_PROBS) {
    const size_t need = stream_workspace_bytes(mode, p.units, p.M, p.d);
    STS_REQUIRE(ws && ws_bytes >= need, STS_ERR_CONTRACT, "gather workspace too small: need %zu, got %zu", need,
                ws_bytes);
    uint8_t* base = static_cast<uint8_t*>(ws);
    const int64_t slots = (int64_t)max_grid() + p.units;
    p.pieces = reinterpret_cast<int2*>(base);
    p.l_part = reinterpret_cast<float*>(base + pieces_bytes(p.units));
    p.o_part = p.l_part + slots * p.M;
    // float4 merge loads need 16-byte aligned slots
    p.o_part = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(p.o_part) + 15) & ~uintptr_t(15));
  } else {
    p.pieces = nullptr;
  }
  return verify_decode_launch(mode, p, st);
}

}  // namespace sts
