// Parameters shared by the gather kernels (sparse decode, draft capture) and
// the launch helpers implemented in sts_stream.cu.
#pragma once

#include "sts_common.cuh"

namespace sts {

constexpr int KEY_TILE = 16;
constexpr float LOG2E = 1.4426950408889634f;
constexpr int MODE_DECODE = 0, MODE_LSE = 1, MODE_PROBS = 2;

struct DecodeParams {
  const void* q;
  const void* k;
  const void* v;
  int64_t kv_stride;
  int64_t row_stride;  // elements between consecutive K (V) rows
  int64_t units;
  int64_t kv_div;       // units per K/V unit (prefill: query rows share their head's cache); <= 1: one each
  int M;
  int d;
  const int32_t* idx;
  int64_t idx_ld;
  const int32_t* cnt;
  int n_dense;
  const uint32_t* member;
  int causal_base;
  int rows_per_head;
  int pos_offset;
  float scale;
  void* out;      // final output (dtype of q, or fp32 when out_f32)
  int out_f32;
  float* lse;     // final lse (nullable)
  float* o_part;  // partials
  float* l_part;
  int splits;
  int32_t* status;
  // MODE_PROBS
  const float* lse_in;  // [units][M] natural-log LSE
  float* probs_out;
  int64_t out_ld;
  int probs_mode;       // 0: reduced over rows (mode S), 1: per row (mode R), 2: per-row raw logits
  int idx_cap;
  // work schedule of the bf16 kernels: 0 = auto (a thread-block cluster per
  // unit for short key streams, else persistent stream-K), 1 = stream-K,
  // 2..8 = clusters of that many CTAs per unit (sts_verify_decode.cu)
  int schedule;
  int plan_only;  // nonzero: resolve the schedule (1 or the cluster size) without launching
  // pieces[u] = (first, last) schedule range holding unit u's tiles, written
  // by the stream-K kernel, read by the piece-merge kernel
  int2* pieces;
};

// Launch of the bf16 gather kernel in `mode`.
// Workspace layout: piece table [units] int2, then partial (O, lse) slots.
size_t stream_workspace_bytes(int mode, int64_t units, int M, int d);
int stream_launch(int mode, DecodeParams& p, void* ws, size_t ws_bytes, cudaStream_t st);

int lse_merge_launch(const float* o_part, const float* lse_part, int nparts, int64_t rows, int d,
                     int out_dtype, void* out, float* lse_out, cudaStream_t st);

int auto_splits(int64_t units, int64_t keys_per_unit);

// draft-score capture on TMA + tcgen05 (sts_capture.cu): mode 0 = LSE,
// 1 = probabilities (probs_mode 0 S / 1 R / 2 raw scores)
size_t capture_workspace_bytes(int64_t units, int M);
int capture_launch(int mode, const void* q, const void* k, int64_t kv_unit_stride, int64_t units, int G, int R, int d,
                   int n_keys, int pos_offset, int base, float scale, float* lse, const float* lse_in, int probs_mode,
                   float* out, int64_t out_ld, void* ws, size_t ws_bytes, cudaStream_t st);
// bf16 decode of the stacked verification rows (sts_verify_decode.cu): the
// main kernel, then the merge of units split over several schedule ranges
int verify_decode_launch(int mode, DecodeParams& p, cudaStream_t st);

}  // namespace sts
