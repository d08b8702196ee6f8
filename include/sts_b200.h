/*
 * sts_b200.h — C-ABI of the B200-native STS (Speculative Token Sparsity)
 * sparse-attention hot path.  libsts_b200.so exports exactly these symbols.
 *
 * Conventions
 *   - Every pointer argument named *_dev / listed as "device" is a CUDA device
 *     pointer; every function is asynchronous on the given cudaStream_t
 *     (passed as void* so this header needs no CUDA include).
 *   - No function throws.  Return value: 0 ok, 1 input/config error
 *     (reference ConfigError/InputError, src/errors.py:15,27), 2 contract
 *     violation (reference ContractViolation, src/errors.py:19), 3 CUDA error.
 *     The message of the last failure on the calling thread is returned by
 *     sts_last_error().
 *   - Re-entrant per stream; no global mutable device state; the caller owns
 *     every buffer (outputs and workspace are caller-allocated, so nothing is
 *     allocated on the hot path).
 *
 * The reference (pkg/src/specsparse, pure numpy) has no FFI.  Each entry point
 * below replaces the reference Python function(s) named in its comment; the
 * Python host package paper_2605_15508_b200 re-exports the reference names on
 * top of these (see INTEGRATION.md for the ctypes binding).
 */
#ifndef STS_B200_H
#define STS_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define STS_API __attribute__((visibility("default")))
#else
#define STS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define STS_ABI_VERSION 8

#define STS_OK 0
#define STS_ERR_INPUT 1
#define STS_ERR_CONTRACT 2
#define STS_ERR_CUDA 3

#define STS_DTYPE_F32 0
#define STS_DTYPE_BF16 1

/* selection extras (SparsityConfig.include_current / include_sink,
 * src/sparsity.py:46-47) */
#define STS_SEL_CURRENT 0x1u
#define STS_SEL_SINK 0x2u

/* device status word bits (written by kernels into *status_dev, never cleared
 * by them; the host reads it after a sync when validation is wanted) */
#define STS_DEV_IDX_CAPACITY 0x1 /* an index list exceeded idx_ld           */
#define STS_DEV_EMPTY_ROW 0x2    /* a query row had no admissible key       */
#define STS_DEV_BAD_INDEX 0x4    /* an index was outside the cached context */
#define STS_DEV_SELECT_INCONSISTENT 0x8 /* sharded select: the global histogram did not
                                           resolve a row (ranks disagree on k / shards) */

STS_API const char* sts_last_error(void);
STS_API int sts_abi_version(void);
/* kernels this process has launched through the library (a CUDA graph
 * replay re-runs the kernels captured once, without passing here) */
STS_API unsigned long long sts_launch_count(void);

/* ------------------------------------------------------------------------
 * sts_select_topk — sparsity-mask construction.
 * Replaces sparsity._select_row / draft_masks_decode / draft_masks_prefill
 * (src/sparsity.py:86-130), numkit.topk_indices (src/numkit.py:74-86),
 * sparsity.page_aggregate (src/sparsity.py:72-83) and, through row_src, the
 * head remap of remap_masks (src/sparsity.py:133-149) and the mode-S
 * reduction.
 *
 * Logical row r in [0, rows):
 *   n_r   = row_len_dev ? row_len_dev[r] : n_common           (positions)
 *   v_r[j]= fp32 sum, in s order, of scores[src(r,s)*ld + j], s < nsrc,
 *           src(r,s) = row_src_dev ? row_src_dev[r*nsrc+s] : r (nsrc==1)
 *   b_r   = budget_is_fraction ? max(1, ceil(budget*n_r)) : (int)budget
 *   out   = sorted unique indices: dense [0,n_r) if b_r >= n_r, else the
 *           top-b_r tokens (page_size==1) or the tokens of the top
 *           ceil(b_r/page_size) pages by fp64 page sum in numpy reduceat
 *           order; plus extras (n_r-1 if CURRENT, 0 if SINK, the last
 *           recent_window positions); then the tail n_r .. n_r+tail_len-1.
 *   Ranking: score descending, ties to the lower index, -0.0 == +0.0, NaN
 *   below everything (identical to the stable argsort of src/numkit.py:84).
 * idx_out_dev[r*idx_ld + i], i < cnt_out_dev[r]: int32 ascending.
 * ---------------------------------------------------------------------- */
STS_API size_t sts_select_workspace_bytes(int64_t rows, int32_t max_len, int32_t page_size);
STS_API int sts_select_topk(const float* scores_dev, int64_t ld, const int32_t* row_src_dev,
                    int32_t nsrc, int64_t rows, const int32_t* row_len_dev,
                    int32_t n_common, double budget, int32_t budget_is_fraction,
                    int32_t page_size, uint32_t flags, int32_t recent_window,
                    int32_t tail_len, int32_t* idx_out_dev, int64_t idx_ld,
                    int32_t* cnt_out_dev, int32_t* status_dev, void* workspace_dev,
                    size_t workspace_bytes, void* stream);

/* sts_page_aggregate — page scores alone (src/sparsity.py:72-83): out[r][pg]
 * = fp64 sum of row r's tokens [pg*ps, min((pg+1)*ps, n_r)) in numpy
 * add.reduceat order (x0 + pairwise(rest)); page_size 1 is the identity. */
STS_API int sts_page_aggregate(const float* scores_dev, int64_t ld, int64_t rows, const int32_t* row_len_dev,
                       int32_t n_common, int32_t page_size, double* out_dev, int64_t out_ld,
                       void* stream);

/* ------------------------------------------------------------------------
 * sts_sparse_decode — gathered-KV sparse flash-decode of the gamma+1
 * verification rows stacked with their GQA group (M = group*rows_per_head).
 * Replaces the masked attention loop of toymodel._run_block
 * (src/toymodel.py:315-348, rows via forward_block :430-455) and
 * sparsity.sparse_attention (src/sparsity.py:152-173).
 *
 * unit u (e.g. (batch, layer, kv-head)): K/V rows at k_cache + u*kv_unit_stride
 *   (elements); row p of d contiguous elements starts kv_row_stride elements
 *   after row p-1 (0 => d).  kv_row_stride = 2d with v = k + d is the
 *   interleaved K|V token layout (one 4d-byte run per gathered bf16 token).
 *   Queries q[u][M][d].
 *   keys: idx_dev[u*idx_ld + j], j < cnt_dev[u]  (idx_dev NULL => dense
 *   0..n_dense-1).  Row r attends key p iff
 *     (causal_base < 0 || pos_offset + p - causal_base <= r % rows_per_head)
 *     && (member_dev == NULL || bit r of member_dev[u*idx_ld + j]).
 *   out[u][M][d] (out_dtype: dtype, or F32 for partials that a later
 *   sts_lse_merge combines, e.g. per-rank results of the sharded path)
 *   = softmax_S(q.k*scale) V ; lse_dev[u][M] = natural
 *   log-sum-exp of the scaled scores (nullable).  dtype F32 computes in fp32
 *   on CUDA cores (parity path); BF16 uses tensor cores with fp32 accumulate.
 *   splits: F32 -> split-K factor (>= 1, partials merged by sts_lse_merge);
 *   BF16 -> work schedule: 0 auto (one thread-block cluster per unit when
 *   the key streams are short, else persistent stream-K), 1 stream-K,
 *   2/3/4/6/8 clusters of exactly that many CTAs per unit (DSMEM merge).
 * ---------------------------------------------------------------------- */
STS_API size_t sts_sparse_decode_workspace_bytes(int64_t units, int32_t M, int32_t d, int32_t splits);
/* split-K factor that fills 148 SMs x 2 CTAs in whole waves (>= 8 key tiles
 * of 16 per CTA); what the host uses when it has no better knowledge. */
STS_API int32_t sts_auto_splits(int64_t units, int64_t keys_per_unit);
/* the BF16 work schedule sts_sparse_decode resolves for `schedule` (0 = auto)
 * with these sizes: 1 = stream-K, C >= 2 = clusters of C CTAs; 0 if the shape
 * is unsupported.  Launches nothing. */
STS_API int32_t sts_sparse_decode_schedule(int64_t units, int32_t M, int32_t d, int64_t keys_per_unit,
                                           int32_t schedule);
STS_API int sts_sparse_decode(int32_t dtype, int32_t out_dtype, const void* q_dev, const void* k_cache_dev,
                      const void* v_cache_dev, int64_t kv_unit_stride, int64_t kv_row_stride, int64_t units,
                      int32_t M, int32_t d, const int32_t* idx_dev, int64_t idx_ld,
                      const int32_t* cnt_dev, int32_t n_dense, const uint32_t* member_dev,
                      int32_t causal_base, int32_t rows_per_head, int32_t pos_offset,
                      float scale, void* out_dev, float* lse_dev, int32_t splits,
                      int32_t* status_dev, void* workspace_dev, size_t workspace_bytes,
                      void* stream);

/* ------------------------------------------------------------------------
 * sts_sparse_prefill — sparse prefill attention (STS-PD):
 * every query row has its own key list.  Replaces the masked prefill of
 * toymodel._run_block (src/toymodel.py:315-348 reached through
 * forward_prefill(masks=...) :370-399, masks from draft_masks_prefill
 * src/sparsity.py:122-130) and a per-row loop of sparse_attention.
 * Unit (g, t) = g*rows + t: queries q[(g*rows+t)][M][d] (M = the heads that
 * share g's K/V and the mask, 1 for MHA), keys idx_dev[(g*rows+t)*idx_ld + j],
 * j < cnt_dev[g*rows+t], positions into K/V block g (k_cache + g*kv_unit_stride);
 * every listed key is attended (lists are causal by construction).
 * out[(g*rows+t)][M][d] (out_dtype), lse (nullable).  Workspace:
 * sts_sparse_decode_workspace_bytes(kv_units*rows, M, d, 1).
 * ---------------------------------------------------------------------- */
STS_API int sts_sparse_prefill(int32_t dtype, int32_t out_dtype, const void* q_dev, const void* k_cache_dev,
                               const void* v_cache_dev, int64_t kv_unit_stride, int64_t kv_row_stride,
                               int64_t kv_units, int32_t rows, int32_t M, int32_t d, const int32_t* idx_dev,
                               int64_t idx_ld, const int32_t* cnt_dev, float scale, void* out_dev, float* lse_dev,
                               int32_t* status_dev, void* workspace_dev, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------
 * sts_draft_scores — draft-score capture (ForwardRecord.attention of the
 * draft's decode, src/toymodel.py:349-350 via specdec.propose
 * src/specdec.py:150-167), computed for the R speculative rows at once.
 *
 * unit u = (draft layer, draft kv-head); q[u][G*R][d] with row index
 * hh*R + i (hh = q-head within the GQA group, i = speculative row); row i sits
 * at global position base+i and sees keys with global position <= base+i.
 * The unit's n_keys K rows hold global positions pos_offset .. .
 *   lse_dev[u][G*R]: natural log-sum-exp of the scaled scores over the local
 *                    keys (sts_draft_lse), or the global one (input to
 *                    sts_draft_probs when the KV is sequence-sharded).
 *   mode 0 (S): out[u][hh][j] = sum_i p_{hh,i}[j], fp32, i ascending, for
 *               local j with global position < base (committed prefix).
 *   mode 1 (R): out[(u*G+hh)*R + i][j] = p_{hh,i}[j] for pos <= base+i.
 *   (row stride out_ld floats)
 * ---------------------------------------------------------------------- */
STS_API size_t sts_draft_workspace_bytes(int64_t units, int32_t GR, int32_t n_keys);
STS_API int sts_draft_lse(int32_t dtype, const void* q_dev, const void* k_cache_dev,
                  int64_t kv_unit_stride, int64_t units, int32_t G, int32_t R, int32_t d,
                  int32_t n_keys, int32_t pos_offset, int32_t base, float scale,
                  float* lse_dev, void* workspace_dev, size_t workspace_bytes, void* stream);
STS_API int sts_draft_probs(int32_t dtype, const void* q_dev, const void* k_cache_dev,
                    int64_t kv_unit_stride, int64_t units, int32_t G, int32_t R, int32_t d,
                    int32_t n_keys, int32_t pos_offset, int32_t base, float scale,
                    const float* lse_dev, int32_t mode, float* out_dev, int64_t out_ld,
                    void* stream);
/* Raw pre-softmax scores (ForwardRecord.scores / record_scores,
 * src/toymodel.py:225-240, :351-352): out[(u*G+hh)*R + i][j] = scale * q.k_j
 * (fp32, natural units) for local j with global position <= base+i; other
 * entries are left untouched.  Same geometry as sts_draft_probs mode 1. */
STS_API int sts_draft_scores(int32_t dtype, const void* q_dev, const void* k_cache_dev,
                     int64_t kv_unit_stride, int64_t units, int32_t G, int32_t R, int32_t d,
                     int32_t n_keys, int32_t pos_offset, int32_t base, float scale,
                     float* out_dev, int64_t out_ld, void* stream);

/* ------------------------------------------------------------------------
 * sts_lse_merge — merge P partial attention results (split-K or
 * sequence shards): LSE = log sum_p exp(LSE_p), O = sum_p exp(LSE_p-LSE) O_p.
 * o_part[p][rows][d] fp32 (nullable => only the LSE), lse_part[p][rows].
 * out dtype F32 or BF16 [rows][d] (nullable), lse_out[rows] (nullable).
 * ---------------------------------------------------------------------- */
STS_API int sts_lse_merge(const float* o_part_dev, const float* lse_part_dev, int32_t nparts,
                  int64_t rows, int32_t d, int32_t out_dtype, void* out_dev,
                  float* lse_out_dev, void* stream);

/* sts_lse_merge_ptrs — the same merge with part q read at part_ptrs_dev[q]
 * (a device array of nparts float pointers, e.g. every rank's symmetric-memory
 * buffer mapped over NVLink): O_q at ptr + o_offset ([rows][d] floats), LSE_q
 * at ptr + l_offset ([rows]).  One kernel = all-gather + merge over peer
 * memory; results identical to sts_lse_merge on the same parts. */
STS_API int sts_lse_merge_ptrs(const void* part_ptrs_dev, int32_t nparts, int64_t rows, int32_t d,
                               int64_t o_offset, int64_t l_offset, int32_t out_dtype, void* out_dev,
                               float* lse_out_dev, void* stream);

/* ------------------------------------------------------------------------
 * sts_row_union — mode R (reference-exact per-row masks) under GQA: build,
 * for each unit, the sorted union of the M per-row index lists together with
 * a membership bit per (row, key) for sts_sparse_decode.
 * lists: row m of unit u is list src_dev[u*M+m] of a selection output
 * (idx_in_dev[list*in_ld + i], i < cnt_in_dev[list]) — the src table is the
 * remap of remap_masks (src/sparsity.py:141).  M <= 32.
 * bitmap_ws: units*n_max uint32 scratch (zeroed by this call).
 * ---------------------------------------------------------------------- */
STS_API int sts_row_union(const int32_t* idx_in_dev, int64_t in_ld, const int32_t* cnt_in_dev,
                  const int32_t* src_dev, int64_t units, int32_t M, int32_t n_max,
                  uint32_t* bitmap_ws_dev, int32_t* idx_out_dev, uint32_t* member_out_dev,
                  int64_t out_ld, int32_t* cnt_out_dev, int32_t* status_dev, void* stream);

/* ------------------------------------------------------------------------
 * Algorithm 1 (offline head mapping): replaces the bitmask
 * overlap of headmap.find_head_mapping (src/headmap.py:76-125).
 * sts_topk_bitsets: row r's index list (idx_dev[r*idx_ld + j], j < cnt_dev[r])
 *   -> bits_out[r][words] (bit i set iff i listed; zeroed first).
 * sts_bitset_overlap: scores[ia][ib] += sum_w popc(a[ia][w] & b[ib][w]) over
 *   W words per head (16-byte aligned, W % 4 == 0), uint64, deterministic.
 * ---------------------------------------------------------------------- */
STS_API int sts_topk_bitsets(const int32_t* idx_dev, int64_t idx_ld, const int32_t* cnt_dev, int64_t rows,
                             int32_t words, uint32_t* bits_out_dev, void* stream);
STS_API int sts_bitset_overlap(const uint32_t* a_dev, int32_t Ta, const uint32_t* b_dev, int32_t Tb, int64_t W,
                               unsigned long long* scores_dev, void* stream);

#define STS_BLOCK_INCLUDE_SELF 0x1

/* ------------------------------------------------------------------------
 * sts_block_attention_f64 — reference-exact masked block attention with
 * attention / score recording: the per-head loop of toymodel._run_block
 * (src/toymodel.py:315-352) for every head of one layer in one launch, math
 * in fp64 as the reference states it.  Replaces the attention of
 * forward_prefill / forward_decode / forward_block (:359-455) with
 * record_attention / record_scores (ForwardRecord.attention / .scores,
 * :226-240), used by the model-level drop-in (model.py, specdec.py).
 *   q_dev      fp32 [heads][m][d]: rows r at global position start_pos + r
 *   k/v_cache  fp32, head h row j at h*kv_head_stride + j*kv_row_stride
 *   idx/cnt    optional per-row key lists (ascending, <= the row's position);
 *              row (h, r) uses list list_of_row[h*m + r] (-1: dense causal),
 *              or list h*m + r when list_of_row is NULL; idx NULL: all dense
 *   flags      STS_BLOCK_INCLUDE_SELF: a listed row also attends its own
 *              position (the decode mask ∪ {current} of src/toymodel.py:467-475
 *              and specdec._clamp_current, src/specdec.py:212-216)
 *   out_dev    fp32 [m][out_ld], head h at columns [h*d, (h+1)*d)
 *   probs_dev  nullable fp32 [heads*m][rec_ld]: the row's softmax weights over
 *              [0, start_pos+m) (zero outside its allowed set)
 *   scores_dev nullable fp32 [heads*m][rec_ld]: raw q.k*scale over the causal
 *              prefix, zero beyond the row's position (dense for masked rows)
 * Limits: d <= 256, start_pos + m <= ~28K (a row's fp64 scores in shared
 * memory).  Device status bits: STS_DEV_BAD_INDEX for list entries outside
 * [0, position], STS_DEV_EMPTY_ROW for an empty list.
 * ---------------------------------------------------------------------- */
STS_API int sts_block_attention_f64(const float* q_dev, const float* k_cache_dev, const float* v_cache_dev,
                                    int64_t kv_head_stride, int64_t kv_row_stride, int32_t heads, int32_t m,
                                    int32_t d, int32_t start_pos, double scale, const int32_t* idx_dev,
                                    int64_t idx_ld, const int32_t* cnt_dev, const int32_t* list_of_row_dev,
                                    int32_t flags, float* out_dev, int64_t out_ld, float* probs_dev, float* scores_dev,
                                    int64_t rec_ld, int32_t* status_dev, void* stream);

/* ------------------------------------------------------------------------
 * Mask-driven KV prefetch into an HBM page pool: the
 * strategies of src/offloadsim.py:153-211 ("on_demand" / "prefetch" with
 * lookahead), pages as in src/specdec.py:236-255 (page = position / P).
 *
 * sts_page_plan — per unit, the ascending unique pages of its key list
 *   (pages_dev[u][0 .. npages_dev[u]), at most pages_ld; overflow sets
 *   STS_DEV_IDX_CAPACITY) and the list re-expressed as rows of the unit's
 *   pool slice: idx_pool[u][i] = rank(page(idx[u][i])) * P + idx[u][i] % P.
 *   Pages >= tail_page0 (the in-block tail; -1: none) take the fixed ranks
 *   tail_rank0 + (page - tail_page0) in every unit, so pool rows of the tail
 *   are position - (tail_page0 - tail_rank0) * P for all units and the
 *   decode's causal test runs with causal_base' = base - that shift.
 * sts_page_copy — copies the planned pages of units [unit_begin, unit_end)
 *   from K/V in pinned, device-mapped host memory ([unit][row][d], strides in
 *   elements) into the pool ([unit][pages_ld * P][d]), with `ctas` CTAs (one
 *   warp per page, 16-byte loads over the host link) so it runs beside the
 *   attention of units already resident.  slots_dev (NULL: page w of a
 *   unit's list goes to pool rank w) gives each listed page its pool slot.
 * sts_page_cache_plan — the "prefetch" strategy's residency across steps
 *   (src/offloadsim.py:173-209, per unit with a capacity of `slots` pages):
 *   slot_page / slot_last ([units][slots_ld], persistent, -1 = empty) hold
 *   each pool slot's page and the step that last used it.  The step's
 *   committed pages already resident keep their slots; the missing ones
 *   (ascending) are listed in copy_pages / copy_slots (ncopy per unit) and
 *   take free slots in the reference's LRU eviction order (empty first,
 *   then by (last use, page)); the key list is re-expressed in pool rows as
 *   in sts_page_plan (tail pages at fixed ranks >= tail_rank0 >= slots).
 *   A step needing more than `slots` committed pages sets
 *   STS_DEV_IDX_CAPACITY.
 * ---------------------------------------------------------------------- */
STS_API int sts_page_plan(const int32_t* idx_dev, int64_t idx_ld, const int32_t* cnt_dev, int64_t units,
                          int32_t page_size, int32_t tail_page0, int32_t tail_rank0, int32_t* pages_dev,
                          int64_t pages_ld, int32_t* npages_dev, int32_t* idx_pool_dev, int32_t* status_dev,
                          void* stream);
STS_API int sts_page_copy(const void* host_k, const void* host_v, int64_t host_unit_stride,
                          int64_t host_row_stride, int32_t n_rows_host, void* pool_k, void* pool_v,
                          int64_t pool_unit_stride, int32_t d, int32_t elem_bytes, const int32_t* pages_dev,
                          int64_t pages_ld, const int32_t* npages_dev, const int32_t* slots_dev,
                          int64_t unit_begin, int64_t unit_end, int32_t page_size, int32_t tail_page0,
                          int32_t tail_rank0, int32_t ctas, void* stream);
STS_API int sts_page_cache_plan(const int32_t* idx_dev, int64_t idx_ld, const int32_t* cnt_dev, int64_t units,
                                int32_t page_size, int32_t tail_page0, int32_t tail_rank0, int32_t* slot_page_dev,
                                int32_t* slot_last_dev, int64_t slots_ld, int32_t slots, int32_t step,
                                int32_t* copy_pages_dev, int32_t* copy_slots_dev, int32_t* ncopy_dev,
                                int32_t* idx_pool_dev, int32_t* status_dev, void* stream);

/* sts_kv_prefetch_l2 — L2 prefetch of selected K/V rows (no result depends
 * on it): for each unit, the rows of the first keys_per_part keys of each of
 * `parts` contiguous shares of its idx list (cnt keys; idx null = keys
 * 0..cnt-1). Used by the host-buffer verify step to pull the attention's
 * first rows into L2 while the queries are still crossing the host link. */
STS_API int sts_kv_prefetch_l2(const void* k_cache_dev, const void* v_cache_dev, int64_t kv_unit_stride,
                               int64_t kv_row_stride, int64_t units, int32_t d, int32_t elem_bytes,
                               const int32_t* idx_dev, int64_t idx_ld, const int32_t* cnt_dev, int32_t parts,
                               int32_t keys_per_part, void* stream);

/* ------------------------------------------------------------------------
 * sts_prefill_blocksparse — block-sparse prefill attention on tcgen05
 * (STS-PD): the masked prefill of toymodel._run_block
 * (src/toymodel.py:315-348 via forward_prefill(masks=...) :370-399) with
 * tile-granular masks: per (kv-head, 128-row query tile T) the committed
 * 64-key blocks a selection picked (all before the tile) plus the tile's
 * diagonal blocks under the causal mask; row t sees the selected keys and
 * the diagonal keys <= t.  idx/cnt: per (kv-head, tile) row hv*tiles + T, the
 * selected committed tokens as whole 64-key blocks, ascending (page-mode
 * sts_select_topk output, page_size 64, no extras); idx NULL = dense causal.
 *   q_dev [heads_q][n][d], k/v_dev [heads_kv][n][d] bf16 (head / row strides
 *   in elements, rows 16-byte aligned); out_dev [heads_q][n][d] bf16.
 * d in {64, 128}.  CTA = (tile, q-head): TMA tiles, S = Q.K^T and O += P.V
 * on tcgen05 with TMEM accumulators, softmax warps one thread per row.
 * ---------------------------------------------------------------------- */
STS_API int sts_prefill_blocksparse(const void* q_dev, const void* k_dev, const void* v_dev, int32_t heads_q,
                                    int32_t heads_kv, int32_t n, int32_t d, int64_t q_head_stride,
                                    int64_t kv_head_stride, int64_t row_stride, float scale, const int32_t* idx_dev,
                                    int64_t idx_ld, const int32_t* cnt_dev, void* out_dev, int32_t* status_dev,
                                    void* stream);

/* ------------------------------------------------------------------------
 * Sequence-sharded selection (context-parallel decode): the
 * global top-k of a row whose positions are split over P ranks, without
 * moving scores.  Replaces numkit.topk_indices / sparsity._select_row
 * (src/numkit.py:74-86, src/sparsity.py:86-112) when the row is sharded.
 * The union over ranks of the emitted sets equals sts_select_topk on the
 * concatenated row, bit for bit (ties to the lowest GLOBAL index).
 *
 * This rank holds global positions [lo, lo + n_local) (lo page-aligned) of
 * rows whose committed length is n_global; k_top counts tokens
 * (page_size 1) or pages.  Row values are formed as in sts_select_topk
 * (fp32 sum of nsrc source rows).  Host protocol, identical on every rank:
 *
 *   begin(g, hist)                                   local keys + digit-0 hist
 *   for r in 0 .. sts_dist_select_rounds(ps)-1:
 *       hist_g = allreduce_sum(hist)                 (NCCL, int32 [rows][2048])
 *       round(g, r, hist_g, hist, r == last ? ties : NULL)
 *   ties_all = allgather(ties)                       (int32 [P][rows])
 *   finish(g, rank, P, ties_all, ...)                local index lists
 * Digits are 11 bits from the top (the last one takes the rest): 3 rounds
 * for fp32 token keys, 6 for fp64 page keys.  With P = 1, hist_g may be the
 * same buffer as hist (no copy, no collective).  A row the global histogram
 * cannot resolve (ranks disagree on k_top / n_global / shard geometry) sets
 * STS_DEV_SELECT_INCONSISTENT in finish's status word.
 *
 * Output: ascending LOCAL offsets (global = lo + offset) of the selected
 * committed positions, the extras (sink = global 0, recent window, current =
 * n_global-1; flags as sts_select_topk) held here, and the in-block tail
 * [n_global, n_global + tail_len) ∩ [lo, lo + n_kv_local).
 * ---------------------------------------------------------------------- */
typedef struct sts_dist_rows {
  const float* scores_dev;   /* [S][ld] fp32 local score rows (columns = local positions) */
  int64_t ld;
  const int32_t* row_src_dev; /* [rows][nsrc] or NULL (nsrc == 1, identity) */
  int32_t nsrc;
  int64_t rows;
  int32_t n_global;          /* committed positions of every logical row */
  int32_t lo;                /* first global position held here */
  int32_t n_local;           /* positions held here */
  int32_t k_top;             /* tokens (page_size 1) or pages to keep */
  int32_t page_size;
} sts_dist_rows;

#define STS_DIST_BINS 2048

STS_API int32_t sts_dist_select_rounds(int32_t page_size);
/* histogram bins per radix round (the width of hist_local/hist_global rows) */
STS_API int32_t sts_dist_select_bins(void);
STS_API size_t sts_dist_select_workspace_bytes(int64_t rows, int32_t n_local, int32_t page_size);
STS_API int sts_dist_select_begin(const sts_dist_rows* g, int32_t* hist_local_dev, void* workspace_dev,
                                  size_t workspace_bytes, void* stream);
STS_API int sts_dist_select_round(const sts_dist_rows* g, int32_t round, const int32_t* hist_global_dev,
                                  int32_t* hist_local_dev, int32_t* ties_local_dev, void* workspace_dev,
                                  size_t workspace_bytes, void* stream);
STS_API int sts_dist_select_finish(const sts_dist_rows* g, int32_t rank, int32_t nranks,
                                   const int32_t* ties_all_dev, uint32_t flags, int32_t recent_window,
                                   int32_t tail_len, int32_t n_kv_local, int32_t* idx_out_dev, int64_t idx_ld,
                                   int32_t* cnt_out_dev, int32_t* status_dev, void* workspace_dev,
                                   size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* STS_B200_H */
