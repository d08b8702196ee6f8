// sts_sparse_decode.cu — gathered-KV sparse flash-decode for the gamma+1
// verification rows (x GQA group) on sm_100a.
//
// BF16 path (the product path).  Per CTA: one (unit, split) — a contiguous
// slice of the unit's selected-key list.  Each warp owns a private
// cp.async ring of STAGES tiles of 16 gathered keys (K and V rows, 16-byte
// copies, XOR-swizzled so ldmatrix is conflict-free) and its own online
// softmax state, so the steady state needs no CTA barrier.  The math runs on
// the tensor cores "transposed": S^T = K.Q^T and O^T += V^T.P^T with
// mma.sync m16n8k16 (keys / head-dim as M, the stacked query rows as N in
// steps of 8), so M = 20 (gamma+1 = 5 rows x GQA 4) costs 3 n-tiles instead
// of padding rows to 32; P^T is re-laid out for the second MMA with
// movmatrix.trans.  At the end the warps are merged through shared memory and
// either the final rows (splits == 1) or fp32 partials + LSE (merged by
// sts_lse_merge) are written.
//
// F32 path (parity): CUDA-core fp32, one warp per query row, lanes over keys.
#include "sts_common.cuh"

namespace sts {
namespace {

constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;
constexpr int KEY_TILE = 16;

struct DecodeParams {
  const void* q;
  const void* k;
  const void* v;
  int64_t kv_stride;
  int64_t row_stride;  // elements between consecutive K (V) rows
  int64_t units;
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
  void* out;      // final output (splits == 1)
  float* lse;     // final lse (nullable)
  float* o_part;  // [splits][units][M][d] (splits > 1)
  float* l_part;  // [splits][units][M]
  int splits;
  int32_t* status;
  // MODE_PROBS
  const float* lse_in;  // [units][M] natural-log LSE
  float* probs_out;
  int64_t out_ld;
  int probs_mode;       // 0: reduced over rows (mode S), 1: per row (mode R)
  int idx_cap;          // keys of the CTA slice staged in shared memory
};

__device__ __forceinline__ int unit_count(const DecodeParams& p, int64_t u) {
  return p.idx ? p.cnt[u] : p.n_dense;
}

// Shared-memory plan of one CTA.  A warp's stage holds KT = 16*SUB keys
// (K, plus V in MODE_DECODE).  The CTA's slice of the index list (and of the
// membership bits) is preloaded once into shared memory so a gather never
// waits on a dependent index load.
template <int D, int NT, int STAGES, int WARPS, int MODE, int SUB>
struct Bf16Layout {
  static constexpr bool K_ONLY = MODE != 0;
  static constexpr int KT = KEY_TILE * SUB;
  static constexpr int MP = 8 * NT;                        // padded rows
  static constexpr int ROW_BYTES = D * 2;
  static constexpr int Q_BYTES = MP * ROW_BYTES;
  static constexpr int SUB_BYTES = KEY_TILE * ROW_BYTES;   // one 16-key K (or V) sub-tile
  static constexpr int STAGE_BYTES = (K_ONLY ? 1 : 2) * SUB * SUB_BYTES;
  static constexpr int PROB_BYTES = MODE == 2 ? KEY_TILE * MP * 4 : 0;  // MODE_PROBS scratch
  static constexpr int WARP_BYTES = STAGES * STAGE_BYTES + PROB_BYTES;
  static constexpr int MERGE_BYTES = WARPS * MP * (K_ONLY ? 0 : D) * 4 + WARPS * MP * 2 * 4;
  static constexpr int PIPE_BYTES = WARPS * WARP_BYTES;
  static constexpr int BODY = PIPE_BYTES > MERGE_BYTES ? PIPE_BYTES : MERGE_BYTES;
  static constexpr int FIXED = Q_BYTES + BODY;             // + idx slice (runtime)
};

__device__ __forceinline__ uint32_t swz(int row, int chunk) { return (uint32_t)((chunk ^ (row & 7)) << 4); }

// MODE_DECODE: K+V gather, online softmax, O = P.V  (sts_sparse_decode)
// MODE_LSE:    K only, online (max, sum) -> LSE     (sts_draft_lse)
// MODE_PROBS:  K only, p = exp(s - LSE), written as probability rows or
//              reduced over the speculative rows of each head (sts_draft_probs)
constexpr int MODE_DECODE = 0, MODE_LSE = 1, MODE_PROBS = 2;

template <int D, int NT, int STAGES, int WARPS, int MODE, int SUB>
__global__ void __launch_bounds__(WARPS * 32, 2) sparse_decode_bf16_kernel(DecodeParams p) {
  using L = Bf16Layout<D, NT, STAGES, WARPS, MODE, SUB>;
  constexpr int CH = D / 8;  // 16-byte chunks per row
  constexpr int KT = L::KT;
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t u = blockIdx.y;
  const int split = blockIdx.x;
  const int M = p.M;

  // ---- key range of this CTA ----
  const int cnt = unit_count(p, u);
  const int ntiles_all = (cnt + KT - 1) / KT;
  const int t0 = (int)((int64_t)split * ntiles_all / p.splits);
  const int t1 = (int)((int64_t)(split + 1) * ntiles_all / p.splits);
  const int key0 = t0 * KT;
  const int key1 = min(t1 * KT, cnt);

  // ---- Q -> smem (zero-padded rows); idx / member slice -> smem ----
  const __nv_bfloat16* qg = static_cast<const __nv_bfloat16*>(p.q) + u * (int64_t)M * D;
  for (int c = threadIdx.x; c < L::MP * CH; c += WARPS * 32) {
    const int r = c / CH, ch = c % CH;
    uint4 val = make_uint4(0, 0, 0, 0);
    if (r < M) val = *reinterpret_cast<const uint4*>(qg + (int64_t)r * D + ch * 8);
    *reinterpret_cast<uint4*>(smem + r * L::ROW_BYTES + swz(r, ch)) = val;
  }
  int* sidx = reinterpret_cast<int*>(smem + L::FIXED);
  uint32_t* smem_bits = reinterpret_cast<uint32_t*>(sidx + p.idx_cap);
  const int32_t* idxg = p.idx ? p.idx + u * p.idx_ld : nullptr;
  const uint32_t* memg = p.member ? p.member + u * p.idx_ld : nullptr;
  const bool idx_in_smem = idxg != nullptr && (key1 - key0) <= p.idx_cap;
  if (idx_in_smem) {
    for (int j = threadIdx.x; j < key1 - key0; j += WARPS * 32) {
      sidx[j] = idxg[key0 + j];
      if (memg) smem_bits[j] = memg[key0 + j];
    }
  }
  __syncthreads();
  const uint32_t q_base = smem_u32(smem);
  uint8_t* wbase = smem + L::Q_BYTES + warp * L::WARP_BYTES;
  const uint32_t wbase_u = smem_u32(wbase);
  float* pscr = reinterpret_cast<float*>(wbase + STAGES * L::STAGE_BYTES);  // [16][MP]

  const __nv_bfloat16* kg = static_cast<const __nv_bfloat16*>(p.k) + u * p.kv_stride;
  const __nv_bfloat16* vg = MODE == MODE_DECODE ? static_cast<const __nv_bfloat16*>(p.v) + u * p.kv_stride : nullptr;

  // position of key j of the list (-1 if past the CTA range)
  auto key_pos = [&](int j) -> int {
    if (j >= key1) return -1;
    if (!idxg) return j;
    return idx_in_smem ? sidx[j - key0] : idxg[j];
  };
  auto key_mem = [&](int j) -> uint32_t {
    if (!memg || j >= key1) return 0xffffffffu;
    return idx_in_smem ? smem_bits[j - key0] : memg[j];
  };

  // number of tiles this warp owns: t = t0 + warp + WARPS*i
  const int my_n = (t1 - t0 - warp + WARPS - 1) / WARPS > 0 ? (t1 - t0 - warp + WARPS - 1) / WARPS : 0;

  auto issue = [&](int i) {
    if (i < my_n) {
      const int stage = i % STAGES;
      const int kbase = (t0 + warp + WARPS * i) * KT;
      const uint32_t st_k = wbase_u + stage * L::STAGE_BYTES;
      constexpr int ROWS_PER_IT = 32 / CH;
#pragma unroll
      for (int it = 0; it < KT / ROWS_PER_IT; ++it) {
        const int r = it * ROWS_PER_IT + lane / CH;  // row within the stage (0..KT)
        const int ch = lane % CH;
        const int pr = key_pos(kbase + r);
        const bool ok = pr >= 0;
        const int64_t off = (int64_t)(ok ? pr : 0) * p.row_stride + ch * 8;
        const uint32_t sk = st_k + (r >> 4) * L::SUB_BYTES;
        const int rr = r & 15;
        cp_async_16_zfill(sk + rr * L::ROW_BYTES + swz(rr, ch), kg + off, ok);
        if constexpr (MODE == MODE_DECODE)
          cp_async_16_zfill(sk + SUB * L::SUB_BYTES + rr * L::ROW_BYTES + swz(rr, ch), vg + off, ok);
      }
    }
    cp_async_commit();
  };

  float o[MODE == MODE_DECODE ? D / 16 : 1][NT][4];
#pragma unroll
  for (int a = 0; a < (MODE == MODE_DECODE ? D / 16 : 1); ++a)
#pragma unroll
    for (int b = 0; b < NT; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) o[a][b][c] = 0.f;
  float m_run[NT][2], l_run[NT][2];
  int rmod[NT][2];
  float lse2[NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      m_run[nt][c] = -INFINITY;
      l_run[nt][c] = 0.f;
      const int r = nt * 8 + 2 * (lane & 3) + c;
      rmod[nt][c] = r % p.rows_per_head;
      lse2[nt][c] = (MODE == MODE_PROBS && r < M) ? p.lse_in[u * M + r] * LOG2E : 0.f;
    }
  const float sl2 = p.scale * LOG2E;
  const int causal_shift = p.pos_offset - p.causal_base;  // pos_rel = pos + shift
  const bool causal = p.causal_base >= 0;
  const int mi = lane >> 3, ri = lane & 7;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) issue(s);

  for (int i = 0; i < my_n; ++i) {
    issue(i + STAGES - 1);
    cp_async_wait<STAGES - 1>();
    __syncwarp();
    const int stage = i % STAGES;
    const int kbase = (t0 + warp + WARPS * i) * KT;

#pragma unroll 1
    for (int sub = 0; sub < SUB; ++sub) {
      const uint32_t sk = wbase_u + stage * L::STAGE_BYTES + sub * L::SUB_BYTES;
      const uint32_t sv = sk + SUB * L::SUB_BYTES;
      const int kb = kbase + sub * KEY_TILE;
      if (kb >= key1) break;

      // ---- S^T = K . Q^T  (16 keys x 8NT rows) ----
      float s[NT][4];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int c = 0; c < 4; ++c) s[nt][c] = 0.f;
#pragma unroll
      for (int kk = 0; kk < D / 16; kk += 2) {
        uint32_t a0[4], a1[4];
        const int key = (mi & 1) * 8 + ri;
        ldmatrix_x4(a0[0], a0[1], a0[2], a0[3], sk + key * L::ROW_BYTES + swz(key, 2 * kk + (mi >> 1)));
        ldmatrix_x4(a1[0], a1[1], a1[2], a1[3], sk + key * L::ROW_BYTES + swz(key, 2 * kk + 2 + (mi >> 1)));
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int row = nt * 8 + ri;
          uint32_t b[4];
          ldmatrix_x4(b[0], b[1], b[2], b[3], q_base + row * L::ROW_BYTES + swz(row, 2 * kk + mi));
          const uint32_t b0[2] = {b[0], b[1]};
          const uint32_t b1[2] = {b[2], b[3]};
          mma_bf16_16816(s[nt], a0, b0);
          mma_bf16_16816(s[nt], a1, b1);
        }
      }

      // ---- masking ----
      const int kA = lane >> 2, kB = kA + 8;
      const int posA = key_pos(kb + kA);
      const int posB = key_pos(kb + kB);
      const uint32_t memA = key_mem(kb + kA);
      const uint32_t memB = key_mem(kb + kB);
      bool okA[NT][2], okB[NT][2];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int r = nt * 8 + 2 * (lane & 3) + c;
          bool a_ = posA >= 0, b_ = posB >= 0;
          if (causal) {
            a_ = a_ && (posA + causal_shift <= rmod[nt][c]);
            b_ = b_ && (posB + causal_shift <= rmod[nt][c]);
          }
          okA[nt][c] = a_ && ((memA >> (r & 31)) & 1u);
          okB[nt][c] = b_ && ((memB >> (r & 31)) & 1u);
        }

      if constexpr (MODE == MODE_PROBS) {
        // p = exp2(s*sl2 - lse2[row]) -> scratch [key][row]
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int r = nt * 8 + 2 * (lane & 3) + c;
            pscr[kA * L::MP + r] = okA[nt][c] ? fast_exp2(s[nt][c] * sl2 - lse2[nt][c]) : 0.f;
            pscr[kB * L::MP + r] = okB[nt][c] ? fast_exp2(s[nt][2 + c] * sl2 - lse2[nt][c]) : 0.f;
          }
        __syncwarp();
        const int R = p.rows_per_head;
        const int G = M / R;
        if (p.probs_mode == 0) {
          // mode S: D[u][hh][j] = sum_i p_{hh,i}[j] (i ascending), committed keys only
          for (int e = lane; e < KEY_TILE * G; e += 32) {
            const int key = e % KEY_TILE, hh = e / KEY_TILE;
            const int pos = key_pos(kb + key);
            if (pos >= 0 && pos + p.pos_offset < p.causal_base) {
              float acc = pscr[key * L::MP + hh * R];
              for (int ii = 1; ii < R; ++ii) acc = __fadd_rn(acc, pscr[key * L::MP + hh * R + ii]);
              p.probs_out[(u * G + hh) * p.out_ld + kb + key] = acc;
            }
          }
        } else {
          // mode R: one probability row per (head, speculative row)
          for (int e = lane; e < KEY_TILE * M; e += 32) {
            const int key = e % KEY_TILE, r = e / KEY_TILE;
            const int pos = key_pos(kb + key);
            if (pos >= 0 && pos + p.pos_offset <= p.causal_base + r % R)
              p.probs_out[(u * M + r) * p.out_ld + kb + key] = pscr[key * L::MP + r];
          }
        }
        __syncwarp();
      } else {
        // ---- online softmax (log2 domain) ----
        uint32_t pb[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          float pv[4];
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const float vA = okA[nt][c] ? s[nt][c] * sl2 : -INFINITY;
            const float vB = okB[nt][c] ? s[nt][2 + c] * sl2 : -INFINITY;
            float tmax = fmaxf(vA, vB);
            tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 4));
            tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 8));
            tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 16));
            const float m_old = m_run[nt][c];
            const float m_new = fmaxf(m_old, tmax);
            float alpha, pA, pB;
            if (m_new == -INFINITY) {
              alpha = 1.f;
              pA = 0.f;
              pB = 0.f;
            } else {
              alpha = fast_exp2(m_old - m_new);
              pA = fast_exp2(vA - m_new);
              pB = fast_exp2(vB - m_new);
            }
            m_run[nt][c] = m_new;
            l_run[nt][c] = l_run[nt][c] * alpha + pA + pB;
            if constexpr (MODE == MODE_DECODE) {
#pragma unroll
              for (int mt = 0; mt < D / 16; ++mt) {
                o[mt][nt][c] *= alpha;
                o[mt][nt][2 + c] *= alpha;
              }
            }
            pv[c] = pA;
            pv[2 + c] = pB;
          }
          if constexpr (MODE == MODE_DECODE) {
            pb[nt][0] = movmatrix_trans(pack_bf16(pv[0], pv[1]));
            pb[nt][1] = movmatrix_trans(pack_bf16(pv[2], pv[3]));
          }
        }

        // ---- O^T += V^T . P^T ----
        if constexpr (MODE == MODE_DECODE) {
#pragma unroll
          for (int mt = 0; mt < D / 16; ++mt) {
            uint32_t a[4];
            const int key = (mi >> 1) * 8 + ri;
            ldmatrix_x4_trans(a[0], a[1], a[2], a[3], sv + key * L::ROW_BYTES + swz(key, 2 * mt + (mi & 1)));
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              const uint32_t b[2] = {pb[nt][0], pb[nt][1]};
              mma_bf16_16816(o[mt][nt], a, b);
            }
          }
        }
      }
    }
    __syncwarp();
  }
  cp_async_wait<0>();

  if constexpr (MODE != MODE_PROBS) {
    // ---- finish per-warp row sums ----
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        float l = l_run[nt][c];
        l += __shfl_xor_sync(0xffffffffu, l, 4);
        l += __shfl_xor_sync(0xffffffffu, l, 8);
        l += __shfl_xor_sync(0xffffffffu, l, 16);
        l_run[nt][c] = l;
      }
    __syncthreads();  // all warps done with their rings: reuse as merge buffer

    float* mo = reinterpret_cast<float*>(smem + L::Q_BYTES);          // [WARPS][MP][D]
    float* mml = mo + (MODE == MODE_DECODE ? WARPS * L::MP * D : 0);  // [WARPS][MP][2]
    if (lane < 4) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int r = nt * 8 + 2 * lane + c;
          mml[(warp * L::MP + r) * 2 + 0] = m_run[nt][c];
          mml[(warp * L::MP + r) * 2 + 1] = l_run[nt][c];
        }
    }
    if constexpr (MODE == MODE_DECODE) {
#pragma unroll
      for (int mt = 0; mt < D / 16; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int dd = mt * 16 + (lane >> 2) + (c >= 2 ? 8 : 0);
            const int r = nt * 8 + 2 * (lane & 3) + (c & 1);
            mo[(warp * L::MP + r) * D + dd] = o[mt][nt][c];
          }
    }
    __syncthreads();

    constexpr int DO = MODE == MODE_DECODE ? D : 1;
    for (int e = threadIdx.x; e < M * DO; e += WARPS * 32) {
      const int r = e / DO, dd = e % DO;
      float mstar = -INFINITY;
#pragma unroll
      for (int w = 0; w < WARPS; ++w) mstar = fmaxf(mstar, mml[(w * L::MP + r) * 2]);
      float acc = 0.f, lsum = 0.f;
      if (mstar != -INFINITY) {
#pragma unroll
        for (int w = 0; w < WARPS; ++w) {
          const float mw = mml[(w * L::MP + r) * 2];
          const float f = mw == -INFINITY ? 0.f : fast_exp2(mw - mstar);
          if constexpr (MODE == MODE_DECODE) acc += f * mo[(w * L::MP + r) * D + dd];
          lsum += f * mml[(w * L::MP + r) * 2 + 1];
        }
      }
      const float val = lsum > 0.f ? acc / lsum : 0.f;
      const float lse = lsum > 0.f ? (mstar + __log2f(lsum)) * LN2 : -INFINITY;
      if (p.splits == 1) {
        if constexpr (MODE == MODE_DECODE) {
          __nv_bfloat16* og = static_cast<__nv_bfloat16*>(p.out) + (u * M + r) * (int64_t)D;
          og[dd] = __float2bfloat16_rn(val);
        }
        if (dd == 0) {
          if (p.lse) p.lse[u * M + r] = lse;
          if (MODE == MODE_DECODE && lsum <= 0.f) set_status(p.status, STS_DEV_EMPTY_ROW);
        }
      } else {
        const int64_t base = ((int64_t)split * p.units + u) * M + r;
        if constexpr (MODE == MODE_DECODE) p.o_part[base * D + dd] = val;
        if (dd == 0) p.l_part[base] = lse;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// F32 parity path: one warp per query row; lanes stride over keys.
// ---------------------------------------------------------------------------
constexpr int F32_WARPS = 4;

__global__ void __launch_bounds__(F32_WARPS * 32) sparse_decode_f32_kernel(DecodeParams p) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t u = blockIdx.y;
  const int split = blockIdx.x;
  const int D = p.d;
  const int M = p.M;
  const int cnt = unit_count(p, u);
  const int c0 = (int)((int64_t)split * cnt / p.splits);
  const int c1 = (int)((int64_t)(split + 1) * cnt / p.splits);
  const float* kg = static_cast<const float*>(p.k) + u * p.kv_stride;
  const float* vg = static_cast<const float*>(p.v) + u * p.kv_stride;
  const int32_t* idxg = p.idx ? p.idx + u * p.idx_ld : nullptr;
  const uint32_t* memg = p.member ? p.member + u * p.idx_ld : nullptr;

  for (int r = warp; r < M; r += F32_WARPS) {
    const float* q = static_cast<const float*>(p.q) + (u * M + r) * (int64_t)D;
    float m = -INFINITY, l = 0.f;
    float acc[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) acc[t] = 0.f;
    const int rm = r % p.rows_per_head;
    for (int base = c0; base < c1; base += 32) {
      const int j = base + lane;
      bool ok = j < c1;
      int pos = 0;
      float s = -INFINITY;
      if (ok) {
        pos = idxg ? idxg[j] : j;
        if (p.causal_base >= 0) ok = ok && (pos + p.pos_offset - p.causal_base <= rm);
        if (memg) ok = ok && ((memg[j] >> (r & 31)) & 1u);
      }
      if (ok) {
        const float* kr = kg + (int64_t)pos * p.row_stride;
        float dot = 0.f;
        for (int e = 0; e < D; ++e) dot = fmaf(q[e], kr[e], dot);
        s = dot * p.scale;
      }
      float tmax = s;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
      const float m_new = fmaxf(m, tmax);
      if (m_new == -INFINITY) continue;
      const float alpha = expf(m - m_new);
      const float pj = ok ? expf(s - m_new) : 0.f;
      float psum = pj;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) psum += __shfl_xor_sync(0xffffffffu, psum, o);
      l = l * alpha + psum;
      m = m_new;
#pragma unroll
      for (int t = 0; t < 8; ++t) acc[t] *= alpha;
      for (int src = 0; src < 32; ++src) {
        const float pk = __shfl_sync(0xffffffffu, pj, src);
        const int posk = __shfl_sync(0xffffffffu, pos, src);
        if (pk == 0.f) continue;
        const float* vr = vg + (int64_t)posk * p.row_stride;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const int e = lane + 32 * t;
          if (e < D) acc[t] = fmaf(pk, vr[e], acc[t]);
        }
      }
    }
    const float lse = l > 0.f ? m + logf(l) : -INFINITY;
    if (p.splits == 1) {
      float* og = static_cast<float*>(p.out) + (u * M + r) * (int64_t)D;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int e = lane + 32 * t;
        if (e < D) og[e] = l > 0.f ? acc[t] / l : 0.f;
      }
      if (lane == 0) {
        if (p.lse) p.lse[u * M + r] = lse;
        if (!(l > 0.f)) set_status(p.status, STS_DEV_EMPTY_ROW);
      }
    } else {
      const int64_t base = ((int64_t)split * p.units + u) * M + r;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int e = lane + 32 * t;
        if (e < D) p.o_part[base * D + e] = l > 0.f ? acc[t] / l : 0.f;
      }
      if (lane == 0) p.l_part[base] = lse;
    }
  }
}

template <int D, int NT, int MODE>
int launch_bf16(DecodeParams p, cudaStream_t st) {
  constexpr int WARPS = 4;
  // K-only draft passes move 16*SUB keys per stage so one stage is ~8 KB.
  constexpr int SUB = MODE == MODE_DECODE ? (D == 64 ? 2 : 1) : (D == 64 ? 4 : 2);
  constexpr int STAGES = 3;
  using L = Bf16Layout<D, NT, STAGES, WARPS, MODE, SUB>;
  auto kern = sparse_decode_bf16_kernel<D, NT, STAGES, WARPS, MODE, SUB>;
  // index slice per CTA (+ membership bits): sized from the largest CTA range
  int64_t max_keys = 0;
  if (p.idx) {
    const int64_t tiles = (p.idx_ld + L::KT - 1) / L::KT;
    max_keys = ((tiles + p.splits - 1) / p.splits + 1) * L::KT;
    if (max_keys > 8192) max_keys = 8192;  // larger slices read the list from global
  }
  p.idx_cap = (int)max_keys;
  const int smem = L::FIXED + (int)max_keys * (p.member ? 8 : 4);
  STS_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  dim3 grid(p.splits, (unsigned)p.units);
  kern<<<grid, WARPS * 32, smem, st>>>(p);
  STS_LAUNCH_CHECK();
  return STS_OK;
}

template <int D, int MODE>
int dispatch_nt(const DecodeParams& p, cudaStream_t st) {
  const int nt = (p.M + 7) / 8;
  switch (nt) {
    case 1: return launch_bf16<D, 1, MODE>(p, st);
    case 2: return launch_bf16<D, 2, MODE>(p, st);
    case 3: return launch_bf16<D, 3, MODE>(p, st);
    case 4: return launch_bf16<D, 4, MODE>(p, st);
    case 5: return launch_bf16<D, 5, MODE>(p, st);
    default: set_error("bf16 gather kernels support M <= 40 stacked rows, got %d", p.M); return STS_ERR_CONTRACT;
  }
}

template <int MODE>
int dispatch_d(const DecodeParams& p, cudaStream_t st) {
  if (p.d == 128) return dispatch_nt<128, MODE>(p, st);
  if (p.d == 64) return dispatch_nt<64, MODE>(p, st);
  set_error("bf16 gather kernels support d in {64, 128}, got %d", p.d);
  return STS_ERR_CONTRACT;
}

// splits so that units*splits CTAs fill the chip in whole waves of 2 CTAs/SM
int auto_splits(int64_t units, int64_t keys_per_unit) {
  const int64_t slots = 2LL * num_sms();
  int64_t tiles = (keys_per_unit + KEY_TILE * 8 - 1) / (KEY_TILE * 8);  // >= 8 tiles per CTA
  int64_t best = 1;
  double best_eff = 0.0;
  for (int64_t s = 1; s <= 64 && s <= (tiles > 0 ? tiles : 1); ++s) {
    const int64_t ctas = units * s;
    const int64_t waves = (ctas + slots - 1) / slots;
    const double eff = (double)ctas / (double)(waves * slots);
    // prefer fuller last waves, then more parallelism up to ~8 waves
    const double score = eff - 0.002 * (double)s;
    if (waves <= 16 && score > best_eff) {
      best_eff = score;
      best = s;
    }
  }
  return (int)best;
}

}  // namespace

int lse_merge_launch(const float* o_part, const float* lse_part, int nparts, int64_t rows, int d,
                     int out_dtype, void* out, float* lse_out, cudaStream_t st);

}  // namespace sts

using namespace sts;

extern "C" size_t sts_sparse_decode_workspace_bytes(int64_t units, int32_t M, int32_t d, int32_t splits) {
  if (splits <= 1) return 0;
  return (size_t)splits * units * M * ((size_t)d + 1) * sizeof(float) + 256;
}

extern "C" int sts_sparse_decode(int32_t dtype, const void* q_dev, const void* k_cache_dev,
                                 const void* v_cache_dev, int64_t kv_unit_stride, int64_t kv_row_stride,
                                 int64_t units,
                                 int32_t M, int32_t d, const int32_t* idx_dev, int64_t idx_ld,
                                 const int32_t* cnt_dev, int32_t n_dense,
                                 const uint32_t* member_dev, int32_t causal_base,
                                 int32_t rows_per_head, int32_t pos_offset, float scale,
                                 void* out_dev, float* lse_dev, int32_t splits,
                                 int32_t* status_dev, void* workspace_dev,
                                 size_t workspace_bytes, void* stream) {
  STS_REQUIRE(units >= 0, STS_ERR_CONTRACT, "units must be >= 0");
  if (units == 0) return STS_OK;
  STS_REQUIRE(q_dev && k_cache_dev && v_cache_dev && out_dev, STS_ERR_CONTRACT, "null buffer");
  STS_REQUIRE(M >= 1, STS_ERR_CONTRACT, "M must be >= 1");
  STS_REQUIRE(!member_dev || M <= 32, STS_ERR_CONTRACT, "row membership bits need M <= 32");
  STS_REQUIRE(rows_per_head >= 1, STS_ERR_CONTRACT, "rows_per_head must be >= 1");
  STS_REQUIRE(idx_dev ? (cnt_dev != nullptr) : (n_dense >= 0), STS_ERR_CONTRACT,
              "index list needs counts / dense needs n_dense");
  STS_REQUIRE(splits >= 1 && splits <= 4096, STS_ERR_CONTRACT, "splits must be in [1, 4096]");
  STS_REQUIRE(units <= 65535, STS_ERR_CONTRACT, "units must be <= 65535 (grid.y)");
  cudaStream_t st = static_cast<cudaStream_t>(stream);

  DecodeParams p;
  p.q = q_dev;
  p.k = k_cache_dev;
  p.v = v_cache_dev;
  p.kv_stride = kv_unit_stride;
  p.row_stride = kv_row_stride > 0 ? kv_row_stride : d;
  STS_REQUIRE(p.row_stride >= d, STS_ERR_CONTRACT, "kv_row_stride must be >= d");
  p.units = units;
  p.M = M;
  p.d = d;
  p.idx = idx_dev;
  p.idx_ld = idx_ld;
  p.cnt = cnt_dev;
  p.n_dense = n_dense;
  p.member = member_dev;
  p.causal_base = causal_base;
  p.rows_per_head = rows_per_head;
  p.pos_offset = pos_offset;
  p.scale = scale;
  p.out = out_dev;
  p.lse = lse_dev;
  p.splits = splits;
  p.status = status_dev;
  p.o_part = nullptr;
  p.l_part = nullptr;
  p.lse_in = nullptr;
  p.probs_out = nullptr;
  p.out_ld = 0;
  p.probs_mode = 0;
  if (splits > 1) {
    size_t need = sts_sparse_decode_workspace_bytes(units, M, d, splits);
    STS_REQUIRE(workspace_dev && workspace_bytes >= need, STS_ERR_CONTRACT,
                "sparse decode workspace too small: need %zu, got %zu", need, workspace_bytes);
    p.o_part = static_cast<float*>(workspace_dev);
    p.l_part = p.o_part + (size_t)splits * units * M * d;
  }

  int rc;
  if (dtype == STS_DTYPE_BF16) {
    rc = dispatch_d<MODE_DECODE>(p, st);
  } else if (dtype == STS_DTYPE_F32) {
    STS_REQUIRE(d >= 1 && d <= 256, STS_ERR_CONTRACT, "f32 sparse decode supports d <= 256");
    dim3 grid(splits, (unsigned)units);
    sparse_decode_f32_kernel<<<grid, F32_WARPS * 32, 0, st>>>(p);
    STS_LAUNCH_CHECK();
    rc = STS_OK;
  } else {
    set_error("unknown dtype %d", dtype);
    return STS_ERR_CONTRACT;
  }
  if (rc != STS_OK || splits == 1) return rc;
  return lse_merge_launch(p.o_part, p.l_part, splits, units * M, d, dtype, out_dev, lse_dev, st);
}

extern "C" int32_t sts_auto_splits(int64_t units, int64_t keys_per_unit) {
  return auto_splits(units, keys_per_unit);
}

// ---------------------------------------------------------------------------
// draft-score capture
// ---------------------------------------------------------------------------
static void draft_params(DecodeParams& p, const void* q_dev, const void* k_cache_dev,
                         int64_t kv_unit_stride, int64_t units, int32_t G, int32_t R, int32_t d,
                         int32_t n_keys, int32_t pos_offset, int32_t base, float scale) {
  memset(&p, 0, sizeof(p));
  p.q = q_dev;
  p.k = k_cache_dev;
  p.v = nullptr;
  p.kv_stride = kv_unit_stride;
  p.row_stride = d;
  p.units = units;
  p.M = G * R;
  p.d = d;
  p.idx = nullptr;
  p.n_dense = n_keys;
  p.member = nullptr;
  p.causal_base = base;
  p.rows_per_head = R;
  p.pos_offset = pos_offset;
  p.scale = scale;
}

extern "C" size_t sts_draft_workspace_bytes(int64_t units, int32_t GR, int32_t n_keys) {
  const int s = auto_splits(units, n_keys);
  return s <= 1 ? 0 : (size_t)s * units * GR * sizeof(float) + 256;
}

extern "C" int sts_draft_lse(int32_t dtype, const void* q_dev, const void* k_cache_dev,
                             int64_t kv_unit_stride, int64_t units, int32_t G, int32_t R,
                             int32_t d, int32_t n_keys, int32_t pos_offset, int32_t base,
                             float scale, float* lse_dev, void* workspace_dev,
                             size_t workspace_bytes, void* stream) {
  STS_REQUIRE(dtype == STS_DTYPE_BF16, STS_ERR_CONTRACT, "draft scores run in bf16");
  STS_REQUIRE(units >= 0 && G >= 1 && R >= 1 && n_keys >= 0, STS_ERR_CONTRACT, "bad draft shape");
  STS_REQUIRE(units <= 65535, STS_ERR_CONTRACT, "units must be <= 65535");
  STS_REQUIRE(q_dev && k_cache_dev && lse_dev, STS_ERR_CONTRACT, "null buffer");
  if (units == 0) return STS_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DecodeParams p;
  draft_params(p, q_dev, k_cache_dev, kv_unit_stride, units, G, R, d, n_keys, pos_offset, base, scale);
  p.splits = auto_splits(units, n_keys);
  p.lse = lse_dev;
  if (p.splits > 1) {
    const size_t need = (size_t)p.splits * units * p.M * sizeof(float);
    STS_REQUIRE(workspace_dev && workspace_bytes >= need, STS_ERR_CONTRACT,
                "draft workspace too small: need %zu, got %zu", need, workspace_bytes);
    p.l_part = static_cast<float*>(workspace_dev);
  }
  int rc = dispatch_d<MODE_LSE>(p, st);
  if (rc != STS_OK || p.splits == 1) return rc;
  return lse_merge_launch(nullptr, p.l_part, p.splits, units * p.M, d, STS_DTYPE_F32, nullptr, lse_dev, st);
}

extern "C" int sts_draft_probs(int32_t dtype, const void* q_dev, const void* k_cache_dev,
                               int64_t kv_unit_stride, int64_t units, int32_t G, int32_t R,
                               int32_t d, int32_t n_keys, int32_t pos_offset, int32_t base,
                               float scale, const float* lse_dev, int32_t mode, float* out_dev,
                               int64_t out_ld, void* stream) {
  STS_REQUIRE(dtype == STS_DTYPE_BF16, STS_ERR_CONTRACT, "draft scores run in bf16");
  STS_REQUIRE(units >= 0 && G >= 1 && R >= 1 && n_keys >= 0, STS_ERR_CONTRACT, "bad draft shape");
  STS_REQUIRE(units <= 65535, STS_ERR_CONTRACT, "units must be <= 65535");
  STS_REQUIRE(q_dev && k_cache_dev && lse_dev && out_dev, STS_ERR_CONTRACT, "null buffer");
  STS_REQUIRE(mode == 0 || mode == 1, STS_ERR_CONTRACT, "mode must be 0 (S) or 1 (R)");
  STS_REQUIRE(out_ld >= n_keys, STS_ERR_CONTRACT, "out_ld must be >= n_keys");
  if (units == 0) return STS_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DecodeParams p;
  draft_params(p, q_dev, k_cache_dev, kv_unit_stride, units, G, R, d, n_keys, pos_offset, base, scale);
  p.splits = auto_splits(units, n_keys);
  p.lse_in = lse_dev;
  p.probs_out = out_dev;
  p.out_ld = out_ld;
  p.probs_mode = mode;
  return dispatch_d<MODE_PROBS>(p, st);
}
