// sts_stream.cu — persistent stream-K gather kernel (bf16, tensor cores).
//
// One warp per CTA, grid = SMs x occupancy.  The key tiles of all units
// (unit = (batch, layer, kv-head); 16*SUB keys per tile) form one global tile
// space that is cut into equal contiguous ranges, one per warp, so every warp
// streams the same number of bytes no matter how ragged the per-unit key
// counts are (mode R unions, page mode, extras).  A warp runs ONE cp.async
// pipeline across its whole range: index slices are prefetched STAGES tiles
// ahead of the K/V gathers into a shared-memory ring, gathers run STAGES-1
// tiles ahead of the math, and crossing into the next unit only flushes the
// running softmax state and reloads Q — the pipeline never drains.  Units that
// span several warps are finished by the last warp to arrive (per-unit atomic
// counter), which merges the fp32 partials in warp order (deterministic).
//
// Math per 16-key sub-tile (MODE_DECODE): S^T = K.Q^T and O^T += V^T.P^T on
// mma.sync m16n8k16 with the stacked query rows as N (M = 20 -> 3 n-tiles),
// online softmax in the log2 domain, P^T re-laid out with movmatrix.trans.
// MODE_LSE drops V and P.V (draft-row log-sum-exp); MODE_PROBS turns scores
// into probabilities with a known LSE and writes them (per row, or summed
// over the speculative rows of each head).
#include <stdlib.h>

#include "sts_decode.cuh"

namespace sts {
namespace {

constexpr float LN2 = 0.6931471805599453f;

template <int D, int NT, int STAGES, int MODE, int SUB>
struct SL {
  static constexpr bool K_ONLY = MODE != MODE_DECODE;
  static constexpr int KT = KEY_TILE * SUB;
  static constexpr int MP = 8 * NT;
  static constexpr int ROW_BYTES = D * 2;
  static constexpr int CH = D / 8;
  static constexpr int Q_BYTES = MP * ROW_BYTES;
  static constexpr int SUB_BYTES = KEY_TILE * ROW_BYTES;
  static constexpr int STAGE_BYTES = (K_ONLY ? 1 : 2) * SUB * SUB_BYTES;
  static constexpr int RING = 2 * STAGES;
  static constexpr int IDX_BYTES = RING * KT * 4;
  static constexpr int META_BYTES = RING * 16;
  static constexpr int PROB_BYTES = MODE == MODE_PROBS ? KEY_TILE * MP * 4 : 0;
  static constexpr int SMEM = Q_BYTES + STAGES * STAGE_BYTES + 2 * IDX_BYTES + META_BYTES + PROB_BYTES;
};

__device__ __forceinline__ uint32_t swz(int row, int chunk) { return (uint32_t)((chunk ^ (row & 7)) << 4); }

__device__ __forceinline__ void cp_async_4_zfill(uint32_t dst, const void* src, bool valid) {
  int sz = valid ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src), "r"(sz));
}

template <int KT>
__device__ __forceinline__ int unit_tiles(const DecodeParams& p, int64_t u) {
  const int c = p.idx ? p.cnt[u] : p.n_dense;
  return (c + KT - 1) / KT;
}

// warp owning global tile t when T tiles are cut into W equal ranges
__device__ __forceinline__ int warp_of(int64_t t, int64_t T, int W) {
  return (int)(((t + 1) * W - 1) / T);
}

template <int D, int NT, int STAGES, int MODE, int SUB>
__global__ void __launch_bounds__(32, 1) stream_kernel(DecodeParams p) {
  using L = SL<D, NT, STAGES, MODE, SUB>;
  constexpr int KT = L::KT, CH = L::CH, MP = L::MP;
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x;
  const int w = blockIdx.x;
  const int M = p.M;
  const int64_t U = p.units;

  uint8_t* s_q = smem;
  uint8_t* s_stage = smem + L::Q_BYTES;
  int* s_idx = reinterpret_cast<int*>(s_stage + STAGES * L::STAGE_BYTES);  // [RING][KT]
  uint32_t* s_mem = reinterpret_cast<uint32_t*>(s_idx + L::RING * KT);     // [RING][KT]
  int* s_meta = reinterpret_cast<int*>(s_mem + L::RING * KT);              // [RING][4]
  float* s_prob = reinterpret_cast<float*>(s_meta + L::RING * 4);          // [16][MP]
  const uint32_t q_base = smem_u32(s_q);
  const uint32_t stage_base = smem_u32(s_stage);
  const uint32_t idx_base = smem_u32(s_idx);
  const uint32_t mem_base = smem_u32(s_mem);

  // ---- units with no keys: striped over warps (output zeros / LSE -inf) ----
  for (int64_t u = w; u < U; u += gridDim.x) {
    if (unit_tiles<KT>(p, u) != 0) continue;
    if constexpr (MODE == MODE_DECODE) {
      __nv_bfloat16* og = static_cast<__nv_bfloat16*>(p.out) + u * (int64_t)M * D;
      for (int e = lane; e < M * D; e += 32) og[e] = __float2bfloat16_rn(0.f);
      if (lane == 0 && M > 0) set_status(p.status, STS_DEV_EMPTY_ROW);
    }
    if constexpr (MODE != MODE_PROBS)
      if (p.lse)
        for (int r = lane; r < M; r += 32) p.lse[u * M + r] = -INFINITY;
  }

  // ---- total tiles and this warp's range ----
  int64_t T = 0;
  for (int64_t u = lane; u < U; u += 32) T += unit_tiles<KT>(p, u);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) T += __shfl_xor_sync(0xffffffffu, T, o);
  if (T == 0) return;
  // never more warps than tiles: every active warp owns >= 1 tile, so the
  // warps touching a unit are exactly warp_of(first)..warp_of(last)
  const int W = (int)(T < (int64_t)gridDim.x ? T : (int64_t)gridDim.x);
  if (w >= W) return;
  const int64_t s_w = (int64_t)w * T / W;
  const int64_t e_w = (int64_t)(w + 1) * T / W;
  if (s_w >= e_w) return;

  // ---- locate the unit holding tile s_w ----
  int64_t iu = 0, iP = 0;
  {
    int64_t base = 0;
    for (int64_t u0 = 0; u0 < U; u0 += 32) {
      const int64_t u = u0 + lane;
      const int t_u = u < U ? unit_tiles<KT>(p, u) : 0;
      int64_t incl = t_u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int64_t x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += x;
      }
      const int64_t tot = __shfl_sync(0xffffffffu, incl, 31);
      if (base + tot > s_w) {
        const uint32_t hit = __ballot_sync(0xffffffffu, base + incl > s_w);
        const int src = __ffs(hit) - 1;
        iu = u0 + src;
        iP = base + __shfl_sync(0xffffffffu, incl - t_u, src);
        break;
      }
      base += tot;
    }
  }
  int icnt = p.idx ? p.cnt[iu] : p.n_dense;
  int64_t iPn = iP + (icnt + KT - 1) / KT;

  // idx cursor: prefetch the index slice of tile t into ring slot (t - s_w) % RING
  auto issue_idx = [&](int64_t t) {
    if (t < e_w) {
      while (t >= iPn) {
        ++iu;
        iP = iPn;
        icnt = p.idx ? p.cnt[iu] : p.n_dense;
        iPn = iP + (icnt + KT - 1) / KT;
      }
      const int slot = (int)((t - s_w) % L::RING);
      const int j0 = (int)(t - iP) * KT;
      if (lane == 0) {
        s_meta[slot * 4 + 0] = (int)iu;
        s_meta[slot * 4 + 1] = j0;
        s_meta[slot * 4 + 2] = icnt;
        s_meta[slot * 4 + 3] = (int)iP;
      }
      if (p.idx) {
        const int32_t* ig = p.idx + iu * p.idx_ld;
        for (int e = lane; e < KT; e += 32) {
          const bool ok = j0 + e < icnt;
          cp_async_4_zfill(idx_base + (slot * KT + e) * 4, ig + (ok ? j0 + e : 0), ok);
          if (p.member) cp_async_4_zfill(mem_base + (slot * KT + e) * 4, p.member + iu * p.idx_ld + (ok ? j0 + e : 0), ok);
        }
      }
    }
  };
  // position of row r of ring slot `slot` (-1 when past the unit's list)
  auto slot_pos = [&](int slot, int r) -> int {
    const int j = s_meta[slot * 4 + 1] + r;
    if (j >= s_meta[slot * 4 + 2]) return -1;
    return p.idx ? s_idx[slot * KT + r] : j;
  };
  auto slot_mem = [&](int slot, int r) -> uint32_t { return p.member ? s_mem[slot * KT + r] : 0xffffffffu; };

  const int64_t ntile = e_w - s_w;
  auto issue_data = [&](int64_t i) {
    if (i < ntile) {
      const int slot = (int)(i % L::RING);
      const int stage = (int)(i % STAGES);
      const int64_t u = s_meta[slot * 4 + 0];
      const int jb = s_meta[slot * 4 + 1], cu = s_meta[slot * 4 + 2];
      const __nv_bfloat16* kg = static_cast<const __nv_bfloat16*>(p.k) + u * p.kv_stride;
      const __nv_bfloat16* vg = static_cast<const __nv_bfloat16*>(p.v) + u * p.kv_stride;
      const uint32_t st_k = stage_base + stage * L::STAGE_BYTES;
      constexpr int ROWS_PER_IT = 32 / CH;
#pragma unroll
      for (int it = 0; it < KT / ROWS_PER_IT; ++it) {
        const int r = it * ROWS_PER_IT + lane / CH;
        const int ch = lane % CH;
        const bool ok = jb + r < cu;
        const int pr = ok ? (p.idx ? s_idx[slot * KT + r] : jb + r) : 0;
        const int64_t off = (int64_t)pr * p.row_stride + ch * 8;
        const uint32_t sk = st_k + (r >> 4) * L::SUB_BYTES;
        const int rr = r & 15;
        cp_async_16_zfill(sk + rr * L::ROW_BYTES + swz(rr, ch), kg + off, ok);
        if constexpr (MODE == MODE_DECODE)
          cp_async_16_zfill(sk + SUB * L::SUB_BYTES + rr * L::ROW_BYTES + swz(rr, ch), vg + off, ok);
      }
    }
  };

  // ---- per-unit running state ----
  float o[MODE == MODE_DECODE ? D / 16 : 1][NT][4];
  float m_run[NT][2], l_run[NT][2], lse2[NT][2];
  int rmod[NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int c = 0; c < 2; ++c) rmod[nt][c] = (nt * 8 + 2 * (lane & 3) + c) % p.rows_per_head;
  const float sl2 = p.scale * LOG2E;
  const int causal_shift = p.pos_offset - p.causal_base;
  const bool causal = p.causal_base >= 0;
  const int mi = lane >> 3, ri = lane & 7;
  int64_t cur_u = -1;
  int cur_P = 0, cur_cnt = 0;

  auto reset_state = [&]() {
#pragma unroll
    for (int a = 0; a < (MODE == MODE_DECODE ? D / 16 : 1); ++a)
#pragma unroll
      for (int b = 0; b < NT; ++b)
#pragma unroll
        for (int c = 0; c < 4; ++c) o[a][b][c] = 0.f;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        m_run[nt][c] = -INFINITY;
        l_run[nt][c] = 0.f;
      }
  };

  auto load_q = [&](int64_t u) {
    const __nv_bfloat16* qg = static_cast<const __nv_bfloat16*>(p.q) + u * (int64_t)M * D;
    for (int c = lane; c < MP * CH; c += 32) {
      const int r = c / CH, ch = c % CH;
      uint4 val = make_uint4(0, 0, 0, 0);
      if (r < M) val = *reinterpret_cast<const uint4*>(qg + (int64_t)r * D + ch * 8);
      *reinterpret_cast<uint4*>(s_q + r * L::ROW_BYTES + swz(r, ch)) = val;
    }
    if constexpr (MODE == MODE_PROBS) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int r = nt * 8 + 2 * (lane & 3) + c;
          lse2[nt][c] = r < M ? p.lse_in[u * M + r] * LOG2E : 0.f;
        }
    }
    __syncwarp();
  };

  // finish unit u: write final rows, or a partial + merge when last to arrive
  auto flush = [&](int64_t u, int P_u, int cnt_u) {
    if constexpr (MODE != MODE_PROBS) {
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
    const int64_t tiles = (cnt_u + KT - 1) / KT;
    const int wf = warp_of(P_u, T, W);
    const int wl = warp_of(P_u + tiles - 1, T, W);
    const bool single = wf == wl;
    const int64_t slot = (int64_t)w + u;  // unique per (warp, unit) pair
    float* part_o = p.o_part + slot * (int64_t)M * D;
    float* part_l = p.l_part + slot * (int64_t)M;
    // rows' normalised values
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int r = nt * 8 + 2 * (lane & 3) + c;
        if (r >= M) continue;
        const float l = l_run[nt][c];
        const float inv = l > 0.f ? 1.f / l : 0.f;
        const float lse = l > 0.f ? (m_run[nt][c] + __log2f(l)) * LN2 : -INFINITY;
        if constexpr (MODE == MODE_DECODE) {
#pragma unroll
          for (int mt = 0; mt < D / 16; ++mt) {
            const int d0 = mt * 16 + (lane >> 2);
            if (single) {
              __nv_bfloat16* og = static_cast<__nv_bfloat16*>(p.out) + (u * M + r) * (int64_t)D;
              og[d0] = __float2bfloat16_rn(o[mt][nt][c] * inv);
              og[d0 + 8] = __float2bfloat16_rn(o[mt][nt][2 + c] * inv);
            } else {
              part_o[r * D + d0] = o[mt][nt][c] * inv;
              part_o[r * D + d0 + 8] = o[mt][nt][2 + c] * inv;
            }
          }
        }
        if (lane < 4) {
          if (single) {
            if (p.lse) p.lse[u * M + r] = lse;
            if (MODE == MODE_DECODE && !(l > 0.f)) set_status(p.status, STS_DEV_EMPTY_ROW);
          } else {
            part_l[r] = lse;
          }
        }
      }
    if (single) return;
    __threadfence();
    __syncwarp();
    int last = 0;
    if (lane == 0) {
      const int old = atomicAdd(p.counters + u, 1);
      last = old == wl - wf;
      if (last) __threadfence();
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) return;
    // merge contributors wf..wl (slots w' + u) in warp order.  Per-row max and
    // weights are computed once (lanes over rows, independent loads) into the
    // Q buffer, then lanes stream the float4 partials with no dependent loads.
    const int n = wl - wf + 1;
    float* s_w8 = reinterpret_cast<float*>(s_q);  // [n][M] weights, then [M] lse
    const bool fits = (n + 1) * M * 4 <= L::Q_BYTES;
    for (int r = lane; r < M; r += 32) {
      float mstar = -INFINITY;
      for (int ww = 0; ww < n; ++ww) mstar = fmaxf(mstar, __ldcg(p.l_part + ((int64_t)wf + ww + u) * M + r));
      float tot = 0.f;
      if (mstar != -INFINITY)
        for (int ww = 0; ww < n; ++ww) {
          const float l = __ldcg(p.l_part + ((int64_t)wf + ww + u) * M + r);
          tot += l == -INFINITY ? 0.f : expf(l - mstar);
        }
      if (p.lse) p.lse[u * M + r] = tot > 0.f ? mstar + logf(tot) : -INFINITY;
      if (MODE == MODE_DECODE && !(tot > 0.f)) set_status(p.status, STS_DEV_EMPTY_ROW);
      if constexpr (MODE == MODE_DECODE) {
        if (fits) {
          for (int ww = 0; ww < n; ++ww) {
            const float l = __ldcg(p.l_part + ((int64_t)wf + ww + u) * M + r);
            s_w8[ww * M + r] = (tot > 0.f && l != -INFINITY) ? expf(l - mstar) / tot : 0.f;
          }
        } else {
          s_w8[r] = mstar;  // slow path: recompute weights per element
          s_w8[M + r] = tot;
        }
      }
    }
    if constexpr (MODE == MODE_DECODE) {
      __syncwarp();
      constexpr int D4 = D / 4;
      for (int e = lane; e < M * D4; e += 32) {
        const int r = e / D4, d4 = e % D4;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
        for (int ww = 0; ww < n; ++ww) {
          const int64_t sl = (int64_t)wf + ww + u;
          float f;
          if (fits) {
            f = s_w8[ww * M + r];
          } else {
            const float l = __ldcg(p.l_part + sl * M + r);
            f = (s_w8[M + r] > 0.f && l != -INFINITY) ? expf(l - s_w8[r]) / s_w8[M + r] : 0.f;
          }
          const float4 x = __ldcg(reinterpret_cast<const float4*>(p.o_part + (sl * M + r) * D) + d4);
          acc.x += f * x.x;
          acc.y += f * x.y;
          acc.z += f * x.z;
          acc.w += f * x.w;
        }
        __nv_bfloat16* og = static_cast<__nv_bfloat16*>(p.out) + (u * M + r) * (int64_t)D + 4 * d4;
        *reinterpret_cast<__nv_bfloat162*>(og) = __floats2bfloat162_rn(acc.x, acc.y);
        *reinterpret_cast<__nv_bfloat162*>(og + 2) = __floats2bfloat162_rn(acc.z, acc.w);
      }
      __syncwarp();
    }
    }
  };

  // ---- pipeline prologue: index slices STAGES tiles ahead of the gathers ----
  for (int k = 0; k < STAGES; ++k) issue_idx(s_w + k);
  cp_async_commit();
  cp_async_wait<0>();
  __syncwarp();
#pragma unroll
  for (int sidx = 0; sidx < STAGES - 1; ++sidx) {
    issue_data(sidx);
    issue_idx(s_w + sidx + STAGES);
    cp_async_commit();
  }

  for (int64_t i = 0; i < ntile; ++i) {
    // group c = i + STAGES - 1: gathers of tile c (its indices landed: group c-STAGES)
    issue_data(i + STAGES - 1);
    issue_idx(s_w + i + 2 * STAGES - 1);
    cp_async_commit();
    cp_async_wait<STAGES - 1>();
    __syncwarp();

    const int slot = (int)(i % L::RING);
    const int stage = (int)(i % STAGES);
    const int64_t u = s_meta[slot * 4 + 0];
    if (u != cur_u) {
      if (cur_u >= 0) flush(cur_u, cur_P, cur_cnt);
      cur_u = u;
      cur_P = s_meta[slot * 4 + 3];
      cur_cnt = s_meta[slot * 4 + 2];
      reset_state();
      load_q(u);
    }
    const int j0 = s_meta[slot * 4 + 1];

    // ---- S^T = K . Q^T for every 16-key sub-tile of the stage ----
    float s[SUB][NT][4];
    bool okA[SUB][NT][2], okB[SUB][NT][2];
#pragma unroll
    for (int sub = 0; sub < SUB; ++sub) {
      const bool live = j0 + sub * KEY_TILE < cur_cnt;
      const uint32_t sk = stage_base + stage * L::STAGE_BYTES + sub * L::SUB_BYTES;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int c = 0; c < 4; ++c) s[sub][nt][c] = 0.f;
      if (live) {
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
            mma_bf16_16816(s[sub][nt], a0, b0);
            mma_bf16_16816(s[sub][nt], a1, b1);
          }
        }
      }
      // masking (keys past the list, causal tail, mode-R membership)
      const int kA = (lane >> 2) + sub * KEY_TILE, kB = kA + 8;
      const int posA = live ? slot_pos(slot, kA) : -1;
      const int posB = live ? slot_pos(slot, kB) : -1;
      const uint32_t memA = slot_mem(slot, kA);
      const uint32_t memB = slot_mem(slot, kB);
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
          okA[sub][nt][c] = a_ && ((memA >> (r & 31)) & 1u);
          okB[sub][nt][c] = b_ && ((memB >> (r & 31)) & 1u);
        }
    }

    if constexpr (MODE == MODE_PROBS) {
      const int lk = lane >> 2;
      const int R = p.rows_per_head;
      const int G = M / R;
#pragma unroll
      for (int sub = 0; sub < SUB; ++sub) {
        if (j0 + sub * KEY_TILE >= cur_cnt) break;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int r = nt * 8 + 2 * (lane & 3) + c;
            s_prob[lk * MP + r] = okA[sub][nt][c] ? fast_exp2(s[sub][nt][c] * sl2 - lse2[nt][c]) : 0.f;
            s_prob[(lk + 8) * MP + r] = okB[sub][nt][c] ? fast_exp2(s[sub][nt][2 + c] * sl2 - lse2[nt][c]) : 0.f;
          }
        __syncwarp();
        const int jb = j0 + sub * KEY_TILE;
        if (p.probs_mode == 0) {
          for (int e = lane; e < KEY_TILE * G; e += 32) {
            const int key = e % KEY_TILE, hh = e / KEY_TILE;
            const int pos = slot_pos(slot, sub * KEY_TILE + key);
            if (pos >= 0 && pos + p.pos_offset < p.causal_base) {
              float acc = s_prob[key * MP + hh * R];
              for (int ii = 1; ii < R; ++ii) acc = __fadd_rn(acc, s_prob[key * MP + hh * R + ii]);
              p.probs_out[(u * G + hh) * p.out_ld + jb + key] = acc;
            }
          }
        } else {
          for (int e = lane; e < KEY_TILE * M; e += 32) {
            const int key = e % KEY_TILE, r = e / KEY_TILE;
            const int pos = slot_pos(slot, sub * KEY_TILE + key);
            if (pos >= 0 && pos + p.pos_offset <= p.causal_base + r % R)
              p.probs_out[(u * M + r) * p.out_ld + jb + key] = s_prob[key * MP + r];
          }
        }
        __syncwarp();
      }
    } else {
      // ---- one online-softmax step over all SUB*16 keys (log2 domain) ----
      float pv[SUB][NT][4];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          float tmax = -INFINITY;
#pragma unroll
          for (int sub = 0; sub < SUB; ++sub) {
            const float vA = okA[sub][nt][c] ? s[sub][nt][c] * sl2 : -INFINITY;
            const float vB = okB[sub][nt][c] ? s[sub][nt][2 + c] * sl2 : -INFINITY;
            s[sub][nt][c] = vA;
            s[sub][nt][2 + c] = vB;
            tmax = fmaxf(tmax, fmaxf(vA, vB));
          }
          tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 4));
          tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 8));
          tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 16));
          const float m_old = m_run[nt][c];
          const float m_new = fmaxf(m_old, tmax);
          float alpha = 1.f, psum = 0.f;
          if (m_new != -INFINITY) {
            alpha = fast_exp2(m_old - m_new);
#pragma unroll
            for (int sub = 0; sub < SUB; ++sub) {
              pv[sub][nt][c] = fast_exp2(s[sub][nt][c] - m_new);
              pv[sub][nt][2 + c] = fast_exp2(s[sub][nt][2 + c] - m_new);
              psum += pv[sub][nt][c] + pv[sub][nt][2 + c];
            }
          } else {
#pragma unroll
            for (int sub = 0; sub < SUB; ++sub) {
              pv[sub][nt][c] = 0.f;
              pv[sub][nt][2 + c] = 0.f;
            }
          }
          m_run[nt][c] = m_new;
          l_run[nt][c] = l_run[nt][c] * alpha + psum;
          if constexpr (MODE == MODE_DECODE) {
            if (alpha != 1.f) {
#pragma unroll
              for (int mt = 0; mt < D / 16; ++mt) {
                o[mt][nt][c] *= alpha;
                o[mt][nt][2 + c] *= alpha;
              }
            }
          }
        }
      // ---- O^T += V^T . P^T ----
      if constexpr (MODE == MODE_DECODE) {
#pragma unroll
        for (int sub = 0; sub < SUB; ++sub) {
          if (j0 + sub * KEY_TILE >= cur_cnt) break;
          const uint32_t sv = stage_base + stage * L::STAGE_BYTES + (SUB + sub) * L::SUB_BYTES;
          uint32_t pb[NT][2];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            pb[nt][0] = movmatrix_trans(pack_bf16(pv[sub][nt][0], pv[sub][nt][1]));
            pb[nt][1] = movmatrix_trans(pack_bf16(pv[sub][nt][2], pv[sub][nt][3]));
          }
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
  if (cur_u >= 0) flush(cur_u, cur_P, cur_cnt);
}

template <int D, int NT, int MODE>
struct Cfg {
  static constexpr int STAGES = 3;
  static constexpr int SUB = MODE == MODE_DECODE ? (D == 64 ? 2 : 1) : (D == 64 ? 4 : 2);
  using L = SL<D, NT, STAGES, MODE, SUB>;
};

int occupancy_for(int smem_bytes) {
  const int per_sm = 227 * 1024;
  int occ = per_sm / (smem_bytes + 1024);
  if (occ > 16) occ = 16;
  return occ < 1 ? 1 : occ;
}

template <int D, int NT, int MODE>
int launch_stream(DecodeParams& p, cudaStream_t st) {
  using C = Cfg<D, NT, MODE>;
  using L = typename C::L;
  auto kern = stream_kernel<D, NT, C::STAGES, MODE, C::SUB>;
  STS_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM));
  const int grid = num_sms() * occupancy_for(L::SMEM);
  kern<<<grid, 32, L::SMEM, st>>>(p);
  STS_LAUNCH_CHECK();
  return STS_OK;
}

template <int D, int MODE>
int dispatch_nt(DecodeParams& p, cudaStream_t st) {
  switch ((p.M + 7) / 8) {
    case 1: return launch_stream<D, 1, MODE>(p, st);
    case 2: return launch_stream<D, 2, MODE>(p, st);
    case 3: return launch_stream<D, 3, MODE>(p, st);
    case 4: return launch_stream<D, 4, MODE>(p, st);
    case 5: return launch_stream<D, 5, MODE>(p, st);
    default: set_error("bf16 gather kernels support M <= 40 stacked rows, got %d", p.M); return STS_ERR_CONTRACT;
  }
}

template <int MODE>
int dispatch_d(DecodeParams& p, cudaStream_t st) {
  if (p.d == 128) return dispatch_nt<128, MODE>(p, st);
  if (p.d == 64) return dispatch_nt<64, MODE>(p, st);
  set_error("bf16 gather kernels support d in {64, 128}, got %d", p.d);
  return STS_ERR_CONTRACT;
}

// largest grid any (D, NT) config of a mode can use (bounds the partial slots)
int max_grid() { return num_sms() * 16; }

}  // namespace

size_t stream_workspace_bytes(int mode, int64_t units, int M, int d) {
  if (mode == MODE_PROBS) return 0;
  const int64_t slots = (int64_t)max_grid() + units;
  const size_t counters = ((size_t)units * 4 + 255) & ~size_t(255);
  const size_t per_slot = (size_t)M * ((mode == MODE_DECODE ? d : 0) + 1) * sizeof(float);
  return counters + (size_t)slots * per_slot + 256;
}

int stream_launch(int mode, DecodeParams& p, void* ws, size_t ws_bytes, cudaStream_t st) {
  const size_t need = stream_workspace_bytes(mode, p.units, p.M, p.d);
  if (mode != MODE_PROBS) {
    STS_REQUIRE(ws && ws_bytes >= need, STS_ERR_CONTRACT, "gather workspace too small: need %zu, got %zu", need,
                ws_bytes);
    const size_t counters = ((size_t)p.units * 4 + 255) & ~size_t(255);
    p.counters = static_cast<int*>(ws);
    const int64_t slots = (int64_t)max_grid() + p.units;
    p.l_part = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + counters);
    p.o_part = p.l_part + slots * p.M;
    // float4 merge loads need 16-byte aligned slots
    p.o_part = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(p.o_part) + 15) & ~uintptr_t(15));
    STS_CUDA_CHECK(cudaMemsetAsync(p.counters, 0, (size_t)p.units * 4, st));
  }
  // warp-specialised TMA gather (sts_gather.cu) unless STS_GATHER=stream
  static int use_stream = -1;
  if (use_stream < 0) {
    const char* e = getenv("STS_GATHER");
    use_stream = (e && strcmp(e, "stream") == 0) ? 1 : 0;
  }
  if (!use_stream) return gather_launch(mode, p, st);
  if (mode == MODE_DECODE) return dispatch_d<MODE_DECODE>(p, st);
  if (mode == MODE_LSE) return dispatch_d<MODE_LSE>(p, st);
  return dispatch_d<MODE_PROBS>(p, st);
}

}  // namespace sts
