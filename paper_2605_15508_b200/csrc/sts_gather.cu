// sts_gather.cu — persistent row-split gather kernel (bf16, sm_100a tensor cores).
//
// Work decomposition
//  * Unit = (batch, layer, kv-head).  The key tiles of all units (KT keys per
//    tile) form one global tile space, cut into equal contiguous ranges, one
//    per CTA (stream-K): every CTA streams the same number of gathered bytes no
//    matter how ragged the per-unit key lists are (mode-R unions, page mode).
//  * A CTA has one warp per 8-row n-tile of the stacked query block
//    (M = GQA group x (gamma+1) rows; M = 20 -> 3 warps).  All warps consume
//    the SAME gathered K/V tile, each for its own 8 query rows, so the tile is
//    fetched once, no math is duplicated, and a warp carries only its rows'
//    accumulators (32 fp32 registers at d = 128) and its Q fragments (16
//    registers).  That keeps registers low enough for 4+ CTAs (12+ warps) per
//    SM — the latency hiding a 256-byte random-row gather needs.
//  * One cp.async pipeline per CTA, STAGES deep, continuous across unit
//    boundaries: index slices are prefetched STAGES tiles ahead into a ring,
//    K/V rows (16-byte cp.async into padded rows) STAGES-1 tiles ahead of the
//    math, one CTA barrier per tile.  Entering a new unit flushes each warp's
//    softmax state and reloads its Q fragments; units spanning several CTAs are
//    merged by the last CTA to arrive (per-unit counter), in CTA order
//    (deterministic).
//  * Instruction economy: rows are padded to 2d+16 bytes (conflict-free
//    ldmatrix without an XOR swizzle), so every ldmatrix / cp.async address is
//    a per-lane constant plus a compile-time offset; tiles fully inside the
//    committed prefix skip per-element masking; the O rescale is skipped when
//    no row's running max moved.
//
// (A warp-specialised variant — one producer warp issuing one cp.async.bulk
// per gathered row into mbarrier rings — was measured 3-4x slower: 256-byte
// bulk copies saturate the per-SM TMA unit.  See DESIGN.md §4.)
//
// Modes: DECODE (K+V, online softmax, O = P.V), LSE (K only, draft-row
// log-sum-exp), PROBS (K only, probabilities from a known LSE, per row or
// summed over the speculative rows of each head).
#include <stdlib.h>

#include "sts_decode.cuh"

namespace sts {
namespace {

constexpr float LN2f = 0.6931471805599453f;

template <int D, int NT, int MODE, int SUB, int STAGES>
struct GL {
  static constexpr bool K_ONLY = MODE != MODE_DECODE;
  static constexpr int KT = KEY_TILE * SUB;
  static constexpr int MP = 8 * NT;
  static constexpr int CH = D / 8;
  static constexpr int PITCH = D * 2 + 16;        // padded row: ldmatrix conflict-free
  static constexpr int SUBB = KEY_TILE * PITCH;   // one 16-key K (or V) block
  static constexpr int KV = KT * PITCH;           // K block -> V block
  static constexpr int STAGE = (K_ONLY ? 1 : 2) * KV;
  static constexpr int RING = STAGES <= 2 ? 4 : 8;  // index ring (power of 2, >= 2*STAGES)
  static constexpr int IDX_BYTES = RING * KT * 4;
  static constexpr int META_BYTES = RING * 16;
  static constexpr int PROB = MODE == MODE_PROBS ? KT * MP * 4 : 0;
  static constexpr int MERGE = MP * 2 * 4;
  static constexpr int SMEM = STAGES * STAGE + 2 * IDX_BYTES + META_BYTES + PROB + MERGE + 16;
  static constexpr int THREADS = NT * 32;
  static constexpr int GROWS = THREADS / CH;      // rows per gather pass
};

__device__ __forceinline__ void cp_async_4_zfill(uint32_t dst, const void* src, bool valid) {
  int sz = valid ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src), "r"(sz));
}

__device__ __forceinline__ int tiles_of(const DecodeParams& p, int64_t u, int KT) {
  const int c = p.idx ? p.cnt[u] : p.n_dense;
  return (c + KT - 1) / KT;
}

__device__ __forceinline__ int owner_of(int64_t t, int64_t T, int W) { return (int)(((t + 1) * W - 1) / T); }

#ifndef STS_GATHER_MINB3
#define STS_GATHER_MINB3 5
#endif
// resident CTAs the register allocation must allow (NT = 3 is the c2 / c4
// decode shape: 5 -> 128 registers, 6 -> 112)
template <int NT>
constexpr int gather_min_blocks() { return NT == 3 ? STS_GATHER_MINB3 : 16 / NT; }

template <int D, int NT, int MODE, int SUB, int STAGES>
__global__ void __launch_bounds__(NT * 32, gather_min_blocks<NT>()) gather_kernel(DecodeParams p) {
  using L = GL<D, NT, MODE, SUB, STAGES>;
  constexpr int KT = L::KT, MP = L::MP, CH = L::CH, NTH = L::THREADS, PITCH = L::PITCH;
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;  // this warp's n-tile: query rows 8*warp .. 8*warp+7
  const int M = p.M;
  const int64_t U = p.units;

  uint8_t* s_stage = smem;
  int* s_idx = reinterpret_cast<int*>(s_stage + STAGES * L::STAGE);
  uint32_t* s_mem = reinterpret_cast<uint32_t*>(s_idx + L::RING * KT);
  int* s_meta = reinterpret_cast<int*>(s_mem + L::RING * KT);
  float* s_prob = reinterpret_cast<float*>(s_meta + L::RING * 4);
  float* s_merge = s_prob + (L::PROB / 4);
  int* s_flag = reinterpret_cast<int*>(s_merge + L::MERGE / 4);
  const uint32_t stage_base = smem_u32(s_stage);
  const uint32_t idx_base = smem_u32(s_idx);
  const uint32_t mem_base = smem_u32(s_mem);

  // ---- units with no keys (striped over CTAs): zero rows, LSE -inf ----
  for (int64_t u = blockIdx.x; u < U; u += gridDim.x) {
    if (tiles_of(p, u, KT) != 0) continue;
    if constexpr (MODE == MODE_DECODE) {
      if (p.out_f32) {
        float* og = static_cast<float*>(p.out) + u * (int64_t)M * D;
        for (int e = tid; e < M * D; e += NTH) og[e] = 0.f;
      } else {
        __nv_bfloat16* og = static_cast<__nv_bfloat16*>(p.out) + u * (int64_t)M * D;
        for (int e = tid; e < M * D; e += NTH) og[e] = __float2bfloat16_rn(0.f);
      }
      if (tid == 0 && M > 0) set_status(p.status, STS_DEV_EMPTY_ROW);
    }
    if constexpr (MODE != MODE_PROBS)
      if (p.lse)
        for (int r = tid; r < M; r += NTH) p.lse[u * M + r] = -INFINITY;
  }

  // ---- tile space and this CTA's range: block-parallel scan of the unit
  // tile counts (thread t owns units [t*cpt, (t+1)*cpt); its count loads are
  // independent, so the whole prologue is ~one memory round trip) ----
  __shared__ long long s_scan[NT + 2];
  const int64_t cpt = (U + NTH - 1) / NTH;
  const int64_t ub = (int64_t)tid * cpt, ue = ub + cpt < U ? ub + cpt : U;
  int64_t mine = 0;
  for (int64_t u0 = ub; u0 < ue; u0 += 4) {
    int t4[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) t4[j] = u0 + j < ue ? tiles_of(p, u0 + j, KT) : 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) mine += t4[j];
  }
  int64_t incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t x = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += x;
  }
  if (lane == 31) s_scan[warp] = incl;
  __syncthreads();
  int64_t before = 0, T = 0;
#pragma unroll
  for (int ww = 0; ww < NT; ++ww) {
    const int64_t v = s_scan[ww];
    before += ww < warp ? v : 0;
    T += v;
  }
  if (T == 0) return;
  const int W = (int)(T < (int64_t)gridDim.x ? T : (int64_t)gridDim.x);
  const int w = blockIdx.x;
  if (w >= W) return;
  const int64_t s_w = (int64_t)w * T / W;
  const int64_t e_w = (int64_t)(w + 1) * T / W;
  const int ntile = (int)(e_w - s_w);
  {
    // the thread whose units contain tile s_w finds the unit and its first tile
    int64_t acc = before + incl - mine;
    if (acc <= s_w && s_w < acc + mine) {
      for (int64_t u = ub; u < ue; ++u) {
        const int t_u = tiles_of(p, u, KT);
        if (s_w < acc + t_u) {
          s_scan[NT] = u;
          s_scan[NT + 1] = acc;
          break;
        }
        acc += t_u;
      }
    }
  }
  __syncthreads();
  int64_t iu = s_scan[NT], iP = s_scan[NT + 1];
  int icnt = p.idx ? p.cnt[iu] : p.n_dense;
  int64_t iPn = iP + (icnt + KT - 1) / KT;

  // index cursor: slice of relative tile i -> next ring slot (+ meta)
  auto issue_idx = [&](int i) {
    const int slot = i & (L::RING - 1);
    if (i >= ntile) return;
    const int64_t t = s_w + i;
    while (t >= iPn) {
      ++iu;
      iP = iPn;
      icnt = p.idx ? p.cnt[iu] : p.n_dense;
      iPn = iP + (icnt + KT - 1) / KT;
    }
    const int j0 = (int)(t - iP) * KT;
    if (tid == 0) {
      s_meta[slot * 4 + 0] = (int)iu;
      s_meta[slot * 4 + 1] = j0;
      s_meta[slot * 4 + 2] = icnt;
      s_meta[slot * 4 + 3] = (int)iP;
    }
    if (p.idx) {
      for (int e = tid; e < KT; e += NTH) {
        const bool ok = j0 + e < icnt;
        cp_async_4_zfill(idx_base + (slot * KT + e) * 4, p.idx + iu * p.idx_ld + (ok ? j0 + e : 0), ok);
        if (p.member)
          cp_async_4_zfill(mem_base + (slot * KT + e) * 4, p.member + iu * p.idx_ld + (ok ? j0 + e : 0), ok);
      }
    }
  };
  auto slot_pos = [&](int slot, int r) -> int {
    const int j = s_meta[slot * 4 + 1] + r;
    if (j >= s_meta[slot * 4 + 2]) return -1;
    return p.idx ? s_idx[slot * KT + r] : j;
  };

  // K/V gather: thread -> (chunk g_ch, rows g_r0 + GROWS*j); K and V of a
  // (row, chunk) share the index lookup.  Row offsets are 32-bit (a unit spans
  // < 4 GiB, checked by the host), so each 16-byte copy costs one
  // IMAD.WIDE.U32 + LDGSTS; full tiles skip the bounds test and the zero-fill.
  constexpr int GROWS = L::GROWS;
  constexpr int GJ = (KT + GROWS - 1) / GROWS;
  const int g_ch = tid % CH, g_r0 = tid / CH;
  const int g_n = (KT - g_r0 + GROWS - 1) / GROWS;  // rows this thread copies per tile
  const uint32_t g_dst = (uint32_t)(g_r0 * PITCH + g_ch * 16);
  const uint32_t row_bytes = (uint32_t)p.row_stride * 2u;
  int64_t g_u = -1;
  const char* g_kb = nullptr;
  const char* g_vb = nullptr;
  auto issue_data = [&](int i, int slot, int stage) {
    if (i >= ntile) return;
    const int64_t u = s_meta[slot * 4 + 0];
    const int jb = s_meta[slot * 4 + 1], cu = s_meta[slot * 4 + 2];
    if (u != g_u) {
      g_u = u;
      // the math side will load this unit's Q fragments when it gets here:
      // pull them into L2 now (M*D*2 bytes, one 128-byte line per thread)
      if (tid * 128 < M * D * 2)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(static_cast<const char*>(p.q) + u * (int64_t)M * D * 2 + tid * 128));
      g_kb = static_cast<const char*>(p.k) + ((p.kv_div > 1 ? u / p.kv_div : u) * p.kv_stride + g_ch * 8) * 2;
      g_vb = MODE == MODE_DECODE ? static_cast<const char*>(p.v) + ((p.kv_div > 1 ? u / p.kv_div : u) * p.kv_stride + g_ch * 8) * 2 : g_kb;
    }
    const uint32_t dst0 = stage_base + stage * L::STAGE + g_dst;
    const int* ring = s_idx + slot * KT;
    if (jb + KT <= cu) {
#pragma unroll
      for (int j = 0; j < GJ; ++j) {
        if (KT % GROWS != 0 && j == GJ - 1 && j >= g_n) break;
        const int r = g_r0 + j * GROWS;
        const uint32_t pr = p.idx ? (uint32_t)ring[r] : (uint32_t)(jb + r);
        const uint32_t dst = dst0 + j * GROWS * PITCH;
        cp_async_16(dst, g_kb + (uint64_t)pr * row_bytes);
        if constexpr (MODE == MODE_DECODE) cp_async_16(dst + L::KV, g_vb + (uint64_t)pr * row_bytes);
      }
    } else {
#pragma unroll
      for (int j = 0; j < GJ; ++j) {
        if (KT % GROWS != 0 && j == GJ - 1 && j >= g_n) break;
        const int r = g_r0 + j * GROWS;
        const bool ok = jb + r < cu;
        const uint32_t pr = ok ? (p.idx ? (uint32_t)ring[r] : (uint32_t)(jb + r)) : 0u;
        const uint32_t dst = dst0 + j * GROWS * PITCH;
        cp_async_16_zfill(dst, g_kb + (uint64_t)pr * row_bytes, ok);
        if constexpr (MODE == MODE_DECODE) cp_async_16_zfill(dst + L::KV, g_vb + (uint64_t)pr * row_bytes, ok);
      }
    }
  };

  // ---- per-warp running state (its 8 rows) ----
  float o[MODE == MODE_DECODE ? D / 16 : 1][4];
  float m_run[2], l_run[2], lse2[2];
  int rmod[2];
#pragma unroll
  for (int c = 0; c < 2; ++c) rmod[c] = (warp * 8 + 2 * (lane & 3) + c) % p.rows_per_head;
  const float sl2 = p.scale * LOG2E;
  const int causal_shift = p.pos_offset - p.causal_base;
  const bool causal = p.causal_base >= 0;
  const int mi = lane >> 3, ri = lane & 7;
  // per-lane ldmatrix offsets inside a 16-key block (padded rows)
  const uint32_t offK = (uint32_t)(((mi & 1) * 8 + ri) * PITCH + (mi >> 1) * 16);
  const uint32_t offV = (uint32_t)(((mi >> 1) * 8 + ri) * PITCH + (mi & 1) * 16);
  uint32_t qf[D / 16][2];  // this warp's Q^T B-fragments (loaded per unit)
  int64_t cur_u = -1;
  int cur_P = 0, cur_cnt = 0;

  auto reset_state = [&]() {
#pragma unroll
    for (int a = 0; a < (MODE == MODE_DECODE ? D / 16 : 1); ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c) o[a][c] = 0.f;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      m_run[c] = -INFINITY;
      l_run[c] = 0.f;
    }
  };

  // Q^T B-fragments straight from global: lane holds Q[row][k-step cols]
  auto load_q = [&](int64_t u) {
    const int row = warp * 8 + (lane >> 2);
    const uint32_t* qg = reinterpret_cast<const uint32_t*>(static_cast<const __nv_bfloat16*>(p.q) +
                                                           (u * M + row) * (int64_t)D) + (lane & 3);
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      qf[kk][0] = row < M ? __ldg(qg + kk * 8) : 0u;
      qf[kk][1] = row < M ? __ldg(qg + kk * 8 + 4) : 0u;
    }
    if constexpr (MODE == MODE_PROBS) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int r = warp * 8 + 2 * (lane & 3) + c;
        lse2[c] = r < M ? p.lse_in[u * M + r] * LOG2E : 0.f;
      }
    }
  };

  // finish unit u for this CTA: final rows, or partial + (last CTA) merge
  auto flush = [&](int64_t u, int P_u, int cnt_u) {
    if constexpr (MODE != MODE_PROBS) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        float l = l_run[c];
        l += __shfl_xor_sync(0xffffffffu, l, 4);
        l += __shfl_xor_sync(0xffffffffu, l, 8);
        l += __shfl_xor_sync(0xffffffffu, l, 16);
        l_run[c] = l;
      }
      const int64_t tiles = (cnt_u + KT - 1) / KT;
      const int wf = owner_of(P_u, T, W);
      const int wl = owner_of(P_u + tiles - 1, T, W);
      const bool single = wf == wl;
      const int64_t slot = (int64_t)w + u;
      float* part_o = p.o_part + slot * (int64_t)M * D;
      float* part_l = p.l_part + slot * (int64_t)M;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int r = warp * 8 + 2 * (lane & 3) + c;
        if (r >= M) continue;
        const float l = l_run[c];
        const float inv = l > 0.f ? 1.f / l : 0.f;
        const float lse = l > 0.f ? (m_run[c] + __log2f(l)) * LN2f : -INFINITY;
        if constexpr (MODE == MODE_DECODE) {
#pragma unroll
          for (int mt = 0; mt < D / 16; ++mt) {
            const int d0 = mt * 16 + (lane >> 2);
            if (single) {
              if (p.out_f32) {
                float* og = static_cast<float*>(p.out) + (u * M + r) * (int64_t)D;
                og[d0] = o[mt][c] * inv;
                og[d0 + 8] = o[mt][2 + c] * inv;
              } else {
                __nv_bfloat16* og = static_cast<__nv_bfloat16*>(p.out) + (u * M + r) * (int64_t)D;
                og[d0] = __float2bfloat16_rn(o[mt][c] * inv);
                og[d0 + 8] = __float2bfloat16_rn(o[mt][2 + c] * inv);
              }
            } else {
              part_o[r * D + d0] = o[mt][c] * inv;
              part_o[r * D + d0 + 8] = o[mt][2 + c] * inv;
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
      if (single) return;  // uniform across the CTA
      __threadfence();
      __syncthreads();
      if (tid == 0) {
        const int old = atomicAdd(p.counters + u, 1);
        const int last = old == wl - wf;
        if (last) __threadfence();
        *s_flag = last;
      }
      __syncthreads();
      const int last = *s_flag;
      if (!last) return;
      // merge CTAs wf..wl in order, the whole CTA at once: every load below is
      // independent of the others (batches of 8 / 4 partials in flight per
      // thread), so the merge costs ~3 L2 round trips instead of a serial
      // chain of 2n per row
      const int n = wl - wf + 1;
      const float* lp = p.l_part + ((int64_t)wf + u) * M;  // partial slot ww at lp + ww*M
      for (int r = tid; r < M; r += NTH) {
        float mstar = -INFINITY;
        for (int w0 = 0; w0 < n; w0 += 8) {
          float l8[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) l8[j] = w0 + j < n ? __ldcg(lp + (int64_t)(w0 + j) * M + r) : -INFINITY;
#pragma unroll
          for (int j = 0; j < 8; ++j) mstar = fmaxf(mstar, l8[j]);
        }
        float tot = 0.f;
        if (mstar != -INFINITY)
          for (int w0 = 0; w0 < n; w0 += 8) {
            float l8[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) l8[j] = w0 + j < n ? __ldcg(lp + (int64_t)(w0 + j) * M + r) : -INFINITY;
#pragma unroll
            for (int j = 0; j < 8; ++j) tot += l8[j] == -INFINITY ? 0.f : expf(l8[j] - mstar);
          }
        if (p.lse) p.lse[u * M + r] = tot > 0.f ? mstar + logf(tot) : -INFINITY;
        if (MODE == MODE_DECODE && !(tot > 0.f)) set_status(p.status, STS_DEV_EMPTY_ROW);
        s_merge[r * 2 + 0] = mstar;
        s_merge[r * 2 + 1] = tot > 0.f ? 1.f / tot : 0.f;
      }
      if constexpr (MODE == MODE_DECODE) {
        __syncthreads();
        constexpr int D4 = D / 4;
        const float* op = p.o_part + ((int64_t)wf + u) * M * D;  // slot ww at op + ww*M*D
        for (int e = tid; e < M * D4; e += NTH) {
          const int r = e / D4, d4 = e % D4;
          const float mstar = s_merge[r * 2], inv = s_merge[r * 2 + 1];
          float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
          if (inv > 0.f) {
            for (int w0 = 0; w0 < n; w0 += 4) {
              float l4[4];
              float4 x4[4];
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const bool ok = w0 + j < n;
                l4[j] = ok ? __ldcg(lp + (int64_t)(w0 + j) * M + r) : -INFINITY;
                x4[j] = ok ? __ldcg(reinterpret_cast<const float4*>(op + ((int64_t)(w0 + j) * M + r) * D) + d4)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
              }
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float f = l4[j] == -INFINITY ? 0.f : expf(l4[j] - mstar) * inv;
                acc.x += f * x4[j].x;
                acc.y += f * x4[j].y;
                acc.z += f * x4[j].z;
                acc.w += f * x4[j].w;
              }
            }
          }
          if (p.out_f32) {
            *reinterpret_cast<float4*>(static_cast<float*>(p.out) + (u * M + r) * (int64_t)D + 4 * d4) = acc;
          } else {
            __nv_bfloat16* og = static_cast<__nv_bfloat16*>(p.out) + (u * M + r) * (int64_t)D + 4 * d4;
            *reinterpret_cast<__nv_bfloat162*>(og) = __floats2bfloat162_rn(acc.x, acc.y);
            *reinterpret_cast<__nv_bfloat162*>(og + 2) = __floats2bfloat162_rn(acc.z, acc.w);
          }
        }
      }
      __syncthreads();  // s_merge / the stage buffers are reused by the caller
    }
  };

  // ---- pipeline: idx slices STAGES tiles ahead, K/V STAGES-1 tiles ahead ----
  for (int kk = 0; kk < STAGES; ++kk) issue_idx(kk);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
#pragma unroll
  for (int s0 = 0; s0 < STAGES - 1; ++s0) {
    issue_data(s0, s0, s0);
    issue_idx(s0 + STAGES);
    cp_async_commit();
  }

  for (int i = 0; i < ntile; ++i) {
    const int slot = i & (L::RING - 1), stage = i % STAGES;
    cp_async_wait<STAGES - 2>();  // this thread's gathers of tile i landed (and idx of tile i+STAGES-1)
    __syncthreads();              // ... everyone's; everyone is done with tile i-1
    issue_data(i + STAGES - 1, (i + STAGES - 1) & (L::RING - 1), (i + STAGES - 1) % STAGES);  // refill tile i-1's stage
    issue_idx(i + 2 * STAGES - 1);
    cp_async_commit();

    const int64_t u = s_meta[slot * 4 + 0];
    const int j0 = s_meta[slot * 4 + 1];
    if (u != cur_u) {
      if (cur_u >= 0) flush(cur_u, cur_P, cur_cnt);
      cur_u = u;
      cur_cnt = s_meta[slot * 4 + 2];
      cur_P = s_meta[slot * 4 + 3];
      reset_state();
      load_q(u);
    }
    const uint32_t sk0 = stage_base + stage * L::STAGE;
    // fast path: all keys valid, no membership bits, tile inside the committed
    // prefix (positions ascending) -> no per-element masking
    const bool simple = (j0 + KT <= cur_cnt) && !p.member && (!causal || slot_pos(slot, KT - 1) + causal_shift <= 0);

    float s[SUB][4];
    bool okA[SUB][2], okB[SUB][2];
#pragma unroll
    for (int sub = 0; sub < SUB; ++sub) {
      const bool live = j0 + sub * KEY_TILE < cur_cnt;
      const uint32_t ak = sk0 + sub * L::SUBB + offK;
#pragma unroll
      for (int c = 0; c < 4; ++c) s[sub][c] = 0.f;
      if (live) {
        // two independent accumulators halve the MMA dependency chain
        float s1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int kk = 0; kk < D / 16; kk += 2) {
          uint32_t a0[4], a1[4];
          ldmatrix_x4(a0[0], a0[1], a0[2], a0[3], ak + kk * 32);
          ldmatrix_x4(a1[0], a1[1], a1[2], a1[3], ak + kk * 32 + 32);
          mma_bf16_16816(s[sub], a0, qf[kk]);
          mma_bf16_16816(s1, a1, qf[kk + 1]);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) s[sub][c] += s1[c];
      }
      if (simple) {
        okA[sub][0] = okA[sub][1] = okB[sub][0] = okB[sub][1] = true;
      } else {
        const int kA = (lane >> 2) + sub * KEY_TILE, kB = kA + 8;
        const int posA = live ? slot_pos(slot, kA) : -1;
        const int posB = live ? slot_pos(slot, kB) : -1;
        const uint32_t memA = p.member ? s_mem[slot * KT + kA] : 0xffffffffu;
        const uint32_t memB = p.member ? s_mem[slot * KT + kB] : 0xffffffffu;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int r = warp * 8 + 2 * (lane & 3) + c;
          bool a_ = posA >= 0, b_ = posB >= 0;
          if (causal) {
            a_ = a_ && (posA + causal_shift <= rmod[c]);
            b_ = b_ && (posB + causal_shift <= rmod[c]);
          }
          okA[sub][c] = a_ && ((memA >> (r & 31)) & 1u);
          okB[sub][c] = b_ && ((memB >> (r & 31)) & 1u);
        }
      }
    }

    if constexpr (MODE == MODE_PROBS) {
      // every warp writes its rows' probabilities; the CTA then reduces over
      // the speculative rows of each head (a head's rows can span warps)
      const int lk = lane >> 2;
#pragma unroll
      for (int sub = 0; sub < SUB; ++sub)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int r = warp * 8 + 2 * (lane & 3) + c;
          s_prob[(sub * 16 + lk) * MP + r] = okA[sub][c] ? fast_exp2(s[sub][c] * sl2 - lse2[c]) : 0.f;
          s_prob[(sub * 16 + lk + 8) * MP + r] = okB[sub][c] ? fast_exp2(s[sub][2 + c] * sl2 - lse2[c]) : 0.f;
        }
      __syncthreads();
      const int R = p.rows_per_head;
      const int G = M / R;
      if (p.probs_mode == 0) {
        for (int e2 = tid; e2 < KT * G; e2 += NTH) {
          const int key = e2 % KT, hh = e2 / KT;
          const int pos = slot_pos(slot, key);
          if (pos >= 0 && pos + p.pos_offset < p.causal_base) {
            float acc = s_prob[key * MP + hh * R];
            for (int ii = 1; ii < R; ++ii) acc = __fadd_rn(acc, s_prob[key * MP + hh * R + ii]);
            p.probs_out[(u * G + hh) * p.out_ld + j0 + key] = acc;
          }
        }
      } else {
        for (int e2 = tid; e2 < KT * M; e2 += NTH) {
          const int key = e2 % KT, r = e2 / KT;
          const int pos = slot_pos(slot, key);
          if (pos >= 0 && pos + p.pos_offset <= p.causal_base + r % R)
            p.probs_out[(u * M + r) * p.out_ld + j0 + key] = s_prob[key * MP + r];
        }
      }
      // the next iteration's barrier orders these reads before s_prob reuse
    } else {
      float pv[SUB][4];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        float tmax = -INFINITY;
#pragma unroll
        for (int sub = 0; sub < SUB; ++sub) {
          const float vA = okA[sub][c] ? s[sub][c] * sl2 : -INFINITY;
          const float vB = okB[sub][c] ? s[sub][2 + c] * sl2 : -INFINITY;
          s[sub][c] = vA;
          s[sub][2 + c] = vB;
          tmax = fmaxf(tmax, fmaxf(vA, vB));
        }
        tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 4));
        tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 8));
        tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 16));
        const float m_old = m_run[c];
        const float m_new = fmaxf(m_old, tmax);
        float alpha = 1.f, psum = 0.f;
        if (m_new != -INFINITY) {
          alpha = fast_exp2(m_old - m_new);
#pragma unroll
          for (int sub = 0; sub < SUB; ++sub) {
            pv[sub][c] = fast_exp2(s[sub][c] - m_new);
            pv[sub][2 + c] = fast_exp2(s[sub][2 + c] - m_new);
            psum += pv[sub][c] + pv[sub][2 + c];
          }
        } else {
#pragma unroll
          for (int sub = 0; sub < SUB; ++sub) pv[sub][c] = pv[sub][2 + c] = 0.f;
        }
        m_run[c] = m_new;
        l_run[c] = l_run[c] * alpha + psum;
        if constexpr (MODE == MODE_DECODE) {
          if (__any_sync(0xffffffffu, alpha != 1.f)) {  // the running max rarely moves
#pragma unroll
            for (int mt = 0; mt < D / 16; ++mt) {
              o[mt][c] *= alpha;
              o[mt][2 + c] *= alpha;
            }
          }
        }
      }
      if constexpr (MODE == MODE_DECODE) {
#pragma unroll
        for (int sub = 0; sub < SUB; ++sub) {
          if (j0 + sub * KEY_TILE >= cur_cnt) break;
          const uint32_t av = sk0 + L::KV + sub * L::SUBB + offV;
          const uint32_t b[2] = {movmatrix_trans(pack_bf16(pv[sub][0], pv[sub][1])),
                                 movmatrix_trans(pack_bf16(pv[sub][2], pv[sub][3]))};
#pragma unroll
          for (int mt = 0; mt < D / 16; ++mt) {
            uint32_t a[4];
            ldmatrix_x4_trans(a[0], a[1], a[2], a[3], av + mt * 32);
            mma_bf16_16816(o[mt], a, b);
          }
        }
      }
    }
  }
  cp_async_wait<0>();
  if (cur_u >= 0) flush(cur_u, cur_P, cur_cnt);
}

template <int D, int NT, int MODE>
struct GCfg {
  static constexpr int SUB = MODE == MODE_DECODE ? 2 : (D == 64 ? 4 : 2);
  // measured on B200 (d=128, M=20): 32-key stages x2 (6 CTAs/SM) > x3 (4/SM) > 16 x4
  static constexpr int STAGES = MODE == MODE_DECODE && D == 128 ? 2 : 4;
  using L = GL<D, NT, MODE, SUB, STAGES>;
};

template <int D, int NT, int MODE, int SUB, int STAGES>
int launch_cfg(DecodeParams& p, cudaStream_t st) {
  using L = GL<D, NT, MODE, SUB, STAGES>;
  static_assert(L::SMEM <= 227 * 1024, "gather kernel shared memory");
  auto kern = gather_kernel<D, NT, MODE, SUB, STAGES>;
  // attribute + occupancy once per instantiation (thread-safe static init);
  // the launch path is then a single <<<>>> (cheap enough for per-step calls)
  static const int per_sm = [&]() {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM) != cudaSuccess) return -1;
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, L::THREADS, L::SMEM) != cudaSuccess) return -1;
    return n < 1 ? 1 : n;
  }();
  STS_REQUIRE(per_sm > 0, STS_ERR_CUDA, "gather kernel setup failed: %s", cudaGetErrorString(cudaGetLastError()));
  kern<<<num_sms() * per_sm, L::THREADS, L::SMEM, st>>>(p);
  STS_LAUNCH_CHECK();
  return STS_OK;
}

// pipeline shape of the d=128, M<=24 decode (the headline configuration):
// STS_GATHER_CFG = 0: 32-key stages x2 (default), 1: 32 x3, 2: 16 x4, 3: 64 x2
int decode_cfg() {
  static int cfg = -1;
  if (cfg < 0) {
    const char* e = getenv("STS_GATHER_CFG");
    cfg = e ? atoi(e) : 0;
    if (cfg < 0 || cfg > 3) cfg = 0;
  }
  return cfg;
}

template <int D, int NT, int MODE>
int launch_gather(DecodeParams& p, cudaStream_t st) {
  if constexpr (D == 128 && NT == 3 && MODE == MODE_DECODE) {
    switch (decode_cfg()) {
      case 1: return launch_cfg<D, NT, MODE, 2, 3>(p, st);
      case 2: return launch_cfg<D, NT, MODE, 1, 4>(p, st);
      case 3: return launch_cfg<D, NT, MODE, 4, 2>(p, st);
      default: break;
    }
  }
  using C = GCfg<D, NT, MODE>;
  return launch_cfg<D, NT, MODE, C::SUB, C::STAGES>(p, st);
}

template <int D, int MODE>
int gdispatch_nt(DecodeParams& p, cudaStream_t st) {
  switch ((p.M + 7) / 8) {
    case 1: return launch_gather<D, 1, MODE>(p, st);
    case 2: return launch_gather<D, 2, MODE>(p, st);
    case 3: return launch_gather<D, 3, MODE>(p, st);
    case 4: return launch_gather<D, 4, MODE>(p, st);
    case 5: return launch_gather<D, 5, MODE>(p, st);
    default: set_error("bf16 gather kernels support M <= 40 stacked rows, got %d", p.M); return STS_ERR_CONTRACT;
  }
}

template <int MODE>
int gdispatch_d(DecodeParams& p, cudaStream_t st) {
  if (p.d == 128) return gdispatch_nt<128, MODE>(p, st);
  if (p.d == 64) return gdispatch_nt<64, MODE>(p, st);
  set_error("bf16 gather kernels support d in {64, 128}, got %d", p.d);
  return STS_ERR_CONTRACT;
}

}  // namespace

int gather_launch(int mode, DecodeParams& p, cudaStream_t st) {
  // product path: sts_verify_decode.cu; STS_DECODE_LEGACY=1 selects the
  // row-split kernels below (kept for A/B measurements)
  static const bool legacy = getenv("STS_DECODE_LEGACY") && atoi(getenv("STS_DECODE_LEGACY")) == 1;
  if (!legacy) return verify_decode_launch(mode, p, st);
  if (mode == MODE_DECODE) return gdispatch_d<MODE_DECODE>(p, st);
  if (mode == MODE_LSE) return gdispatch_d<MODE_LSE>(p, st);
  return gdispatch_d<MODE_PROBS>(p, st);
}

}  // namespace sts
