// sts_verify_decode.cu — gathered-KV sparse flash-decode of the stacked
// verification rows (bf16, sm_100a).  The product kernel of sts_sparse_decode.
//
// Work decomposition (as the gather kernel of sts_gather.cu): unit = (batch,
// layer, kv-head); the key tiles of all units form one global tile space cut
// into equal contiguous ranges, one per CTA (persistent stream-K, grid = SMs x
// resident CTAs); units split over CTAs are merged by the last CTA to arrive.
//
// Math layout: one warp per 16 stacked query rows (M = GQA group x (gamma+1);
// M = 20 -> 2 warps, M = 40 -> 3), each warp walks ALL keys of the tile:
//   S (16 rows x 8 keys) = Q (A, registers, loaded once per unit) . K^T
//     (B fragments: ldmatrix of the gathered K rows, 4 independent n-tiles)
//   P stays in registers: the S accumulator layout IS the A-fragment layout of
//     the next MMA (no shared-memory round trip, no transpose)
//   O (16 rows x D) += P . V  (B fragments: ldmatrix.trans of the gathered V)
// Softmax statistics are per row, reduced over the 4 lanes of a quad, so a
// 32-key tile costs each thread 16 exponentials and 2 shuffles per row.
//
// Gather: 16-byte cp.async into padded rows (2d+16 bytes: conflict-free
// ldmatrix), one IMAD.WIDE + LDGSTS per copy (32-bit row offsets), STAGES
// deep, continuous across unit boundaries; index slices prefetched a ring ahead.
#include "sts_decode.cuh"

namespace sts {
namespace {

constexpr float LN2 = 0.6931471805599453f;

// Optional per-CTA timeline (tuning builds only: -DSTS_TRACE, read back with
// sts_debug_trace): entry, first issue, first tile ready, loop end, exit,
// ns spent in unit flushes, flush count, tiles.
#ifdef STS_TRACE
__device__ unsigned long long g_trace[8192 * 8];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define STS_TRACE_AT(k) \
  if (threadIdx.x == 0 && blockIdx.x < 8192) g_trace[blockIdx.x * 8 + (k)] = gtimer()
#define STS_TRACE_ADD(k, v) \
  if (threadIdx.x == 0 && blockIdx.x < 8192) g_trace[blockIdx.x * 8 + (k)] += (v)
#else
#define STS_TRACE_AT(k)
#define STS_TRACE_ADD(k, v)
#endif

__device__ __forceinline__ void cp_async_4z(uint32_t dst, const void* src, bool valid) {
  int sz = valid ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src), "r"(sz));
}

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cta address -> the same offset in CTA `rank` of this cluster
__device__ __forceinline__ uint32_t dsmem_map(uint32_t addr, unsigned rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ float4 dsmem_ld4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr) : "memory");
  return v;
}

__device__ __forceinline__ int unit_tiles(const DecodeParams& p, int64_t u, int KT) {
  const int c = p.idx ? p.cnt[u] : p.n_dense;
  return (c + KT - 1) / KT;
}


// resident warps per SM the draft (K-only) kernels' register budget targets
#ifndef STS_DRAFT_WARPS
#define STS_DRAFT_WARPS 16
#endif

template <int D, int NW, int KT, int STAGES, int MODE>
struct VL {
  static constexpr bool K_ONLY = MODE != MODE_DECODE;
  static constexpr int THREADS = NW * 32;
  static constexpr int CH = D / 8;                // 16-byte chunks per row
  static constexpr int PITCH = D * 2 + 16;        // padded row
  static constexpr int KV = KT * PITCH;           // K block -> V block
  static constexpr int STAGE = (K_ONLY ? 1 : 2) * KV;
  static constexpr int RING = STAGES <= 2 ? 4 : 8;  // index ring (power of 2, >= 2*STAGES)
  static constexpr int IDX_BYTES = RING * KT * 4;
  static constexpr int META_BYTES = RING * 32;
  static constexpr int MERGE = NW * 16 * 2 * 4;
  static constexpr int SMEM = STAGES * STAGE + 2 * IDX_BYTES + META_BYTES + MERGE + 16;
  // resident CTAs per SM the register allocation must allow: the shared-memory
  // limit, capped so a warp keeps ~168 registers (O, Q fragments, S, P)
  static constexpr int SMEM_CTAS = (227 * 1024) / (SMEM + 1024);
  static constexpr int REG_CTAS = K_ONLY ? STS_DRAFT_WARPS / NW : (NW == 1 ? 12 : (NW == 2 ? 6 : 3));
  static constexpr int MINB = SMEM_CTAS < REG_CTAS ? (SMEM_CTAS < 1 ? 1 : SMEM_CTAS) : REG_CTAS;
  static constexpr int GROWS = THREADS / CH;      // rows per gather pass
  static constexpr int GJ = (KT + GROWS - 1) / GROWS;
  static_assert(THREADS % CH == 0, "gather mapping");
  static_assert(KT % 16 == 0, "key tile");
};

template <int D, int NW, int KT, int STAGES, int MODE, int CS>
__global__ void __launch_bounds__(NW * 32, (VL<D, NW, KT, STAGES, MODE>::MINB)) verify_decode_kernel(DecodeParams p) {
  using L = VL<D, NW, KT, STAGES, MODE>;
  constexpr int NTH = L::THREADS, PITCH = L::PITCH, CH = L::CH;
  constexpr int NT = KT / 8;   // 8-key n-tiles of S per tile
  constexpr int KS = KT / 16;  // 16-key k-steps of P.V per tile
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int M = p.M;
  const int64_t U = p.units;
  // let the (programmatically dependent) merge grid launch now; it waits for
  // this grid's completion before reading anything
  asm volatile("griddepcontrol.launch_dependents;");
#ifdef STS_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 8192)
    for (int k = 0; k < 8; ++k) g_trace[blockIdx.x * 8 + k] = 0;
#endif
  STS_TRACE_AT(0);

  uint8_t* s_stage = smem;
  int* s_idx = reinterpret_cast<int*>(s_stage + STAGES * L::STAGE);
  uint32_t* s_mem = reinterpret_cast<uint32_t*>(s_idx + L::RING * KT);
  int* s_meta = reinterpret_cast<int*>(s_mem + L::RING * KT);
  float* s_merge = reinterpret_cast<float*>(s_meta + L::RING * 8);
  int* s_flag = reinterpret_cast<int*>(s_merge + L::MERGE / 4);
  const uint32_t stage_base = smem_u32(s_stage);
  const uint32_t idx_base = smem_u32(s_idx);
  const uint32_t mem_base = smem_u32(s_mem);

  // ---- units with no keys (striped over CTAs): zero rows, LSE -inf ----
  for (int64_t u = blockIdx.x; u < U; u += gridDim.x) {
    if (unit_tiles(p, u, KT) != 0) continue;
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
    if (p.lse)
      for (int r = tid; r < M; r += NTH) p.lse[u * M + r] = -INFINITY;
  }

  // ---- tile space and this CTA's range (block-parallel scan) ----
  // (the cluster schedule needs none of this: each cluster knows its unit)
  __shared__ long long s_scan[NW + 3];
  const int64_t cpt = (U + NTH - 1) / NTH;
  const int64_t ub = (int64_t)tid * cpt, ue = CS > 1 ? ub : (ub + cpt < U ? ub + cpt : U);
  int64_t mine = 0;
  for (int64_t u0 = ub; u0 < ue; u0 += 4) {
    int t4[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) t4[j] = u0 + j < ue ? unit_tiles(p, u0 + j, KT) : 0;
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
  for (int ww = 0; ww < NW; ++ww) {
    const int64_t v = s_scan[ww];
    before += ww < warp ? v : 0;
    T += v;
  }
  if (CS == 1 && T == 0) return;

  // ---- schedule.  CS == 1: one contiguous tile range per CTA (stream-K); a
  // piece of a unit is (CTA range, unit), its partial slot is range + unit, and
  // units split over several ranges are merged afterwards in range order
  // (merge_pieces_kernel) — deterministic.  CS > 1: a thread-block cluster of
  // CS CTAs per unit, each taking an equal contiguous share of the unit's
  // tiles; the shares are merged through distributed shared memory at the end
  // (no global partials, no second kernel).
  int W, w;
  int64_t s_w, iu, iP;
  int ntile, icnt;
  [[maybe_unused]] unsigned crank = 0;
  if constexpr (CS > 1) {
    crank = cluster_rank();
    iu = blockIdx.x / CS;
    icnt = iu < U ? (p.idx ? p.cnt[iu] : p.n_dense) : 0;
    const int64_t T_u = (icnt + KT - 1) / KT;
    W = CS;
    w = (int)crank;
    s_w = (int64_t)w * T_u / CS;
    ntile = (int)((int64_t)(w + 1) * T_u / CS - s_w);
    iP = 0;
  } else {
    W = (int)(T < (int64_t)gridDim.x ? T : (int64_t)gridDim.x);
    w = blockIdx.x;
    if (w >= W) return;
    s_w = (int64_t)w * T / W;
    ntile = (int)((int64_t)(w + 1) * T / W - s_w);
    int64_t acc = before + incl - mine;
    if (acc <= s_w && s_w < acc + mine) {
      for (int64_t u = ub; u < ue; ++u) {
        const int t_u = unit_tiles(p, u, KT);
        if (s_w < acc + t_u) {
          s_scan[NW] = u;
          s_scan[NW + 1] = acc;
          s_scan[NW + 2] = p.idx ? p.cnt[u] : p.n_dense;  // (an L1 hit: just loaded)
          break;
        }
        acc += t_u;
      }
    }
    __syncthreads();
    iu = s_scan[NW];
    iP = s_scan[NW + 1];
    icnt = (int)s_scan[NW + 2];
  }
  auto owner = [&](int64_t t) -> int64_t { return ((t + 1) * W - 1) / T; };
  // uniform cursor of the index side (every thread holds the same values)
  int64_t iPn = iP + (icnt + KT - 1) / KT;

  // ---- index slices: tile i of this CTA -> ring slot i & (RING-1) (+ meta) ----
  auto issue_idx = [&](int i) {
    const int slot = i & (L::RING - 1);
    int* meta = s_meta + slot * 8;
    if (i >= ntile) {
      if (tid == 0) meta[0] = -1;
      return;
    }
    const int64_t t = s_w + i;
    while (t >= iPn) {
      ++iu;
      iP = iPn;
      icnt = p.idx ? p.cnt[iu] : p.n_dense;
      iPn = iP + (icnt + KT - 1) / KT;
    }
    const int j0 = (int)(t - iP) * KT;
    if (tid == 0) {
      meta[0] = (int)iu;
      meta[1] = j0;
      meta[2] = icnt;
      meta[3] = (int)iP;
      meta[4] = w;
    }
    if (p.idx) {
      for (int e = tid; e < KT; e += NTH) {
        const bool ok = j0 + e < icnt;
        cp_async_4z(idx_base + (slot * KT + e) * 4, p.idx + iu * p.idx_ld + (ok ? j0 + e : 0), ok);
        if (p.member)
          cp_async_4z(mem_base + (slot * KT + e) * 4, p.member + iu * p.idx_ld + (ok ? j0 + e : 0), ok);
      }
    }
  };

  // ---- K/V gather (thread -> chunk g_ch of rows g_r0 + GROWS*j) ----
  constexpr int GROWS = L::GROWS, GJ = L::GJ;
  const int g_ch = tid % CH, g_r0 = tid / CH;
  const int g_n = (KT - g_r0 + GROWS - 1) / GROWS;
  const uint32_t g_dst = (uint32_t)(g_r0 * PITCH + g_ch * 16);
  const uint32_t row_bytes = (uint32_t)p.row_stride * 2u;
  int64_t g_u = -1;
  const char* g_kb = nullptr;
  const char* g_vb = nullptr;
  auto issue_data = [&](int i) {
    const int slot = i & (L::RING - 1), stage = i % STAGES;
    const int64_t u = s_meta[slot * 8 + 0];
    if (u < 0) return;
    const int jb = s_meta[slot * 8 + 1], cu = s_meta[slot * 8 + 2];
    if (u != g_u) {
      g_u = u;
      if (tid * 128 < M * D * 2)  // this unit's Q into L2 ahead of the math side
        asm volatile("prefetch.global.L2 [%0];" ::"l"(static_cast<const char*>(p.q) + u * (int64_t)M * D * 2 + tid * 128));
      const int64_t ukv = p.kv_div > 1 ? u / p.kv_div : u;  // the unit's K/V block
      g_kb = static_cast<const char*>(p.k) + (ukv * p.kv_stride + g_ch * 8) * 2;
      if constexpr (MODE == MODE_DECODE) g_vb = static_cast<const char*>(p.v) + (ukv * p.kv_stride + g_ch * 8) * 2;
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

  // ---- per-warp state: rows rA = 16*warp + lane/4 and rB = rA + 8 ----
  const int rA = warp * 16 + (lane >> 2), rB = rA + 8;
  const int rmodA = rA % p.rows_per_head, rmodB = rB % p.rows_per_head;
  const bool rB_live = warp * 16 + 8 < M;  // warp-uniform: this warp's rB rows hold queries
  const float sl2 = p.scale * LOG2E;
  const int causal_shift = p.pos_offset - p.causal_base;
  const bool causal = p.causal_base >= 0;
  float o[MODE == MODE_DECODE ? D / 8 : 1][4];
  float m_a = -INFINITY, m_b = -INFINITY, l_a = 0.f, l_b = 0.f;
  uint32_t qa[D / 16][4];
  // ldmatrix lane offsets: K (B of QK^T, non-trans): key (lane&7), dim block (lane>>3)*8
  const uint32_t offK = (uint32_t)((lane & 7) * PITCH + (lane >> 3) * 16);
  // V (B of P.V, trans): key (lane&7) + ((lane>>3)&1)*8, dim block (lane>>4)*8
  const uint32_t offV = (uint32_t)(((lane & 7) + ((lane >> 3) & 1) * 8) * PITCH + (lane >> 4) * 16);
  int64_t cur_u = -1;
  int cur_P = 0, cur_cnt = 0;

  auto reset_state = [&]() {
#pragma unroll
    for (int a = 0; a < (MODE == MODE_DECODE ? D / 8 : 1); ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c) o[a][c] = 0.f;
    m_a = m_b = -INFINITY;
    l_a = l_b = 0.f;
  };
  auto load_q = [&](int64_t u) {
    const uint32_t* qA = reinterpret_cast<const uint32_t*>(static_cast<const __nv_bfloat16*>(p.q) +
                                                           (u * M + rA) * (int64_t)D) + (lane & 3);
    const uint32_t* qB = qA + 8 * D / 2;
    const bool okA = rA < M, okB = rB < M;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      qa[kk][0] = okA ? __ldg(qA + kk * 8) : 0u;
      qa[kk][1] = okB ? __ldg(qB + kk * 8) : 0u;
      qa[kk][2] = okA ? __ldg(qA + kk * 8 + 4) : 0u;
      qa[kk][3] = okB ? __ldg(qB + kk * 8 + 4) : 0u;
    }
  };

  // ---- finish unit u for this CTA: final rows, or partial + last-CTA merge ----
  auto flush = [&](int64_t u, int P_u, int cnt_u, int64_t range) {
    float la = l_a, lb = l_b;
    la += __shfl_xor_sync(0xffffffffu, la, 1);
    la += __shfl_xor_sync(0xffffffffu, la, 2);
    lb += __shfl_xor_sync(0xffffffffu, lb, 1);
    lb += __shfl_xor_sync(0xffffffffu, lb, 2);
    const int64_t tiles = (cnt_u + KT - 1) / KT;
    const int64_t wf = owner(P_u);
    const int64_t wl = owner(P_u + tiles - 1);
    const bool single = wf == wl;
    const int64_t pslot = range + u;
    const float inv_a = la > 0.f ? 1.f / la : 0.f, inv_b = lb > 0.f ? 1.f / lb : 0.f;
    const float lse_a = la > 0.f ? (m_a + __log2f(la)) * LN2 : -INFINITY;
    const float lse_b = lb > 0.f ? (m_b + __log2f(lb)) * LN2 : -INFINITY;
    const int dc = 2 * (lane & 3);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = h ? rB : rA;
      if (r >= M) continue;
      const float inv = h ? inv_b : inv_a;
      if constexpr (MODE != MODE_DECODE) {
        (void)inv;
      } else if (single) {
        if (p.out_f32) {
          float* og = static_cast<float*>(p.out) + (u * M + r) * (int64_t)D + dc;
#pragma unroll
          for (int nt = 0; nt < D / 8; ++nt)
            *reinterpret_cast<float2*>(og + nt * 8) = make_float2(o[nt][2 * h] * inv, o[nt][2 * h + 1] * inv);
        } else {
          __nv_bfloat16* og = static_cast<__nv_bfloat16*>(p.out) + (u * M + r) * (int64_t)D + dc;
#pragma unroll
          for (int nt = 0; nt < D / 8; ++nt)
            *reinterpret_cast<__nv_bfloat162*>(og + nt * 8) =
                __floats2bfloat162_rn(o[nt][2 * h] * inv, o[nt][2 * h + 1] * inv);
        }
      } else {
        float* og = p.o_part + (pslot * M + r) * (int64_t)D + dc;
#pragma unroll
        for (int nt = 0; nt < D / 8; ++nt)
          *reinterpret_cast<float2*>(og + nt * 8) = make_float2(o[nt][2 * h] * inv, o[nt][2 * h + 1] * inv);
      }
      if ((lane & 3) == 0) {
        const float lse = h ? lse_b : lse_a;
        const bool empty = !((h ? lb : la) > 0.f);
        if (single) {
          if (p.lse) p.lse[u * M + r] = lse;
          if (MODE == MODE_DECODE && empty) set_status(p.status, STS_DEV_EMPTY_ROW);
        } else {
          p.l_part[pslot * M + r] = lse;
        }
      }
    }
    // the piece holding the unit's first tile records the unit's range span;
    // split units are merged by merge_pieces_kernel after this kernel
    if (range == wf && tid == 0) p.pieces[u] = make_int2((int)wf, (int)wl);
  };

  // ---- pipeline: idx slices STAGES tiles ahead, K/V STAGES-1 tiles ahead ----
  STS_TRACE_AT(1);
#ifdef STS_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 8192) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_trace[blockIdx.x * 8 + 7] = (unsigned long long)ntile | ((unsigned long long)smid << 32);
  }
#endif
  for (int kk = 0; kk < STAGES; ++kk) {
    if (kk) __syncthreads();
    issue_idx(kk);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
#pragma unroll
  for (int s0 = 0; s0 < STAGES - 1; ++s0) {
    if (s0) __syncthreads();
    issue_data(s0);
    issue_idx(s0 + STAGES);
    cp_async_commit();
  }

  int64_t cur_range = -1;
  reset_state();  // (a cluster CTA with no tiles still contributes an empty share)
  for (int i = 0;; ++i) {
    const int slot = i & (L::RING - 1), stage = i % STAGES;
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    issue_data(i + STAGES - 1);
    issue_idx(i + 2 * STAGES - 1);
    cp_async_commit();

#ifdef STS_TRACE
    if (i == 0) STS_TRACE_AT(2);
#endif
    const int64_t u = s_meta[slot * 8 + 0];
    if (u < 0) break;
    const int j0 = s_meta[slot * 8 + 1];
    const int64_t range = s_meta[slot * 8 + 4];
    if (u != cur_u || range != cur_range) {
#ifdef STS_TRACE
      const unsigned long long tf0 = gtimer();
#endif
      if (cur_u >= 0) flush(cur_u, cur_P, cur_cnt, cur_range);
#ifdef STS_TRACE
      if (cur_u >= 0) {
        STS_TRACE_ADD(5, gtimer() - tf0);
        STS_TRACE_ADD(6, 1);
      }
#endif
      const bool new_unit = u != cur_u;
      cur_u = u;
      cur_range = range;
      cur_cnt = s_meta[slot * 8 + 2];
      cur_P = s_meta[slot * 8 + 3];
      reset_state();
      if (new_unit) load_q(u);
    }
    const uint32_t sk = stage_base + stage * L::STAGE;
    const int* ring = s_idx + slot * KT;
    const int nvalid = cur_cnt - j0;  // keys of this tile that exist (>= 1)
    // fast path: all keys valid, no membership bits, tile entirely at or
    // before the causal base (positions ascending)
    const int last_pos = p.idx ? ring[KT - 1] : j0 + KT - 1;
    const bool simple = nvalid >= KT && !p.member && (!causal || last_pos + causal_shift <= 0);

    // S = Q K^T : NT independent 16x8 accumulators
    float s[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
      for (int c = 0; c < 4; ++c) s[nt][c] = 0.f;
      const uint32_t ak = sk + nt * 8 * PITCH + offK;
#pragma unroll
      for (int kk = 0; kk < D / 16; kk += 2) {
        uint32_t b[4];
        ldmatrix_x4(b[0], b[1], b[2], b[3], ak + kk * 32);
        const uint32_t b0[2] = {b[0], b[1]}, b1[2] = {b[2], b[3]};
        mma_bf16_16816(s[nt], qa[kk], b0);
        mma_bf16_16816(s[nt], qa[kk + 1], b1);
      }
    }
    // scale to log2 units
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int c = 0; c < 4; ++c) s[nt][c] *= sl2;

    if (!simple) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int key = nt * 8 + 2 * (lane & 3) + e;
          const bool valid = key < nvalid;
          const int pos = valid ? (p.idx ? ring[key] : j0 + key) : 0;
          const uint32_t mem = p.member ? s_mem[slot * KT + key] : 0xffffffffu;
          bool okA = valid && ((mem >> (rA & 31)) & 1u);
          bool okB = valid && ((mem >> (rB & 31)) & 1u);
          if (causal) {
            okA = okA && (pos + causal_shift <= rmodA);
            okB = okB && (pos + causal_shift <= rmodB);
          }
          if (!okA) s[nt][e] = -INFINITY;
          if (!okB) s[nt][2 + e] = -INFINITY;
        }
    }
    // online softmax (rows rA: s[.][0..1], rB: s[.][2..3])
    float tA = -INFINITY, tB = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      tA = fmaxf(tA, fmaxf(s[nt][0], s[nt][1]));
      tB = fmaxf(tB, fmaxf(s[nt][2], s[nt][3]));
    }
    tA = fmaxf(tA, __shfl_xor_sync(0xffffffffu, tA, 1));
    tA = fmaxf(tA, __shfl_xor_sync(0xffffffffu, tA, 2));
    if (rB_live) {
      tB = fmaxf(tB, __shfl_xor_sync(0xffffffffu, tB, 1));
      tB = fmaxf(tB, __shfl_xor_sync(0xffffffffu, tB, 2));
    } else {
      tB = 0.f;  // padding rows: keep their state constant (m = 0, nothing accumulated)
    }
    const float nA = fmaxf(m_a, tA), nB = rB_live ? fmaxf(m_b, tB) : 0.f;
    // rows with no admissible key yet keep everything at zero
    const float bA = nA == -INFINITY ? 0.f : nA, bB = nB == -INFINITY ? 0.f : nB;
    const float alA = fast_exp2(m_a - bA), alB = rB_live ? fast_exp2(m_b - bB) : 1.f;
    m_a = nA;
    m_b = nB;
    float sumA = 0.f, sumB = 0.f;
    uint32_t pa[KS][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const float p0 = fast_exp2(s[nt][0] - bA), p1 = fast_exp2(s[nt][1] - bA);
      // rows rB of the last warp are often all padding (M = 20: rows 24..31)
      const float p2 = rB_live ? fast_exp2(s[nt][2] - bB) : 0.f, p3 = rB_live ? fast_exp2(s[nt][3] - bB) : 0.f;
      sumA += p0 + p1;
      sumB += p2 + p3;
      if constexpr (MODE == MODE_DECODE) {
        pa[nt >> 1][(nt & 1) * 2 + 0] = pack_bf16(p0, p1);
        pa[nt >> 1][(nt & 1) * 2 + 1] = pack_bf16(p2, p3);
      }
    }
    l_a = l_a * alA + sumA;
    l_b = l_b * alB + sumB;
    if constexpr (MODE == MODE_DECODE) {
      if (__any_sync(0xffffffffu, alA != 1.f || alB != 1.f)) {
#pragma unroll
        for (int nt = 0; nt < D / 8; ++nt) {
          o[nt][0] *= alA;
          o[nt][1] *= alA;
          o[nt][2] *= alB;
          o[nt][3] *= alB;
        }
      }
      // O += P V
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const uint32_t av = sk + L::KV + ks * 16 * PITCH + offV;
#pragma unroll
        for (int n2 = 0; n2 < D / 16; ++n2) {
          uint32_t b[4];
          ldmatrix_x4_trans(b[0], b[1], b[2], b[3], av + n2 * 32);
          const uint32_t b0[2] = {b[0], b[1]}, b1[2] = {b[2], b[3]};
          mma_bf16_16816(o[2 * n2], pa[ks], b0);
          mma_bf16_16816(o[2 * n2 + 1], pa[ks], b1);
        }
      }
    }
  }
  cp_async_wait<0>();
  STS_TRACE_AT(3);
  if constexpr (CS > 1) {
    // ---- merge the cluster's shares of the unit through DSMEM ----
    constexpr int NO = MODE == MODE_DECODE ? D / 8 : 0;  // float4 of O per thread
    float la = l_a, lb = l_b;
    la += __shfl_xor_sync(0xffffffffu, la, 1);
    la += __shfl_xor_sync(0xffffffffu, la, 2);
    lb += __shfl_xor_sync(0xffffffffu, lb, 1);
    lb += __shfl_xor_sync(0xffffffffu, lb, 2);
    __syncthreads();  // the stage buffers are free: reuse them as the exchange area
    float4* xb = reinterpret_cast<float4*>(smem);  // [NO + 1][NTH] float4
    if (crank != 0) {
      if constexpr (MODE == MODE_DECODE) {
#pragma unroll
        for (int j = 0; j < NO; ++j) xb[j * NTH + tid] = make_float4(o[j][0], o[j][1], o[j][2], o[j][3]);
      }
      xb[NO * NTH + tid] = make_float4(m_a, m_b, la, lb);
    }
    cluster_sync_all();
    if (crank == 0 && iu < U && icnt > 0) {
      const uint32_t xa = smem_u32(xb);
      for (unsigned q = 1; q < (unsigned)CS; ++q) {
        const uint32_t ra = dsmem_map(xa, q);
        const float4 st = dsmem_ld4(ra + (uint32_t)((NO * NTH + tid) * 16));
        const float nA = fmaxf(m_a, st.x), nB = fmaxf(m_b, st.y);
        const float bA = nA == -INFINITY ? 0.f : nA, bB = nB == -INFINITY ? 0.f : nB;
        const float fA = fast_exp2(m_a - bA), gA = fast_exp2(st.x - bA);
        const float fB = fast_exp2(m_b - bB), gB = fast_exp2(st.y - bB);
        la = la * fA + st.z * gA;
        lb = lb * fB + st.w * gB;
        m_a = nA;
        m_b = nB;
        if constexpr (MODE == MODE_DECODE) {
#pragma unroll
          for (int j = 0; j < NO; ++j) {
            const float4 x = dsmem_ld4(ra + (uint32_t)((j * NTH + tid) * 16));
            o[j][0] = o[j][0] * fA + x.x * gA;
            o[j][1] = o[j][1] * fA + x.y * gA;
            o[j][2] = o[j][2] * fB + x.z * gB;
            o[j][3] = o[j][3] * fB + x.w * gB;
          }
        }
      }
      const float inv_a = la > 0.f ? 1.f / la : 0.f, inv_b = lb > 0.f ? 1.f / lb : 0.f;
      const int dc = 2 * (lane & 3);
      const int64_t u = iu;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = h ? rB : rA;
        if (r >= M) continue;
        const float inv = h ? inv_b : inv_a;
        if constexpr (MODE == MODE_DECODE) {
          if (p.out_f32) {
            float* og = static_cast<float*>(p.out) + (u * M + r) * (int64_t)D + dc;
#pragma unroll
            for (int nt = 0; nt < D / 8; ++nt)
              *reinterpret_cast<float2*>(og + nt * 8) = make_float2(o[nt][2 * h] * inv, o[nt][2 * h + 1] * inv);
          } else {
            __nv_bfloat16* og = static_cast<__nv_bfloat16*>(p.out) + (u * M + r) * (int64_t)D + dc;
#pragma unroll
            for (int nt = 0; nt < D / 8; ++nt)
              *reinterpret_cast<__nv_bfloat162*>(og + nt * 8) =
                  __floats2bfloat162_rn(o[nt][2 * h] * inv, o[nt][2 * h + 1] * inv);
          }
        }
        if ((lane & 3) == 0) {
          const float l = h ? lb : la;
          const float m = h ? m_b : m_a;
          if (p.lse) p.lse[u * M + r] = l > 0.f ? (m + __log2f(l)) * LN2 : -INFINITY;
          if (MODE == MODE_DECODE && !(l > 0.f)) set_status(p.status, STS_DEV_EMPTY_ROW);
        }
      }
    }
    cluster_sync_all();  // partners keep their shared memory until rank 0 has read it
  } else {
    if (cur_u >= 0) flush(cur_u, cur_P, cur_cnt, cur_range);
  }
  STS_TRACE_AT(4);
}

// Merge of the units whose tiles were split over several schedule ranges: one
// CTA per unit, pieces in range order (deterministic), every load of a row's
// pieces issued before any is used.
constexpr int MERGE_MAX_THREADS = 1024;

template <int D, int MODE>
__global__ void __launch_bounds__(MERGE_MAX_THREADS) merge_pieces_kernel(DecodeParams p) {
  // weights w[k][r] = exp(lse_k[r] - lse[r]) of piece k for row r, in smem
  constexpr int MAXP = 32;
  __shared__ float s_w[MAXP * 48];
  __shared__ float s_l[MAXP * 48];
  const int nth = blockDim.x;
  const int64_t u = blockIdx.x;
  const int M = p.M;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the main kernel's pieces are complete
  const int2 pr = p.pieces[u];
  if ((p.idx ? p.cnt[u] : p.n_dense) <= 0) return;
  const int n = pr.y - pr.x + 1;
  if (n <= 1) return;
  const float* lp = p.l_part + ((int64_t)pr.x + u) * M;  // piece k at lp + k*M
  const int nb = n < MAXP ? n : MAXP;                    // pieces staged in smem
  for (int e = threadIdx.x; e < nb * M; e += nth) s_l[e] = __ldcg(lp + e);
  __syncthreads();
  for (int r = threadIdx.x; r < M; r += nth) {
    float mstar = -INFINITY, tot = 0.f;
    for (int k = 0; k < n; ++k) mstar = fmaxf(mstar, k < nb ? s_l[k * M + r] : __ldcg(lp + (int64_t)k * M + r));
    if (mstar != -INFINITY)
      for (int k = 0; k < n; ++k) {
        const float l = k < nb ? s_l[k * M + r] : __ldcg(lp + (int64_t)k * M + r);
        tot += l == -INFINITY ? 0.f : expf(l - mstar);
      }
    const float inv = tot > 0.f ? 1.f / tot : 0.f;
    for (int k = 0; k < nb; ++k) {
      const float l = s_l[k * M + r];
      s_w[k * M + r] = l == -INFINITY ? 0.f : expf(l - mstar) * inv;
    }
    s_l[r] = mstar;  // (row r of piece 0 is no longer needed: its weight is in s_w)
    if (p.lse) p.lse[u * M + r] = tot > 0.f ? mstar + logf(tot) : -INFINITY;
    if (MODE == MODE_DECODE && !(tot > 0.f)) set_status(p.status, STS_DEV_EMPTY_ROW);
    if (nb < n) s_w[r] = -1.f - inv;  // marker: pieces beyond MAXP use the slow path (never in practice)
  }
  if constexpr (MODE != MODE_DECODE) return;
  __syncthreads();
  constexpr int D4 = D / 4;
  const float* op = p.o_part + ((int64_t)pr.x + u) * M * D;
  for (int e = threadIdx.x; e < M * D4; e += nth) {
    const int r = e / D4, d4 = e % D4;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (nb == n) {
      for (int k0 = 0; k0 < n; k0 += 8) {
        float4 x8[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          x8[j] = k0 + j < n ? __ldcg(reinterpret_cast<const float4*>(op + ((int64_t)(k0 + j) * M + r) * D) + d4)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float f = k0 + j < n ? s_w[(k0 + j) * M + r] : 0.f;
          acc.x += f * x8[j].x;
          acc.y += f * x8[j].y;
          acc.z += f * x8[j].z;
          acc.w += f * x8[j].w;
        }
      }
    } else {
      // > MAXP pieces (a unit spread over more than 32 CTAs): plain loop
      const float mstar = s_l[r], inv = -1.f - s_w[r];
      for (int k = 0; k < n; ++k) {
        const float l = __ldcg(lp + (int64_t)k * M + r);
        const float f = l == -INFINITY ? 0.f : expf(l - mstar) * inv;
        const float4 x = __ldcg(reinterpret_cast<const float4*>(op + ((int64_t)k * M + r) * D) + d4);
        acc.x += f * x.x;
        acc.y += f * x.y;
        acc.z += f * x.z;
        acc.w += f * x.w;
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

template <int D, int NW, int KT, int STAGES, int MODE>
int launch_verify(DecodeParams& p, cudaStream_t st);

template <int D, int NW, int KT, int STAGES, int MODE, int CS>
int launch_cluster(DecodeParams& p, cudaStream_t st) {
  using L = VL<D, NW, KT, STAGES, MODE>;
  auto kern = verify_decode_kernel<D, NW, KT, STAGES, MODE, CS>;
  static const cudaError_t attr = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
  STS_CUDA_CHECK(attr);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(p.units * CS));
  cfg.blockDim = dim3(L::THREADS);
  cfg.dynamicSmemBytes = L::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  STS_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, p));
  count_launch();
  return STS_OK;
}

// Schedule (DecodeParams::schedule).  Auto (0): a thread-block cluster per
// unit when the resident CTA slots hold >= 2 CTAs per unit and a CTA would
// stream few tiles (fixed per-launch costs dominate): the c2 shape (256 units
// on 888 slots, ~30 tiles per CTA) -> clusters of 3, measured 92.8 vs 98.9 us
// (sparse) and 670 vs 688 us (dense, ~300 tiles per CTA).  At c4 (~950 tiles
// per CTA) the 13% of slots a floor(slots / units) cluster grid leaves idle
// cost more (2.55 vs 2.35 ms), so long streams stay stream-K; the draft LSE
// pass also measured better as stream-K.  1: stream-K.  2..8: clusters of
// exactly that many CTAs (any M; parity tests force every size).
template <int D, int NW, int KT, int STAGES, int MODE>
int try_cluster(DecodeParams& p, cudaStream_t st, int per_sm) {
  if (MODE != MODE_DECODE || p.units <= 0 || p.schedule == 1) return -1;
  int64_t cs = p.schedule;
  if (cs == 0) {
    if (NW != 2) return -1;
    const int64_t slots = (int64_t)num_sms() * per_sm;
    const int64_t cap = p.idx ? p.idx_ld : p.n_dense;  // keys per unit (upper bound)
    const int64_t tiles_per_slot = p.units * ((cap + KT - 1) / KT) / slots;
    if (tiles_per_slot > 600) return -1;
    cs = slots / p.units;
    if (cs > 8) cs = 8;
    cs = cs >= 8 ? 8 : cs >= 6 ? 6 : cs >= 4 ? 4 : cs;
    if (cs < 2) return -1;
  }
  if (p.plan_only) return (int)cs;
  STS_REQUIRE(p.units * cs <= 0x7fffffffLL, STS_ERR_CONTRACT, "too many units for a cluster grid");
  switch (cs) {
    case 2: return launch_cluster<D, NW, KT, STAGES, MODE, 2>(p, st);
    case 3: return launch_cluster<D, NW, KT, STAGES, MODE, 3>(p, st);
    case 4: return launch_cluster<D, NW, KT, STAGES, MODE, 4>(p, st);
    case 6: return launch_cluster<D, NW, KT, STAGES, MODE, 6>(p, st);
    case 8: return launch_cluster<D, NW, KT, STAGES, MODE, 8>(p, st);
    default:
      set_error("unsupported cluster size %d", (int)cs);
      return STS_ERR_CONTRACT;
  }
}

template <int D, int NW, int KT, int STAGES, int MODE>
int launch_verify(DecodeParams& p, cudaStream_t st) {
  using L = VL<D, NW, KT, STAGES, MODE>;
  static_assert(L::SMEM <= 227 * 1024, "verify decode shared memory");
  auto kern = verify_decode_kernel<D, NW, KT, STAGES, MODE, 1>;
  static const int per_sm = [&]() {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM) != cudaSuccess) return -1;
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, L::THREADS, L::SMEM) != cudaSuccess) return -1;
    return n < 1 ? 1 : n;
  }();
  if (per_sm <= 0 && p.plan_only) return -1;
  STS_REQUIRE(per_sm > 0, STS_ERR_CUDA, "verify kernel setup failed: %s", cudaGetErrorString(cudaGetLastError()));
  if constexpr (MODE == MODE_DECODE) {
    const int rc = try_cluster<D, NW, KT, STAGES, MODE>(p, st, per_sm);
    if (rc >= 0) return rc;
  }
  if (p.plan_only) return 1;
  const int smem = L::SMEM;
  kern<<<num_sms() * per_sm, L::THREADS, smem, st>>>(p);
  STS_LAUNCH_CHECK();
  if (p.pieces) {
    // one thread per (row, 4 dims) output element: every piece load in flight at once
    // (optional, -DSTS_PDL) programmatic dependent launch: the merge grid is
    // launched while the main kernel runs and waits (griddepcontrol.wait)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)p.units);
    cfg.blockDim = dim3(MODE == MODE_DECODE ? 256 : 64);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
#ifdef STS_PDL
    attr[0].val.programmaticStreamSerializationAllowed = 1;
#else
    // measured: an early-launched merge grid costs the main kernel ~3 us at c2
    attr[0].val.programmaticStreamSerializationAllowed = 0;
#endif
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    STS_CUDA_CHECK(cudaLaunchKernelEx(&cfg, merge_pieces_kernel<D, MODE>, p));
    count_launch();
  }
  return STS_OK;
}

#ifndef STS_VERIFY_KT
#define STS_VERIFY_KT 32
#endif
#ifndef STS_VERIFY_STAGES
#define STS_VERIFY_STAGES 2
#endif
// draft capture (K only, contiguous keys): bigger tiles, deeper pipeline
#ifndef STS_DRAFT_KT
#define STS_DRAFT_KT 64
#endif
#ifndef STS_DRAFT_STAGES
#define STS_DRAFT_STAGES 2
#endif

// Pipeline shapes were tuned on B200 at c2 (profiles/r01): decode 32-key tiles
// x2 stages (vs 32x3, 16x4, 16x3, 64x2: all within 1-5% slower); draft passes
// 64-key tiles x2 (247 us) < 64x3 (270) < 64x4 (296) < 32x4 (297) < 32x3 (306)
// < 128x2 (316) < 128x3 (415).

template <int D, int MODE>
int verify_dispatch(DecodeParams& p, cudaStream_t st) {
  constexpr bool DEC = MODE == MODE_DECODE;
  constexpr int KT = DEC ? STS_VERIFY_KT : STS_DRAFT_KT, S = DEC ? STS_VERIFY_STAGES : STS_DRAFT_STAGES;
  switch ((p.M + 15) / 16) {
    case 1: return launch_verify<D, 1, KT, S, MODE>(p, st);
    case 2: return launch_verify<D, 2, KT, S, MODE>(p, st);
    case 3: return launch_verify<D, 3, KT, S, MODE>(p, st);
    default:
      set_error("bf16 gather kernels support M <= 48 stacked rows, got %d", p.M);
      return STS_ERR_CONTRACT;
  }
}

template <int MODE>
int verify_dispatch_d(DecodeParams& p, cudaStream_t st) {
  if (p.d == 128) return verify_dispatch<128, MODE>(p, st);
  if (p.d == 64) return verify_dispatch<64, MODE>(p, st);
  set_error("bf16 gather kernels support d in {64, 128}, got %d", p.d);
  return STS_ERR_CONTRACT;
}

}  // namespace

#ifdef STS_TRACE
extern "C" STS_API int sts_debug_trace(void* host, size_t bytes) {
  return cudaMemcpyFromSymbol(host, g_trace, bytes < sizeof(g_trace) ? bytes : sizeof(g_trace)) == cudaSuccess ? 0 : 3;
}
#endif

int verify_decode_launch(int mode, DecodeParams& p, cudaStream_t st) {
  if (mode == MODE_DECODE) return verify_dispatch_d<MODE_DECODE>(p, st);
  // the draft capture runs on TMA + tcgen05 (sts_capture.cu); the LSE / PROBS
  // instantiations of this kernel are not built
  set_error("verify_decode_launch: mode %d is served by sts_capture.cu", mode);
  return STS_ERR_CONTRACT;
}

}  // namespace sts
