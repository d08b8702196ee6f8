// sts_gather.cu — warp-specialised persistent gather kernel (bf16, sm_100a).
//
// One CTA per SM: warp 0 is a TMA producer, warps 1..NC are math consumers.
//
//  * The key tiles of all units (unit = (batch, layer, kv-head); KT keys per
//    tile) form one global tile space cut into equal contiguous ranges, one
//    per consumer warp (stream-K), so every consumer streams the same bytes
//    however ragged the per-unit key lists are.
//  * The producer walks the consumers round-robin.  For each tile it waits for
//    a free slot in that consumer's SPC-deep ring (mbarrier `empty`), writes
//    the tile's key positions into the slot, arms the slot's `full` mbarrier
//    with the byte count and issues one cp.async.bulk (TMA) copy per gathered
//    K / V row (D*2 bytes each) straight into padded shared-memory rows.  The
//    index slice of a consumer's next tile is loaded one round ahead, so the
//    gather never waits on a dependent index load.  Up to NC*SPC tiles
//    (~160 KB at D=128) are in flight per SM.
//  * Consumers issue no loads at all: wait `full`, run the tile math on the
//    tensor cores (mma.sync m16n8k16, stacked query rows as N), release the
//    slot.  Crossing into a new unit flushes the softmax state (final rows, or
//    an fp32 partial merged in warp order by the last consumer to arrive).
//
// Modes: DECODE (K+V, online softmax, O = P.V), LSE (K only, draft-row
// log-sum-exp), PROBS (K only, probabilities from a known LSE, per row or
// summed over the speculative rows of each head).
#include "sts_decode.cuh"

namespace sts {
namespace {

constexpr float LN2f = 0.6931471805599453f;

template <int D, int NT, int MODE, int SUB, int NC, int SPC>
struct GL {
  static constexpr bool K_ONLY = MODE != MODE_DECODE;
  static constexpr int KT = KEY_TILE * SUB;
  static constexpr int MP = 8 * NT;
  static constexpr int CH = D / 8;
  static constexpr int PITCH = D * 2 + 16;  // padded rows: ldmatrix conflict-free
  static constexpr int ROWS_BYTES = KT * PITCH;
  static constexpr int DATA = (K_ONLY ? 1 : 2) * ROWS_BYTES;
  static constexpr int META = KT * 8 + 16;  // pos[KT], mem[KT], info[4]
  static constexpr int STAGE = (DATA + META + 15) & ~15;
  static constexpr int Q_BYTES = MP * D * 2;
  static constexpr int PROB = MODE == MODE_PROBS ? KEY_TILE * MP * 4 : 0;
  static constexpr int PER_C = SPC * STAGE + Q_BYTES + PROB;
  static constexpr int BAR = ((NC * SPC * 2 * 8) + 127) & ~127;
  static constexpr int SMEM = BAR + NC * PER_C;
  static constexpr int THREADS = (NC + 1) * 32;
};

__device__ __forceinline__ uint32_t swz(int row, int chunk) { return (uint32_t)((chunk ^ (row & 7)) << 4); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

__device__ __forceinline__ int tiles_of(const DecodeParams& p, int64_t u, int KT) {
  const int c = p.idx ? p.cnt[u] : p.n_dense;
  return (c + KT - 1) / KT;
}

__device__ __forceinline__ int owner_of(int64_t t, int64_t T, int W) { return (int)(((t + 1) * W - 1) / T); }

// Warp-cooperative: total tiles T and the unit containing tile `t0`
// (returns unit index and the unit's first tile).
__device__ void locate(const DecodeParams& p, int KT, int64_t t0, int64_t& u_out, int64_t& P_out) {
  const int lane = threadIdx.x & 31;
  int64_t base = 0;
  u_out = 0;
  P_out = 0;
  for (int64_t u0 = 0; u0 < p.units; u0 += 32) {
    const int64_t u = u0 + lane;
    const int t_u = u < p.units ? tiles_of(p, u, KT) : 0;
    int64_t incl = t_u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t x = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += x;
    }
    const int64_t tot = __shfl_sync(0xffffffffu, incl, 31);
    if (base + tot > t0) {
      const uint32_t hit = __ballot_sync(0xffffffffu, base + incl > t0);
      const int src = __ffs(hit) - 1;
      u_out = u0 + src;
      P_out = base + __shfl_sync(0xffffffffu, incl - t_u, src);
      return;
    }
    base += tot;
  }
}

template <int D, int NT, int MODE, int SUB, int NC, int SPC>
__global__ void __launch_bounds__((NC + 1) * 32, 1) gather_kernel(DecodeParams p) {
  using L = GL<D, NT, MODE, SUB, NC, SPC>;
  constexpr int KT = L::KT, MP = L::MP, CH = L::CH, PITCH = L::PITCH;
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int M = p.M;
  const int64_t U = p.units;
  const uint32_t bar_base = smem_u32(smem);  // full[k][s] then empty[k][s]
  auto full_bar = [&](int k, int s) { return bar_base + (uint32_t)((k * SPC + s) * 8); };
  auto empty_bar = [&](int k, int s) { return bar_base + (uint32_t)((NC * SPC + k * SPC + s) * 8); };
  uint8_t* cbase = smem + L::BAR;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NC * SPC; ++i) {
      mbar_init(bar_base + i * 8, 1);
      mbar_init(bar_base + (NC * SPC + i) * 8, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // ---- units with no keys (striped over CTAs): zero rows, LSE -inf ----
  if (warp == 0) {
    for (int64_t u = blockIdx.x; u < U; u += gridDim.x) {
      if (tiles_of(p, u, KT) != 0) continue;
      if constexpr (MODE == MODE_DECODE) {
        __nv_bfloat16* og = static_cast<__nv_bfloat16*>(p.out) + u * (int64_t)M * D;
        for (int e = lane; e < M * D; e += 32) og[e] = __float2bfloat16_rn(0.f);
        if (lane == 0 && M > 0) set_status(p.status, STS_DEV_EMPTY_ROW);
      }
      if constexpr (MODE != MODE_PROBS)
        if (p.lse)
          for (int r = lane; r < M; r += 32) p.lse[u * M + r] = -INFINITY;
    }
  }

  // ---- tile space and consumer ranges ----
  int64_t T = 0;
  for (int64_t u = lane; u < U; u += 32) T += tiles_of(p, u, KT);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) T += __shfl_xor_sync(0xffffffffu, T, o);
  if (T == 0) return;
  const int W = (int)(T < (int64_t)gridDim.x * NC ? T : (int64_t)gridDim.x * NC);
  auto range_of = [&](int gw, int64_t& s, int64_t& e) {
    if (gw >= W) {
      s = e = 0;
      return;
    }
    s = (int64_t)gw * T / W;
    e = (int64_t)(gw + 1) * T / W;
  };

  if (warp == 0) {
    // =========================== PRODUCER ===========================
    int64_t t[NC], e[NC], cu[NC], cP[NC], cPn[NC];
    int ccnt[NC], n_used[NC];
    int pos_n[NC];
    uint32_t mem_n[NC];
    int nu[NC], nj0[NC], ncnt[NC], nP[NC];  // info of the prefetched tile t[k]
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      range_of(blockIdx.x * NC + k, t[k], e[k]);
      n_used[k] = 0;
      cu[k] = 0;
      cP[k] = 0;
      if (t[k] < e[k]) {
        int64_t uu, PP;
        locate(p, KT, t[k], uu, PP);
        cu[k] = uu;
        cP[k] = PP;
      }
      ccnt[k] = t[k] < e[k] ? (p.idx ? p.cnt[cu[k]] : p.n_dense) : 0;
      cPn[k] = cP[k] + (ccnt[k] + KT - 1) / KT;
    }
    // prefetch the positions of tile t[k] into registers (lane = row)
    auto prefetch = [&](int k) {
      if (t[k] >= e[k]) return;
      while (t[k] >= cPn[k]) {
        ++cu[k];
        cP[k] = cPn[k];
        ccnt[k] = p.idx ? p.cnt[cu[k]] : p.n_dense;
        cPn[k] = cP[k] + (ccnt[k] + KT - 1) / KT;
      }
      nu[k] = (int)cu[k];
      nj0[k] = (int)(t[k] - cP[k]) * KT;
      ncnt[k] = ccnt[k];
      nP[k] = (int)cP[k];
      const int j = nj0[k] + lane;
      pos_n[k] = -1;
      mem_n[k] = 0xffffffffu;
      if (lane < KT && j < ncnt[k]) {
        pos_n[k] = p.idx ? __ldg(p.idx + cu[k] * p.idx_ld + j) : j;
        if (p.member) mem_n[k] = __ldg(p.member + cu[k] * p.idx_ld + j);
      }
    };
#pragma unroll
    for (int k = 0; k < NC; ++k) prefetch(k);

    const int row_bytes = D * 2;
    bool more = true;
    while (more) {
      more = false;
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        if (t[k] >= e[k]) continue;
        more = true;
        const int s = n_used[k] % SPC;
        const uint32_t ph = (uint32_t)((n_used[k] / SPC) & 1);
        mbar_wait(empty_bar(k, s), ph ^ 1u);
        uint8_t* st = cbase + k * L::PER_C + s * L::STAGE;
        int* m_pos = reinterpret_cast<int*>(st + L::DATA);
        uint32_t* m_mem = reinterpret_cast<uint32_t*>(m_pos + KT);
        int* m_info = reinterpret_cast<int*>(m_mem + KT);
        const int valid = min(KT, ncnt[k] - nj0[k]);
        const int pos = pos_n[k];
        if (lane < KT) {
          m_pos[lane] = pos;
          m_mem[lane] = mem_n[k];
        }
        if (lane == 0) {
          m_info[0] = nu[k];
          m_info[1] = nj0[k];
          m_info[2] = ncnt[k];
          m_info[3] = nP[k];
        }
        __syncwarp();
        const uint32_t fb = full_bar(k, s);
        if (lane == 0) mbar_arrive_expect_tx(fb, (uint32_t)(valid * row_bytes * (L::K_ONLY ? 1 : 2)));
        __syncwarp();
        const int64_t u = nu[k];
        const __nv_bfloat16* kg = static_cast<const __nv_bfloat16*>(p.k) + u * p.kv_stride;
        const __nv_bfloat16* vg = static_cast<const __nv_bfloat16*>(p.v) + u * p.kv_stride;
        const uint32_t dst = smem_u32(st);
        constexpr int COPIES = (L::K_ONLY ? 1 : 2) * KT;
#pragma unroll
        for (int c0 = 0; c0 < COPIES; c0 += 32) {
          const int c = c0 + lane;
          const int r = c % KT;
          const int isv = c / KT;
          const int pr = __shfl_sync(0xffffffffu, pos, r & 31);
          if (c < COPIES && r < valid) {
            const __nv_bfloat16* src = (isv ? vg : kg) + (int64_t)pr * p.row_stride;
            bulk_g2s(dst + isv * L::ROWS_BYTES + r * PITCH, src, row_bytes, fb);
          }
        }
        // next tile of consumer k: its index slice lands during the next round
        ++t[k];
        ++n_used[k];
        prefetch(k);
      }
    }
    return;
  }

  // =========================== CONSUMERS ===========================
  const int k = warp - 1;
  const int gw = blockIdx.x * NC + k;
  int64_t s_w, e_w;
  range_of(gw, s_w, e_w);
  if (s_w >= e_w) return;
  uint8_t* my = cbase + k * L::PER_C;
  uint8_t* s_q = my + SPC * L::STAGE;
  float* s_prob = reinterpret_cast<float*>(s_q + L::Q_BYTES);
  const uint32_t q_base = smem_u32(s_q);

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
      *reinterpret_cast<uint4*>(s_q + r * (D * 2) + swz(r, ch)) = val;
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
      const int wf = owner_of(P_u, T, W);
      const int wl = owner_of(P_u + tiles - 1, T, W);
      const bool single = wf == wl;
      const int64_t slot = (int64_t)gw + u;
      float* part_o = p.o_part + slot * (int64_t)M * D;
      float* part_l = p.l_part + slot * (int64_t)M;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int r = nt * 8 + 2 * (lane & 3) + c;
          if (r >= M) continue;
          const float l = l_run[nt][c];
          const float inv = l > 0.f ? 1.f / l : 0.f;
          const float lse = l > 0.f ? (m_run[nt][c] + __log2f(l)) * LN2f : -INFINITY;
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
      const int n = wl - wf + 1;
      float* s_w8 = reinterpret_cast<float*>(s_q);
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
            s_w8[r] = mstar;
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

  int n_used = 0;
  for (int64_t i = 0; i < e_w - s_w; ++i) {
    const int slot = n_used % SPC;
    mbar_wait(full_bar(k, slot), (uint32_t)((n_used / SPC) & 1));
    const uint8_t* st = my + slot * L::STAGE;
    const int* m_pos = reinterpret_cast<const int*>(st + L::DATA);
    const uint32_t* m_mem = reinterpret_cast<const uint32_t*>(m_pos + KT);
    const int* m_info = reinterpret_cast<const int*>(m_mem + KT);
    const int64_t u = m_info[0];
    const int j0 = m_info[1];
    if (u != cur_u) {
      if (cur_u >= 0) flush(cur_u, cur_P, cur_cnt);
      cur_u = u;
      cur_cnt = m_info[2];
      cur_P = m_info[3];
      reset_state();
      load_q(u);
    }
    const uint32_t sk0 = smem_u32(st);
    // fast path: every row valid, no membership bits, whole tile in the
    // committed prefix (positions ascending) -> no per-element masking
    const int last_pos = m_pos[KT - 1];
    const bool simple = (j0 + KT <= cur_cnt) && !p.member && (!causal || last_pos + causal_shift <= 0);

    float s[SUB][NT][4];
    bool okA[SUB][NT][2], okB[SUB][NT][2];
#pragma unroll
    for (int sub = 0; sub < SUB; ++sub) {
      const bool live = j0 + sub * KEY_TILE < cur_cnt;
      const uint32_t sk = sk0 + sub * KEY_TILE * PITCH;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int c = 0; c < 4; ++c) s[sub][nt][c] = 0.f;
      if (live) {
#pragma unroll
        for (int kk = 0; kk < D / 16; kk += 2) {
          uint32_t a0[4], a1[4];
          const int key = (mi & 1) * 8 + ri;
          ldmatrix_x4(a0[0], a0[1], a0[2], a0[3], sk + key * PITCH + (2 * kk + (mi >> 1)) * 16);
          ldmatrix_x4(a1[0], a1[1], a1[2], a1[3], sk + key * PITCH + (2 * kk + 2 + (mi >> 1)) * 16);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const int row = nt * 8 + ri;
            uint32_t b[4];
            ldmatrix_x4(b[0], b[1], b[2], b[3], q_base + row * (D * 2) + swz(row, 2 * kk + mi));
            const uint32_t b0[2] = {b[0], b[1]};
            const uint32_t b1[2] = {b[2], b[3]};
            mma_bf16_16816(s[sub][nt], a0, b0);
            mma_bf16_16816(s[sub][nt], a1, b1);
          }
        }
      }
      if (simple) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int c = 0; c < 2; ++c) okA[sub][nt][c] = okB[sub][nt][c] = true;
      } else {
        const int kA = (lane >> 2) + sub * KEY_TILE, kB = kA + 8;
        const int posA = m_pos[kA], posB = m_pos[kB];
        const uint32_t memA = m_mem[kA], memB = m_mem[kB];
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
          for (int e2 = lane; e2 < KEY_TILE * G; e2 += 32) {
            const int key = e2 % KEY_TILE, hh = e2 / KEY_TILE;
            const int pos = m_pos[sub * KEY_TILE + key];
            if (pos >= 0 && pos + p.pos_offset < p.causal_base) {
              float acc = s_prob[key * MP + hh * R];
              for (int ii = 1; ii < R; ++ii) acc = __fadd_rn(acc, s_prob[key * MP + hh * R + ii]);
              p.probs_out[(u * G + hh) * p.out_ld + jb + key] = acc;
            }
          }
        } else {
          for (int e2 = lane; e2 < KEY_TILE * M; e2 += 32) {
            const int key = e2 % KEY_TILE, r = e2 / KEY_TILE;
            const int pos = m_pos[sub * KEY_TILE + key];
            if (pos >= 0 && pos + p.pos_offset <= p.causal_base + r % R)
              p.probs_out[(u * M + r) * p.out_ld + jb + key] = s_prob[key * MP + r];
          }
        }
        __syncwarp();
      }
    } else {
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
      if constexpr (MODE == MODE_DECODE) {
#pragma unroll
        for (int sub = 0; sub < SUB; ++sub) {
          if (j0 + sub * KEY_TILE >= cur_cnt) break;
          const uint32_t sv = sk0 + L::ROWS_BYTES + sub * KEY_TILE * PITCH;
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
            ldmatrix_x4_trans(a[0], a[1], a[2], a[3], sv + key * PITCH + (2 * mt + (mi & 1)) * 16);
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
    if (lane == 0) mbar_arrive(empty_bar(k, slot));
    ++n_used;
  }
  if (cur_u >= 0) flush(cur_u, cur_P, cur_cnt);
}

template <int D, int NT, int MODE>
struct GCfg {
  static constexpr int SUB = MODE == MODE_DECODE ? (D == 64 ? 2 : 1) : 2;
  static constexpr int SPC = 3;
  // as many consumer warps (<= 6) as fit in 227 KB of shared memory
  static constexpr int NC = GL<D, NT, MODE, SUB, 6, SPC>::SMEM <= 227 * 1024 ? 6 : 5;
  using L = GL<D, NT, MODE, SUB, NC, SPC>;
};

template <int D, int NT, int MODE>
int launch_gather(DecodeParams& p, cudaStream_t st) {
  using C = GCfg<D, NT, MODE>;
  using L = typename C::L;
  static_assert(L::SMEM <= 227 * 1024, "gather kernel shared memory");
  static_assert(L::KT <= 32, "producer keeps one key position per lane");
  auto kern = gather_kernel<D, NT, MODE, C::SUB, C::NC, C::SPC>;
  STS_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM));
  kern<<<num_sms(), L::THREADS, L::SMEM, st>>>(p);
  STS_LAUNCH_CHECK();
  return STS_OK;
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

int gather_consumers_per_sm() { return 6; }

int gather_launch(int mode, DecodeParams& p, cudaStream_t st) {
  if (mode == MODE_DECODE) return gdispatch_d<MODE_DECODE>(p, st);
  if (mode == MODE_LSE) return gdispatch_d<MODE_LSE>(p, st);
  return gdispatch_d<MODE_PROBS>(p, st);
}

}  // namespace sts
