// decode_tc.cu — measurement prototype (not part of the library): the
// gathered mode-S verify decode on tcgen05, for the tcgen05-versus-mma.sync
// comparison at M > 32 stacked rows (c3: 35).  Keys are the MMA's M = 128
// (TMEM lanes), the unit's rows its N = 48:
//   S^T = K_tile . Q^T            (A = K tile, K-major; B = Q, K-major)
//   O^T += V_tile^T . P           (A = V tile as an MN-major operand; B = P,
//                                  written by the softmax threads, MN-major)
// Warps 0-1 gather the tile's K / V rows with cp.async (16-byte chunks into
// the 128B-swizzled layout, zero-filled past the list), warp 2 issues the
// MMAs, warps 3-6 (thread = key) do the softmax.  The row maxima are one
// CTA-wide reference per row that moves only when a score exceeds it by 2^16
// (then O^T and the row sums are rescaled), so a tile needs no cross-thread
// reduction; the row sums stay per thread until the unit's end.  One CTA per
// SM, persistent over units; output bf16 [U][M][128] + LSE.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC \
//        -I paper_2605_15508_b200/csrc -o tools/_build/decode_tc.so tools/decode_tc.cu
#include "sts_common.cuh"

namespace {
using sts::fast_exp2;
using sts::pack_bf16;

constexpr int D = 128, NC = 48, KT = 128, KS = 3, VS = 2;  // K ring freed after S, V ring after PV
constexpr int THREADS = 224;                   // 2 producer warps, 1 MMA warp, 4 softmax warps (<= 2 per SMSP)
constexpr int Q_SLAB = NC * 128;               // 6 KB per 64-d slab of Q (48 rows x 128 B)
constexpr int KV_SLAB = KT * 128;              // 16 KB per slab of a K or V tile
constexpr int KV_TILE = 2 * KV_SLAB;           // 32 KB
constexpr int P_TILE = KT * 128;               // [key][64 rows] bf16, 16 KB
constexpr int OFF_Q = 0;
constexpr int OFF_K = OFF_Q + 2 * Q_SLAB;      // 12 KB (1024-aligned)
constexpr int OFF_V = OFF_K + KS * KV_TILE;
constexpr int OFF_P = OFF_V + VS * KV_TILE;
constexpr int OFF_RED = OFF_P + 2 * P_TILE;    // [4 warps][48] floats + flags
constexpr int OFF_BAR = OFF_RED + 5 * NC * 4 + 64;  // + the row references [48]
constexpr int NBAR = 2 * KS + 2 * VS + 2 + 2 + 2 + 2 + 2 + 2;
constexpr int SMEM = OFF_BAR + NBAR * 8 + 16 + 1024;
constexpr int S_COL = 0, O_COL = 128;          // TMEM: S slots at 0 / 48, O^T at 128
constexpr float JUMP = 16.f;

struct P {
  const __nv_bfloat16 *q, *k, *v;
  int64_t kv_stride, units;
  int M, R, base;
  const int32_t *idx, *cnt;
  int64_t idx_ld;
  float sl2;
  __nv_bfloat16* out;
  float* lse;
  long long* dbg;  // (optional) per-role wait / busy cycle counters of CTA 0
};

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void minit(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su(b)), "r"(c));
}
__device__ __forceinline__ void marrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su(b)) : "memory");
}
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t par) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done)
                 : "r"(su(b)), "r"(par)
                 : "memory");
}
__device__ __forceinline__ void fb() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fa() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su(b)) : "memory");
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
               "l"(a), "l"(b), "r"(id), "r"(acc)
               : "memory");
}
// K-major SW128: 8-row groups 1024 B apart
__device__ __forceinline__ uint64_t dk(const void* p) {
  return ((su(p) >> 4) & 0x3FFFull) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
// MN-major SW128: atoms of 64 MN elements x 8 K rows; lbo between MN atoms, sbo between K groups
__device__ __forceinline__ uint64_t dmn(const void* p, uint32_t lbo, uint32_t sbo) {
  return ((su(p) >> 4) & 0x3FFFull) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) |
         (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void ld16(uint32_t t, float* v) {
  uint32_t r[16];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(t));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void st16(uint32_t t, const float* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(t),
               "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
               "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
               "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
               "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
               "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
               "r"(__float_as_uint(v[15]))
               : "memory");
}
__device__ __forceinline__ void wld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void wst() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void cpa16(uint32_t dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0) : "memory");
}
__device__ __forceinline__ void proxy() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// CTA-wide (over the 128 softmax threads) max of v[r] per row; result in v
__device__ __forceinline__ void rows_max(float* v, float* red, int sw, int lane) {
#pragma unroll
  for (int r = 0; r < NC; ++r) {
    float x = v[r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
    v[r] = x;
  }
  if (lane == 0)
#pragma unroll
    for (int r = 0; r < NC; ++r) red[sw * NC + r] = v[r];
  asm volatile("bar.sync 1, 128;\n" ::: "memory");
#pragma unroll
  for (int r = 0; r < NC; ++r) v[r] = fmaxf(fmaxf(red[r], red[NC + r]), fmaxf(red[2 * NC + r], red[3 * NC + r]));
  asm volatile("bar.sync 1, 128;\n" ::: "memory");
}

__global__ void __launch_bounds__(THREADS, 1) decode_tc_kernel(P p) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + OFF_BAR);
  uint64_t* kfull = bars;
  uint64_t* kempty = kfull + KS;
  uint64_t* vfull = kempty + KS;
  uint64_t* vempty = vfull + VS;
  uint64_t* sfull = vempty + VS;
  uint64_t* sempty = sfull + 2;
  uint64_t* pfull = sempty + 2;
  uint64_t* pempty = pfull + 2;
  uint64_t* qfull = pempty + 2;   // [0]
  uint64_t* qempty = qfull + 1;
  uint64_t* odone = qempty + 1;
  uint64_t* oempty = odone + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + NBAR);
  float* red = reinterpret_cast<float*>(sm + OFF_RED);
  int* flag = reinterpret_cast<int*>(red + 4 * NC);
  float* mref = red + 4 * NC + 16;  // [48] the CTA's row references (log2 units)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < KS; ++i) {
      minit(&kfull[i], 32);  // producer warp 0
      minit(&kempty[i], 1);
    }
    for (int i = 0; i < VS; ++i) {
      minit(&vfull[i], 32);  // producer warp 1
      minit(&vempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      minit(&sfull[i], 1);
      minit(&sempty[i], 128);
      minit(&pfull[i], 128);
      minit(&pempty[i], 1);
    }
    minit(qfull, 64);
    minit(qempty, 1);
    minit(odone, 1);
    minit(oempty, 128);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(su(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  fb();
  __syncthreads();
  fa();
  const uint32_t tmem = *tslot;
  const int M = p.M;

  if (warp < 2) {
    // ---------------- producers: Q per unit, K / V rows per tile ----------------
    const int t = threadIdx.x;  // keys t and t + 64 of the tile
    uint32_t gj = 0;            // tiles loaded so far (ring position)
    int n_u = 0;
    for (int64_t u = blockIdx.x; u < p.units; u += gridDim.x, ++n_u) {
      const int n = p.cnt[u];
      const int nt = (n + KT - 1) / KT;
      if (n_u > 0) mwait(qempty, (n_u - 1) & 1);
      // Q: rows 0..47 x 16 chunks, K-major SW128 per 64-d slab, zero past M
      for (int e = t; e < NC * 16; e += 64) {
        const int r = e >> 4, c = e & 15;
        uint4 x = make_uint4(0, 0, 0, 0);
        if (r < M) x = *reinterpret_cast<const uint4*>(p.q + ((u * M + r) * (int64_t)D) + c * 8);
        *reinterpret_cast<uint4*>(sm + OFF_Q + (c >> 3) * Q_SLAB + r * 128 + (((c & 7) ^ (r & 7)) * 16)) = x;
      }
      proxy();
      marrive(qfull);
      const int32_t* il = p.idx + u * p.idx_ld;
      const __nv_bfloat16* kb = p.k + u * p.kv_stride;
      const __nv_bfloat16* vb = p.v + u * p.kv_stride;
      // warp 0 streams the K tiles (ring of KS, freed by S), warp 1 the V tiles
      // (ring of VS, freed by PV); each keeps two tiles in flight and publishes a
      // tile once the next one is issued (and at the unit's end)
      const bool isK = warp == 0;
      const int NS = isK ? KS : VS;
      uint64_t* fullb = isK ? kfull : vfull;
      uint64_t* emptyb = isK ? kempty : vempty;
      const __nv_bfloat16* src = isK ? kb : vb;
      const uint32_t base = su(sm + (isK ? OFF_K : OFF_V));
      for (int j = 0; j < nt; ++j) {
        const uint32_t g = gj + j;
        const int st = g % NS;
        mwait(&emptyb[st], ((g / NS) & 1) ^ 1);
        const uint32_t dst = base + st * KV_TILE;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int key = lane + 32 * h;
          const int kk = j * KT + key;
          const bool ok = kk < n;
          const int pos = ok ? il[kk] : 0;
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const uint32_t off = (c >> 3) * KV_SLAB + key * 128 + (((c & 7) ^ (key & 7)) * 16);
            cpa16(dst + off, src + (int64_t)pos * D + c * 8, ok);
          }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        if (j > 0) {
          asm volatile("cp.async.wait_group 1;\n" ::: "memory");
          proxy();
          marrive(&fullb[(g - 1) % NS]);
        }
      }
      if (nt > 0) {
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        proxy();
        marrive(&fullb[(gj + nt - 1) % NS]);
      }
      gj += nt;
    }
  } else if (warp == 2) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t id_s = idesc(128, NC, false, false);
      constexpr uint32_t id_o = idesc(128, NC, true, true);
      uint32_t gj = 0, sc = 0;
      int n_u = 0;
      for (int64_t u = blockIdx.x; u < p.units; u += gridDim.x, ++n_u) {
        const int n = p.cnt[u];
        const int nt = (n + KT - 1) / KT;
        mwait(qfull, n_u & 1);
        fa();
        auto issue_s = [&](uint32_t g) {  // S of ring tile g into slot g & 1
          const int st = g % KS;
          long long a0_ = clock64();
          mwait(&sempty[g & 1], ((g >> 1) & 1) ^ 1);
          long long a1_ = clock64();
          mwait(&kfull[st], (g / KS) & 1);
          if (p.dbg && blockIdx.x == 0) {
            p.dbg[4] += a1_ - a0_;          // MMA: waiting for the S slot
            p.dbg[5] += clock64() - a1_;    // MMA: waiting for K
          }
          fa();
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            const uint64_t a = dk(sm + OFF_K + st * KV_TILE + s * KV_SLAB);
            const uint64_t b = dk(sm + OFF_Q + s * Q_SLAB);
#pragma unroll
            for (int k = 0; k < 4; ++k) mma(tmem + S_COL + (g & 1) * NC, a + 2 * k, b + 2 * k, id_s, (s | k) != 0);
          }
          commit(&sfull[g & 1]);
          commit(&kempty[st]);  // the K stage is free once S is done
        };
        if (nt > 0) issue_s(gj);
        for (int j = 0; j < nt; ++j) {
          const uint32_t g = gj + j;
          if (j + 1 < nt) issue_s(g + 1);
          if (j + 1 == nt) commit(qempty);  // every S of the unit issued: Q may be replaced
          long long b0_ = clock64();
          mwait(&pfull[g & 1], (g >> 1) & 1);
          long long b1_ = clock64();
          if (j == 0 && n_u > 0) mwait(oempty, (n_u - 1) & 1);  // O^T drained by the last unit's epilogue
          if (p.dbg && blockIdx.x == 0) {
            p.dbg[6] += b1_ - b0_;          // MMA: waiting for P
            p.dbg[7] += clock64() - b1_;    // MMA: waiting for O drained
          }
          fa();
          const int st = g % VS;
          long long v0_ = clock64();
          mwait(&vfull[st], (g / VS) & 1);
          if (p.dbg && blockIdx.x == 0) p.dbg[8] += clock64() - v0_;  // MMA: waiting for V
          fa();
          // O^T += V^T . P: A = V tile (MN-major: 64-d atoms 16 KB apart, 8-key groups 1 KB apart),
          // B = P (MN-major: rows 0..47 of a 64-wide atom, 8-key groups 1 KB apart); K = 16 keys per MMA
          const uint64_t a = dmn(sm + OFF_V + st * KV_TILE, KV_SLAB, 1024);
          const uint64_t b = dmn(sm + OFF_P + (g & 1) * P_TILE, 128 * 128, 1024);
#pragma unroll
          for (int k = 0; k < KT / 16; ++k)
            mma(tmem + O_COL, a + (uint64_t)(2048 >> 4) * k, b + (uint64_t)(2048 >> 4) * k, id_o, (j > 0 || k > 0) ? 1u : 0u);
          commit(&vempty[st]);
          commit(&pempty[g & 1]);
        }
        if (nt == 0) commit(qempty);
        commit(odone);
        gj += nt;
        ++sc;
      }
    }
  } else {
    // ---------------- softmax: thread = key of the tile (TMEM lane) ----------------
    const int sw = warp - 3;             // 0..3
    const int quad = warp & 3;           // TMEM lane quadrant of this warp
    const int t = quad * 32 + lane;      // key in tile = TMEM lane
    const uint32_t loff = (uint32_t)(quad * 32) << 16;
    uint32_t gj = 0;
    int n_u = 0;
    for (int64_t u = blockIdx.x; u < p.units; u += gridDim.x, ++n_u) {
      const int n = p.cnt[u];
      const int nt = (n + KT - 1) / KT;
      const int32_t* il = p.idx + u * p.idx_ld;
      float lt[NC];
#pragma unroll
      for (int r = 0; r < NC; ++r) lt[r] = 0.f;
      for (int j = 0; j < nt; ++j) {
        const uint32_t g = gj + j;
        const int kk = j * KT + t;
        const bool ok = kk < n;
        const int pos = ok ? il[kk] : 0;
        long long c0_ = clock64();
        mwait(&sfull[g & 1], (g >> 1) & 1);
        long long c1_ = clock64();
        fa();
        float x[NC];
        ld16(tmem + loff + S_COL + (g & 1) * NC, x);
        ld16(tmem + loff + S_COL + (g & 1) * NC + 16, x + 16);
        ld16(tmem + loff + S_COL + (g & 1) * NC + 32, x + 32);
        wld();
        fb();
        marrive(&sempty[g & 1]);
        // committed keys are seen by every row; an in-block key by the rows of
        // each head at or after its offset (gamma + 1 = 5 rows per head, compiled in)
        const int toff = pos - p.base;  // < 0: committed
#pragma unroll
        for (int r = 0; r < NC; ++r) {
          const bool vis = ok && r < M && toff <= (r % 5);
          x[r] = vis ? x[r] * p.sl2 : -INFINITY;
        }
        bool need = j == 0;
        if (j > 0) {
          // the reference moves only when some score tops it by 2^16
#pragma unroll
          for (int r = 0; r < NC; ++r) need |= x[r] > mref[r] + JUMP;
        }
        const int any = __any_sync(0xffffffffu, need);
        if (lane == 0) flag[sw] = any;
        asm volatile("bar.sync 1, 128;\n" ::: "memory");
        const bool cta_need = flag[0] | flag[1] | flag[2] | flag[3];
        if (cta_need) {
          float tm[NC];
#pragma unroll
          for (int r = 0; r < NC; ++r) tm[r] = x[r];
          rows_max(tm, red, sw, lane);  // (its barriers also order the flag reads)
          if (j > 0) {
            // O^T holds PV up to tile j-1: wait for it, rescale this thread's O^T lane (d = t)
            mwait(&pempty[(g - 1) & 1], ((g - 1) >> 1) & 1);
            fa();
#pragma unroll
            for (int c0 = 0; c0 < NC; c0 += 16) {
              float o[16];
              ld16(tmem + loff + O_COL + c0, o);
              wld();
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const float mo = mref[c0 + i], mn = fmaxf(mo, tm[c0 + i]);
                const float f = mn == -INFINITY ? 1.f : fast_exp2(mo - mn);
                o[i] *= f;
                lt[c0 + i] *= f;
              }
              st16(tmem + loff + O_COL + c0, o);
            }
            wst();
          }
          asm volatile("bar.sync 1, 128;\n" ::: "memory");  // every thread has read the old references
          if (t == 0)
#pragma unroll
            for (int r = 0; r < NC; ++r) mref[r] = j == 0 ? tm[r] : fmaxf(mref[r], tm[r]);
          asm volatile("bar.sync 1, 128;\n" ::: "memory");
        } else {
          asm volatile("bar.sync 1, 128;\n" ::: "memory");  // the flags are read before the next tile's writes
        }
        // P = 2^(x - ref) in bf16, row r at column r of the key's 128-byte row
        uint32_t w[NC / 2];
#pragma unroll
        for (int e = 0; e < NC / 2; ++e) {
          const float r0 = mref[2 * e], r1 = mref[2 * e + 1];
          const float a0 = x[2 * e] == -INFINITY ? 0.f : fast_exp2(x[2 * e] - (r0 == -INFINITY ? 0.f : r0));
          const float a1 = x[2 * e + 1] == -INFINITY ? 0.f : fast_exp2(x[2 * e + 1] - (r1 == -INFINITY ? 0.f : r1));
          lt[2 * e] += a0;
          lt[2 * e + 1] += a1;
          w[e] = pack_bf16(a0, a1);
        }
        long long c2_ = clock64();
        mwait(&pempty[g & 1], ((g >> 1) & 1) ^ 1);  // PV two tiles back has read this P buffer
        long long c3_ = clock64();
        if (p.dbg && blockIdx.x == 0 && t == 0) {
          p.dbg[0] += c1_ - c0_;  // softmax: waiting for S
          p.dbg[1] += c2_ - c1_;  // softmax: compute
          p.dbg[2] += c3_ - c2_;  // softmax: waiting for the P buffer
          p.dbg[3] += 1;
        }
        uint8_t* prow = sm + OFF_P + (g & 1) * P_TILE + t * 128;
#pragma unroll
        for (int c = 0; c < NC / 8; ++c)
          *reinterpret_cast<uint4*>(prow + ((c ^ (t & 7)) * 16)) = make_uint4(w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
        proxy();
        fb();
        marrive(&pfull[g & 1]);
      }
      // ---- unit epilogue: row sums over the CTA, O^T / l -> out, lse ----
#pragma unroll
      for (int r = 0; r < NC; ++r) {
        float s = lt[r];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        lt[r] = s;
      }
      if (lane == 0)
#pragma unroll
        for (int r = 0; r < NC; ++r) red[sw * NC + r] = lt[r];
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
#pragma unroll
      for (int r = 0; r < NC; ++r) lt[r] = (red[r] + red[NC + r]) + (red[2 * NC + r] + red[3 * NC + r]);
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
      mwait(odone, n_u & 1);
      fa();
#pragma unroll
      for (int c0 = 0; c0 < NC; c0 += 16) {
        float o[16];
        ld16(tmem + loff + O_COL + c0, o);
        wld();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int r = c0 + i;
          if (r < M) {
            const float l = lt[r];
            p.out[(u * M + r) * (int64_t)D + t] = __float2bfloat16_rn(l > 0.f ? o[i] / l : 0.f);
          }
        }
      }
      if (t == 0 && p.lse) {
#pragma unroll
        for (int r = 0; r < NC; ++r)
          if (r < M) {
            const float l = lt[r], m = mref[r];
            p.lse[u * M + r] = l > 0.f ? (m + __log2f(l)) * 0.6931471805599453f : -INFINITY;
          }
      }
      fb();
      marrive(oempty);
      gj += nt;
    }
  }
  fb();
  __syncthreads();
  if (warp == 2) {
    fa();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tmem));
  }
}

}  // namespace

extern "C" int decode_tc(const void* q, const void* k, const void* v, long long kv_stride, long long units, int M,
                         int R, int base, const int* idx, long long idx_ld, const int* cnt, float scale, void* out,
                         float* lse, int sms, void* stream, long long* dbg) {
  if (M > NC || R != 5) return 2;
  P p;
  p.q = (const __nv_bfloat16*)q;
  p.k = (const __nv_bfloat16*)k;
  p.v = (const __nv_bfloat16*)v;
  p.kv_stride = kv_stride;
  p.units = units;
  p.M = M;
  p.R = R;
  p.base = base;
  p.idx = idx;
  p.idx_ld = idx_ld;
  p.cnt = cnt;
  p.sl2 = scale * 1.4426950408889634f;
  p.out = (__nv_bfloat16*)out;
  p.lse = lse;
  p.dbg = dbg;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(decode_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    attr = true;
  }
  const int grid = (int)(units < sms ? units : sms);
  decode_tc_kernel<<<grid, THREADS, SMEM, (cudaStream_t)stream>>>(p);
  return (int)cudaGetLastError();
}
