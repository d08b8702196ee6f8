// sts_capture.cu — draft-score capture on the Blackwell tensor-core path:
// TMA tensor-tile loads of the contiguous draft K, S^T = K.Q^T on tcgen05
// (keys as M = 128, the unit's stacked query rows as N, fp32 accumulator in
// TMEM), epilogue warps reading TMEM with tcgen05.ld.
//
// Replaces the draft attention record of the reference (`_run_block`
// record_attention, src/toymodel.py:315-352, reached via specdec.propose,
// src/specdec.py:150-167) in two passes over the draft K:
//   LSE   — per (unit, row) log-sum-exp of scale * q.k over the row's causal
//           keys; CTAs own contiguous ranges of the global (unit, key-tile)
//           space, write per-piece partials, the last CTA of a unit merges;
//   PROBS — p = exp(s - lse): summed over each head's speculative rows for
//           the committed positions (mode S), per row (mode R), or the raw
//           scores (ForwardRecord.scores).
//
// Warp roles (192 threads, one CTA per SM, persistent over its tile range):
//   warp 0   TMA producer (one lane): Q of each unit (double buffered) and a
//            STAGES-deep ring of 128-key K tiles (128B swizzle)
//   warp 1   MMA issuer (one lane): per tile D/16 tcgen05.mma.kind::f16 into
//            one of NACC TMEM accumulators, tcgen05.commit to the barriers
//   warps 2-5 epilogue: thread = key (TMEM lane), registers = the N rows
#include <cuda.h>

#include "sts_decode.cuh"

namespace sts {
namespace {

// epilogue warps: groups of four (one warp per TMEM lane quadrant) taking
// alternate tiles; two groups for N = 32 (registers allow), one for N = 48
// (the LSE pass at N = 48 keeps 3 x 48 row registers per thread: one group)
constexpr int cap_epi_warps(int ncol, int mode) { return (ncol <= 32 || mode != 0) ? 8 : 4; }
constexpr int cap_threads(int ncol, int mode) { return 64 + 32 * cap_epi_warps(ncol, mode); }
constexpr int CAP_KEYS = 128;  // keys per tile = MMA M = TMEM lanes
constexpr int CAP_MODE_LSE = 0, CAP_MODE_PROBS = 1;
constexpr float CAP_LN2 = 0.6931471805599453f;

// ---------------------------------------------------------------------------
// PTX wrappers: mbarrier, TMA, tcgen05
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(
          d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// 32 lanes x 32 consecutive 32-bit columns: thread t of the warp gets lane
// (quadrant*32 + t), columns [col, col + 32)
__device__ __forceinline__ void tc_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tc_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// UMMA shared-memory descriptor: K-major operand, 128-byte swizzle, rows of
// 128 bytes in 8-row (1024 B) core-matrix groups
__device__ __forceinline__ uint64_t umma_desc_sw128(const void* smem) {
  const uint64_t addr = smem_u32(smem);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;          // start address
  d |= (uint64_t)1 << 16;                // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;      // stride byte offset: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                // SWIZZLE_128B
  return d;
}
// instruction descriptor: bf16 x bf16 -> f32, both K-major, M = 128, N
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N) {
  return (1u << 4)                       // D format f32
         | (1u << 7)                     // A bf16
         | (1u << 10)                    // B bf16
         | ((uint32_t)(N >> 3) << 17)    // N
         | ((uint32_t)(M >> 4) << 24);   // M
}

struct CapParams {
  int64_t units;
  int M;            // stacked rows per unit (G * R)
  int N;            // MMA N (M rounded up to 16)
  int R;            // rows per head
  int n_keys;       // keys per unit
  int tiles_per_unit;
  int64_t tiles;    // units * tiles_per_unit
  int pos_offset;
  int causal_base;  // rows r at global position causal_base + r % R
  float scale;
  int mode;         // CAP_MODE_LSE / CAP_MODE_PROBS
  int probs_mode;   // 0: S (summed rows, committed keys), 1: R (per row), 2: raw scores
  float* lse_out;   // LSE: final natural-log lse [units][M]
  float* l_part;    // LSE: per-piece partial lse [grid + units][M]
  int* counters;    // LSE: per-unit arrival counters (zeroed per launch)
  const float* lse_in;  // PROBS
  float* out;
  int64_t out_ld;
};

__device__ __forceinline__ int64_t range_begin(int64_t c, int64_t tiles, int64_t grid) { return c * tiles / grid; }

// CTA holding global tile t under the static partition
__device__ __forceinline__ int64_t owner_of(int64_t t, int64_t tiles, int64_t grid) {
  int64_t c = (t * grid) / tiles;
  while (c + 1 < grid && range_begin(c + 1, tiles, grid) <= t) ++c;
  while (c > 0 && range_begin(c, tiles, grid) > t) --c;
  return c;
}

template <int D, int NCOL, int MODE>
struct CapLayout {
  static constexpr int SLABS = D / 64;                    // 128-byte K-major slabs
  static constexpr int KTILE = CAP_KEYS * 128 * SLABS;    // bytes per K tile
  // tiles per pipeline step: one TMA barrier, TPS*D/16 MMAs, one commit and
  // one epilogue hand-off per step (the per-hand-off cost is fixed)
  static constexpr int TPS = (D == 64 && NCOL == 32) ? 4 : 2;
  static constexpr int STEP = TPS * KTILE;
  static constexpr int STAGES = (192 * 1024) / STEP;      // K bytes in flight: 192 KB
  static constexpr int SLOT_COLS = TPS * NCOL;            // TMEM columns per step
  static constexpr int NSLOT = (512 / SLOT_COLS) < 8 ? (512 / SLOT_COLS) : 8;
  static constexpr int TMEM_COLS = NSLOT * SLOT_COLS <= 256 ? 256 : 512;
  static constexpr int QTILE = NCOL * 128 * SLABS;        // bytes per Q tile (N rows)
  static constexpr int OFF_K = 0;
  static constexpr int OFF_Q = OFF_K + STAGES * STEP;
  static constexpr int EPI = cap_epi_warps(NCOL, MODE);
  static constexpr int GROUPS = EPI / 4;
  static constexpr int THREADS = cap_threads(NCOL, MODE);
  static constexpr int OFF_RED = OFF_Q + 2 * QTILE;       // [epilogue warps][NCOL] (m, l) float2
  static constexpr int OFF_BAR = OFF_RED + EPI * NCOL * 8;
  static constexpr int NBAR = 2 * STAGES + 2 * NSLOT + 4;
  static constexpr int SMEM = OFF_BAR + NBAR * 8 + 16 + 1024;  // + TMEM address, + 1024 alignment slack
};

// the step sequence every role walks: steps never span a unit (one Q per step)
struct StepIter {
  int64_t t, t_end, u;
  int kt, tpu, n;
  __device__ __forceinline__ StepIter(int64_t t0, int64_t t1, int tpu_, int tps) : t(t0), t_end(t1), tpu(tpu_) {
    u = t0 / tpu_;
    kt = (int)(t0 - u * tpu_);
    size(tps);
  }
  __device__ __forceinline__ void size(int tps) {
    const int64_t left = t_end - t;
    n = tps;
    if (left < n) n = (int)left;
    if (tpu - kt < n) n = tpu - kt;
  }
  __device__ __forceinline__ bool valid() const { return t < t_end; }
  __device__ __forceinline__ bool unit_first(int64_t t_begin) const { return t == t_begin || kt == 0; }
  __device__ __forceinline__ bool unit_last() const { return t + n == t_end || kt + n == tpu; }
  __device__ __forceinline__ void next(int tps) {
    t += n;
    kt += n;
    if (kt == tpu) {
      kt = 0;
      ++u;
    }
    size(tps);
  }
};

// RT: rows per head at compile time (5 = gamma 4, the configured depth), 0 = runtime p.R;
// MODE: CAP_MODE_LSE or CAP_MODE_PROBS (p.mode is ignored);
// MC: the unit's stacked rows G*R at compile time (0 = runtime p.M): the
// per-score loops then skip the MMA's padding columns (c2: 20 of 32, c3: 35 of 48)
template <int D, int NCOL, int RT, int MODE, int MC = 0>
__global__ void __launch_bounds__(cap_threads(NCOL, MODE), 1)
    capture_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap qmap, CapParams p) {
  using L = CapLayout<D, NCOL, MODE>;
  constexpr int TPS = L::TPS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* full = bars;                    // TMA -> MMA (per stage)
  uint64_t* empty = bars + L::STAGES;       // epilogue (MMA done) -> TMA
  uint64_t* accf = bars + 2 * L::STAGES;    // MMA commit -> epilogue (per slot)
  uint64_t* acce = accf + L::NSLOT;         // epilogue -> MMA
  uint64_t* qfull = acce + L::NSLOT;
  uint64_t* qempty = qfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + L::NBAR);
  float2* red = reinterpret_cast<float2*>(smem + L::OFF_RED);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t grid = gridDim.x;
  const int64_t t_begin = range_begin(blockIdx.x, p.tiles, grid);
  const int64_t t_end = range_begin(blockIdx.x + 1, p.tiles, grid);
  const int TPU = p.tiles_per_unit;

  if (threadIdx.x == 0) {
    for (int i = 0; i < L::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < L::NSLOT; ++i) {
      mbar_init(&accf[i], 1);
      mbar_init(&acce[i], 128);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&qfull[i], 1);
      mbar_init(&qempty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    tma_prefetch_desc(&kmap);
    tma_prefetch_desc(&qmap);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "n"(L::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // programmatic dependent launch: the probability pass may start its
  // prologue and K stream while this grid finishes; it waits (griddepcontrol.
  // wait) only before reading the LSE this grid writes
  if (MODE == CAP_MODE_LSE) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");

  if (warp == 0) {
    // ===== TMA producer =====
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int qb = 0;
      uint32_t qphase[2] = {0, 0};
      for (StepIter it(t_begin, t_end, TPU, TPS); it.valid(); it.next(TPS)) {
        if (it.unit_first(t_begin)) {
          mbar_wait(&qempty[qb], qphase[qb] ^ 1);
          qphase[qb] ^= 1;
          mbar_expect_tx(&qfull[qb], L::QTILE);
#pragma unroll
          for (int s = 0; s < L::SLABS; ++s)
            tma_load_3d(smem + L::OFF_Q + qb * L::QTILE + s * NCOL * 128, &qmap, &qfull[qb], s * 64,
                        (int)(it.u * p.M), 0);
          qb ^= 1;
        }
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_expect_tx(&full[stage], it.n * L::KTILE);
        for (int i = 0; i < it.n; ++i)
#pragma unroll
          for (int s = 0; s < L::SLABS; ++s)
            tma_load_3d(smem + L::OFF_K + stage * L::STEP + i * L::KTILE + s * CAP_KEYS * 128, &kmap, &full[stage],
                        s * 64, (it.kt + i) * CAP_KEYS, (int)it.u);
        if (++stage == L::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer =====
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(CAP_KEYS, NCOL);
      int stage = 0, slot = 0;
      uint32_t phase = 0, sphase = 0;
      int qb = 0, qcur = 0;
      uint32_t qphase[2] = {0, 0};
      for (StepIter it(t_begin, t_end, TPU, TPS); it.valid(); it.next(TPS)) {
        if (it.unit_first(t_begin)) {
          mbar_wait(&qfull[qb], qphase[qb]);
          qphase[qb] ^= 1;
          qcur = qb;
          qb ^= 1;
        }
        mbar_wait(&acce[slot], sphase ^ 1);
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        for (int i = 0; i < it.n; ++i) {
          const uint32_t d_tmem = tmem + (uint32_t)(slot * L::SLOT_COLS + i * NCOL);
#pragma unroll
          for (int s = 0; s < L::SLABS; ++s) {
            const uint64_t ad = umma_desc_sw128(smem + L::OFF_K + stage * L::STEP + i * L::KTILE + s * CAP_KEYS * 128);
            const uint64_t bd = umma_desc_sw128(smem + L::OFF_Q + qcur * L::QTILE + s * NCOL * 128);
#pragma unroll
            for (int k = 0; k < 4; ++k)  // 4 x K=16 bf16 = the 128-byte slab: +32 B per step
              tc_mma(d_tmem, ad + (uint64_t)(2 * k), bd + (uint64_t)(2 * k), idesc, (s | k) != 0);
          }
        }
        tc_commit(&accf[slot]);  // MMA done: accumulators ready AND the K stage reusable
        if (it.unit_last()) tc_commit(&qempty[qcur]);
        if (++stage == L::STAGES) {
          stage = 0;
          phase ^= 1;
        }
        if (++slot == L::NSLOT) {
          slot = 0;
          sphase ^= 1;
        }
      }
    }
  } else {
    // ===== epilogue: thread = key =====
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    const int key_in_tile = quad * 32 + lane;
    const int ew = warp - 2;    // epilogue warp index
    const int grp = ew >> 2;    // steps with index % GROUPS == grp
    const int M = MC > 0 ? MC : p.M, R = p.R;
    constexpr int MR = MC > 0 ? MC : NCOL;  // columns the per-score loops visit
    const int lim = p.causal_base - p.pos_offset;  // row r sees local keys j <= lim + r % R
    const float sl2 = p.scale * LOG2E;
    int slot = 0, stage = 0;
    uint32_t sphase = 0;
    // LSE: per-thread, per-row running (reference m, sum of 2^(x - m)); the
    // reference only moves when a score exceeds it by 2^32 (or on the first
    // score), so the steady state is one FADD + MUFU + FADD per score
    float mx[NCOL], ls[NCOL];
    bool fresh = true;  // some row of this unit has no score yet in this thread (LSE)
    bool lse_ready = false;
    int64_t step_i = 0;
    for (StepIter it(t_begin, t_end, TPU, TPS); it.valid(); it.next(TPS), ++step_i) {
      const int64_t u = it.u;
      if (it.unit_first(t_begin)) {
        fresh = true;
        if (MODE == CAP_MODE_LSE) {
#pragma unroll
          for (int r = 0; r < NCOL; ++r) {
            mx[r] = -INFINITY;
            ls[r] = 0.f;
          }
        } else {
          // this unit's final lse (log2 units) for every row: registers (written
          // by the LSE grid this launch may overlap: wait for it, once)
          if (!lse_ready) {
            asm volatile("griddepcontrol.wait;\n" ::: "memory");
            lse_ready = true;
          }
#pragma unroll
          for (int r = 0; r < NCOL; ++r) mx[r] = (r < M && p.lse_in) ? p.lse_in[u * M + r] * LOG2E : 0.f;
        }
      }
      const bool mine = (step_i % L::GROUPS) == grp;
      if (mine) {
        mbar_wait(&accf[slot], sphase);
        tc_fence_after();
        if (ew == grp * 4 && lane == 0) mbar_arrive(&empty[stage]);  // the MMAs read their K stage: free it
        for (int i = 0; i < it.n; ++i) {
          float s[NCOL];
          const uint32_t ta = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(slot * L::SLOT_COLS + i * NCOL);
          tc_ld32(ta, s);
          if constexpr (NCOL == 48) tc_ld16(ta + 32, s + 32);
          tc_wait_ld();
          const int kt = it.kt + i;
          const int j = kt * CAP_KEYS + key_in_tile;  // local key index
          const bool in_range = j < p.n_keys;
          // every row sees every key of this tile (the common case): no per-row tests
          const int tile_last = kt * CAP_KEYS + CAP_KEYS - 1;
          const bool full_tile = tile_last < p.n_keys && tile_last <= lim;
          if (MODE == CAP_MODE_LSE && full_tile && !fresh) {
            // steady state: x = s*scale*log2e - m (one FFMA), 2^x (MUFU), sum (FADD)
            bool need = false;
#pragma unroll
            for (int r = 0; r < MR; ++r) {
              const float x = fmaf(s[r], sl2, -mx[r]);
              s[r] = x;
              need |= x > 32.f;
            }
            if (__any_sync(0xffffffffu, need)) {  // warp-uniform and rare: a jump of 2^32 moves the reference
#pragma unroll
              for (int r = 0; r < MR; ++r) {
                const float real = s[r] + mx[r];
                const float mn = fmaxf(mx[r], real);
                ls[r] *= fast_exp2(mx[r] - mn);
                mx[r] = mn;
                s[r] = real - mn;
              }
            }
#pragma unroll
            for (int r = 0; r < MR; ++r)
              if (r < M) ls[r] += fast_exp2(s[r]);
            continue;
          }
          if (MODE != CAP_MODE_LSE && full_tile) {
            // probabilities: 2^(s*scale*log2e - lse2) in one FFMA + MUFU
            if (in_range && p.probs_mode != 2) {
#pragma unroll
              for (int r = 0; r < MR; ++r) s[r] = fast_exp2(fmaf(s[r], sl2, -mx[r]));
            } else {
#pragma unroll
              for (int r = 0; r < MR; ++r) s[r] *= p.scale;
            }
          } else {
            // masked tile (a unit's causal tail / past the last key) or the
            // unit's first tile: log2-unit scores, -inf where the row may not look
#pragma unroll
            for (int r = 0; r < NCOL; ++r) {
              const int rm = RT ? r % (RT ? RT : 1) : r % R;
              s[r] = (in_range && j <= lim + rm) ? s[r] * sl2 : -INFINITY;
            }
            if (MODE == CAP_MODE_LSE) {
              bool need = false;
#pragma unroll
              for (int r = 0; r < NCOL; ++r)
                if (r < M) need |= s[r] > mx[r] + 32.f;
              if (__any_sync(0xffffffffu, need)) {
#pragma unroll
                for (int r = 0; r < NCOL; ++r) {
                  const float mn = fmaxf(mx[r], s[r]);
                  ls[r] = mn == -INFINITY ? 0.f : ls[r] * fast_exp2(mx[r] - mn);
                  mx[r] = mn;
                }
              }
              bool any_empty = false;
#pragma unroll
              for (int r = 0; r < NCOL; ++r) {
                const float e = fast_exp2(s[r] - mx[r]);  // NaN only for (-inf) - (-inf): no key yet
                ls[r] += (r < M && mx[r] != -INFINITY) ? e : 0.f;
                if (r < M) any_empty |= mx[r] == -INFINITY;
              }
              fresh = __any_sync(0xffffffffu, any_empty);
              continue;
            }
            if (in_range && p.probs_mode != 2) {
#pragma unroll
              for (int r = 0; r < NCOL; ++r) s[r] = s[r] == -INFINITY ? -INFINITY : fast_exp2(s[r] - mx[r]);
            } else {
#pragma unroll
              for (int r = 0; r < NCOL; ++r) s[r] = s[r] == -INFINITY ? -INFINITY : s[r] * CAP_LN2;
            }
          }
          // s[r]: probabilities (modes S / R) or raw natural-unit scores (mode
          // raw); -inf marks a key the row may not see
          if (in_range) {
            if (p.probs_mode == 0) {
              if (j < lim) {  // committed positions only (every row sees them)
                float* outp = p.out + (u * (M / R)) * p.out_ld + j;
                if constexpr (RT > 0) {
#pragma unroll
                  for (int g = 0; g < NCOL / (RT ? RT : 1); ++g) {
                    if (g * RT >= M) continue;
                    float a = s[g * RT];
#pragma unroll
                    for (int ii = 1; ii < RT; ++ii) a = __fadd_rn(a, s[g * RT + ii]);  // the head's rows in order
                    outp[g * p.out_ld] = a;
                  }
                } else {
                  float a = 0.f;
                  int rm = 0, g = 0;
#pragma unroll
                  for (int r = 0; r < NCOL; ++r) {
                    if (r >= M) continue;
                    a = rm == 0 ? s[r] : __fadd_rn(a, s[r]);
                    if (++rm == R) {
                      outp[g * p.out_ld] = a;
                      ++g;
                      rm = 0;
                    }
                  }
                }
              }
            } else {
              float* outp = p.out + (u * M) * p.out_ld + j;
#pragma unroll
              for (int r = 0; r < NCOL; ++r) {
                if (r >= M || s[r] == -INFINITY) continue;
                outp[r * p.out_ld] = s[r];
              }
            }
          }
        }
        tc_fence_before();
        mbar_arrive(&acce[slot]);
      }
      if (++slot == L::NSLOT) {
        slot = 0;
        sphase ^= 1;
      }
      if (++stage == L::STAGES) stage = 0;
      if (MODE == CAP_MODE_LSE && it.unit_last()) {
        // reduce (m, l) per row over the 128 keys x epilogue groups of this
        // CTA, publish the piece, the last arriving piece of the unit merges
#pragma unroll
        for (int r = 0; r < NCOL; ++r) {
          if (r >= M) continue;
          float m = mx[r], l = ls[r];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
            const float l2 = __shfl_xor_sync(0xffffffffu, l, o);
            const float mn = fmaxf(m, m2);
            l = (mn == -INFINITY) ? 0.f : l * fast_exp2(m - mn) + l2 * fast_exp2(m2 - mn);
            m = mn;
          }
          if (lane == 0) red[ew * NCOL + r] = make_float2(m, l);
        }
        asm volatile("bar.sync 1, %0;\n" ::"n"(32 * L::EPI) : "memory");
        const int64_t first = u * TPU, last = first + TPU - 1;
        const int64_t c0 = owner_of(first, p.tiles, grid), c1 = owner_of(last, p.tiles, grid);
        if (ew == 0 && lane < M) {
          const int r = lane;
          float m = -INFINITY, l = 0.f;
          for (int w = 0; w < L::EPI; ++w) {
            const float2 x = red[w * NCOL + r];
            const float mn = fmaxf(m, x.x);
            l = (mn == -INFINITY) ? 0.f : l * fast_exp2(m - mn) + x.y * fast_exp2(x.x - mn);
            m = mn;
          }
          const float lse = l > 0.f ? (m + __log2f(l)) * CAP_LN2 : -INFINITY;
          if (c0 == c1) {
            p.lse_out[u * M + r] = lse;
          } else {
            p.l_part[(blockIdx.x + u) * M + r] = lse;
            __threadfence();
          }
        }
        asm volatile("bar.sync 1, %0;\n" ::"n"(32 * L::EPI) : "memory");
        if (ew == 0 && c0 != c1) {
          int prev = 0;
          if (lane == 0) prev = atomicAdd(&p.counters[u], 1);
          prev = __shfl_sync(0xffffffffu, prev, 0);
          if (prev == (int)(c1 - c0)) {  // last piece: merge all pieces of u
            __threadfence();
            for (int r = lane; r < M; r += 32) {
              float m = -INFINITY, l = 0.f;
              for (int64_t c = c0; c <= c1; ++c) {
                const float x = __ldcg(&p.l_part[(c + u) * M + r]);
                const float mn = fmaxf(m, x);
                l = (mn == -INFINITY) ? 0.f : l * __expf(m - mn) + __expf(x - mn);
                m = mn;
              }
              p.lse_out[u * M + r] = l > 0.f ? m + __logf(l) : -INFINITY;
            }
            if (lane == 0) p.counters[u] = 0;  // ready for the next launch
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(L::TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
// host side: tensor maps via the driver entry point (no -lcuda link)
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(f);
  }
  return fn;
}

// 3-D bf16 map over [units][rows][d] (unit stride in elements), box {64, box_rows, 1}, 128B swizzle
int make_map(CUtensorMap* map, const void* base, int64_t units, int64_t rows, int d, int64_t unit_stride,
             int64_t row_stride, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  STS_REQUIRE(fn, STS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)rows, (cuuint64_t)units};
  const cuuint64_t strides[2] = {(cuuint64_t)row_stride * 2, (cuuint64_t)unit_stride * 2};
  const cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  STS_REQUIRE(r == CUDA_SUCCESS, STS_ERR_CONTRACT,
              "tensor map encode failed (%d): base %p must be 16-byte aligned, strides multiples of 16 bytes", (int)r,
              base);
  return STS_OK;
}

template <int D, int NCOL, int RT, int MODE, int MC>
int launch_m(const CUtensorMap& km, const CUtensorMap& qm, const CapParams& p, cudaStream_t st) {
  using L = CapLayout<D, NCOL, MODE>;
  static_assert(L::SMEM <= 227 * 1024, "capture shared memory");
  STS_CUDA_CHECK(cudaFuncSetAttribute(capture_kernel<D, NCOL, RT, MODE, MC>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM));
  const int64_t grid = p.tiles < num_sms() ? p.tiles : num_sms();
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(L::THREADS);
  cfg.dynamicSmemBytes = L::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = MODE == CAP_MODE_PROBS ? 1 : 0;  // the probability pass overlaps the LSE pass's tail
  STS_CUDA_CHECK(cudaLaunchKernelEx(&cfg, capture_kernel<D, NCOL, RT, MODE, MC>, km, qm, p));
  count_launch();
  return STS_OK;
}

template <int D, int NCOL, int RT, int MC = 0>
int launch_t(const CUtensorMap& km, const CUtensorMap& qm, const CapParams& p, cudaStream_t st) {
  return p.mode == CAP_MODE_LSE ? launch_m<D, NCOL, RT, CAP_MODE_LSE, MC>(km, qm, p, st)
                                : launch_m<D, NCOL, RT, CAP_MODE_PROBS, MC>(km, qm, p, st);
}

template <int D, int NCOL>
int launch_r(const CUtensorMap& km, const CUtensorMap& qm, const CapParams& p, cudaStream_t st) {
  if (p.R != 5) return launch_t<D, NCOL, 0>(km, qm, p, st);
  // the measured shapes' stacked rows at compile time (4 or 7 q-heads per kv-head, gamma 4)
  if constexpr (D == 64 && NCOL == 32) {
    if (p.M == 20) return launch_t<D, NCOL, 5, 20>(km, qm, p, st);
  }
  if constexpr (D == 64 && NCOL == 48) {
    if (p.M == 35) return launch_t<D, NCOL, 5, 35>(km, qm, p, st);
  }
  return launch_t<D, NCOL, 5>(km, qm, p, st);
}

}  // namespace

size_t capture_workspace_bytes(int64_t units, int M) {
  const int64_t slots = (int64_t)num_sms() + units;
  return ((size_t)units * 4 + 255) / 256 * 256 + (size_t)slots * M * sizeof(float) + 256;
}

// mode: 0 LSE, 1 PROBS; probs_mode as DecodeParams
int capture_launch(int mode, const void* q, const void* k, int64_t kv_unit_stride, int64_t units, int G, int R, int d,
                   int n_keys, int pos_offset, int base, float scale, float* lse, const float* lse_in, int probs_mode,
                   float* out, int64_t out_ld, void* ws, size_t ws_bytes, cudaStream_t st) {
  const int M = G * R;
  STS_REQUIRE(d == 64 || d == 128, STS_ERR_CONTRACT, "draft capture supports head_dim 64 or 128, got %d", d);
  STS_REQUIRE(M >= 1 && M <= 48, STS_ERR_CONTRACT, "draft capture supports G*R <= 48 stacked rows, got %d", M);
  STS_REQUIRE(kv_unit_stride % 8 == 0, STS_ERR_CONTRACT, "draft K unit stride must be a multiple of 8 elements");
  STS_REQUIRE((reinterpret_cast<uintptr_t>(k) & 15) == 0 && (reinterpret_cast<uintptr_t>(q) & 15) == 0,
              STS_ERR_CONTRACT, "draft q / K must be 16-byte aligned");
  if (units == 0 || n_keys == 0) return STS_OK;
  CapParams p;
  memset(&p, 0, sizeof(p));
  p.units = units;
  p.M = M;
  p.N = M <= 32 ? 32 : 48;
  p.R = R;
  p.n_keys = n_keys;
  p.tiles_per_unit = (n_keys + CAP_KEYS - 1) / CAP_KEYS;
  p.tiles = units * p.tiles_per_unit;
  p.pos_offset = pos_offset;
  p.causal_base = base;
  p.scale = scale;
  p.mode = mode;
  p.probs_mode = probs_mode;
  p.lse_out = lse;
  p.lse_in = lse_in;
  p.out = out;
  p.out_ld = out_ld;
  if (mode == CAP_MODE_LSE) {
    const size_t need = capture_workspace_bytes(units, M);
    STS_REQUIRE(ws && ws_bytes >= need, STS_ERR_CONTRACT, "capture workspace too small: need %zu, got %zu", need,
                ws_bytes);
    p.counters = static_cast<int*>(ws);
    p.l_part = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + ((size_t)units * 4 + 255) / 256 * 256);
    STS_CUDA_CHECK(cudaMemsetAsync(p.counters, 0, (size_t)units * 4, st));
  }
  CUtensorMap km, qm;
  int rc = make_map(&km, k, units, n_keys, d, kv_unit_stride, d, CAP_KEYS);
  if (rc != STS_OK) return rc;
  // Q as one [units*M][d] matrix: a box of N >= M rows starting at unit u's
  // first row (rows past M belong to the next unit or are zero-filled; the
  // epilogue ignores columns >= M)
  rc = make_map(&qm, q, 1, units * M, d, units * M * (int64_t)d, d, p.N);
  if (rc != STS_OK) return rc;
  if (d == 64) return p.N == 32 ? launch_r<64, 32>(km, qm, p, st) : launch_r<64, 48>(km, qm, p, st);
  return p.N == 32 ? launch_r<128, 32>(km, qm, p, st) : launch_r<128, 48>(km, qm, p, st);
}

}  // namespace sts
