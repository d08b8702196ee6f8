// sts_prefill_tc.cu — block-sparse prefill attention on tcgen05 (STS-PD,
// SURVEY §8f row 1): masked prefill of the reference (`forward_prefill(masks=
// ...)` -> `_run_block`, src/toymodel.py:315-348, :370-399) with the masks of
// `draft_masks_prefill` (src/sparsity.py:122-130) made tile-granular:
//
//   one key-block set per (kv-head, 128-row query tile): the committed blocks
//   (64 keys, all before the tile) the selection picked for the tile, plus the
//   tile's two diagonal blocks under the causal mask.  Row t of tile T sees
//   the selected committed keys and the diagonal keys <= t.
//
// Persistent CTAs (one per SM) walk the work items (q-head, query tile) in
// snake order, heavy tiles first; a tile's 128 rows = the 128 TMEM lanes.
// Warp roles:
//   warp 0   TMA producer: Q tile once, then K and V blocks of the list
//            (128B swizzle; ring of STAGES (K, V) blocks)
//   warps 1-2 MMA issuers, one per softmax group (even / odd key blocks):
//            S_j = Q.K_j^T (M=128 rows, N=64 keys, K=d) into the group's
//            TMEM S slot, issued as soon as the group has read S_{j-2};
//            O_g += P_j.V_j (M=128, N=d, K=64; V as an MN-major operand)
//   warps 3-10 softmax (two groups of 4), thread = query row: tcgen05.ld of
//            its S row, causal mask on diagonal blocks, online max with lazy
//            rescale (O rows in TMEM rescaled only when the max grows by
//            > 2^8), P in bf16 written back to TMEM (tcgen05.st: the A operand
//            of PV comes from TMEM, no shared-memory round trip), row sums in
//            fp32; at the end O / l to global (bf16)
#include <cuda.h>

#include "sts_decode.cuh"

namespace sts {
namespace {

constexpr int PF_ROWS = 128;   // query tile = MMA M = TMEM lanes
constexpr int PF_BLK = 64;     // keys per block = MMA N of S, K of PV
constexpr int PF_STAGES = 5;  // P lives in TMEM: shared memory holds two Q tiles + 5 K/V stages
constexpr int PF_THREADS = 352;  // TMA, two MMA issuers, two softmax warp groups (even / odd key blocks)
constexpr float PF_RESCALE = 8.f;  // log2 growth of the row max that forces an O rescale

__device__ __forceinline__ void pf_mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void pf_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void pf_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void pf_wait(uint64_t* bar, uint32_t parity) {
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
__device__ __forceinline__ void pf_tma3(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void pf_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void pf_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void pf_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void pf_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(
          d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void pf_ld32(uint32_t taddr, float* v) {
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
__device__ __forceinline__ void pf_st32(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
      "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])),
      "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])),
      "r"(__float_as_uint(v[17])), "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])),
      "r"(__float_as_uint(v[20])), "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])),
      "r"(__float_as_uint(v[23])), "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])),
      "r"(__float_as_uint(v[26])), "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])),
      "r"(__float_as_uint(v[29])), "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
      : "memory");
}
// D += A.B with A (M x 16, bf16 pairs per 32-bit column) in TMEM, B from shared memory
__device__ __forceinline__ void pf_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(
          d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void pf_st32u(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void pf_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void pf_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// K-major operand, 128B swizzle: 8-row groups of 1024 B (SBO), LBO unused
__device__ __forceinline__ uint64_t pf_desc_k(const void* p) {
  const uint64_t a = smem_u32(p);
  return ((a >> 4) & 0x3FFFull) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
// MN-major operand, 128B swizzle: atoms of 64 elements (MN) x 8 rows (K);
// LBO = bytes between MN atoms, SBO = bytes between 8-row K groups
__device__ __forceinline__ uint64_t pf_desc_mn(const void* p, uint32_t lbo, uint32_t sbo) {
  const uint64_t a = smem_u32(p);
  return ((a >> 4) & 0x3FFFull) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) |
         (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t pf_idesc(int M, int N, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

struct PfParams {
  int n;             // keys = query rows of the layer
  int heads_q, group;  // q-heads, q-heads per kv-head
  int tiles;         // ceil(n / 128)
  float scale;
  const int32_t* idx;  // [kv_heads * tiles][idx_ld] committed tokens (whole 64-key blocks, ascending); null = dense
  int64_t idx_ld;
  const int32_t* cnt;
  __nv_bfloat16* out;  // [heads_q][n][d]
  int32_t* status;
};

template <int D>
struct PfLayout {
  static constexpr int SLABS = D / 64;
  static constexpr int Q_BYTES = PF_ROWS * 128 * SLABS;
  static constexpr int KB_BYTES = PF_BLK * 128 * SLABS;     // one K block (= one V block)
  static constexpr int OFF_Q = 0;                            // two Q tiles (consecutive work items)
  static constexpr int OFF_K = OFF_Q + 2 * Q_BYTES;
  static constexpr int OFF_V = OFF_K + PF_STAGES * KB_BYTES;
  static constexpr int OFF_X = OFF_V + PF_STAGES * KB_BYTES;  // [128 rows] (m, l) of the odd group
  static constexpr int OFF_BAR = OFF_X + PF_ROWS * 8;
  // full[S], empty[S], sfull[2], sempty[2], pfull[2], odone[2], qfull[2], qempty[2], oempty
  static constexpr int NBAR = 2 * PF_STAGES + 13;
  static constexpr int SMEM = OFF_BAR + NBAR * 8 + 16 + 1024;
  static constexpr int S_COLS = PF_BLK;                       // per S slot
  static constexpr int O_COL = 2 * PF_BLK;                    // O_even, O_odd after the two S slots
  static constexpr int P_COL = O_COL + 2 * D;                  // P_even, P_odd: bf16 pairs, PF_BLK / 2 columns each
  static constexpr int TMEM_COLS = P_COL + PF_BLK <= 256 ? 256 : 512;
  static_assert(P_COL + PF_BLK <= 512, "TMEM columns");
  static_assert(SMEM <= 227 * 1024, "prefill shared memory exceeds the 227 KB per-CTA limit");
};

// the tile's block list: committed blocks from the selection, then the diagonal
__device__ __forceinline__ int pf_nblocks(const PfParams& p, int kvh, int T, int& ncommit) {
  const int diag0 = 2 * T;
  const int nblk_total = (p.n + PF_BLK - 1) / PF_BLK;
  const int ndiag = min(2, nblk_total - diag0);
  if (!p.idx) {
    ncommit = diag0;
  } else {
    ncommit = p.cnt[(int64_t)kvh * p.tiles + T] / PF_BLK;
  }
  return ncommit + ndiag;
}
__device__ __forceinline__ int pf_block(const PfParams& p, int kvh, int T, int ncommit, int j) {
  if (j >= ncommit) return 2 * T + (j - ncommit);
  if (!p.idx) return j;
  return p.idx[((int64_t)kvh * p.tiles + T) * p.idx_ld + (int64_t)j * PF_BLK] / PF_BLK;
}

// the n-th work item of this CTA: rounds of gridDim.x items in snake order
// (CTA b takes item b of even rounds, item G-1-b of odd rounds), so with
// heavy tiles first every CTA gets an even share of the work
__device__ __forceinline__ int pf_item_index(int n, int n_items) {
  const int G = gridDim.x, b = blockIdx.x;
  const int i = n * G + ((n & 1) ? G - 1 - b : b);
  return i < n_items ? i : n_items;
}

// work item i of the persistent grid: heavy (late) tiles first, heads inner
struct PfItem {
  int T, hq, kvh, ncommit, nb;
};
__device__ __forceinline__ PfItem pf_item(const PfParams& p, int i) {
  PfItem it;
  it.T = p.tiles - 1 - i / p.heads_q;
  it.hq = i % p.heads_q;
  it.kvh = it.hq / p.group;
  it.nb = pf_nblocks(p, it.kvh, it.T, it.ncommit);
  return it;
}

// Persistent: one CTA per SM walks the work items (tile, q-head) i = blockIdx.x,
// blockIdx.x + gridDim.x, ... (heavy tiles first).  Every barrier phase is
// counted across items, the K/V ring and the S slots flow from one item into
// the next, and the Q tile is double-buffered, so an item's loads and first
// scores overlap the previous item's last blocks and epilogue.
template <int D>
__global__ void __launch_bounds__(PF_THREADS, 1) prefill_tc_kernel(const __grid_constant__ CUtensorMap qmap,
                                                                   const __grid_constant__ CUtensorMap kmap,
                                                                   const __grid_constant__ CUtensorMap vmap,
                                                                   PfParams p) {
  using L = PfLayout<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* full = bars;
  uint64_t* empty = bars + PF_STAGES;
  uint64_t* sfull = bars + 2 * PF_STAGES;
  uint64_t* sempty = sfull + 2;
  uint64_t* pfull = sempty + 2;
  uint64_t* odone = pfull + 2;   // odone[g]: group g's latest PV landed in O_g
  uint64_t* qfull = odone + 2;   // qfull[b] / qempty[b]: Q buffer b loaded / no longer read
  uint64_t* qempty = qfull + 2;
  uint64_t* oempty = qempty + 2;  // the item's epilogue has read O_0 and O_1
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + L::NBAR);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = p.tiles * p.heads_q;

  if (threadIdx.x == 0) {
    for (int i = 0; i < PF_STAGES; ++i) {
      pf_mbar_init(&full[i], 1);
      pf_mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      pf_mbar_init(&sfull[i], 1);
      pf_mbar_init(&sempty[i], 128);
      pf_mbar_init(&pfull[i], 128);
      pf_mbar_init(&odone[i], 1);
      pf_mbar_init(&qfull[i], 1);
      pf_mbar_init(&qempty[i], 2);  // both MMA issuers
    }
    pf_mbar_init(oempty, 128);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "n"(L::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  pf_fence_before();
  __syncthreads();
  pf_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // the whole warp walks the items: the block ids of 32 blocks at a time
    // come in one load across the lanes (a selection's list is a dependent
    // read, one per block would serialise the producer), lane 0 issues
    uint32_t kv = 0;  // blocks loaded so far (ring position)
    int n_it = 0;
    for (int i = pf_item_index(0, n_items); i < n_items; i = pf_item_index(n_it + 1, n_items), ++n_it) {
      const PfItem it = pf_item(p, i);
      const int qb = n_it & 1;
      if (lane == 0) {
        if (n_it >= 2) pf_wait(&qempty[qb], ((n_it >> 1) - 1) & 1);  // item n_it - 2 done with this Q buffer
        pf_expect_tx(&qfull[qb], L::Q_BYTES);
#pragma unroll
        for (int s = 0; s < L::SLABS; ++s)
          pf_tma3(smem + L::OFF_Q + qb * L::Q_BYTES + s * PF_ROWS * 128, &qmap, &qfull[qb], s * 64,
                  it.T * PF_ROWS, it.hq);
      }
      for (int j0 = 0; j0 < it.nb; j0 += 32) {
        const int bid = j0 + lane < it.nb ? pf_block(p, it.kvh, it.T, it.ncommit, j0 + lane) : 0;
        const int cnt32 = min(32, it.nb - j0);
        for (int jl = 0; jl < cnt32; ++jl, ++kv) {
          const int b = __shfl_sync(0xffffffffu, bid, jl);
          if (lane == 0) {
            const int stage = kv % PF_STAGES;
            pf_wait(&empty[stage], ((kv / PF_STAGES) & 1) ^ 1);
            pf_expect_tx(&full[stage], 2 * L::KB_BYTES);
#pragma unroll
            for (int s = 0; s < L::SLABS; ++s) {
              pf_tma3(smem + L::OFF_K + stage * L::KB_BYTES + s * PF_BLK * 128, &kmap, &full[stage], s * 64,
                      b * PF_BLK, it.kvh);
              pf_tma3(smem + L::OFF_V + stage * L::KB_BYTES + s * PF_BLK * 128, &vmap, &full[stage], s * 64,
                      b * PF_BLK, it.kvh);
            }
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == 1 || warp == 2) {
    // one MMA issuer per softmax group (warp 1: even blocks, warp 2: odd
    // blocks), so neither group's next S waits behind the other group's P
    if (lane == 0) {
      const int g = warp - 1;
      constexpr uint32_t id_s = pf_idesc(PF_ROWS, PF_BLK, false);
      constexpr uint32_t id_o = pf_idesc(PF_ROWS, D, true);
      uint32_t sc = 0, pc = 0;  // S / PV issued by this issuer (slot g uses)
      uint32_t kv0 = 0;         // ring position of the item's block 0
      int n_it = 0;
      for (int i = pf_item_index(0, n_items); i < n_items; i = pf_item_index(n_it + 1, n_items), ++n_it) {
        const PfItem it = pf_item(p, i);
        const int nb = it.nb;
        const int qb = n_it & 1;
        pf_wait(&qfull[qb], (n_it >> 1) & 1);
        pf_fence_after();
        auto issue_s = [&](int j) {  // S_j into TMEM slot g
          const uint32_t kv = kv0 + j;
          const int stage = kv % PF_STAGES;
          pf_wait(&sempty[g], (sc & 1) ^ 1);  // the group has read its previous S
          pf_wait(&full[stage], (kv / PF_STAGES) & 1);
          pf_fence_after();
          const uint32_t d_tmem = tmem + g * L::S_COLS;
#pragma unroll
          for (int s = 0; s < L::SLABS; ++s) {
            const uint64_t ad = pf_desc_k(smem + L::OFF_Q + qb * L::Q_BYTES + s * PF_ROWS * 128);
            const uint64_t bd = pf_desc_k(smem + L::OFF_K + stage * L::KB_BYTES + s * PF_BLK * 128);
#pragma unroll
            for (int k = 0; k < 4; ++k) pf_mma(d_tmem, ad + 2 * k, bd + 2 * k, id_s, (s | k) != 0);
          }
          pf_commit(&sfull[g]);
          ++sc;
        };
        // S_{j+2} reuses S_j's slot: issued as soon as the group has read S_j
        // (early in softmax j), so its next scores are ready when it finishes
        if (g < nb) issue_s(g);
        for (int j = g; j < nb; j += 2) {
          if (j + 2 < nb) issue_s(j + 2);
          const uint32_t kv = kv0 + j;
          const int stage = kv % PF_STAGES;
          pf_wait(&pfull[g], pc & 1);
          if (j < 2 && n_it > 0) pf_wait(oempty, (n_it - 1) & 1);  // O_g drained by the last epilogue
          pf_fence_after();
          const uint32_t a_tmem = tmem + L::P_COL + g * (PF_BLK / 2);  // P_j as the A operand, from TMEM
          // V block [64 keys][D] as an MN-major B operand: MN atoms (64 d) are
          // the slabs (LBO), K groups of 8 keys are 1024 B apart (SBO)
          const uint64_t bd = pf_desc_mn(smem + L::OFF_V + stage * L::KB_BYTES, PF_BLK * 128, 1024);
#pragma unroll
          for (int k = 0; k < PF_BLK / 16; ++k)
            pf_mma_ts(tmem + L::O_COL + g * D, a_tmem + 8 * k, bd + (uint64_t)((16 * 128) >> 4) * k, id_o,
                      (j >= 2 || k != 0) ? 1u : 0u);
          pf_commit(&empty[stage]);  // K and V of this block no longer read
          pf_commit(&odone[g]);      // O_g holds the group's blocks up to j (frees P buffer g)
          ++pc;
        }
        pf_commit(&qempty[qb]);  // this issuer's reads of Q buffer qb are done
        kv0 += nb;
      }
    }
  } else {
    // ===== softmax: thread = query row; group g takes the blocks j = g mod 2 =====
    const int quad = warp & 3;
    const int grp = (warp - 3) >> 2;
    const int r = quad * 32 + lane;  // row within the tile (TMEM lane)
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const uint32_t o_col = L::O_COL + grp * D;
    const float sl2 = p.scale * LOG2E;
    float2* xch = reinterpret_cast<float2*>(smem + L::OFF_X);
    uint32_t u0 = 0, u1 = 0;  // blocks processed so far by group 0 / group 1 (barrier phases)
    int n_it = 0;
    for (int i = pf_item_index(0, n_items); i < n_items; i = pf_item_index(n_it + 1, n_items), ++n_it) {
      const PfItem it = pf_item(p, i);
      const int nb = it.nb;
      const int row = it.T * PF_ROWS + r;  // query position
      uint32_t& u = grp ? u1 : u0;
      float m = -INFINITY, l = 0.f;
      for (int j = grp; j < nb; j += 2, ++u) {
        const int b = 2 * it.T + (j - it.ncommit);  // (used for the diagonal blocks only)
        pf_wait(&sfull[grp], u & 1);
        pf_fence_after();
        float s[PF_BLK];
        pf_ld32(tmem + lane_off + grp * L::S_COLS, s);
        pf_ld32(tmem + lane_off + grp * L::S_COLS + 32, s + 32);
        pf_wait_ld();
        pf_fence_before();
        pf_arrive(&sempty[grp]);
        // row max of the raw scores (the scale is folded into the exponent's FFMA)
        float mx = -INFINITY;
        if (j >= it.ncommit) {  // diagonal block: causal mask (and the ragged end of the prompt)
#pragma unroll
          for (int c = 0; c < PF_BLK; ++c) {
            const int key = b * PF_BLK + c;
            s[c] = (key <= row && key < p.n) ? s[c] : -INFINITY;
            mx = fmaxf(mx, s[c]);
          }
        } else {
          float m8[8];  // 8 independent chains: the max is not a 64-long dependency
#pragma unroll
          for (int c = 0; c < 8; ++c) m8[c] = s[c];
#pragma unroll
          for (int c = 8; c < PF_BLK; ++c) m8[c & 7] = fmaxf(m8[c & 7], s[c]);
          mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])), fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
        }
        mx *= sl2;
        // lazy rescale, warp-uniform (tcgen05.ld/st are warp-collective): rows
        // whose max grew by > 2^8 rescale their O row
        const bool need = mx > m + PF_RESCALE;
        const bool any = __any_sync(0xffffffffu, need);
        float m_new = m, f = 1.f;
        if (any) {
          if (j < 2) {
            m_new = mx;  // the group's first block of the item: its PV overwrites O_grp
          } else if (need) {
            f = fast_exp2(m - mx);
            m_new = mx;
          }
        }
        const float mb = m_new == -INFINITY ? 0.f : m_new;  // a row with no key yet: P = 0, not NaN
        // P = 2^(s - m) in bf16 (before waiting for the group's previous PV)
        uint32_t w[PF_BLK / 2];
        float rs4[4] = {0.f, 0.f, 0.f, 0.f};  // 4 independent sum chains
#pragma unroll
        for (int e = 0; e < PF_BLK / 2; ++e) {
          const float a0 = fast_exp2(fmaf(s[2 * e], sl2, -mb)), a1 = fast_exp2(fmaf(s[2 * e + 1], sl2, -mb));
          rs4[e & 3] += a0 + a1;
          const __nv_bfloat162 h = __floats2bfloat162_rn(a0, a1);
          w[e] = *reinterpret_cast<const uint32_t*>(&h);
        }
        const float rs = (rs4[0] + rs4[1]) + (rs4[2] + rs4[3]);
        // the group's previous PV (maybe the last item's) read P buffer grp and wrote O_grp
        if (u > 0) pf_wait(&odone[grp], (u - 1) & 1);
        if (any) {
          if (j < 2) {
            l = 0.f;
          } else {
            pf_fence_after();
#pragma unroll
            for (int c0 = 0; c0 < D; c0 += 32) {
              float o[32];
              pf_ld32(tmem + lane_off + o_col + c0, o);
              pf_wait_ld();
#pragma unroll
              for (int c = 0; c < 32; ++c) o[c] *= f;
              pf_st32(tmem + lane_off + o_col + c0, o);
            }
            pf_wait_st();
            l *= f;
          }
        }
        m = m_new;
        // the row's P into its TMEM lane: the A operand of PV_j
        pf_st32u(tmem + lane_off + L::P_COL + grp * (PF_BLK / 2), w);
        pf_wait_st();
        l += rs;
        pf_fence_before();
        pf_arrive(&pfull[grp]);
      }
      // both groups track both counts: the other group's blocks of this item
      if (grp == 1) u0 += (nb + 1) / 2;
      else u1 += nb / 2;
      // epilogue: the odd group hands its (m, l) to the even group, which
      // merges O_even and O_odd (both in its TMEM lanes) and writes O / l
      if (grp == 1) {
        if (n_it > 0) asm volatile("bar.sync 2, 256;\n" ::: "memory");  // group 0 has read the last (m, l)
        xch[r] = make_float2(m, l);
      }
      asm volatile("bar.sync 1, 256;\n" ::: "memory");
      if (grp == 0) {
        const bool has1 = nb >= 2;
        // the last PVs of both groups in this item (group 0: u0 - 1, group 1: u1 - 1)
        pf_wait(&odone[0], (u0 - 1) & 1);
        if (has1) pf_wait(&odone[1], (u1 - 1) & 1);
        pf_fence_after();
        const float2 x1 = xch[r];
        if (pf_item_index(n_it + 1, n_items) < n_items) asm volatile("bar.arrive 2, 256;\n" ::: "memory");
        const float m1 = has1 ? x1.x : -INFINITY, l1 = has1 ? x1.y : 0.f;
        const float mm = fmaxf(m, m1);
        const float a0 = (m == -INFINITY) ? 0.f : fast_exp2(m - mm);
        const float a1 = (m1 == -INFINITY) ? 0.f : fast_exp2(m1 - mm);
        const float Lsum = l * a0 + l1 * a1;
        const float inv = Lsum > 0.f ? 1.f / Lsum : 0.f;
        const float w0 = a0 * inv, w1 = a1 * inv;
        __nv_bfloat16* orow = p.out + ((int64_t)it.hq * p.n + row) * D;
#pragma unroll
        for (int c0 = 0; c0 < D; c0 += 32) {
          float o[32], o1[32];
          pf_ld32(tmem + lane_off + L::O_COL + c0, o);  // warp-collective: every row loads
          pf_ld32(tmem + lane_off + L::O_COL + D + c0, o1);
          pf_wait_ld();
          if (row < p.n) {
#pragma unroll
            for (int c = 0; c < 32; c += 8) {
              uint4 wv;
              wv.x = pack_bf16(o[c] * w0 + (has1 ? o1[c] * w1 : 0.f), o[c + 1] * w0 + (has1 ? o1[c + 1] * w1 : 0.f));
              wv.y = pack_bf16(o[c + 2] * w0 + (has1 ? o1[c + 2] * w1 : 0.f),
                               o[c + 3] * w0 + (has1 ? o1[c + 3] * w1 : 0.f));
              wv.z = pack_bf16(o[c + 4] * w0 + (has1 ? o1[c + 4] * w1 : 0.f),
                               o[c + 5] * w0 + (has1 ? o1[c + 5] * w1 : 0.f));
              wv.w = pack_bf16(o[c + 6] * w0 + (has1 ? o1[c + 6] * w1 : 0.f),
                               o[c + 7] * w0 + (has1 ? o1[c + 7] * w1 : 0.f));
              *reinterpret_cast<uint4*>(orow + c0 + c) = wv;
            }
          }
        }
        if (row < p.n && !(Lsum > 0.f)) set_status(p.status, STS_DEV_EMPTY_ROW);
        pf_fence_before();
        pf_arrive(oempty);  // the next item's first PVs may overwrite O_0 / O_1
      }
    }
  }
  pf_fence_before();
  __syncthreads();
  if (warp == 1) {
    pf_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(L::TMEM_COLS));
  }
}

typedef CUresult (*PfEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int pf_map(CUtensorMap* map, const void* base, int64_t heads, int64_t rows, int d, int64_t head_stride,
           int64_t row_stride, int box_rows) {
  static PfEncodeFn fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PfEncodeFn>(f);
  }
  STS_REQUIRE(fn, STS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)rows, (cuuint64_t)heads};
  const cuuint64_t strides[2] = {(cuuint64_t)row_stride * 2, (cuuint64_t)head_stride * 2};
  const cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  STS_REQUIRE(r == CUDA_SUCCESS, STS_ERR_CONTRACT, "tensor map encode failed (%d)", (int)r);
  return STS_OK;
}

}  // namespace
}  // namespace sts

using namespace sts;

extern "C" int sts_prefill_blocksparse(const void* q_dev, const void* k_dev, const void* v_dev, int32_t heads_q,
                                       int32_t heads_kv, int32_t n, int32_t d, int64_t q_head_stride,
                                       int64_t kv_head_stride, int64_t row_stride, float scale,
                                       const int32_t* idx_dev, int64_t idx_ld, const int32_t* cnt_dev, void* out_dev,
                                       int32_t* status_dev, void* stream) {
  STS_REQUIRE(d == 128 || d == 64, STS_ERR_CONTRACT, "block-sparse prefill supports head_dim 64 or 128");
  STS_REQUIRE(heads_q >= 1 && heads_kv >= 1 && heads_q % heads_kv == 0 && n >= 0, STS_ERR_CONTRACT,
              "bad prefill shape");
  if (n == 0) return STS_OK;
  STS_REQUIRE(q_dev && k_dev && v_dev && out_dev, STS_ERR_CONTRACT, "null buffer");
  STS_REQUIRE(!idx_dev || cnt_dev, STS_ERR_CONTRACT, "block lists need counts");
  STS_REQUIRE(row_stride % 8 == 0 && q_head_stride % 8 == 0 && kv_head_stride % 8 == 0, STS_ERR_CONTRACT,
              "strides must be multiples of 8 elements");
  PfParams p;
  memset(&p, 0, sizeof(p));
  p.n = n;
  p.heads_q = heads_q;
  p.group = heads_q / heads_kv;
  p.tiles = (n + PF_ROWS - 1) / PF_ROWS;
  p.scale = scale;
  p.idx = idx_dev;
  p.idx_ld = idx_ld;
  p.cnt = cnt_dev;
  p.out = static_cast<__nv_bfloat16*>(out_dev);
  p.status = status_dev;
  CUtensorMap qm, km, vm;
  int rc = pf_map(&qm, q_dev, heads_q, n, d, q_head_stride, row_stride, PF_ROWS);
  if (rc == STS_OK) rc = pf_map(&km, k_dev, heads_kv, n, d, kv_head_stride, row_stride, PF_BLK);
  if (rc == STS_OK) rc = pf_map(&vm, v_dev, heads_kv, n, d, kv_head_stride, row_stride, PF_BLK);
  if (rc != STS_OK) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t items = (int64_t)p.tiles * heads_q;
  STS_REQUIRE(items <= 0x7fffffffLL, STS_ERR_CONTRACT, "too many prefill tiles");
  const unsigned grid = (unsigned)(items < num_sms() ? items : num_sms());  // persistent: one CTA per SM
  if (d == 128) {
    STS_CUDA_CHECK(cudaFuncSetAttribute(prefill_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        PfLayout<128>::SMEM));
    prefill_tc_kernel<128><<<grid, PF_THREADS, PfLayout<128>::SMEM, st>>>(qm, km, vm, p);
  } else {
    STS_CUDA_CHECK(cudaFuncSetAttribute(prefill_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        PfLayout<64>::SMEM));
    prefill_tc_kernel<64><<<grid, PF_THREADS, PfLayout<64>::SMEM, st>>>(qm, km, vm, p);
  }
  STS_LAUNCH_CHECK();
  return STS_OK;
}
