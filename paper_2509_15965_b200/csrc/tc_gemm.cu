// Tensor-core path of the head (bf16 in, fp32 accumulate) for sm_100a:
// one persistent, warp-specialised tcgen05 GEMM with four fused epilogues.
//
//   warp 0  : TMA producer (one elected lane): A/B k-blocks -> smem ring
//             (128-B swizzle), mbarrier complete_tx.
//   warp 1  : TMEM allocator + MMA issuer (one lane): tcgen05.mma kind::f16,
//             N = 256, K = 16; fp32 accumulators in TMEM, two 256-column
//             accumulators (double buffered) so the epilogue of tile i
//             overlaps the MMAs of tile i+1; tcgen05.commit frees smem stages
//             and signals the epilogue.
//   warps 4-7: epilogue (thread = accumulator row = TMEM lane):
//     EPI_LSE (H3+H4, N3): online log-sum-exp of the 256 logits of the tile
//             -> per-row split-V partial (m, sum e^{z-m}, sum e^{z-m}(z-m)),
//             target logit captured in the tile that holds it. The logits
//             never leave TMEM/registers (BASELINE.json north_star).
//     EPI_DZ  (H6, N5): recompute the same logits (same tile/K order),
//             dZ = tau^-1 g (onehot(y) - exp(z - lse)) -> bf16 dZ chunk.
//     EPI_ROWS(H7, N6): dH = dZ W, rows scattered back to the packed layout.
//     EPI_ACC (H8, N7): dW += dZ^T H (fp32; TMA reduce-add of smem boxes).
//
// Tiles are claimed in order from a per-launch global counter (dynamic
// scheduler, one tile ahead), so the tiles that share A/B panels run together.
//
// CG = 1: one CTA per 128 x 256 tile (tcgen05 cta_group::1, M = 128).
// CG = 2: a cluster of two CTAs (a TPC pair) per 256 x 256 tile
//   (cta_group::2, M = 256): each CTA loads its 128 rows of A and its 128
//   columns of B with 2-SM TMA (complete_tx on the leader's barrier), the
//   leader issues the pair MMA, commits are multicast to both CTAs, each CTA
//   drains its own TMEM half. Per-SM operand traffic per MMA drops from
//   12 KB to 8 KB, so smem stages shrink to 32 KB and the ring deepens to 6.
//
// Operand majors: fwd/dZ  A = Hc [T,h] K-major,  B = W [V,h] K-major;
//                 dH      A = dZ [T,V] K-major,  B = W [V,h] MN-major;
//                 dW      A = dZ [T,V] MN-major, B = Hc [T,h] MN-major.
// Tiles are rasterised in groups of GROUP_M row-tiles so the CTAs resident
// at any time share A and B panels in L2.
#include "kernels.h"
#include "ptx.cuh"

#include <cstdlib>
#include <mutex>

namespace rlh {

constexpr int TC_THREADS = 256;
constexpr int TC_TMEM_COLS = 512;  // 2 x 256 fp32 accumulators
constexpr float LOG2E = 1.4426950408889634f;

// CG: CTAs per tile (cta_group). NB: 256-column accumulators per tile (1 =
// 256-wide tile, TMEM double buffered; 2 = 512-wide tile filling all 512
// TMEM columns, single buffered -- for the long-K dH/dW GEMMs whose
// epilogue is rare, it halves the A re-reads).
template <int CG, int NB>
struct TcCfg {
  static constexpr int A_BYTES = TC_BM * TC_BK * 2;            // 16 KB: this CTA's 128 rows
  static constexpr int PART_ROWS = TC_BN / CG;                 // B rows per CTA per 256-col part
  static constexpr int PART_BYTES = PART_ROWS * TC_BK * 2;     // 32 KB | 16 KB
  static constexpr int B_BYTES = NB * PART_BYTES;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;        // 48 KB | 32 KB | 48 KB
  static constexpr int STAGES = (200 * 1024) / STAGE_BYTES;    // 4 | 6 | 4
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
  static constexpr int TILE_M = TC_BM * CG;
  static constexpr int TILE_N = TC_BN * NB;
  static constexpr int ACC_STAGES = NB == 1 ? 2 : 1;
  // dW epilogue staging for the TMA reduce-add (acc_red == 2): 4 warps x 2 x
  // [32 rows][32 fp32], 128-B swizzled; placed after the barrier block.
  static constexpr int STG_OFF = STAGES * STAGE_BYTES + 1024;
  static constexpr int STG_BYTES = 4 * 2 * 4096;
};
// extra dynamic smem of an epilogue's TMA staging buffers (after the barriers)
template <int CG, int NB, int EPI>
constexpr int tc_smem_bytes() {
  return TcCfg<CG, NB>::SMEM_BYTES +
         ((EPI == 3 /*EPI_ACC*/ || EPI == 4 /*EPI_BWD*/) && NB == 2
              ? 1024 + TcCfg<CG, NB>::STG_BYTES
          : (EPI == 1 /*EPI_DZ*/ || EPI == 0 /*EPI_LSE: q stores*/) ? 1024 + 4 * 2 * 2048
                                          : 0);
}

// EPI_BWD: problem 0 = dH (A K-major, EPI_ROWS), problem 1 = dW (A MN-major,
// EPI_ACC), both with MN-major B, in one persistent launch.
enum { EPI_LSE = 0, EPI_DZ = 1, EPI_ROWS = 2, EPI_ACC = 3, EPI_BWD = 4 };

struct TcArgs {
  int64_t M, K;        // host values (used unless m_dyn / k_dyn)
  int32_t N;           // output columns (V or h)
  int32_t n_tiles;
  int32_t m_dyn, k_dyn;
  int32_t group_m;
  // second problem of EPI_BWD (the dW GEMM)
  int64_t M2, K2;
  int32_t n_tiles2, m_dyn2, k_dyn2, group_m2;
  int32_t l2_pol_a;    // TMA L2 hint of the A operand: 0 normal, 1 evict_last, 2 evict_first
  int32_t l2_pol_b;    // same for B (A/B can differ: a streamed panel vs a reused one)
  const WsHeader* hdr;
  uint32_t* sched;     // dynamic tile scheduler {claimed, retired} (NULL = static schedule)
  float inv_temp;
  int32_t vocab;       // columns of this (shard of the) head
  int64_t y_off;       // global id of column 0 (vocab-parallel shard offset)
  // EPI_LSE
  float *pm, *ps, *pu, *zy;
  const int32_t* tgt_c;
  int64_t ldp;         // (unused by the row-blocked partial layout)
  // EPI_DZ
  const float *lse_c, *g_c;
  const float *ge_c, *ez_c;  // entropy bonus (NULL = off): w c_ent and E_p[z]
  __nv_bfloat16* dz;
  int64_t ld_dz;
  // EPI_ROWS
  __nv_bfloat16* out;
  int64_t ld_out;
  const int32_t* row_idx;
  float* out_f32;      // non-NULL: fp32 rows [R, N] instead (vocab-parallel partial dL/dH
                       // written straight into a symmetric NVLink-mapped buffer)
  int32_t out_mc;      // out_f32 is an NVLS multicast address: multimem.red.add the tile
                       // into every rank's copy (the TP all-reduce inside the epilogue)
  // EPI_ACC
  float* acc;
  int64_t ld_acc;
  // EPI_ACC reduce-scatter (DP dW, last micro-batch): row j
  // belongs to rank o = min(j / rs_rows, rs_world - 1); the epilogue stores
  // (local partial + tile) into slot [rs_rank][j - o rs_rows] of the owner's
  // staging buffer over NVLink (plain stores; the owner sums the slots in
  // rank order afterwards, so the result is deterministic).
  int32_t dz_tma;      // EPI_DZ: stage bf16 32x32 boxes in smem, TMA-store them (tmA2 = dZ map)
  int32_t dyn_bwd;     // m_dyn / k_dyn read the backward-row count (hdr->n_bwd, skip mode)
  // q stores are skipped for a warp's 32 rows when every one has advantage 0
  // (no gradient, never read back in skip mode); NULL = store every box
  const float* q_adv;  // advantages, per sequence (seq_c) or per packed row (active_idx)
  const int32_t* q_row;  // seq_c or active_idx
  int32_t q_tma;       // EPI_LSE: also store q = e^{z - m_tile} (0 at the target) as bf16
                       // 32x32 boxes by TMA (tmA2 = map of the dZ buffer): the backward then
                       // needs no logits recompute (k_dz_from_q rescales q into dZ in place)
  int32_t k_serp2;     // k_serp of EPI_BWD's second problem (dW), waves counted from its start
  int32_t k_serp;      // tiles of odd waves (tile / clusters) walk K backwards: the next wave
                       // starts on the operand rows the previous one read last, still in L2
  int32_t acc_red;     // EPI_ACC: 0 load+add+store, 1 red.global.add (L2), 2 TMA reduce-add
                       // of 32x32 smem boxes (tmA2 = fp32 map of acc; 512-wide tiles only)
  int32_t rs_world;    // 0 = off
  int32_t rs_no_partial;  // acc holds no partial: send the tile alone, do not read acc
  int32_t rs_bulk;     // 512-wide tiles: each lane stages its 128-B row piece in smem and
                       // ships it with a 1-D bulk copy (whole NVLink lines, asynchronous)
                       // instead of 16-B stores from registers
  int32_t rs_rank;
  int64_t rs_rows;
  float* rs_peer[8];   // every rank's staging buffer [rs_world][rs_rows][ld_acc]
};

__device__ __forceinline__ void tile_coords(int64_t tile, int64_t m_tiles, int n_tiles,
                                            int group_m, int64_t& mb, int& nb) {
  const int64_t gsz = static_cast<int64_t>(group_m) * n_tiles;
  const int64_t g = tile / gsz;
  const int64_t first_m = g * group_m;
  const int64_t rem = m_tiles - first_m;
  const int64_t gm = rem < group_m ? rem : group_m;
  const int64_t local = tile - g * gsz;
  mb = first_m + local % gm;
  nb = static_cast<int>(local / gm);
}

// One GEMM problem of a launch: rows, K blocks and its share of the tile space.
struct Prob {
  int64_t M = 0, num_k = 0, m_tiles = 0, tiles = 0;
  int32_t n_tiles = 1, group_m = 1;
  // keep_empty: run the epilogue even when K == 0 (its accumulator reads as
  // 0) -- the dW reduce-scatter must still send this rank's partial.
  __device__ void init(int64_t M_, int64_t K_, int tile_m, int32_t n_tiles_, int32_t group_m_,
                       bool keep_empty = false) {
    M = M_;
    m_tiles = (M_ + tile_m - 1) / tile_m;
    num_k = (K_ + TC_BK - 1) / TC_BK;
    n_tiles = n_tiles_;
    group_m = group_m_;
    tiles = (num_k > 0 || keep_empty) ? m_tiles * n_tiles_ : 0;
  }
};

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

template <int CG, int NB, int AMN, int BMN, int EPI>
__global__ void __launch_bounds__(TC_THREADS, 1)
k_tc_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
          const __grid_constant__ CUtensorMap tmA2, const __grid_constant__ CUtensorMap tmB2,
          const __grid_constant__ CUtensorMap tmC, const TcArgs args) {
  using C = TcCfg<CG, NB>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;   // dynamic scheduler: tile id ring (2 slots)
  uint64_t* sempty = sfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sempty + 2);
  int32_t* ring = reinterpret_cast<int32_t*>(tmem_slot + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if constexpr (EPI == EPI_BWD) {
      tma_prefetch_desc(&tmA2);
      tma_prefetch_desc(&tmB2);
      if (args.acc_red == 2) tma_prefetch_desc(&tmC);
    }
    if constexpr (EPI == EPI_ACC) {
      if (args.acc_red == 2) tma_prefetch_desc(&tmA2);
    }
    if constexpr (EPI == EPI_DZ) {
      if (args.dz_tma) tma_prefetch_desc(&tmA2);
    }
    if constexpr (EPI == EPI_LSE) {
      if (args.q_tma) tma_prefetch_desc(&tmA2);
    }
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(full + i, CG);     // CG producers arrive (remote for the peer)
      mbar_init(empty + i, 1);     // one (multicast) commit per phase
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(tfull + i, 1);
      mbar_init(tempty + i, 128 * CG);  // all epilogue threads of the pair
      mbar_init(sfull + i, 1);          // the leader's scheduler thread
      // consumers of a tile id: producer + MMA + 4 epilogue warps (leader),
      // producer + 4 epilogue warps (peer)
      mbar_init(sempty + i, CG == 2 ? 11 : 6);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    if constexpr (CG == 2) tmem_alloc_2sm(tmem_slot, TC_TMEM_COLS);
    else tmem_alloc(tmem_slot, TC_TMEM_COLS);
  }
  tc_fence_before();
  __syncwarp();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // Tile space: problem 0, then (EPI_BWD only) problem 1 -- the dH and dW
  // GEMMs of one backward in a single persistent launch, so the short last
  // wave of one fills with tiles of the other.
  const int64_t T = args.dyn_bwd ? args.hdr->n_bwd : args.hdr->n_active;
  Prob P0, P1;
  P0.init(args.m_dyn ? T : args.M, args.k_dyn ? T : args.K, C::TILE_M, args.n_tiles, args.group_m,
          EPI == EPI_ACC && args.rs_world > 0);
  if constexpr (EPI == EPI_BWD)
    P1.init(args.m_dyn2 ? T : args.M2, args.k_dyn2 ? T : args.K2, C::TILE_M, args.n_tiles2,
            args.group_m2, args.rs_world > 0);
  const int64_t num_tiles = P0.tiles + P1.tiles;
  const int64_t cid = blockIdx.x / CG, ncl = gridDim.x / CG;
  // Tile schedule. Static: cluster c runs tiles c, c + ncl, ... Dynamic
  // (args.sched): the first tile is static, then the leader's scheduler thread
  // claims tiles from a global counter one tile ahead of use and hands the id
  // to both CTAs through a 2-slot ring, so tiles run in claim order and the
  // tiles that share A/B panels in L2 (consecutive ids) run at the same time
  // however far individual pairs drift apart over a long launch.
  const bool dyn = args.sched != nullptr;
  auto next_tile = [&](int64_t it, int64_t& tile) -> bool {
    if (!dyn) {
      tile = cid + it * ncl;
      return tile < num_tiles;
    }
    mbar_wait_acq_cluster(sfull + (it & 1), static_cast<uint32_t>((it >> 1) & 1));
    tile = ring[it & 1];
    return tile >= 0;
  };
  auto tile_read = [&](int64_t it) {  // one thread per consumer role, after next_tile
    if (!dyn) return;
    if (CG == 2 && !leader) mbar_arrive_cluster_release(sempty + (it & 1), 0);
    else mbar_arrive(sempty + (it & 1));
  };
  // per tile: which problem, its coordinates and K extent
  auto locate = [&](int64_t tile, bool& second, int64_t& mb, int& nb) -> const Prob& {
    second = tile >= P0.tiles;
    const Prob& P = second ? P1 : P0;
    tile_coords(second ? tile - P0.tiles : tile, P.m_tiles, P.n_tiles, P.group_m, mb, nb);
    return P;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------ TMA producer
      auto mkpol = [](int code) {
        return code == 1 ? l2_policy_evict_last()
               : code == 2 ? l2_policy_evict_first()
                           : l2_policy_evict_normal();
      };
      const uint64_t pol_a = mkpol(args.l2_pol_a), pol_b = mkpol(args.l2_pol_b);
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t it = 0;; ++it) {
        int64_t tile;
        if (!next_tile(it, tile)) break;
        tile_read(it);
        int64_t mb;
        int nb;
        bool second;
        const Prob& P = locate(tile, second, mb, nb);
        const bool amn = EPI == EPI_BWD ? second : (AMN != 0);
        const bool krev = second ? (args.k_serp2 && (((tile - P0.tiles) / ncl) & 1))
                                 : (args.k_serp && ((tile / ncl) & 1));
        const CUtensorMap* mA = second ? &tmA2 : &tmA;
        const CUtensorMap* mB = second ? &tmB2 : &tmB;
        const int32_t m0 = static_cast<int32_t>(mb * C::TILE_M + rank * TC_BM);
        // part p of this CTA's B: global rows n0 + p*256 + [0, PART_ROWS)
        const int32_t n0 = nb * C::TILE_N + static_cast<int32_t>(rank) * C::PART_ROWS;
        for (int64_t kb = 0; kb < P.num_k; ++kb) {
          mbar_wait(empty + stage, phase ^ 1);
          if (leader) mbar_arrive_expect_tx(full + stage, C::STAGE_BYTES * CG);
          else mbar_arrive_cluster(full + stage, 0);
          uint8_t* a_dst = sA + stage * C::A_BYTES;
          uint8_t* b_dst = sB + stage * C::B_BYTES;
          const int32_t k0 = static_cast<int32_t>((krev ? P.num_k - 1 - kb : kb) * TC_BK);
          auto load = [&](const CUtensorMap* m, void* dst, int32_t c0, int32_t c1) {
            const uint64_t pol = m == mA ? pol_a : pol_b;
            if constexpr (CG == 2) tma_load_2d_2sm(m, full + stage, dst, c0, c1, pol);
            else tma_load_2d(m, full + stage, dst, c0, c1, pol);
          };
          if (amn) {
            load(mA, a_dst, m0, k0);
            load(mA, a_dst + 8192, m0 + 64, k0);
          } else {
            load(mA, a_dst, k0, m0);
          }
#pragma unroll
          for (int p = 0; p < NB; ++p) {
            uint8_t* pd = b_dst + p * C::PART_BYTES;
            const int32_t np = n0 + p * TC_BN;
            if (BMN) {
#pragma unroll
              for (int i = 0; i < C::PART_ROWS / 64; ++i) load(mB, pd + i * 8192, np + 64 * i, k0);
            } else {
              load(mB, pd, k0, np);
            }
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ------------------------------------------------------- MMA issuer
      constexpr uint32_t IDESC_K = umma_idesc_bf16(TC_BM * CG, TC_BN, 0, BMN);
      constexpr uint32_t IDESC_MN = umma_idesc_bf16(TC_BM * CG, TC_BN, 1, BMN);
      const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int64_t it = 0;; ++it) {
        int64_t tile;
        if (!next_tile(it, tile)) break;
        tile_read(it);
        int64_t mb_unused;
        int nb_unused;
        bool second;
        const Prob& P = locate(tile, second, mb_unused, nb_unused);
        const bool amn = EPI == EPI_BWD ? second : (AMN != 0);
        const uint32_t IDESC = amn ? IDESC_MN : IDESC_K;
        mbar_wait(tempty + acc, acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * TC_BN);
        for (int64_t kb = 0; kb < P.num_k; ++kb) {
          mbar_wait(full + stage, phase);
          tc_fence_after();
          const uint32_t a_addr = a_base + stage * C::A_BYTES;
          const uint32_t b_addr = b_base + stage * C::B_BYTES;
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k) {
            const uint64_t ad = amn ? umma_desc_sw128(a_addr + k * 2048, 8192, 1024)
                                    : umma_desc_sw128(a_addr + k * 32, 0, 1024);
            const uint32_t accum = (kb > 0 || k > 0) ? 1u : 0u;
#pragma unroll
            for (int p = 0; p < NB; ++p) {
              const uint32_t bp = b_addr + p * C::PART_BYTES;
              const uint64_t bd = BMN ? umma_desc_sw128(bp + k * 2048, 8192, 1024)
                                      : umma_desc_sw128(bp + k * 32, 0, 1024);
              if constexpr (CG == 2) tc_mma_f16_2sm(d_tmem + p * TC_BN, ad, bd, IDESC, accum);
              else tc_mma_f16(d_tmem + p * TC_BN, ad, bd, IDESC, accum);
            }
          }
          if constexpr (CG == 2) tc_commit_2sm(empty + stage); else tc_commit(empty + stage);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if constexpr (CG == 2) tc_commit_2sm(tfull + acc); else tc_commit(tfull + acc);
        if (++acc == C::ACC_STAGES) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp == 2) {
    if (dyn && lane == 0 && leader) {
      // ------------------------------------------------- tile scheduler
      for (int64_t it = 0;; ++it) {
        mbar_wait(sempty + (it & 1), static_cast<uint32_t>(((it >> 1) & 1) ^ 1));
        int64_t t = it == 0 ? cid : ncl + static_cast<int64_t>(atomicAdd(args.sched, 1u));
        const int32_t v = t < num_tiles ? static_cast<int32_t>(t) : -1;
        ring[it & 1] = v;
        mbar_arrive(sfull + (it & 1));
        if constexpr (CG == 2) st_cluster_u32_arrive(ring + (it & 1), v, sfull + (it & 1), 1);
        if (v < 0) break;
      }
      // the last scheduler to retire resets the counters for the next launch
      __threadfence();
      if (atomicAdd(args.sched + 1, 1u) == static_cast<uint32_t>(ncl - 1)) {
        atomicExch(args.sched, 0u);
        atomicExch(args.sched + 1, 0u);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 4;
    const int rit = ew * 32 + lane;  // row in this CTA's half tile == TMEM lane
    int acc = 0;
    uint32_t acc_phase = 0;
    auto release = [&](int a) {
      tc_fence_before();
      if constexpr (CG == 2) {
        if (leader) mbar_arrive(tempty + a); else mbar_arrive_cluster(tempty + a, 0);
      } else {
        mbar_arrive(tempty + a);
      }
    };
    for (int64_t it = 0;; ++it) {
      int64_t tile;
      if (!next_tile(it, tile)) break;
      __syncwarp();
      if (lane == 0) tile_read(it);
      int64_t mb;
      int nb;
      bool second;
      const Prob& P = locate(tile, second, mb, nb);
      const int64_t row = mb * C::TILE_M + rank * TC_BM + rit;
      const int n0 = nb * C::TILE_N;
      const bool row_ok = row < P.M;
      static_assert(NB == 1 || EPI == EPI_ROWS || EPI == EPI_ACC || EPI == EPI_BWD,
                    "512-wide tiles: dH/dW only");
      mbar_wait(tfull + acc, acc_phase);
      tc_fence_after();
      const uint32_t taddr =
          tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + static_cast<uint32_t>(acc * TC_BN);

      if constexpr (EPI == EPI_LSE) {
        // target column in this shard (or none): local id = global - y_off
        const int64_t yl = row_ok ? static_cast<int64_t>(args.tgt_c[row]) - args.y_off : -1;
        const int yrel = (yl >= 0 && yl < args.vocab) ? static_cast<int>(yl) - n0 : -(1 << 30);
        const int valid = args.vocab - n0;  // columns < valid are real vocab ids
        float m = -INFINITY, s = 0.f, u = 0.f, zyv = 0.f;
        bool has_y = false;
        // Two passes over the TMEM tile. Pass 1: the tile maximum m (and the
        // target logit). Pass 2: e = e^{z - m} and the partial sums s, u;
        // with q_tma also q = e (0 at the target column) -> bf16 32x32 smem
        // boxes (64-B swizzle) -> TMA store into the dZ buffer (evict-
        // first). q is the softmax up to the per-(row, tile) factor
        // e^{m - lse}: k_dz_from_q turns it into dZ after the merge, instead
        // of a recompute GEMM.
        // Lean inner loops (these warps share issue slots with the MMA
        // issuer): the max over raw accumulators (tau^-1 > 0), masking only
        // in the tile that crosses V, the target column patched only in the
        // one chunk that holds it, u summed in log2 units.
        const bool full = valid >= TC_BN;  // warp-uniform: no column beyond V
        float mraw = -INFINITY;
#pragma unroll 1
        for (int c = 0; c < TC_BN / 32; ++c) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(taddr + c * 32, v);
          tmem_ld_wait();
          if (full) {
#pragma unroll
            for (int j = 0; j < 32; ++j) mraw = fmaxf(mraw, __uint_as_float(v[j]));
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (c * 32 + j < valid) mraw = fmaxf(mraw, __uint_as_float(v[j]));
          }
          const int yc = yrel - c * 32;
          if (yc >= 0 && yc < 32) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j == yc) zyv = __uint_as_float(v[j]) * args.inv_temp;
            has_y = true;
          }
        }
        m = mraw * args.inv_temp;
        const uint64_t st_pol = l2_policy_evict_first();
        const float m2 = m * LOG2E, sc2 = args.inv_temp * LOG2E;
        float u2 = 0.f;                  // sum e (z - m) log2 e
        bool skip_q = false;             // warp-uniform
        if (args.q_tma && args.q_adv)
          skip_q = __all_sync(0xffffffffu, !row_ok || args.q_adv[args.q_row[row]] == 0.f);
#pragma unroll 1
        for (int c = 0; c < TC_BN / 32; ++c) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(taddr + c * 32, v);
          tmem_ld_wait();
          if (c == TC_BN / 32 - 1) release(acc);
          float e[32];
          if (full) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float d2 = fmaf(__uint_as_float(v[j]), sc2, -m2);  // <= 0
              e[j] = ex2_approx(d2);
              s += e[j];
              u2 = fmaf(e[j], d2, u2);
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const bool ok = c * 32 + j < valid;
              const float d2 = ok ? fmaf(__uint_as_float(v[j]), sc2, -m2) : 0.f;
              e[j] = ok ? ex2_approx(d2) : 0.f;
              s += e[j];
              u2 = fmaf(e[j], d2, u2);
            }
          }
          if (!args.q_tma || skip_q) continue;  // forward only / all-A = 0 rows: no q
          const int yc = yrel - c * 32;
          if (yc >= 0 && yc < 32) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j == yc) e[j] = 0.f;   // q = 0 at the target: dZ_y comes from z_y
          }
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 32; j += 2) pk[j / 2] = pack_bf16x2(e[j], e[j + 1]);
          uint8_t* buf = smem + C::STG_OFF + ew * 4096 + (c & 1) * 2048;
          if (lane == 0) bulk_wait_group_read<1>();
          __syncwarp();
#pragma unroll
          for (int q = 0; q < 4; ++q)
            *reinterpret_cast<uint4*>(buf + lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4)) =
                make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmA2, buf, n0 + c * 32,
                         static_cast<int32_t>(mb * C::TILE_M + rank * TC_BM + ew * 32), st_pol);
            bulk_commit_group();
          }
        }
        u = u2 * (1.f / LOG2E);
        if (row_ok) {
          // row-blocked partials [Rp/32][n_vt][32]: a warp's 32 rows are 128 B
          // per vocab tile here, and k_merge streams one row block's n_vt
          // tiles contiguously
          const int64_t o = ((row >> 5) * args.n_tiles + nb) * 32 + (row & 31);
          args.pm[o] = m;
          args.ps[o] = s;
          args.pu[o] = u;
          if (has_y) args.zy[row] = zyv;
        }
      } else if constexpr (EPI == EPI_DZ) {
        const float lse = row_ok ? args.lse_c[row] : 0.f;
        const float coef = row_ok ? args.g_c[row] * args.inv_temp : 0.f;
        const int64_t yl = row_ok ? static_cast<int64_t>(args.tgt_c[row]) - args.y_off : -1;
        const int yrel = (yl >= 0 && yl < args.vocab) ? static_cast<int>(yl) - n0 : -(1 << 30);
        const float lse2 = lse * LOG2E, sc2 = args.inv_temp * LOG2E;
        uint4* dst = reinterpret_cast<uint4*>(args.dz + row * args.ld_dz + n0);
        const uint64_t st_pol = l2_policy_evict_first();  // 17 GB stream: keep W/Hc in L2
        // entropy bonus: + tau^-1 w c_ent p (z - E_p z); off -> cent = 0 (warp-uniform)
        const bool ent_on = args.ge_c != nullptr;
        const float cent = (ent_on && row_ok) ? args.ge_c[row] * args.inv_temp : 0.f;
        const float ez = (ent_on && row_ok) ? args.ez_c[row] : 0.f;
#pragma unroll 1
        for (int c = 0; c < TC_BN / 32; ++c) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(taddr + c * 32, v);
          tmem_ld_wait();
          if (c == TC_BN / 32 - 1) release(acc);
          uint32_t pk[16];
          if (!ent_on) {
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              const float p0 = ex2_approx(fmaf(__uint_as_float(v[j]), sc2, -lse2));
              const float p1 = ex2_approx(fmaf(__uint_as_float(v[j + 1]), sc2, -lse2));
              const float d0 = coef * ((c * 32 + j == yrel ? 1.f : 0.f) - p0);
              const float d1 = coef * ((c * 32 + j + 1 == yrel ? 1.f : 0.f) - p1);
              pk[j / 2] = pack_bf16x2(d0, d1);
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              const float z0 = __uint_as_float(v[j]) * args.inv_temp;
              const float z1 = __uint_as_float(v[j + 1]) * args.inv_temp;
              const float p0 = ex2_approx(fmaf(__uint_as_float(v[j]), sc2, -lse2));
              const float p1 = ex2_approx(fmaf(__uint_as_float(v[j + 1]), sc2, -lse2));
              const float d0 = coef * ((c * 32 + j == yrel ? 1.f : 0.f) - p0) + cent * p0 * (z0 - ez);
              const float d1 =
                  coef * ((c * 32 + j + 1 == yrel ? 1.f : 0.f) - p1) + cent * p1 * (z1 - ez);
              pk[j / 2] = pack_bf16x2(d0, d1);
            }
          }
          if (args.dz_tma) {
            // 32 rows x 32 bf16 (64 B) per warp -> smem box, 64-B swizzle
            // (16-B chunk q of row r at q ^ ((r >> 1) & 3): conflict-free),
            // one TMA store of whole lines; two buffers per warp.
            uint8_t* buf = smem + C::STG_OFF + ew * 4096 + (c & 1) * 2048;
            if (lane == 0) bulk_wait_group_read<1>();
            __syncwarp();
#pragma unroll
            for (int q = 0; q < 4; ++q)
              *reinterpret_cast<uint4*>(buf + lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4)) =
                  make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&tmA2, buf, n0 + c * 32,
                           static_cast<int32_t>(mb * C::TILE_M + rank * TC_BM + ew * 32), st_pol);
              bulk_commit_group();
            }
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              st_global_v4_hint(dst + c * 4 + q,
                                make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]),
                                st_pol);
          }
        }
      } else if (EPI == EPI_ROWS || (EPI == EPI_BWD && !second)) {
        const int64_t orow = row_ok ? static_cast<int64_t>(args.row_idx[row]) : 0;
        uint4* dst = reinterpret_cast<uint4*>(args.out + orow * args.ld_out + n0);
#pragma unroll 1
        for (int c = 0; c < C::TILE_N / 32; ++c) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(taddr + c * 32, v);
          tmem_ld_wait();
          if (c == C::TILE_N / 32 - 1) release(acc);
          if (args.out_f32) {
            if (row_ok && n0 + c * 32 < args.N) {
              float4* df = reinterpret_cast<float4*>(args.out_f32 + orow * args.N + n0 + c * 32);
              if (args.out_mc) {
#pragma unroll
                for (int q = 0; q < 8; ++q)
                  multimem_red_add_v4_f32(df + q, v[4 * q], v[4 * q + 1], v[4 * q + 2],
                                          v[4 * q + 3]);
              } else {
#pragma unroll
                for (int q = 0; q < 8; ++q)
                  df[q] = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                      __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]));
              }
            }
          } else if (row_ok && n0 + c * 32 < args.N) {
            uint32_t pk[16];
#pragma unroll
            for (int j = 0; j < 32; j += 2)
              pk[j / 2] = pack_bf16x2(__uint_as_float(v[j]), __uint_as_float(v[j + 1]));
#pragma unroll
            for (int q = 0; q < 4; ++q)
              dst[c * 4 + q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
          }
        }
      } else {  // EPI_ACC (or the dW half of EPI_BWD)
        float4* dst = reinterpret_cast<float4*>(args.acc + row * args.ld_acc + n0);
        const bool empty_k = P.num_k == 0;  // keep_empty tile: no MMA ran
        const bool tma_red =
            (EPI == EPI_ACC || EPI == EPI_BWD) && NB == 2 && args.acc_red == 2 && args.rs_world == 0;
#pragma unroll 1
        for (int c = 0; c < C::TILE_N / 32; ++c) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(taddr + c * 32, v);
          tmem_ld_wait();
          if (c == C::TILE_N / 32 - 1) release(acc);
          if (empty_k) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = 0u;
          }
          if constexpr ((EPI == EPI_ACC || EPI == EPI_BWD) && NB == 2) {
            if (args.rs_world > 0 && args.rs_bulk) {
              // (local partial + tile) row piece -> this lane's 128-B line of the
              // warp's staging buffer (written in rotated chunk order: the 8
              // lanes of a quarter-warp hit 8 different bank groups), then one
              // bulk copy per lane into the owner's staging slot over NVLink.
              // Two buffers per warp: chunk c reuses the one of chunk c - 2.
              uint8_t* line = smem + C::STG_OFF + ew * 8192 + (c & 1) * 4096 + lane * 128;
              bulk_wait_group_read<1>();
              if (row_ok && n0 + c * 32 < args.N) {
                int64_t own = row / args.rs_rows;
                own = own < args.rs_world - 1 ? own : args.rs_world - 1;
                float* slot = args.rs_peer[own] +
                              (args.rs_rank * args.rs_rows + (row - own * args.rs_rows)) *
                                  args.ld_acc +
                              n0 + c * 32;
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {
                  const int q = (jj + lane) & 7;
                  float4 o = args.rs_no_partial ? make_float4(0.f, 0.f, 0.f, 0.f) : dst[c * 8 + q];
                  o.x += __uint_as_float(v[4 * q]);
                  o.y += __uint_as_float(v[4 * q + 1]);
                  o.z += __uint_as_float(v[4 * q + 2]);
                  o.w += __uint_as_float(v[4 * q + 3]);
                  *reinterpret_cast<float4*>(line + (q << 4)) = o;
                }
                fence_proxy_async_smem();
                bulk_copy_s2g(slot, line, 128);
                bulk_commit_group();
              }
              continue;
            }
            if (tma_red) {
              // this warp's 32 rows x 32 columns -> a 128-B-swizzled smem box
              // (16-B chunk j of row r at chunk j ^ (r & 7): conflict-free),
              // then one lane adds the box into acc with a TMA reduce (whole
              // L2 lines; out-of-range rows/columns are clipped by the map).
              // Two buffers per warp: chunk c reuses the one of chunk c - 2.
              uint8_t* buf = smem + C::STG_OFF + ew * 8192 + (c & 1) * 4096;
              if (lane == 0) bulk_wait_group_read<1>();
              __syncwarp();
#pragma unroll
              for (int j = 0; j < 8; ++j)
                *reinterpret_cast<uint4*>(buf + lane * 128 + ((j ^ (lane & 7)) << 4)) =
                    make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
              fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_reduce_add_2d(EPI == EPI_BWD ? &tmC : &tmA2, buf, n0 + c * 32,
                                  static_cast<int32_t>(mb * C::TILE_M + rank * TC_BM + ew * 32));
                bulk_commit_group();
              }
              continue;
            }
          }
          if (row_ok && n0 + c * 32 < args.N) {
            if (args.rs_world > 0) {  // local partial + tile -> the owner's slot
              int64_t own = row / args.rs_rows;
              own = own < args.rs_world - 1 ? own : args.rs_world - 1;
              float4* slot = reinterpret_cast<float4*>(
                  args.rs_peer[own] +
                  (args.rs_rank * args.rs_rows + (row - own * args.rs_rows)) * args.ld_acc + n0 +
                  c * 32);
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                float4 o = args.rs_no_partial ? make_float4(0.f, 0.f, 0.f, 0.f) : dst[c * 8 + q];
                o.x += __uint_as_float(v[4 * q]);
                o.y += __uint_as_float(v[4 * q + 1]);
                o.z += __uint_as_float(v[4 * q + 2]);
                o.w += __uint_as_float(v[4 * q + 3]);
                slot[q] = o;
              }
            } else if (args.acc_red) {
              // the add happens in L2: no read on the epilogue's critical path.
              // One add per element per launch, launches stream-ordered: the
              // accumulation order is still fixed (deterministic).
#pragma unroll
              for (int q = 0; q < 8; ++q)
                red_add_v4_f32(dst + c * 8 + q, __uint_as_float(v[4 * q]),
                               __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                               __uint_as_float(v[4 * q + 3]));
            } else {
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                float4 o = dst[c * 8 + q];
                o.x += __uint_as_float(v[4 * q]);
                o.y += __uint_as_float(v[4 * q + 1]);
                o.z += __uint_as_float(v[4 * q + 2]);
                o.w += __uint_as_float(v[4 * q + 3]);
                dst[c * 8 + q] = o;
              }
            }
          }
        }
      }
      if (++acc == C::ACC_STAGES) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  if constexpr ((EPI == EPI_ACC || EPI == EPI_BWD) && NB == 2) {
    if (warp >= 4 && lane == 0 && args.acc_red == 2) bulk_wait_group_all();
    // every lane's bulk copies complete (written at the owner) before exit
    if (warp >= 4 && args.rs_world > 0 && args.rs_bulk) bulk_wait_group_all();
  }
  if constexpr (EPI == EPI_DZ) {
    if (warp >= 4 && lane == 0 && args.dz_tma) bulk_wait_group_all();
  }
  if constexpr (EPI == EPI_LSE) {
    if (warp >= 4 && lane == 0 && args.q_tma) bulk_wait_group_all();
  }
  tc_fence_before();
  __syncwarp();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    if constexpr (CG == 2) tmem_dealloc_2sm(tmem_base, TC_TMEM_COLS);
    else tmem_dealloc(tmem_base, TC_TMEM_COLS);
  }
}

// ------------------------------------------------------------------ host ----
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                      const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                      const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion,
                                      CUtensorMapFloatOOBfill);

static PFN_encodeTiled_t get_encode() {
  static PFN_encodeTiled_t fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(p);
  });
  return fn;
}

// 2-D bf16 tensor map: dims {inner, outer}, row stride in bytes, box
// {64, box_outer}, 128-B swizzle, OOB elements read as zero.
static bool make_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                     uint64_t stride_bytes, uint32_t box_outer) {
  PFN_encodeTiled_t enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {stride_bytes};
  cuuint32_t box[2] = {64, box_outer};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

// 2-D bf16 tensor map with a 32 x 32 box and 64-B swizzle: the dZ chunk as a
// TMA store destination (one epilogue warp's 32 rows x 32 columns).
static bool make_map_bf16_32(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                             uint64_t stride_bytes) {
  PFN_encodeTiled_t enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {stride_bytes};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 2-D fp32 tensor map (dims {inner, outer}, box {box_inner, box_outer},
// 128-B swizzle): the dW accumulator as a TMA reduce-add destination.
static bool make_map_f32(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                         uint64_t stride_bytes, uint32_t box_inner, uint32_t box_outer) {
  PFN_encodeTiled_t enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int num_sms() {
  static int n = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  });
  return n;
}

// Tuning knobs read once from the environment (benchmarks / A-B tests).
static int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return (e && *e) ? std::atoi(e) : dflt;
}

// CTA group of the tensor-core GEMMs: 2 (default) or 1 (RLHEAD_CTA_GROUP=1).
int tc_cta_group() {
  static int cg = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* e = std::getenv("RLHEAD_CTA_GROUP");
    cg = (e && e[0] == '1') ? 1 : 2;
  });
  return cg;
}

template <int CG, int NB, int AMN, int BMN, int EPI>
static rl_status run_gemm(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& a2,
                          const CUtensorMap& b2, const TcArgs& args, int64_t tiles_bound,
                          int kind, cudaStream_t s, bool persistent = true,
                          const CUtensorMap* c = nullptr) {
  using C = TcCfg<CG, NB>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(k_tc_gemm<CG, NB, AMN, BMN, EPI>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    tc_smem_bytes<CG, NB, EPI>());
  });
  if (attr_err != cudaSuccess) return RL_ERR_CUDA;
  if (tiles_bound <= 0) return RL_OK;
  const int64_t clusters_max = num_sms() / CG;
  // persistent: one cluster per TPC pair walks the tile space; otherwise one
  // cluster per tile and the block scheduler hands tiles out in order as
  // clusters retire, so tiles that share operand panels (consecutive ids)
  // start together however far the pairs have drifted apart.
  const int64_t clusters =
      (!persistent || tiles_bound < clusters_max) ? tiles_bound : clusters_max;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(clusters * CG));
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = tc_smem_bytes<CG, NB, EPI>();
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TraceScope ts(kind, s);
  if (cudaLaunchKernelEx(&cfg, k_tc_gemm<CG, NB, AMN, BMN, EPI>, a, b, a2, b2, c ? *c : a,
                         args) != cudaSuccess)
    return RL_ERR_CUDA;
  RLH_CHECK_LAUNCH();
  return RL_OK;
}

// 256-wide tiles (double-buffered TMEM) for the short-K forward/dZ GEMMs.
template <int AMN, int BMN, int EPI>
static rl_status run_narrow(const CUtensorMap& a, const CUtensorMap& b, TcArgs t,
                            int64_t m_extent, int kind, cudaStream_t s,
                            const CUtensorMap* a2 = nullptr) {
  t.n_tiles = static_cast<int32_t>(ceil_div(t.N, TC_BN));
  t.group_m = env_int("RLHEAD_GROUP_M", 32) / tc_cta_group();
  if (t.group_m < 1) t.group_m = 1;
  const int cg = tc_cta_group();
  const int64_t tiles = ceil_div(m_extent, TC_BM * cg) * t.n_tiles;
  const CUtensorMap& x2 = a2 ? *a2 : a;
  if (cg == 2) return run_gemm<2, 1, AMN, BMN, EPI>(a, b, x2, b, t, tiles, kind, s);
  return run_gemm<1, 1, AMN, BMN, EPI>(a, b, x2, b, t, tiles, kind, s);
}

// Long-K dH/dW GEMMs: 256 x 512 pair tiles (all 512 TMEM columns), rastered
// N-fastest so the CTA pairs sharing an A panel run together.
static bool wide_bwd() { return tc_cta_group() == 2 && env_int("RLHEAD_WIDE", 1) != 0; }
// Off by default: in same-box A/B runs of bench.py the fused launch drew more
// power (dH and dW tiles compete for L2 at the transition), lowering clocks
// for the whole step (-2.3% tokens/s, profiles/r1/SUMMARY.md).
static bool fused_bwd() { return wide_bwd() && env_int("RLHEAD_FUSED_BWD", 0) != 0; }
template <int AMN, int BMN, int EPI>
static rl_status run_wide(const CUtensorMap& a, const CUtensorMap& b, TcArgs t, int64_t m_extent,
                          int kind, cudaStream_t s, const CUtensorMap* a2 = nullptr) {
  t.group_m = env_int("RLHEAD_GROUP_M_BWD", 1);
  if (t.group_m < 1) t.group_m = 1;
  // per-GEMM override (A/B of the tile-count quantisation): RLHEAD_WIDE_DH /
  // RLHEAD_WIDE_DW = 0 runs that GEMM on 256-wide tiles
  const bool wide =
      wide_bwd() && env_int(EPI == EPI_ACC ? "RLHEAD_WIDE_DW" : "RLHEAD_WIDE_DH", 1) != 0;
  if (wide) {
    t.n_tiles = static_cast<int32_t>(ceil_div(t.N, 2 * TC_BN));
    const bool persistent =
        env_int(EPI == EPI_ACC ? "RLHEAD_NONPERSIST_DW" : "RLHEAD_NONPERSIST_DH", 0) == 0;
    return run_gemm<2, 2, AMN, BMN, EPI>(a, b, a2 ? *a2 : a, b, t,
                                         ceil_div(m_extent, 2 * TC_BM) * t.n_tiles, kind, s,
                                         persistent);
  }
  if (t.acc_red == 2) t.acc_red = 1;  // TMA reduce: 512-wide tiles only
  t.n_tiles = static_cast<int32_t>(ceil_div(t.N, TC_BN));
  const int cg = tc_cta_group();
  const int64_t tiles = ceil_div(m_extent, TC_BM * cg) * t.n_tiles;
  if (cg == 2) return run_gemm<2, 1, AMN, BMN, EPI>(a, b, a, b, t, tiles, kind, s);
  return run_gemm<1, 1, AMN, BMN, EPI>(a, b, a, b, t, tiles, kind, s);
}

// Per-GEMM-kind L2 hints for (A, B): env RLHEAD_L2_<KIND> = two digits "ab"
// (0 normal, 1 evict_last, 2 evict_first); unset keeps RLHEAD_L2_POLICY for both.
static void kind_policy(TcArgs& t, const char* env, int dflt_ab) {
  const int ab = env_int(env, dflt_ab);
  if (ab < 0) return;
  t.l2_pol_a = (ab / 10) % 10;
  t.l2_pol_b = ab % 10;
}

// Dynamic tile scheduler (default; RLHEAD_DYN_SCHED=0 restores the static
// schedule): one counter slot per GEMM kind. Same-box A/B, Qwen-7B, 1 GPU:
// +3.8% tokens/s; forward/dZ DRAM reads per micro-batch 7.8/9.2 -> 4.5/4.5 GB
// (profiles/r1/SUMMARY.md).
static void use_sched(TcArgs& t, char* ws, const WsLayout& L, int slot) {
  if (env_int("RLHEAD_DYN_SCHED", 1) == 0) return;
  t.sched = reinterpret_cast<WsHeader*>(ws + L.off_hdr)->sched[slot];
}

static TcArgs base_args(const rl_head* hd, const WsLayout& L, char* ws) {
  TcArgs t{};
  t.hdr = reinterpret_cast<const WsHeader*>(ws + L.off_hdr);
  t.inv_temp = hd->inv_temperature;
  t.vocab = hd->vocab;
  t.y_off = hd->vocab_total > 0 ? hd->vocab_offset : 0;
  const int pol = env_int("RLHEAD_L2_POLICY", 1);
  t.l2_pol_a = pol;
  t.l2_pol_b = pol;
  t.tgt_c = reinterpret_cast<const int32_t*>(ws + L.off_tgt);
  t.ldp = L.Rp;
  return t;
}

rl_status launch_tc_fwd(const rl_head* hd, const void* weight, const WsLayout& L, char* ws,
                        cudaStream_t s, bool q_out, const float* q_adv, bool q_adv_per_row) {
  const int h = hd->hidden, V = hd->vocab;
  const int cg = tc_cta_group();
  CUtensorMap ma, mb;
  if (!make_map(&ma, ws + L.off_hc, h, L.Rp, static_cast<uint64_t>(h) * 2, TC_BM) ||
      !make_map(&mb, weight, h, V, static_cast<uint64_t>(h) * 2, TC_BN / cg))
    return RL_ERR_CUDA;
  TcArgs t = base_args(hd, L, ws);
  t.M = L.Rp;
  t.m_dyn = 1;
  t.K = h;
  t.N = V;
  t.pm = reinterpret_cast<float*>(ws + L.off_pm);
  t.ps = reinterpret_cast<float*>(ws + L.off_ps);
  t.pu = reinterpret_cast<float*>(ws + L.off_pu);
  t.zy = reinterpret_cast<float*>(ws + L.off_zy);
  kind_policy(t, "RLHEAD_L2_FWD", -1);
  use_sched(t, ws, L, 0);
  CUtensorMap mq;
  if (q_out) {  // q tiles into the dZ buffer [Rp, Vp] (bf16, 32x32 TMA store boxes)
    t.q_tma = 1;
    t.q_adv = q_adv;
    t.q_row = reinterpret_cast<const int32_t*>(ws + (q_adv_per_row ? L.off_active : L.off_seq));
    if (!make_map_bf16_32(&mq, ws + L.off_dz, V, L.Rp, static_cast<uint64_t>(L.Vp) * 2))
      return RL_ERR_CUDA;
  }
  return run_narrow<0, 0, EPI_LSE>(ma, mb, t, L.Rp, RL_K_GEMM_LSE, s, q_out ? &mq : nullptr);
}

rl_status launch_tc_bwd(const rl_head* hd, const void* weight, void* grad_hidden,
                        float* grad_hidden_f32, bool gh_multicast, float* grad_weight,
                        const rl_peer_group* dw_rs, bool entropy_on, const WsLayout& L, char* ws,
                        cudaStream_t s, bool dz_ready, int bwd_rows) {
  const int h = hd->hidden, V = hd->vocab;
  const int cg = tc_cta_group();
  const bool packed = bwd_rows == BWD_PACKED;
  // packed mode: dZ / Hc rows of the backward rows only (packed by k_dz_from_q)
  __nv_bfloat16* dz = reinterpret_cast<__nv_bfloat16*>(ws + (packed ? L.off_dz2 : L.off_dz));
  char* hc_b = ws + (packed ? L.off_hc2 : L.off_hc);
  rl_status st;
  // N5: recompute logits, dZ = tau^-1 g (onehot - p) -> bf16 [Rp, Vp] (unless
  // k_dz_from_q already built dZ from the forward's q tiles).
  if (!dz_ready) {
    CUtensorMap ma, mb;
    if (!make_map(&ma, ws + L.off_hc, h, L.Rp, static_cast<uint64_t>(h) * 2, TC_BM) ||
        !make_map(&mb, weight, h, V, static_cast<uint64_t>(h) * 2, TC_BN / cg))
      return RL_ERR_CUDA;
    TcArgs t = base_args(hd, L, ws);
    t.M = L.Rp;
    t.m_dyn = 1;
    t.K = h;
    t.N = V;
    t.lse_c = reinterpret_cast<const float*>(ws + L.off_lse);
    t.g_c = reinterpret_cast<const float*>(ws + L.off_g);
    if (entropy_on) {
      t.ge_c = reinterpret_cast<const float*>(ws + L.off_ge);
      t.ez_c = reinterpret_cast<const float*>(ws + L.off_ez);
    }
    t.dz = dz;
    t.ld_dz = L.Vp;
    kind_policy(t, "RLHEAD_L2_DZ", -1);
    use_sched(t, ws, L, 1);
    // TMA stores of the dZ boxes (whole lines) instead of per-row 16-B stores:
    // same-box +0.3% tokens/s (RLHEAD_DZ_TMA=0 restores the per-row stores)
    t.dz_tma = env_int("RLHEAD_DZ_TMA", 1);
    CUtensorMap mdz;
    if (t.dz_tma &&
        !make_map_bf16_32(&mdz, dz, V, L.Rp, static_cast<uint64_t>(L.Vp) * 2))
      return RL_ERR_CUDA;
    st = run_narrow<0, 0, EPI_DZ>(ma, mb, t, L.Rp, RL_K_GEMM_DZ, s, t.dz_tma ? &mdz : nullptr);
    if (st != RL_OK) return st;
  }
  // N6: dH[T, h] = dZ[T, V] W[V, h]; rows -> grad_hidden[active_idx[r]].
  // N7: dW[V, h] += dZ^T[V, T] Hc[T, h].
  CUtensorMap ma6, mb6, ma7, mb7;
  if (!make_map(&ma6, dz, V, L.Rp, static_cast<uint64_t>(L.Vp) * 2, TC_BM) ||
      !make_map(&mb6, weight, h, V, static_cast<uint64_t>(h) * 2, 64) ||
      !make_map(&ma7, dz, V, L.Rp, static_cast<uint64_t>(L.Vp) * 2, 64) ||
      !make_map(&mb7, hc_b, h, L.Rp, static_cast<uint64_t>(h) * 2, 64))
    return RL_ERR_CUDA;
  TcArgs t6 = base_args(hd, L, ws);
  t6.M = L.Rp;
  t6.m_dyn = 1;
  t6.K = V;
  t6.N = h;
  t6.out = static_cast<__nv_bfloat16*>(grad_hidden);
  t6.ld_out = hd->ld_hidden;
  t6.out_f32 = grad_hidden_f32;
  t6.out_mc = gh_multicast ? 1 : 0;
  t6.row_idx = reinterpret_cast<const int32_t*>(ws + (packed ? L.off_oidx2 : L.off_active));
  t6.dyn_bwd = bwd_rows != BWD_DENSE ? 1 : 0;
  kind_policy(t6, "RLHEAD_L2_DH", -1);
  // serpentine K for dH measured neutral (~6 waves per micro-batch): off
  t6.k_serp = env_int("RLHEAD_DH_SERP", 0);
  use_sched(t6, ws, L, 2);
  TcArgs t7 = base_args(hd, L, ws);
  t7.dyn_bwd = bwd_rows != BWD_DENSE ? 1 : 0;
  t7.M = V;
  t7.K = L.Rp;
  t7.k_dyn = 1;
  t7.N = h;
  t7.acc = grad_weight;
  t7.ld_acc = h;
  // accumulate: 2 (default) = TMA reduce-add of 32x32 smem boxes (whole L2
  // lines: dW DRAM reads 30.4 -> 14.9 GB per micro-batch, dW GEMM -9%, +2.1%
  // tokens/s same-box); 1 = per-row red.global.add.v4; 0 = load+add+store
  // (profiles/r1/SUMMARY.md)
  t7.acc_red = env_int("RLHEAD_DW_RED", 2);
  kind_policy(t7, "RLHEAD_L2_DW", -1);
  // serpentine K: dW DRAM reads 20.9 -> 15.7 GB per micro-batch, +0.6% tokens/s
  // same-box (RLHEAD_DW_SERP=0: every tile walks K forwards)
  t7.k_serp = env_int("RLHEAD_DW_SERP", 1);
  use_sched(t7, ws, L, 3);
  if (dw_rs && dw_rs->world > 1) {
    t7.rs_world = dw_rs->world;
    t7.rs_rank = dw_rs->rank;
    t7.rs_rows = dw_rs->rows_per_rank;
    t7.rs_no_partial = dw_rs->no_partial ? 1 : 0;
    for (int q = 0; q < dw_rs->world; ++q) t7.rs_peer[q] = dw_rs->peers[q];
    // bulk copies need 16-B aligned rows (ld_acc % 4 == 0, aligned staging)
    bool al = (t7.ld_acc & 3) == 0;
    for (int q = 0; q < dw_rs->world; ++q)
      al = al && (reinterpret_cast<uintptr_t>(dw_rs->peers[q]) & 15) == 0;
    t7.rs_bulk = al && env_int("RLHEAD_RS_BULK", 1) != 0;
  }
  if (fused_bwd()) {
    // one persistent launch over the dH tiles then the dW tiles: the last
    // (partial) wave of dH fills with dW tiles instead of idling.
    TcArgs t = t6;
    if (t.sched) use_sched(t, ws, L, 4);
    t.n_tiles = static_cast<int32_t>(ceil_div(h, 2 * TC_BN));
    t.group_m = std::max(1, env_int("RLHEAD_GROUP_M_BWD", 1));
    t.M2 = V;
    t.K2 = L.Rp;
    t.k_dyn2 = 1;
    t.n_tiles2 = t.n_tiles;
    t.group_m2 = t.group_m;
    t.acc = grad_weight;
    t.ld_acc = h;
    t.acc_red = t7.acc_red;
    t.k_serp2 = t7.k_serp;   // dW tiles: serpentine K by dW wave, as in the separate launch
    t.rs_world = t7.rs_world;
    t.rs_rank = t7.rs_rank;
    t.rs_rows = t7.rs_rows;
    t.rs_no_partial = t7.rs_no_partial;
    for (int q = 0; q < 8; ++q) t.rs_peer[q] = t7.rs_peer[q];
    const int64_t tiles = (ceil_div(L.Rp, 2 * TC_BM) + ceil_div(V, 2 * TC_BM)) * t.n_tiles;
    // dW accumulation as in the separate launch: TMA reduce-add of 32x32
    // smem boxes (whole L2 lines) unless the reduce-scatter stores plainly
    CUtensorMap macc;
    if (t.acc_red == 2) {
      if (t.rs_world > 0 || (reinterpret_cast<uintptr_t>(grad_weight) & 15) != 0) t.acc_red = 1;
      else if (!make_map_f32(&macc, grad_weight, h, V, static_cast<uint64_t>(h) * 4, 32, 32))
        return RL_ERR_CUDA;
    }
    return run_gemm<2, 2, 0, 1, EPI_BWD>(ma6, mb6, ma7, mb7, t, tiles, RL_K_GEMM_DHDW, s, true,
                                         t.acc_red == 2 ? &macc : nullptr);
  }
  if ((st = run_wide<0, 1, EPI_ROWS>(ma6, mb6, t6, L.Rp, RL_K_GEMM_DH, s)) != RL_OK) return st;
  CUtensorMap macc;
  if (t7.acc_red == 2) {
    // TMA needs a 16-B aligned base; the reduce-scatter epilogue stores plainly
    if (t7.rs_world > 0 || (reinterpret_cast<uintptr_t>(grad_weight) & 15) != 0) t7.acc_red = 1;
    else if (!make_map_f32(&macc, grad_weight, h, V, static_cast<uint64_t>(h) * 4, 32, 32))
      return RL_ERR_CUDA;
  }
  return run_wide<1, 1, EPI_ACC>(ma7, mb7, t7, V, RL_K_GEMM_DW, s,
                                 t7.acc_red == 2 ? &macc : nullptr);
}

}  // namespace rlh
