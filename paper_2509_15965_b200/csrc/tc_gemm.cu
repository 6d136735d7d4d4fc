// Tensor-core path of the head (bf16 in, fp32 accumulate) for sm_100a:
// one persistent, warp-specialised tcgen05 GEMM with four fused epilogues.
//
//   warp 0  : TMA producer (one elected lane): A/B k-blocks -> 4-stage smem
//             ring (128-B swizzle), mbarrier complete_tx.
//   warp 1  : TMEM allocator + MMA issuer (one lane): tcgen05.mma
//             kind::f16, M=128 N=256 K=16, accumulator in TMEM, two 256-col
//             accumulators (double buffered) so the epilogue of tile i
//             overlaps the MMAs of tile i+1; tcgen05.commit frees smem
//             stages and signals the epilogue.
//   warps 4-7: epilogue (thread = accumulator row = TMEM lane):
//     EPI_LSE (H3+H4, N3): online log-sum-exp of the 256 logits of the tile
//             -> per-row split-V partial (m, sum e^{z-m}, sum e^{z-m}(z-m)),
//             target logit captured in the tile that holds it. The logits
//             never leave TMEM/registers (BASELINE.json north_star).
//     EPI_DZ  (H6, N5): recompute the same logits (same tile/K order),
//             dZ = tau^-1 g (onehot(y) - exp(z - lse)) -> bf16 dZ chunk.
//     EPI_ROWS(H7, N6): dH = dZ W, rows scattered back to the packed layout.
//     EPI_ACC (H8, N7): dW += dZ^T H (fp32 read-modify-write).
//
// Operand majors: fwd/dZ  A = Hc [T,h] K-major,  B = W [V,h] K-major;
//                 dH      A = dZ [T,V] K-major,  B = W [V,h] MN-major;
//                 dW      A = dZ [T,V] MN-major, B = Hc [T,h] MN-major.
// Tiles are rasterised in groups of GROUP_M row-tiles so the CTAs resident
// at any time share A and B panels in L2.
#include "kernels.h"
#include "ptx.cuh"

#include <mutex>

namespace rlh {

constexpr int TC_STAGES = 4;
constexpr int TC_A_BYTES = TC_BM * TC_BK * 2;             // 16 KB
constexpr int TC_B_BYTES = TC_BN * TC_BK * 2;             // 32 KB
constexpr int TC_STAGE_BYTES = TC_A_BYTES + TC_B_BYTES;   // 48 KB
constexpr int TC_THREADS = 256;
constexpr int TC_SMEM_BYTES = TC_STAGES * TC_STAGE_BYTES + 1024 + 256;
constexpr int TC_TMEM_COLS = 512;                         // 2 x 256 fp32 accumulators
constexpr float LOG2E = 1.4426950408889634f;

enum { EPI_LSE = 0, EPI_DZ = 1, EPI_ROWS = 2, EPI_ACC = 3 };

struct TcArgs {
  int64_t M, K;        // host values (used unless m_dyn / k_dyn)
  int32_t N;           // output columns (V or h)
  int32_t n_tiles;
  int32_t m_dyn, k_dyn;
  int32_t group_m;
  const WsHeader* hdr;
  float inv_temp;
  int32_t vocab;
  // EPI_LSE
  float *pm, *ps, *pu, *zy;
  const int32_t* tgt_c;
  int64_t ldp;
  // EPI_DZ
  const float *lse_c, *g_c;
  __nv_bfloat16* dz;
  int64_t ld_dz;
  // EPI_ROWS
  __nv_bfloat16* out;
  int64_t ld_out;
  const int32_t* row_idx;
  // EPI_ACC
  float* acc;
  int64_t ld_acc;
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

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

template <int AMN, int BMN, int EPI>
__global__ void __launch_bounds__(TC_THREADS, 1)
k_tc_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
          const TcArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + TC_STAGES * TC_A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + TC_STAGES * TC_STAGE_BYTES);
  uint64_t* empty = full + TC_STAGES;
  uint64_t* tfull = empty + TC_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < TC_STAGES; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(tfull + i, 1);
      mbar_init(tempty + i, 128);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, TC_TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int64_t T = args.hdr->n_active;
  const int64_t M = args.m_dyn ? T : args.M;
  const int64_t K = args.k_dyn ? T : args.K;
  const int64_t m_tiles = (M + TC_BM - 1) / TC_BM;
  const int64_t num_k = (K + TC_BK - 1) / TC_BK;
  const int64_t num_tiles = num_k > 0 ? m_tiles * args.n_tiles : 0;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------ TMA producer
      const uint64_t pol_a = l2_policy_evict_last();
      const uint64_t pol_b = l2_policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int64_t mb;
        int nb;
        tile_coords(tile, m_tiles, args.n_tiles, args.group_m, mb, nb);
        const int32_t m0 = static_cast<int32_t>(mb * TC_BM), n0 = nb * TC_BN;
        for (int64_t kb = 0; kb < num_k; ++kb) {
          mbar_wait(empty + stage, phase ^ 1);
          mbar_arrive_expect_tx(full + stage, TC_STAGE_BYTES);
          uint8_t* a_dst = sA + stage * TC_A_BYTES;
          uint8_t* b_dst = sB + stage * TC_B_BYTES;
          const int32_t k0 = static_cast<int32_t>(kb * TC_BK);
          if (AMN) {
            tma_load_2d(&tmA, full + stage, a_dst, m0, k0, pol_a);
            tma_load_2d(&tmA, full + stage, a_dst + 8192, m0 + 64, k0, pol_a);
          } else {
            tma_load_2d(&tmA, full + stage, a_dst, k0, m0, pol_a);
          }
          if (BMN) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              tma_load_2d(&tmB, full + stage, b_dst + i * 8192, n0 + 64 * i, k0, pol_b);
          } else {
            tma_load_2d(&tmB, full + stage, b_dst, k0, n0, pol_b);
          }
          if (++stage == TC_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------- MMA issuer
      constexpr uint32_t IDESC = umma_idesc_bf16(TC_BM, TC_BN, AMN, BMN);
      const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        mbar_wait(tempty + acc, acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * TC_BN);
        for (int64_t kb = 0; kb < num_k; ++kb) {
          mbar_wait(full + stage, phase);
          tc_fence_after();
          const uint32_t a_addr = a_base + stage * TC_A_BYTES;
          const uint32_t b_addr = b_base + stage * TC_B_BYTES;
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k) {
            const uint64_t ad = AMN ? umma_desc_sw128(a_addr + k * 2048, 8192, 1024)
                                    : umma_desc_sw128(a_addr + k * 32, 0, 1024);
            const uint64_t bd = BMN ? umma_desc_sw128(b_addr + k * 2048, 8192, 1024)
                                    : umma_desc_sw128(b_addr + k * 32, 0, 1024);
            tc_mma_f16(d_tmem, ad, bd, IDESC, (kb > 0 || k > 0) ? 1u : 0u);
          }
          tc_commit(empty + stage);
          if (++stage == TC_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit(tfull + acc);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 4;
    const int rit = ew * 32 + lane;  // row in tile == TMEM lane
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      int64_t mb;
      int nb;
      tile_coords(tile, m_tiles, args.n_tiles, args.group_m, mb, nb);
      const int64_t row = mb * TC_BM + rit;
      const int n0 = nb * TC_BN;
      const bool row_ok = row < M;
      mbar_wait(tfull + acc, acc_phase);
      tc_fence_after();
      const uint32_t taddr =
          tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + static_cast<uint32_t>(acc * TC_BN);

      if constexpr (EPI == EPI_LSE) {
        const int y = row_ok ? args.tgt_c[row] : -1;
        const int yrel = y - n0;
        const int valid = args.vocab - n0;  // columns < valid are real vocab ids
        float m = -INFINITY, s = 0.f, u = 0.f, zyv = 0.f;
        bool has_y = false;
#pragma unroll 1
        for (int c = 0; c < TC_BN / 32; ++c) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(taddr + c * 32, v);
          tmem_ld_wait();
          float z[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            z[j] = __uint_as_float(v[j]) * args.inv_temp;
            if (c * 32 + j >= valid) z[j] = -INFINITY;
          }
          const int yc = yrel - c * 32;
          if (yc >= 0 && yc < 32) {
            has_y = true;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j == yc) zyv = z[j];
          }
          float cm = z[0];
#pragma unroll
          for (int j = 1; j < 32; ++j) cm = fmaxf(cm, z[j]);
          if (cm > m) {
            if (s > 0.f) {
              const float f = ex2_approx((m - cm) * LOG2E);
              u = f * (u + (m - cm) * s);
              s *= f;
            }
            m = cm;
          }
          if (m > -INFINITY) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              // clamp keeps masked (-inf) columns at e = 0, e*d = 0 (not NaN);
              // e^{-200} underflows fp32 anyway.
              const float d = fmaxf(z[j] - m, -200.f);
              const float e = ex2_approx(d * LOG2E);
              s += e;
              u = fmaf(e, d, u);
            }
          }
        }
        tc_fence_before();
        mbar_arrive(tempty + acc);
        if (row_ok) {
          const int64_t o = static_cast<int64_t>(nb) * args.ldp + row;
          args.pm[o] = m;
          args.ps[o] = s;
          args.pu[o] = u;
          if (has_y) args.zy[row] = zyv;
        }
      } else if constexpr (EPI == EPI_DZ) {
        const float lse = row_ok ? args.lse_c[row] : 0.f;
        const float coef = row_ok ? args.g_c[row] * args.inv_temp : 0.f;
        const int yrel = (row_ok ? args.tgt_c[row] : -1) - n0;
        const float lse2 = lse * LOG2E, sc2 = args.inv_temp * LOG2E;
        uint4* dst = reinterpret_cast<uint4*>(args.dz + row * args.ld_dz + n0);
#pragma unroll 1
        for (int c = 0; c < TC_BN / 32; ++c) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(taddr + c * 32, v);
          tmem_ld_wait();
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const float p0 = ex2_approx(fmaf(__uint_as_float(v[j]), sc2, -lse2));
            const float p1 = ex2_approx(fmaf(__uint_as_float(v[j + 1]), sc2, -lse2));
            const float d0 = coef * ((c * 32 + j == yrel ? 1.f : 0.f) - p0);
            const float d1 = coef * ((c * 32 + j + 1 == yrel ? 1.f : 0.f) - p1);
            pk[j / 2] = pack_bf16x2(d0, d1);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q)
            dst[c * 4 + q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
        }
        tc_fence_before();
        mbar_arrive(tempty + acc);
      } else if constexpr (EPI == EPI_ROWS) {
        const int64_t orow = row_ok ? static_cast<int64_t>(args.row_idx[row]) : 0;
        uint4* dst = reinterpret_cast<uint4*>(args.out + orow * args.ld_out + n0);
#pragma unroll 1
        for (int c = 0; c < TC_BN / 32; ++c) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(taddr + c * 32, v);
          tmem_ld_wait();
          if (row_ok && n0 + c * 32 < args.N) {
            uint32_t pk[16];
#pragma unroll
            for (int j = 0; j < 32; j += 2)
              pk[j / 2] = pack_bf16x2(__uint_as_float(v[j]), __uint_as_float(v[j + 1]));
#pragma unroll
            for (int q = 0; q < 4; ++q)
              dst[c * 4 + q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
          }
        }
        tc_fence_before();
        mbar_arrive(tempty + acc);
      } else {  // EPI_ACC
        float4* dst = reinterpret_cast<float4*>(args.acc + row * args.ld_acc + n0);
#pragma unroll 1
        for (int c = 0; c < TC_BN / 32; ++c) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(taddr + c * 32, v);
          tmem_ld_wait();
          if (row_ok && n0 + c * 32 < args.N) {
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
        tc_fence_before();
        mbar_arrive(tempty + acc);
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem_base, TC_TMEM_COLS);
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

template <int AMN, int BMN, int EPI>
static rl_status run_gemm(const CUtensorMap& a, const CUtensorMap& b, const TcArgs& args,
                          int64_t tiles_bound, int kind, cudaStream_t s) {
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(k_tc_gemm<AMN, BMN, EPI>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM_BYTES);
  });
  if (attr_err != cudaSuccess) return RL_ERR_CUDA;
  if (tiles_bound <= 0) return RL_OK;
  const int64_t grid = tiles_bound < num_sms() ? tiles_bound : num_sms();
  TraceScope ts(kind, s);
  k_tc_gemm<AMN, BMN, EPI><<<static_cast<unsigned>(grid), TC_THREADS, TC_SMEM_BYTES, s>>>(a, b,
                                                                                          args);
  RLH_CHECK_LAUNCH();
  return RL_OK;
}

static TcArgs base_args(const rl_head* hd, const WsLayout& L, char* ws) {
  TcArgs t{};
  t.hdr = reinterpret_cast<const WsHeader*>(ws + L.off_hdr);
  t.inv_temp = hd->inv_temperature;
  t.vocab = hd->vocab;
  t.group_m = 16;
  t.tgt_c = reinterpret_cast<const int32_t*>(ws + L.off_tgt);
  t.ldp = L.Rp;
  return t;
}

rl_status launch_tc_fwd(const rl_head* hd, const void* weight, const WsLayout& L, char* ws,
                        cudaStream_t s) {
  const int h = hd->hidden, V = hd->vocab;
  CUtensorMap ma, mb;
  if (!make_map(&ma, ws + L.off_hc, h, L.Rp, static_cast<uint64_t>(h) * 2, TC_BM) ||
      !make_map(&mb, weight, h, V, static_cast<uint64_t>(h) * 2, TC_BN))
    return RL_ERR_CUDA;
  TcArgs t = base_args(hd, L, ws);
  t.M = L.Rp;
  t.m_dyn = 1;
  t.K = h;
  t.N = V;
  t.n_tiles = static_cast<int32_t>(L.n_vt);
  t.pm = reinterpret_cast<float*>(ws + L.off_pm);
  t.ps = reinterpret_cast<float*>(ws + L.off_ps);
  t.pu = reinterpret_cast<float*>(ws + L.off_pu);
  t.zy = reinterpret_cast<float*>(ws + L.off_zy);
  return run_gemm<0, 0, EPI_LSE>(ma, mb, t, (L.Rp / TC_BM) * L.n_vt, RL_K_GEMM_LSE, s);
}

rl_status launch_tc_bwd(const rl_head* hd, const void* weight, void* grad_hidden,
                        float* grad_weight, const WsLayout& L, char* ws, cudaStream_t s) {
  const int h = hd->hidden, V = hd->vocab;
  const int h_tiles = static_cast<int>(ceil_div(h, TC_BN));
  __nv_bfloat16* dz = reinterpret_cast<__nv_bfloat16*>(ws + L.off_dz);
  rl_status st;
  // N5: recompute logits, dZ = tau^-1 g (onehot - p) -> bf16 [Rp, Vp].
  {
    CUtensorMap ma, mb;
    if (!make_map(&ma, ws + L.off_hc, h, L.Rp, static_cast<uint64_t>(h) * 2, TC_BM) ||
        !make_map(&mb, weight, h, V, static_cast<uint64_t>(h) * 2, TC_BN))
      return RL_ERR_CUDA;
    TcArgs t = base_args(hd, L, ws);
    t.M = L.Rp;
    t.m_dyn = 1;
    t.K = h;
    t.N = V;
    t.n_tiles = static_cast<int32_t>(L.n_vt);
    t.lse_c = reinterpret_cast<const float*>(ws + L.off_lse);
    t.g_c = reinterpret_cast<const float*>(ws + L.off_g);
    t.dz = dz;
    t.ld_dz = L.Vp;
    st = run_gemm<0, 0, EPI_DZ>(ma, mb, t, (L.Rp / TC_BM) * L.n_vt, RL_K_GEMM_DZ, s);
    if (st != RL_OK) return st;
  }
  // N6: dH[T, h] = dZ[T, V] W[V, h]; rows -> grad_hidden[active_idx[r]].
  {
    CUtensorMap ma, mb;
    if (!make_map(&ma, dz, V, L.Rp, static_cast<uint64_t>(L.Vp) * 2, TC_BM) ||
        !make_map(&mb, weight, h, V, static_cast<uint64_t>(h) * 2, 64))
      return RL_ERR_CUDA;
    TcArgs t = base_args(hd, L, ws);
    t.M = L.Rp;
    t.m_dyn = 1;
    t.K = V;
    t.N = h;
    t.n_tiles = h_tiles;
    t.out = static_cast<__nv_bfloat16*>(grad_hidden);
    t.ld_out = hd->ld_hidden;
    t.row_idx = reinterpret_cast<const int32_t*>(ws + L.off_active);
    st = run_gemm<0, 1, EPI_ROWS>(ma, mb, t, (L.Rp / TC_BM) * h_tiles, RL_K_GEMM_DH, s);
    if (st != RL_OK) return st;
  }
  // N7: dW[V, h] += dZ^T[V, T] Hc[T, h].
  {
    CUtensorMap ma, mb;
    if (!make_map(&ma, dz, V, L.Rp, static_cast<uint64_t>(L.Vp) * 2, 64) ||
        !make_map(&mb, ws + L.off_hc, h, L.Rp, static_cast<uint64_t>(h) * 2, 64))
      return RL_ERR_CUDA;
    TcArgs t = base_args(hd, L, ws);
    t.M = V;
    t.K = L.Rp;
    t.k_dyn = 1;
    t.N = h;
    t.n_tiles = h_tiles;
    t.acc = grad_weight;
    t.ld_acc = h;
    st = run_gemm<1, 1, EPI_ACC>(ma, mb, t, ceil_div(V, TC_BM) * h_tiles, RL_K_GEMM_DW, s);
    if (st != RL_OK) return st;
  }
  return RL_OK;
}

}  // namespace rlh
