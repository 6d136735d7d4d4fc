// H6 without the logits recompute: dZ from the forward's q tiles.
//
// The forward GEMM (EPI_LSE with q_tma) stored, for every compact row r and
// vocab tile v, q[r, j] = e^{z_rj - m_rv} in bf16 (m_rv the tile maximum it
// also wrote as the split-V partial, q = 0 at the target column), into the
// dZ buffer. After the merge knows lse_r and g_r, the softmax is
// p_rj = q[r, j] e^{m_rv - lse_r}, so
//   dZ[r, j] = tau^-1 g_r (onehot_j(y_r) - p_rj)
//            = -tau^-1 g_r e^{m_rv - lse_r} q[r, j]          (j != y_r)
//            = tau^-1 g_r (1 - p_ry) = -tau^-1 g_r expm1(z_ry - lse_r)   (j = y_r),
// the target column from the fp32 z_y the forward captured (no cancellation
// for confident tokens, p_y -> 1). One pass, in place: 2 B read + 2 B written
// per element of active rows with g != 0; rows with g = 0 (A = 0, clipped,
// padding) are written as zeros without reading q. This replaces the 2hV
// flop/token recompute GEMM (BASELINE.json north_star: the logits
// themselves still never reach HBM -- q is the tile-normalised softmax,
// the same bytes the dZ buffer holds anyway).
#include "kernels.h"

namespace rlh {

constexpr int DZ_THREADS = 256;   // one CTA per row; a warp covers one 256-column vocab tile

__global__ void __launch_bounds__(DZ_THREADS)
k_dz_from_q(uint4* __restrict__ dz, int64_t ld_vec, int32_t V, int64_t n_vt,
            const float* __restrict__ pm, const float* __restrict__ lse_c,
            const float* __restrict__ g_c, const float* __restrict__ zy,
            const int32_t* __restrict__ tgt_c, int64_t y_off, float inv_temp,
            const WsHeader* __restrict__ hdr, int64_t Rp) {
  const int64_t T = hdr->n_active;
  const int64_t Tp = (T + 2 * TC_BM - 1) / (2 * TC_BM) * (2 * TC_BM);  // rows the GEMMs read
  const int64_t nvec = (static_cast<int64_t>(V) + 7) / 8;   // 8 bf16 per 16-B vector
  const int64_t r = blockIdx.x;
  if (r >= Tp || r >= Rp) return;
  uint4* row = dz + r * ld_vec;
  const float g = r < T ? g_c[r] : 0.f;
  if (g == 0.f) {                                          // no gradient: dZ row = 0
    const uint4 z = make_uint4(0, 0, 0, 0);
    for (int64_t i = threadIdx.x; i < nvec; i += DZ_THREADS) row[i] = z;
    return;
  }
  const float coef = inv_temp * g;
  const float lse = lse_c[r];
  const int64_t yl = static_cast<int64_t>(tgt_c[r]) - y_off;
  const int64_t yv = (yl >= 0 && yl < V) ? yl : -1;
  const float dzy = -coef * expm1f(zy[r] - lse);           // tau^-1 g (1 - p_y)
  const float* pmr = pm + (r >> 5) * n_vt * 32 + (r & 31);  // row-blocked partial maxima
#pragma unroll 4
  for (int64_t i = threadIdx.x; i < nvec; i += DZ_THREADS) {
    const int64_t v = i >> 5;                                // 32 vectors per vocab tile
    const float sc = -coef * __expf(pmr[v * 32] - lse);      // -tau^-1 g e^{m_rv - lse}
    uint4 q = row[i];
    uint32_t* w = reinterpret_cast<uint32_t*>(&q);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&w[k]);
      float2 f = __bfloat1622float2(b);
      f.x *= sc;
      f.y *= sc;
      const int64_t j = 8 * i + 2 * k;
      if (j == yv) f.x = dzy;
      if (j + 1 == yv) f.y = dzy;
      const __nv_bfloat162 o = __floats2bfloat162_rn(f.x, f.y);
      w[k] = *reinterpret_cast<const uint32_t*>(&o);
    }
    row[i] = q;
  }
}

rl_status launch_dz_from_q(const rl_head* hd, const WsLayout& L, char* ws, cudaStream_t s) {
  if (L.Rp <= 0) return RL_OK;
  TraceScope ts(RL_K_DZQ, s);
  // one CTA per row (a bounded persistent grid, which would leave room for a
  // GEMM CTA of another micro-batch beside it, measured 1.7x slower alone)
  k_dz_from_q<<<static_cast<unsigned>(L.Rp), DZ_THREADS, 0, s>>>(
      reinterpret_cast<uint4*>(ws + L.off_dz), L.Vp / 8, hd->vocab, L.n_vt,
      reinterpret_cast<const float*>(ws + L.off_pm), reinterpret_cast<const float*>(ws + L.off_lse),
      reinterpret_cast<const float*>(ws + L.off_g), reinterpret_cast<const float*>(ws + L.off_zy),
      reinterpret_cast<const int32_t*>(ws + L.off_tgt),
      hd->vocab_total > 0 ? hd->vocab_offset : 0, hd->inv_temperature,
      reinterpret_cast<const WsHeader*>(ws + L.off_hdr), L.Rp);
  RLH_CHECK_LAUNCH();
  return RL_OK;
}

}  // namespace rlh
