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
constexpr int KEEP_ITEMS = 4;     // backward-row compaction: 1024-row tiles

// Backward rows (skip mode): the compact rows r < T with dL/dlogp g_r != 0, in
// order -> keep[r2] = r, oidx2[r2] = active_idx[r] (the packed row dL/dH goes
// to), hdr->n_bwd = their count. Rows with g = 0 -- every row of a GRPO group
// whose rewards are all equal (A = 0), clipped rows, padding -- have dZ = 0,
// so they contribute exactly nothing to dH (written as zeros elsewhere) or dW.
// Single pass: ballot counts per (item, warp), decoupled look-back across the
// tiles (claimed in order from a counter).
__global__ void __launch_bounds__(DZ_THREADS)
k_keep_compact(const float* __restrict__ g_c, const int32_t* __restrict__ active_idx,
               WsHeader* hdr, unsigned long long* status, int64_t ntiles,
               int32_t* __restrict__ keep, int32_t* __restrict__ oidx2) {
  __shared__ int32_t s_cnt[KEEP_ITEMS][DZ_THREADS / 32];
  __shared__ long long s_prefix;
  __shared__ int32_t s_tile;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = static_cast<int32_t>(atomicAdd(&hdr->tile_ctr2, 1u));
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t T = hdr->n_active;
  const int64_t base = tile * (DZ_THREADS * KEEP_ITEMS) + tid;
  uint32_t kbits = 0;
#pragma unroll
  for (int it = 0; it < KEEP_ITEMS; ++it) {
    const int64_t r = base + static_cast<int64_t>(it) * DZ_THREADS;
    if (r < T && g_c[r] != 0.f) kbits |= 1u << it;
  }
#pragma unroll
  for (int it = 0; it < KEEP_ITEMS; ++it) {
    const uint32_t b = __ballot_sync(0xffffffffu, (kbits >> it) & 1u);
    if (lane == 0) s_cnt[it][warp] = __popc(b);
  }
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the 32 (item, warp) counts, one per lane
    int32_t* flat = &s_cnt[0][0];
    const int c = flat[lane];
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    flat[lane] = incl - c;
    const long long agg = __shfl_sync(0xffffffffu, incl, 31);
    const long long excl = decoupled_lookback(status, tile, agg, lane);
    if (lane == 0) {
      s_prefix = excl;
      if (tile == ntiles - 1) hdr->n_bwd = excl + agg;
    }
  }
  __syncthreads();
  const long long pfx = s_prefix;
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int it = 0; it < KEEP_ITEMS; ++it) {
    const uint32_t b = __ballot_sync(0xffffffffu, (kbits >> it) & 1u);
    if ((kbits >> it) & 1u) {
      const int64_t r = base + static_cast<int64_t>(it) * DZ_THREADS;
      const long long o = pfx + s_cnt[it][warp] + __popc(b & lt);
      keep[o] = static_cast<int32_t>(r);
      oidx2[o] = active_idx[r];
    }
  }
}

// Fused-backward mode (RLHEAD_DZ_FUSED=1): before the forward, reorder the
// compact rows so the rows that can carry a gradient (their sequence's
// advantage A != 0; no KL term) come first, in order, and the A = 0 rows fill
// the tail (in reverse order): active_idx / tgt_c / seq_c are rewritten from
// copies (src_*), hdr->n_bwd = the prefix length. The backward GEMMs then run
// over that prefix of Hc / q in place. One pass: per tile the two classes'
// counts, packed (c1 << 31 | c0) in one decoupled look-back word; T (the
// active count, from H1) places the tail.
__global__ void __launch_bounds__(DZ_THREADS)
k_partition_rows(const int32_t* __restrict__ src_idx, const int32_t* __restrict__ src_tgt,
                 const int32_t* __restrict__ src_seq, const float* __restrict__ adv,
                 WsHeader* hdr, unsigned long long* status, int64_t ntiles,
                 int32_t* __restrict__ active_idx, int32_t* __restrict__ tgt_c,
                 int32_t* __restrict__ seq_c) {
  __shared__ int32_t s_cnt[2][KEEP_ITEMS][DZ_THREADS / 32];
  __shared__ long long s_p1, s_p0;
  __shared__ int32_t s_tile;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = static_cast<int32_t>(atomicAdd(&hdr->tile_ctr2, 1u));
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t T = hdr->n_active;
  const int64_t base = tile * (DZ_THREADS * KEEP_ITEMS) + tid;
  uint32_t vbits = 0, cbits = 0;  // valid row / class 1 (A != 0)
#pragma unroll
  for (int it = 0; it < KEEP_ITEMS; ++it) {
    const int64_t r = base + static_cast<int64_t>(it) * DZ_THREADS;
    if (r < T) {
      vbits |= 1u << it;
      if (adv[src_seq[r]] != 0.f) cbits |= 1u << it;
    }
  }
#pragma unroll
  for (int it = 0; it < KEEP_ITEMS; ++it) {
    const uint32_t b1 = __ballot_sync(0xffffffffu, (cbits >> it) & 1u);
    const uint32_t b0 = __ballot_sync(0xffffffffu, ((vbits & ~cbits) >> it) & 1u);
    if (lane == 0) {
      s_cnt[1][it][warp] = __popc(b1);
      s_cnt[0][it][warp] = __popc(b0);
    }
  }
  __syncthreads();
  if (warp == 0) {  // exclusive scans of the 32 (item, warp) counts of each class
    int32_t* f1 = &s_cnt[1][0][0];
    int32_t* f0 = &s_cnt[0][0][0];
    const int c1 = f1[lane], c0 = f0[lane];
    int i1 = c1, i0 = c0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v1 = __shfl_up_sync(0xffffffffu, i1, o);
      const int v0 = __shfl_up_sync(0xffffffffu, i0, o);
      if (lane >= o) {
        i1 += v1;
        i0 += v0;
      }
    }
    f1[lane] = i1 - c1;
    f0[lane] = i0 - c0;
    const long long a1 = __shfl_sync(0xffffffffu, i1, 31);
    const long long a0 = __shfl_sync(0xffffffffu, i0, 31);
    const long long excl = decoupled_lookback(status, tile, (a1 << 31) | a0, lane);
    if (lane == 0) {
      s_p1 = excl >> 31;
      s_p0 = excl & ((1ll << 31) - 1);
      if (tile == ntiles - 1) hdr->n_bwd = s_p1 + a1;
    }
  }
  __syncthreads();
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int it = 0; it < KEEP_ITEMS; ++it) {
    const uint32_t b1 = __ballot_sync(0xffffffffu, (cbits >> it) & 1u);
    const uint32_t b0 = __ballot_sync(0xffffffffu, ((vbits & ~cbits) >> it) & 1u);
    if ((vbits >> it) & 1u) {
      const int64_t r = base + static_cast<int64_t>(it) * DZ_THREADS;
      const bool c = (cbits >> it) & 1u;
      const long long o = c ? s_p1 + s_cnt[1][it][warp] + __popc(b1 & lt)
                            : T - 1 - (s_p0 + s_cnt[0][it][warp] + __popc(b0 & lt));
      active_idx[o] = src_idx[r];
      tgt_c[o] = src_tgt[r];
      seq_c[o] = src_seq[r];
    }
  }
}

rl_status launch_partition_rows(const WsLayout& L, char* ws, const float* adv, cudaStream_t s) {
  if (L.Rp <= 0) return RL_OK;
  WsHeader* hdr = reinterpret_cast<WsHeader*>(ws + L.off_hdr);
  int32_t* act = reinterpret_cast<int32_t*>(ws + L.off_active);
  int32_t* tgt = reinterpret_cast<int32_t*>(ws + L.off_tgt);
  int32_t* seq = reinterpret_cast<int32_t*>(ws + L.off_seq);
  // sources: copies in the (unused in this mode) packed-row scratch of skip mode
  int32_t* s_act = reinterpret_cast<int32_t*>(ws + L.off_keep);
  int32_t* s_tgt = reinterpret_cast<int32_t*>(ws + L.off_oidx2);
  int32_t* s_seq = reinterpret_cast<int32_t*>(ws + L.off_hc2);
  const size_t nb = static_cast<size_t>(L.Rp) * 4;
  if (cudaMemcpyAsync(s_act, act, nb, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
      cudaMemcpyAsync(s_tgt, tgt, nb, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
      cudaMemcpyAsync(s_seq, seq, nb, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return RL_ERR_CUDA;
  const int64_t ntiles = ceil_div(L.Rp, DZ_THREADS * KEEP_ITEMS);
  TraceScope ts(RL_K_PREPARE, s);
  k_partition_rows<<<static_cast<unsigned>(ntiles), DZ_THREADS, 0, s>>>(
      s_act, s_tgt, s_seq, adv, hdr, reinterpret_cast<unsigned long long*>(ws + L.off_st2),
      ntiles, act, tgt, seq);
  RLH_CHECK_LAUNCH();
  return RL_OK;
}

// dZ rows from the q tiles. Dense mode (keep == NULL): in place, row r of the
// dZ buffer from q row r (zeros when g_r = 0). Skip mode: row r2 < n_bwd of
// the packed buffer dz_out from q row keep[r2] (and Hc2[r2] = Hc[keep[r2]]),
// rows [n_bwd, n_bwd rounded up to the tile) zeroed.
__global__ void __launch_bounds__(DZ_THREADS)
k_dz_from_q(const uint4* q_in, uint4* dz_out, int64_t ld_vec, int32_t V, int64_t n_vt,
            const float* __restrict__ pm, const float* __restrict__ lse_c,
            const float* __restrict__ g_c, const float* __restrict__ zy,
            const int32_t* __restrict__ tgt_c, int64_t y_off, float inv_temp,
            const WsHeader* __restrict__ hdr, int64_t Rp, const int32_t* __restrict__ keep,
            const uint4* __restrict__ hc, uint4* __restrict__ hc2, int32_t h_vec,
            int32_t use_nbwd) {
  const int64_t r2 = blockIdx.x;
  const int64_t T = use_nbwd ? hdr->n_bwd : hdr->n_active;
  const int64_t Tp = (T + 2 * TC_BM - 1) / (2 * TC_BM) * (2 * TC_BM);  // rows the GEMMs read
  if (r2 >= Tp || r2 >= Rp) return;
  const int64_t nvec = (static_cast<int64_t>(V) + 7) / 8;   // 8 bf16 per 16-B vector
  uint4* row = dz_out + r2 * ld_vec;
  const int64_t r = r2 < T ? (keep ? static_cast<int64_t>(keep[r2]) : r2) : -1;
  const float g = r >= 0 ? g_c[r] : 0.f;
  if (keep) {  // Hc row of the packed backward rows (zeros past n_bwd)
    uint4* dst = hc2 + r2 * h_vec;
    if (r >= 0) {
      const uint4* src = hc + r * h_vec;
      for (int i = threadIdx.x; i < h_vec; i += DZ_THREADS) dst[i] = src[i];
    } else {
      for (int i = threadIdx.x; i < h_vec; i += DZ_THREADS) dst[i] = make_uint4(0, 0, 0, 0);
    }
  }
  if (g == 0.f) {                                          // no gradient: dZ row = 0
    const uint4 z = make_uint4(0, 0, 0, 0);
    for (int64_t i = threadIdx.x; i < nvec; i += DZ_THREADS) row[i] = z;
    return;
  }
  const uint4* qrow = q_in + r * ld_vec;
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
    uint4 q = qrow[i];
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

rl_status launch_dz_from_q(const rl_head* hd, const WsLayout& L, char* ws, cudaStream_t s,
                           int bwd_rows) {
  if (L.Rp <= 0) return RL_OK;
  WsHeader* hdr = reinterpret_cast<WsHeader*>(ws + L.off_hdr);
  const bool skip_zero_rows = bwd_rows == BWD_PACKED;
  int32_t* keep = nullptr;
  if (skip_zero_rows) {
    keep = reinterpret_cast<int32_t*>(ws + L.off_keep);
    const int64_t ntiles = ceil_div(L.Rp, DZ_THREADS * KEEP_ITEMS);
    TraceScope ts(RL_K_DZQ, s);
    k_keep_compact<<<static_cast<unsigned>(ntiles), DZ_THREADS, 0, s>>>(
        reinterpret_cast<const float*>(ws + L.off_g),
        reinterpret_cast<const int32_t*>(ws + L.off_active), hdr,
        reinterpret_cast<unsigned long long*>(ws + L.off_st2), ntiles, keep,
        reinterpret_cast<int32_t*>(ws + L.off_oidx2));
    RLH_CHECK_LAUNCH();
  }
  TraceScope ts(RL_K_DZQ, s);
  k_dz_from_q<<<static_cast<unsigned>(L.Rp), DZ_THREADS, 0, s>>>(
      reinterpret_cast<const uint4*>(ws + L.off_dz),
      reinterpret_cast<uint4*>(ws + (skip_zero_rows ? L.off_dz2 : L.off_dz)), L.Vp / 8,
      hd->vocab, L.n_vt, reinterpret_cast<const float*>(ws + L.off_pm),
      reinterpret_cast<const float*>(ws + L.off_lse), reinterpret_cast<const float*>(ws + L.off_g),
      reinterpret_cast<const float*>(ws + L.off_zy),
      reinterpret_cast<const int32_t*>(ws + L.off_tgt),
      hd->vocab_total > 0 ? hd->vocab_offset : 0, hd->inv_temperature, hdr, L.Rp, keep,
      reinterpret_cast<const uint4*>(ws + L.off_hc), reinterpret_cast<uint4*>(ws + L.off_hc2),
      hd->hidden / 8, bwd_rows != BWD_DENSE ? 1 : 0);
  RLH_CHECK_LAUNCH();
  return RL_OK;
}

}  // namespace rlh
