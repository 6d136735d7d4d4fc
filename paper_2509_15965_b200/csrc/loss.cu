// H4 merge + H5 loss head. One thread per active (compact) row:
//  * merge the split-V partials (m_n, s_n = sum e^{z-m_n}, u_n = sum
//    e^{z-m_n}(z-m_n)) into lse = M + log S and entropy = log S - U/S
//    (entropy in the shifted form avoids cancelling M), logp = z_y - lse;
//  * H5 (P:L828 token-level mean, readings DESIGN.md §3 #12-#15):
//    d = logp - old, r = exp(clamp(d)), l = max(-A r, -A clip(r)),
//    g = dL/dlogp = -w A r [unclipped] [|d| <= c]; NEXT-1 variants (#25-#28):
//    dual clip, KL-k3 to ref_logp, entropy bonus (w c_ent and E_p[z] kept for
//    the dZ epilogue), seq-mean-token-mean weights w = 1/(S n_s);
//  * per-block fixed-order reduction of the loss statistics (deterministic),
//    summed by a one-block kernel into the caller's accumulators.
#include "kernels.h"

#include <algorithm>
#include <mutex>

namespace rlh {

constexpr int MERGE_THREADS = 256;
constexpr int MERGE_ROWS = 32;                     // k_merge rows per block
constexpr int MERGE_SPLIT = MERGE_THREADS / 32;    // warps splitting the partials

struct LStat {
  double loss, ratio, ent, kl, obj;
  float rmax;
  long long clo, chi, tok;
};

__device__ __forceinline__ void lstat_add(LStat& a, const LStat& b) {
  a.loss += b.loss;
  a.ratio += b.ratio;
  a.ent += b.ent;
  a.kl += b.kl;
  a.obj += b.obj;
  a.rmax = fmaxf(a.rmax, b.rmax);
  a.clo += b.clo;
  a.chi += b.chi;
  a.tok += b.tok;
}

__device__ __forceinline__ LStat lstat_shfl(const LStat& v, int o) {
  LStat w;
  w.loss = __shfl_xor_sync(0xffffffffu, v.loss, o);
  w.ratio = __shfl_xor_sync(0xffffffffu, v.ratio, o);
  w.ent = __shfl_xor_sync(0xffffffffu, v.ent, o);
  w.kl = __shfl_xor_sync(0xffffffffu, v.kl, o);
  w.obj = __shfl_xor_sync(0xffffffffu, v.obj, o);
  w.rmax = __shfl_xor_sync(0xffffffffu, v.rmax, o);
  w.clo = __shfl_xor_sync(0xffffffffu, v.clo, o);
  w.chi = __shfl_xor_sync(0xffffffffu, v.chi, o);
  w.tok = __shfl_xor_sync(0xffffffffu, v.tok, o);
  return w;
}

template <int NT>
__device__ LStat block_reduce_lstat(LStat v) {
  __shared__ LStat sh[NT / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    LStat w = lstat_shfl(v, o);
    lstat_add(v, w);
  }
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  LStat t = sh[0];
  for (int w = 1; w < NT / 32; ++w) lstat_add(t, sh[w]);
  return t;
}

// First index i in [0, T) with active_idx[i] >= row (active_idx ascending).
__device__ __forceinline__ int64_t lower_bound_rows(const int32_t* __restrict__ a, int64_t T,
                                                   int64_t row) {
  int64_t lo = 0, hi = T;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (static_cast<int64_t>(a[mid]) < row) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Fold one partial (m, s, u) into the running (M, S, U); M = -inf = empty.
__device__ __forceinline__ void lse_fold(float& M, float& S, float& U, float m, float s, float u) {
  if (M == -INFINITY) {
    M = m;
    S = s;
    U = u;
    return;
  }
  if (m > M) {  // rescale the running sums to the new max
    const float f = expf(M - m);
    U = f * (U + (M - m) * S);
    S = f * S;
    M = m;
  }
  const float f2 = expf(m - M);
  S += s * f2;
  U += f2 * (u + (m - M) * s);
}

// Guarded fold of a partial (m, s, u) that may be empty (m = -inf).
__device__ __forceinline__ void lse_fold_g(float& M, float& S, float& U, float m, float s,
                                           float u) {
  if (m != -INFINITY) lse_fold(M, S, U, m, s, u);
}

// Fold a batch of partials j = 0..B-1 (m[j] = -inf: absent) into (M, S, U):
// one rescale to the batch maximum, then one exp per present partial.
template <int B>
__device__ __forceinline__ void lse_fold_batch(float& M, float& S, float& U, const float* m,
                                               const float* sv, const float* u) {
  float Mn = M;
#pragma unroll
  for (int j = 0; j < B; ++j) Mn = fmaxf(Mn, m[j]);
  if (Mn == -INFINITY) return;                 // nothing but empty partials so far
  const bool empty = M == -INFINITY;
  const float dM = empty ? 0.f : M - Mn;
  const float f = empty ? 0.f : expf(dM);
  float Sn = f * S, Un = f * (U + dM * S);
#pragma unroll
  for (int j = 0; j < B; ++j) {
    if (m[j] != -INFINITY) {
      const float d = m[j] - Mn, e = expf(d);
      Sn += e * sv[j];
      Un += e * (u[j] + d * sv[j]);
    }
  }
  M = Mn;
  S = Sn;
  U = Un;
}

// H5 for one active row r (compact) / t (packed): ratio, clipped surrogate
// (+ NEXT-1 variants), dL/dlogp -> g_c (and the entropy-bonus coefficients),
// the row's loss statistics.
__device__ __forceinline__ LStat row_loss(const MergeArgs& a, int64_t r, int32_t t, int64_t T,
                                          float lp, float lse, float ent) {
  const int32_t sq = a.seq_c[r];
  // per-token weight w_t (token mean: 1/N; seq-mean-token-mean: 1/(S n_s))
  double base = a.loss_scale;
  if (a.seq_mean) {
    if (a.n_seqs_global) {
      const long long Sg = *a.n_seqs_global;
      base = Sg > 0 ? 1.0 / static_cast<double>(Sg) : 0.0;
    }
    // active rows of sequence sq are the compact range [lb(cu[sq]), lb(cu[sq+1]))
    const int64_t b0 = lower_bound_rows(a.active_idx, T, a.cu_seqlens[sq]);
    const int64_t b1 = lower_bound_rows(a.active_idx, T, a.cu_seqlens[sq + 1]);
    base /= static_cast<double>(b1 - b0);
  } else if (a.n_global) {
    const long long N = *a.n_global;
    base = N > 0 ? 1.0 / static_cast<double>(N) : 0.0;
  }
  const float A = a.adv_per_token ? a.adv[t] : a.adv[sq];
  const float d = lp - a.old_logp[t];
  const float dc = fminf(fmaxf(d, -a.clamp_c), a.clamp_c);
  const float ratio = expf(dc);
  const float lo = 1.f - a.clip_lo, hi = 1.f + a.clip_hi;
  const float rc = fminf(fmaxf(ratio, lo), hi);
  float loss = fmaxf(-A * ratio, -A * rc);
  const bool chi = (A > 0.f) && (ratio > hi);
  const bool clo = (A < 0.f) && (ratio < lo);
  bool flows = !(chi || clo) && (fabsf(d) <= a.clamp_c);
  if (a.dual_clip > 0.f && A < 0.f) {  // dual clip: cap the loss at -A c_dual
    loss = fminf(loss, -A * a.dual_clip);
    if (ratio > a.dual_clip) flows = false;
  }
  double dl = flows ? -static_cast<double>(A) * ratio : 0.0;
  float kl = 0.f;
  if (a.ref_logp) {  // k3 estimator of KL to the reference policy
    const float q0 = a.ref_logp[t] - lp;
    const float q = fminf(fmaxf(q0, -a.clamp_c), a.clamp_c);
    const float eq = expf(q);
    kl = eq - q - 1.f;
    if (fabsf(q0) <= a.clamp_c) dl += static_cast<double>(a.kl_coef) * (1.0 - eq);
  }
  a.g_c[r] = static_cast<float>(base * dl);
  a.lse_c[r] = lse;
  if (a.ge_c) {
    a.ge_c[r] = static_cast<float>(base * a.entropy_coef);
    a.ez_c[r] = lse - ent;  // E_p[z]
  }
  const double obj = base * (static_cast<double>(loss) + a.kl_coef * static_cast<double>(kl) -
                             a.entropy_coef * static_cast<double>(ent));
  return {static_cast<double>(loss), static_cast<double>(ratio), static_cast<double>(ent),
          static_cast<double>(kl), obj, ratio, clo ? 1ll : 0ll, chi ? 1ll : 0ll, 1ll};
}

// k_merge: persistent over 32-row blocks (grid = resident CTAs, row block rb =
// blockIdx.x, + gridDim.x, ...; every row block's results and stats depend
// only on rb, so the grid size does not change them). Per row block:
//  * fold phase, 8 warps, warp w a contiguous 1/8 of the n_vt partials.
//    Row-blocked layout (this call's own partials): lane l loads float4s --
//    rows 4(l&7)..+3 of partial n0 + (l>>3) + 4k -- so one warp instruction
//    moves 512 contiguous bytes, two k-steps (6 x 16 B) in flight per lane,
//    one rescale per batch; the 4 lanes holding the same rows then combine in
//    a fixed xor-8 / xor-16 order. Strided layout (gathered vocab-parallel
//    parts, few partials): lane = row, scalar loads.
//  * warp 0, lane = row: fold the 8 warps' results in warp order (fixed,
//    deterministic), then logp / entropy / lse and the per-row loss.
constexpr int MERGE_KB = 2;

template <bool LOSS>
__global__ void __launch_bounds__(MERGE_THREADS, 4)
k_merge(MergeArgs a, const WsHeader* __restrict__ hdr, int64_t ldp, int64_t nblk) {
  __shared__ float sh_m[MERGE_SPLIT][MERGE_ROWS], sh_s[MERGE_SPLIT][MERGE_ROWS],
      sh_u[MERGE_SPLIT][MERGE_ROWS];
  const int64_t T = hdr->n_active;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t n_vt = a.nparts, pst = a.part_stride;
  const int64_t per = (n_vt + MERGE_SPLIT - 1) / MERGE_SPLIT;
  const int64_t n0 = wid * per, n1 = n0 + per < n_vt ? n0 + per : n_vt;
  for (int64_t rb = blockIdx.x; rb < nblk; rb += gridDim.x) {
    const int64_t r = rb * MERGE_ROWS + lane;
    if (rb * MERGE_ROWS < T) {
      if (pst == 0) {
        const int q = lane & 7, sub = lane >> 3;
        const float4* pm4 = reinterpret_cast<const float4*>(a.pm);
        const float4* ps4 = reinterpret_cast<const float4*>(a.ps);
        const float4* pu4 = reinterpret_cast<const float4*>(a.pu);
        const int64_t b4 = rb * n_vt * 8 + q;        // float4 index of (rb, n = 0, rows 4q..)
        float M[4], S[4], U[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          M[j] = -INFINITY;
          S[j] = 0.f;
          U[j] = 0.f;
        }
        for (int64_t n = n0 + sub; n < n1; n += 4 * MERGE_KB) {
          float4 m4[MERGE_KB], s4[MERGE_KB], u4[MERGE_KB];
          bool ok[MERGE_KB];
#pragma unroll
          for (int k = 0; k < MERGE_KB; ++k) {   // loads unconditional (index clamped)
            const int64_t nk = n + 4 * k;
            ok[k] = nk < n1;
            const int64_t o = b4 + (ok[k] ? nk : n1 - 1) * 8;
            m4[k] = __ldcs(pm4 + o);
            s4[k] = __ldcs(ps4 + o);
            u4[k] = __ldcs(pu4 + o);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float mj[MERGE_KB], sj[MERGE_KB], uj[MERGE_KB];
#pragma unroll
            for (int k = 0; k < MERGE_KB; ++k) {
              const float mm = j == 0 ? m4[k].x : j == 1 ? m4[k].y : j == 2 ? m4[k].z : m4[k].w;
              mj[k] = ok[k] ? mm : -INFINITY;
              sj[k] = j == 0 ? s4[k].x : j == 1 ? s4[k].y : j == 2 ? s4[k].z : s4[k].w;
              uj[k] = j == 0 ? u4[k].x : j == 1 ? u4[k].y : j == 2 ? u4[k].z : u4[k].w;
            }
            lse_fold_batch<MERGE_KB>(M[j], S[j], U[j], mj, sj, uj);
          }
        }
        // the 4 lanes (sub = 0..3) holding rows 4q..4q+3: fixed xor order
#pragma unroll
        for (int o = 8; o <= 16; o <<= 1) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float m = __shfl_xor_sync(0xffffffffu, M[j], o);
            const float sv = __shfl_xor_sync(0xffffffffu, S[j], o);
            const float u = __shfl_xor_sync(0xffffffffu, U[j], o);
            lse_fold_g(M[j], S[j], U[j], m, sv, u);
          }
        }
        if (sub == 0) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            sh_m[wid][4 * q + j] = M[j];
            sh_s[wid][4 * q + j] = S[j];
            sh_u[wid][4 * q + j] = U[j];
          }
        }
      } else {
        float M = -INFINITY, S = 0.f, U = 0.f;
        if (r < T)
          for (int64_t n = n0; n < n1; ++n)
            lse_fold_g(M, S, U, a.pm[n * pst + r], a.ps[n * pst + r], a.pu[n * pst + r]);
        sh_m[wid][lane] = M;
        sh_s[wid][lane] = S;
        sh_u[wid][lane] = U;
      }
    }
    __syncthreads();
    if (wid == 0) {
      LStat st{0.0, 0.0, 0.0, 0.0, 0.0, 0.f, 0, 0, 0};
      if (r < T) {
        float M = -INFINITY, S = 0.f, U = 0.f;
#pragma unroll
        for (int w = 0; w < MERGE_SPLIT; ++w) lse_fold_g(M, S, U, sh_m[w][lane], sh_s[w][lane],
                                                         sh_u[w][lane]);
        if (a.parts_out) {  // vocab-parallel phase 1: this shard's merged partial
          const int64_t yl = static_cast<int64_t>(a.tgt_c[r]) - a.y_off;
          a.parts_out[r] = M;
          a.parts_out[a.ldo + r] = S;
          a.parts_out[2 * a.ldo + r] = U;
          a.parts_out[3 * a.ldo + r] = (yl >= 0 && yl < a.v_shard) ? a.zy[r] : 0.f;
        } else {
          const float logS = logf(S);
          const float lse = M + logS;
          const float ent = logS - U / S;
          const float lp = a.zy[r] - lse;
          const int32_t t = a.active_idx[r];
          if (a.logp) a.logp[t] = lp;
          if (a.entropy) a.entropy[t] = ent;
          if (a.lse) a.lse[t] = lse;
          if constexpr (LOSS) st = row_loss(a, r, t, T, lp, lse, ent);
        }
      } else if (r < ldp) {
        if constexpr (LOSS) {  // padding rows of the last tile: zero gradient coefficients
          a.g_c[r] = 0.f;
          a.lse_c[r] = 0.f;
          if (a.ge_c) {
            a.ge_c[r] = 0.f;
            a.ez_c[r] = 0.f;
          }
        }
      }
      if constexpr (LOSS) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {  // fixed-order butterfly
          LStat w = lstat_shfl(st, o);
          lstat_add(st, w);
        }
        if (lane == 0) {
          a.st_d[5 * rb] = st.loss;
          a.st_d[5 * rb + 1] = st.ratio;
          a.st_d[5 * rb + 2] = st.ent;
          a.st_d[5 * rb + 3] = st.kl;
          a.st_d[5 * rb + 4] = st.obj;
          a.st_f[rb] = st.rmax;
          a.st_i[3 * rb] = st.clo;
          a.st_i[3 * rb + 1] = st.chi;
          a.st_i[3 * rb + 2] = st.tok;
        }
      }
    }
    __syncthreads();   // smem reused by the next row block
  }
}

rl_status launch_merge(const WsLayout& L, char* ws, const MergeArgs& a_in, cudaStream_t s) {
  const WsHeader* hdr = reinterpret_cast<const WsHeader*>(ws + L.off_hdr);
  if (L.nblk_loss == 0) return RL_OK;
  MergeArgs a = a_in;
  if (a.nparts == 0) {  // this call's own split-V partials in the workspace (row-blocked)
    a.nparts = L.n_vt;
    a.part_stride = 0;
  }
  if (a.parts_out && a.old_logp) return RL_ERR_INVALID_ARG;
  // persistent grid: the CTAs that fit at once (no partial second wave)
  static int occ[2] = {0, 0};
  static std::once_flag once;
  std::call_once(once, [] {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[0], k_merge<false>, MERGE_THREADS, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[1], k_merge<true>, MERGE_THREADS, 0);
  });
  const int64_t resident =
      static_cast<int64_t>(std::max(1, occ[a.old_logp ? 1 : 0])) * num_sms();
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(L.nblk_loss, resident));
  TraceScope ts(RL_K_MERGE, s);
  if (a.old_logp)
    k_merge<true><<<grid, MERGE_THREADS, 0, s>>>(a, hdr, L.Rp, L.nblk_loss);
  else
    k_merge<false><<<grid, MERGE_THREADS, 0, s>>>(a, hdr, L.Rp, L.nblk_loss);
  RLH_CHECK_LAUNCH();
  return RL_OK;
}

__global__ void __launch_bounds__(MERGE_THREADS)
k_zy_combine(const float* __restrict__ parts_all, int64_t nparts, int64_t ldr,
             const WsHeader* __restrict__ hdr, float* __restrict__ zy) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * MERGE_THREADS + threadIdx.x;
  if (r >= hdr->n_active) return;
  float acc = 0.f;  // one shard holds z_y, the others contribute exact zeros
  for (int64_t p = 0; p < nparts; ++p) acc += parts_all[(4 * p + 3) * ldr + r];
  zy[r] = acc;
}

rl_status launch_zy_combine(const float* parts_all, int64_t nparts, int64_t ldr,
                            const WsLayout& L, char* ws, cudaStream_t s) {
  if (L.nblk_loss == 0) return RL_OK;
  TraceScope ts(RL_K_MERGE, s);
  k_zy_combine<<<static_cast<unsigned>(ceil_div(L.Rp, MERGE_THREADS)), MERGE_THREADS, 0, s>>>(
      parts_all, nparts, ldr, reinterpret_cast<const WsHeader*>(ws + L.off_hdr),
      reinterpret_cast<float*>(ws + L.off_zy));
  RLH_CHECK_LAUNCH();
  return RL_OK;
}

__global__ void __launch_bounds__(MERGE_THREADS)
k_stats_reduce(const double* __restrict__ st_d, const float* __restrict__ st_f,
               const long long* __restrict__ st_i, int64_t nblk, rl_loss_stats* out) {
  LStat v{0.0, 0.0, 0.0, 0.0, 0.0, 0.f, 0, 0, 0};
  for (int64_t b = threadIdx.x; b < nblk; b += MERGE_THREADS) {
    LStat w{st_d[5 * b],     st_d[5 * b + 1], st_d[5 * b + 2], st_d[5 * b + 3],
            st_d[5 * b + 4], st_f[b],         st_i[3 * b],     st_i[3 * b + 1],
            st_i[3 * b + 2]};
    lstat_add(v, w);
  }
  v = block_reduce_lstat<MERGE_THREADS>(v);
  if (threadIdx.x == 0) {
    out->loss_sum += v.loss;
    out->ratio_sum += v.ratio;
    out->entropy_sum += v.ent;
    out->kl_sum += v.kl;
    out->objective += v.obj;
    out->ratio_max = fmaxf(out->ratio_max, v.rmax);
    out->clip_lo_count += v.clo;
    out->clip_hi_count += v.chi;
    out->tokens += v.tok;
  }
}

// C4 of the DP step: combine the ranks' gathered stats in rank order.
__global__ void k_stats_ranks(const rl_loss_stats* __restrict__ g, int32_t n,
                              rl_loss_stats* __restrict__ out) {
  rl_loss_stats t = g[0];
  for (int32_t q = 1; q < n; ++q) {
    const rl_loss_stats& v = g[q];
    t.loss_sum += v.loss_sum;
    t.ratio_sum += v.ratio_sum;
    t.entropy_sum += v.entropy_sum;
    t.kl_sum += v.kl_sum;
    t.objective += v.objective;
    t.ratio_max = fmaxf(t.ratio_max, v.ratio_max);
    t.clip_lo_count += v.clip_lo_count;
    t.clip_hi_count += v.clip_hi_count;
    t.tokens += v.tokens;
  }
  *out = t;
}

rl_status launch_stats_ranks(const rl_loss_stats* gathered, int32_t n, rl_loss_stats* out,
                             cudaStream_t s) {
  TraceScope ts(RL_K_REDUCE, s);
  k_stats_ranks<<<1, 1, 0, s>>>(gathered, n, out);
  RLH_CHECK_LAUNCH();
  return RL_OK;
}

rl_status launch_stats_reduce(const WsLayout& L, char* ws, rl_loss_stats* stats, cudaStream_t s) {
  if (!stats || L.nblk_loss == 0) return RL_OK;
  TraceScope ts(RL_K_REDUCE, s);
  k_stats_reduce<<<1, MERGE_THREADS, 0, s>>>(reinterpret_cast<const double*>(ws + L.off_st_d),
                                            reinterpret_cast<const float*>(ws + L.off_st_f),
                                            reinterpret_cast<const long long*>(ws + L.off_st_i),
                                            L.nblk_loss, stats);
  RLH_CHECK_LAUNCH();
  return RL_OK;
}

}  // namespace rlh
