// NEXT-4: PPO pieces for the embodied / RLHF workflows (PAPER.md P:L184,
// P:L836): generalised advantage estimation over packed trajectories, and the
// value head (v = <w_v, h> + b_v) with the clipped value loss and its
// backward (DESIGN.md §3 #30-#32; oracle/ppo.py).
//  * k_gae: one thread per trajectory, the reverse recurrence in fp64
//    (latency-bound: 256 trajectories x 448 steps is microseconds).
//  * k_value_loss: 8 warps per 64-row block; warp-per-row dot products with
//    16-B loads, per-row clipped loss and dL/dv, dL/dh += g w (accumulated
//    into the policy's grad_hidden), then a fixed-order per-block partial of
//    dL/dw; k_value_reduce sums the partials in block order (deterministic).
#include "kernels.h"

namespace rlh {

constexpr int VAL_THREADS = 256;
constexpr int VAL_ROWS = 64;

__global__ void k_gae(const float* __restrict__ r, const float* __restrict__ v,
                      const uint8_t* __restrict__ dones, const float* __restrict__ boot,
                      const int32_t* __restrict__ cu, int32_t S, float gamma, float lam,
                      float* __restrict__ adv, float* __restrict__ ret) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  const double g = gamma, gl = static_cast<double>(gamma) * lam;
  double next_v = boot ? static_cast<double>(boot[s]) : 0.0, next_a = 0.0;
  for (int t = cu[s + 1] - 1; t >= cu[s]; --t) {
    const double nonterm = (dones && dones[t]) ? 0.0 : 1.0;
    const double vt = v[t];
    const double delta = static_cast<double>(r[t]) + g * nonterm * next_v - vt;
    next_a = delta + gl * nonterm * next_a;
    adv[t] = static_cast<float>(next_a);
    ret[t] = static_cast<float>(next_a + vt);
    next_v = vt;
  }
}

__device__ __forceinline__ float ld_f(const float* p) { return *p; }
__device__ __forceinline__ float ld_f(const __nv_bfloat16* p) { return __bfloat162float(*p); }
__device__ __forceinline__ void add_f(float* p, float x) { *p += x; }
__device__ __forceinline__ void add_f(__nv_bfloat16* p, float x) {
  *p = __float2bfloat16_rn(__bfloat162float(*p) + x);
}

template <typename T>
__global__ void __launch_bounds__(VAL_THREADS)
k_value_loss(const T* __restrict__ hidden, int64_t ld, int h, const T* __restrict__ w,
             float b, const uint8_t* __restrict__ mask, int64_t R,
             const float* __restrict__ returns, const float* __restrict__ old_values,
             float clip_eps, double scale_host, const int64_t* __restrict__ n_global,
             float* __restrict__ values, T* __restrict__ grad_hidden, float* __restrict__ part_dw,
             double* __restrict__ part_st) {
  __shared__ float g_s[VAL_ROWS];
  __shared__ double st_s[VAL_THREADS / 32][3];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * VAL_ROWS;
  double scale = scale_host;
  if (n_global) {
    const long long N = *n_global;
    scale = N > 0 ? 1.0 / static_cast<double>(N) : 0.0;
  }
  double loss_w = 0.0, clip_w = 0.0, tok_w = 0.0;
  for (int i = warp; i < VAL_ROWS; i += VAL_THREADS / 32) {
    const int64_t t = r0 + i;
    float g = 0.f;
    if (t < R && mask[t]) {
      const T* hrow = hidden + t * ld;
      float acc = 0.f;
      for (int k = lane; k < h; k += 32) acc = fmaf(ld_f(hrow + k), ld_f(w + k), acc);
      acc = warp_sum(acc);
      const float v = acc + b;
      const float ret = returns[t], vo = old_values[t];
      const float lo = vo - clip_eps, hi = vo + clip_eps;
      const float vc = fminf(fmaxf(v, lo), hi);
      const float a = (v - ret) * (v - ret), c = (vc - ret) * (vc - ret);
      float dv;
      if (a >= c) {
        dv = v - ret;
      } else {
        dv = (v >= lo && v <= hi) ? vc - ret : 0.f;
        clip_w += (lane == 0) ? 1.0 : 0.0;
      }
      g = static_cast<float>(scale * dv);
      if (lane == 0) {
        values[t] = v;
        loss_w += 0.5 * static_cast<double>(fmaxf(a, c));
        tok_w += 1.0;
      }
      T* grow = grad_hidden + t * ld;
      for (int k = lane; k < h; k += 32) add_f(grow + k, g * ld_f(w + k));
    } else if (t < R && lane == 0) {
      values[t] = 0.f;
    }
    if (lane == 0) g_s[i] = g;
  }
  if (lane == 0) {
    st_s[warp][0] = loss_w;
    st_s[warp][1] = clip_w;
    st_s[warp][2] = tok_w;
  }
  __syncthreads();
  // fixed-order per-block partial of dL/dw = sum_t g_t h_t
  for (int k = threadIdx.x; k < h; k += VAL_THREADS) {
    float acc = 0.f;
    for (int i = 0; i < VAL_ROWS; ++i) {
      const int64_t t = r0 + i;
      if (t < R && g_s[i] != 0.f) acc = fmaf(g_s[i], ld_f(hidden + t * ld + k), acc);
    }
    part_dw[static_cast<int64_t>(blockIdx.x) * h + k] = acc;
  }
  if (threadIdx.x == 0) {
    double l = 0.0, c = 0.0, n = 0.0, gs = 0.0;
    for (int w2 = 0; w2 < VAL_THREADS / 32; ++w2) {
      l += st_s[w2][0];
      c += st_s[w2][1];
      n += st_s[w2][2];
    }
    for (int i = 0; i < VAL_ROWS; ++i) gs += g_s[i];
    part_st[4 * blockIdx.x] = l;
    part_st[4 * blockIdx.x + 1] = gs;
    part_st[4 * blockIdx.x + 2] = c;
    part_st[4 * blockIdx.x + 3] = n;
  }
}

__global__ void __launch_bounds__(VAL_THREADS)
k_value_reduce(const float* __restrict__ part_dw, const double* __restrict__ part_st,
               int64_t nblk, int h, double scale_host, const int64_t* __restrict__ n_global,
               float* __restrict__ grad_w, float* __restrict__ grad_b, rl_loss_stats* stats) {
  const int k = blockIdx.x * VAL_THREADS + threadIdx.x;
  if (k < h) {
    float acc = 0.f;
    for (int64_t b = 0; b < nblk; ++b) acc += part_dw[b * h + k];
    grad_w[k] += acc;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double l = 0.0, gs = 0.0, c = 0.0, n = 0.0;
    for (int64_t b = 0; b < nblk; ++b) {
      l += part_st[4 * b];
      gs += part_st[4 * b + 1];
      c += part_st[4 * b + 2];
      n += part_st[4 * b + 3];
    }
    if (grad_b) *grad_b += static_cast<float>(gs);
    if (stats) {
      double scale = scale_host;
      if (n_global) {
        const long long N = *n_global;
        scale = N > 0 ? 1.0 / static_cast<double>(N) : 0.0;
      }
      stats->loss_sum += l;
      stats->objective += l * scale;
      stats->clip_hi_count += static_cast<long long>(c);
      stats->tokens += static_cast<long long>(n);
    }
  }
}

}  // namespace rlh

using namespace rlh;

extern "C" {

rl_status rl_gae(const float* rewards, const float* values, const uint8_t* dones,
                 const float* bootstrap, const int32_t* cu_steps, int32_t num_traj, float gamma,
                 float lam, float* adv, float* returns, rl_stream_t stream) {
  if (num_traj < 0 || !(gamma >= 0.f) || !(lam >= 0.f) || !cu_steps) return RL_ERR_INVALID_ARG;
  if (num_traj > 0 && (!rewards || !values || !adv || !returns)) return RL_ERR_INVALID_ARG;
  if (num_traj == 0) return RL_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  TraceScope ts(RL_K_MISC, s);
  k_gae<<<static_cast<unsigned>(ceil_div(num_traj, 128)), 128, 0, s>>>(
      rewards, values, dones, bootstrap, cu_steps, num_traj, gamma, lam, adv, returns);
  RLH_CHECK_LAUNCH();
  return RL_OK;
}

size_t rl_value_workspace_size(int32_t hidden, int64_t num_rows) {
  if (hidden < 1 || num_rows < 0) return 0;
  const int64_t nblk = ceil_div(num_rows, VAL_ROWS);
  return static_cast<size_t>(nblk) * hidden * 4 + static_cast<size_t>(nblk) * 4 * 8 + 256;
}

rl_status rl_value_loss_fwd_bwd(const rl_head* hd, const void* hidden, const void* w_v,
                                float b_v, const rl_batch* b, const float* returns,
                                const float* old_values, const rl_value_params* p,
                                float* values, void* grad_hidden, float* grad_w, float* grad_b,
                                rl_loss_stats* stats, void* ws, size_t ws_bytes,
                                rl_stream_t stream) {
  if (!hd || !b || !p || !w_v || !grad_w || hd->hidden < 1 || hd->ld_hidden < hd->hidden ||
      (hd->dtype != RL_F32 && hd->dtype != RL_BF16) || b->num_rows < 0 || !(p->clip_eps >= 0.f))
    return RL_ERR_INVALID_ARG;
  const int64_t R = b->num_rows;
  if (R > 0 && (!hidden || !b->mask || !returns || !old_values || !values || !grad_hidden))
    return RL_ERR_INVALID_ARG;
  if (ws_bytes < rl_value_workspace_size(hd->hidden, R) || (R > 0 && !ws))
    return RL_ERR_WORKSPACE;
  if (R == 0) return RL_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t nblk = ceil_div(R, VAL_ROWS);
  float* part_dw = static_cast<float*>(ws);
  double* part_st = reinterpret_cast<double*>(
      static_cast<char*>(ws) + ((static_cast<size_t>(nblk) * hd->hidden * 4 + 255) & ~size_t(255)));
  {
    TraceScope ts(RL_K_MISC, s);
    if (hd->dtype == RL_BF16)
      k_value_loss<__nv_bfloat16><<<static_cast<unsigned>(nblk), VAL_THREADS, 0, s>>>(
          static_cast<const __nv_bfloat16*>(hidden), hd->ld_hidden, hd->hidden,
          static_cast<const __nv_bfloat16*>(w_v), b_v, b->mask, R, returns, old_values,
          p->clip_eps, p->loss_scale, p->n_tokens_global, values,
          static_cast<__nv_bfloat16*>(grad_hidden), part_dw, part_st);
    else
      k_value_loss<float><<<static_cast<unsigned>(nblk), VAL_THREADS, 0, s>>>(
          static_cast<const float*>(hidden), hd->ld_hidden, hd->hidden,
          static_cast<const float*>(w_v), b_v, b->mask, R, returns, old_values, p->clip_eps,
          p->loss_scale, p->n_tokens_global, values, static_cast<float*>(grad_hidden), part_dw,
          part_st);
  }
  RLH_CHECK_LAUNCH();
  {
    TraceScope ts(RL_K_REDUCE, s);
    k_value_reduce<<<static_cast<unsigned>(ceil_div(hd->hidden, VAL_THREADS)), VAL_THREADS, 0,
                     s>>>(part_dw, part_st, nblk, hd->hidden, p->loss_scale, p->n_tokens_global,
                          grad_w, grad_b, stats);
  }
  RLH_CHECK_LAUNCH();
  return RL_OK;
}

}  // extern "C"
