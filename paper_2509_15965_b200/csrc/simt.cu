// CUDA-core (SIMT) path of the head: exact fp32 FFMA arithmetic for fp32
// inputs (the tiny config, BASELINE.json configs[0], |dlogp| <= 1e-5; tcgen05
// has no exact-fp32 kind) and a bf16 cross-check path. Same outputs and
// workspace contract as the tensor-core path: it writes one split-V partial
// per row (n_vt = 1) that the shared merge/loss kernel consumes.
//   fwd: one CTA per active row, z_v = tau^-1 <h_t, W_v> in fp32, online
//        (max, sum e^{z-m}, sum e^{z-m}(z-m)) per thread, fixed-order merge.
//   bwd: dZ = tau^-1 g (onehot - p) into an fp32 workspace (logits
//        recomputed with the identical FMA order), then two tiled SIMT GEMMs
//        dH = dZ W (rows scattered to grad_hidden) and dW += dZ^T H.
#include "kernels.h"

namespace rlh {

constexpr int SIMT_THREADS = 256;

__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

// tau^-1 <h, W_v>, k ascending (the fwd and bwd recompute share it).
template <typename T>
__device__ __forceinline__ float simt_logit(const float* __restrict__ hs,
                                            const T* __restrict__ wrow, int h, float inv_temp) {
  float acc = 0.f;
  for (int k = 0; k < h; ++k) acc = fmaf(hs[k], to_f(wrow[k]), acc);
  return acc * inv_temp;
}

struct MSU {
  float m, s, u;
};
// Merge two (max, sum e^{z-m}, sum e^{z-m}(z-m)) triples.
__device__ __forceinline__ MSU msu_merge(MSU a, MSU b) {
  if (b.m > a.m) { MSU t = a; a = b; b = t; }
  if (b.s == 0.f) return a;
  const float f = expf(b.m - a.m);
  return {a.m, a.s + f * b.s, a.u + f * (b.u + (b.m - a.m) * b.s)};
}

template <typename T>
__global__ void __launch_bounds__(SIMT_THREADS)
k_simt_fwd(const T* __restrict__ hidden, int64_t ld, const T* __restrict__ W, int h, int V,
           float inv_temp, int64_t y_off, const int32_t* __restrict__ active_idx,
           const int32_t* __restrict__ tgt_c, const WsHeader* __restrict__ hdr,
           float* __restrict__ pm, float* __restrict__ ps, float* __restrict__ pu,
           float* __restrict__ zy) {
  extern __shared__ float hs[];
  __shared__ MSU red[SIMT_THREADS];
  const int64_t T_ = hdr->n_active;
  for (int64_t r = blockIdx.x; r < T_; r += gridDim.x) {
    const T* hrow = hidden + static_cast<int64_t>(active_idx[r]) * ld;
    for (int k = threadIdx.x; k < h; k += SIMT_THREADS) hs[k] = to_f(hrow[k]);
    __syncthreads();
    const int64_t y = static_cast<int64_t>(tgt_c[r]) - y_off;  // local id in this shard
    MSU acc{-INFINITY, 0.f, 0.f};
    for (int v = threadIdx.x; v < V; v += SIMT_THREADS) {
      const float z = simt_logit(hs, W + static_cast<int64_t>(v) * h, h, inv_temp);
      if (v == y) zy[r] = z;
      acc = msu_merge(acc, MSU{z, 1.f, 0.f});
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int o = SIMT_THREADS / 2; o > 0; o >>= 1) {
      if (threadIdx.x < o) red[threadIdx.x] = msu_merge(red[threadIdx.x], red[threadIdx.x + o]);
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      pm[r] = red[0].m;
      ps[r] = red[0].s;
      pu[r] = red[0].u;
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void __launch_bounds__(SIMT_THREADS)
k_simt_dz(const T* __restrict__ hidden, int64_t ld, const T* __restrict__ W, int h, int V,
          float inv_temp, int64_t y_off, const int32_t* __restrict__ active_idx,
          const int32_t* __restrict__ tgt_c, const WsHeader* __restrict__ hdr,
          const float* __restrict__ lse_c, const float* __restrict__ g_c,
          const float* __restrict__ ge_c, const float* __restrict__ ez_c,
          float* __restrict__ dz) {
  extern __shared__ float hs[];
  const int64_t T_ = hdr->n_active;
  for (int64_t r = blockIdx.x; r < T_; r += gridDim.x) {
    const T* hrow = hidden + static_cast<int64_t>(active_idx[r]) * ld;
    for (int k = threadIdx.x; k < h; k += SIMT_THREADS) hs[k] = to_f(hrow[k]);
    __syncthreads();
    const int64_t y = static_cast<int64_t>(tgt_c[r]) - y_off;  // local id in this shard
    const float lse = lse_c[r], coef = g_c[r] * inv_temp;
    const float cent = ge_c ? ge_c[r] * inv_temp : 0.f, ez = ge_c ? ez_c[r] : 0.f;
    for (int v = threadIdx.x; v < V; v += SIMT_THREADS) {
      const float z = simt_logit(hs, W + static_cast<int64_t>(v) * h, h, inv_temp);
      const float p = expf(z - lse);
      // g (onehot - p) + w c_ent p (z - E_p z)  (entropy bonus; 0 when off)
      dz[r * V + v] = coef * ((v == y ? 1.f : 0.f) - p) + cent * p * (z - ez);
    }
    __syncthreads();
  }
}

// C[m, n] (=|+=) sum_k A(m,k) B(k,n); 64x64 tile, 16 k per step, 4x4 per
// thread, k ascending (deterministic).
template <class LA, class LB, class ST>
__global__ void __launch_bounds__(SIMT_THREADS)
k_simt_gemm(int64_t M_bound, int N, int64_t K_fixed, int m_is_T, int k_is_T,
            const WsHeader* __restrict__ hdr, LA la, LB lb, ST st) {
  __shared__ float As[16][64 + 4];
  __shared__ float Bs[16][64 + 4];
  const int64_t T_ = hdr->n_active;
  const int64_t M = m_is_T ? T_ : M_bound;
  const int64_t K = k_is_T ? T_ : K_fixed;
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * 64;
  const int n0 = blockIdx.x * 64;
  if (m0 >= M) return;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4] = {};
  for (int64_t k0 = 0; k0 < K; k0 += 16) {
    for (int i = threadIdx.x; i < 16 * 64; i += SIMT_THREADS) {
      const int kk = i / 64, mm = i % 64;
      const int64_t m = m0 + mm, k = k0 + kk;
      As[kk][mm] = (m < M && k < K) ? la(m, k) : 0.f;
      const int n = n0 + mm;
      Bs[kk][mm] = (n < N && k < K) ? lb(k, n) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(As[kk][ty * 4 + i], Bs[kk][tx * 4 + j], acc[i][j]);
    }
    __syncthreads();
  }
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      const int64_t m = m0 + ty * 4 + i;
      const int n = n0 + tx * 4 + j;
      if (m < M && n < N) st(m, n, acc[i][j]);
    }
}

// dH: A(r, v) = dZ[r, v], B(v, n) = W[v, n], C row r -> grad_hidden[active_idx[r]].
struct LA_dz_rows {
  const float* dz; int64_t V;
  __device__ float operator()(int64_t r, int64_t v) const { return dz[r * V + v]; }
};
template <typename T> struct LB_w {
  const T* W; int h;
  __device__ float operator()(int64_t v, int n) const { return to_f(W[v * h + n]); }
};
template <typename T> struct ST_rows {
  T* out; int64_t ld; const int32_t* idx;
  __device__ void operator()(int64_t r, int n, float x) const {
    out[static_cast<int64_t>(idx[r]) * ld + n] = from_f<T>(x);
  }
};
// dW: A(v, r) = dZ[r, v], B(r, n) = hidden[active_idx[r], n], C += into dW.
struct LA_dz_cols {
  const float* dz; int64_t V;
  __device__ float operator()(int64_t v, int64_t r) const { return dz[r * V + v]; }
};
template <typename T> struct LB_hid {
  const T* H; int64_t ld; const int32_t* idx;
  __device__ float operator()(int64_t r, int n) const {
    return to_f(H[static_cast<int64_t>(idx[r]) * ld + n]);
  }
};
struct ST_acc {
  float* dW; int h;
  __device__ void operator()(int64_t v, int n, float x) const { dW[v * h + n] += x; }
};

template <typename T>
static rl_status simt_fwd_t(const rl_head* hd, const void* hidden, const void* weight,
                            const WsLayout& L, char* ws, cudaStream_t s) {
  const WsHeader* hdr = reinterpret_cast<const WsHeader*>(ws + L.off_hdr);
  const int blocks = static_cast<int>(L.R < 8192 ? (L.R > 0 ? L.R : 1) : 8192);
  const size_t smem = static_cast<size_t>(hd->hidden) * sizeof(float);
  if (smem > 48 * 1024) {
    if (cudaFuncSetAttribute(k_simt_fwd<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem)) != cudaSuccess)
      return RL_ERR_CUDA;
  }
  TraceScope ts(RL_K_SIMT_FWD, s);
  k_simt_fwd<T><<<blocks, SIMT_THREADS, smem, s>>>(
      static_cast<const T*>(hidden), hd->ld_hidden, static_cast<const T*>(weight), hd->hidden,
      hd->vocab, hd->inv_temperature, hd->vocab_total > 0 ? hd->vocab_offset : 0,
      reinterpret_cast<const int32_t*>(ws + L.off_active),
      reinterpret_cast<const int32_t*>(ws + L.off_tgt), hdr,
      reinterpret_cast<float*>(ws + L.off_pm), reinterpret_cast<float*>(ws + L.off_ps),
      reinterpret_cast<float*>(ws + L.off_pu), reinterpret_cast<float*>(ws + L.off_zy));
  RLH_CHECK_LAUNCH();
  return RL_OK;
}

template <typename T>
static rl_status simt_bwd_t(const rl_head* hd, const void* hidden, const void* weight,
                            void* grad_hidden, float* grad_weight, bool entropy_on,
                            const WsLayout& L, char* ws, cudaStream_t s) {
  const WsHeader* hdr = reinterpret_cast<const WsHeader*>(ws + L.off_hdr);
  const int32_t* active_idx = reinterpret_cast<const int32_t*>(ws + L.off_active);
  float* dz = reinterpret_cast<float*>(ws + L.off_dz);
  const int h = hd->hidden, V = hd->vocab;
  const int blocks = static_cast<int>(L.R < 8192 ? (L.R > 0 ? L.R : 1) : 8192);
  const size_t smem = static_cast<size_t>(h) * sizeof(float);
  if (smem > 48 * 1024) {
    if (cudaFuncSetAttribute(k_simt_dz<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem)) != cudaSuccess)
      return RL_ERR_CUDA;
  }
  {
    TraceScope ts(RL_K_SIMT_BWD, s);
    k_simt_dz<T><<<blocks, SIMT_THREADS, smem, s>>>(
        static_cast<const T*>(hidden), hd->ld_hidden, static_cast<const T*>(weight), h, V,
        hd->inv_temperature, hd->vocab_total > 0 ? hd->vocab_offset : 0, active_idx,
        reinterpret_cast<const int32_t*>(ws + L.off_tgt), hdr,
        reinterpret_cast<const float*>(ws + L.off_lse), reinterpret_cast<const float*>(ws + L.off_g),
        entropy_on ? reinterpret_cast<const float*>(ws + L.off_ge) : nullptr,
        entropy_on ? reinterpret_cast<const float*>(ws + L.off_ez) : nullptr, dz);
  }
  RLH_CHECK_LAUNCH();
  {
    dim3 grid(static_cast<unsigned>(ceil_div(h, 64)), static_cast<unsigned>(ceil_div(L.R, 64)));
    if (grid.y > 0) {
      TraceScope ts(RL_K_SIMT_BWD, s);
      k_simt_gemm<<<grid, SIMT_THREADS, 0, s>>>(
          L.R, h, static_cast<int64_t>(V), 1, 0, hdr, LA_dz_rows{dz, V},
          LB_w<T>{static_cast<const T*>(weight), h},
          ST_rows<T>{static_cast<T*>(grad_hidden), hd->ld_hidden, active_idx});
    }
  }
  RLH_CHECK_LAUNCH();
  {
    dim3 grid(static_cast<unsigned>(ceil_div(h, 64)), static_cast<unsigned>(ceil_div(V, 64)));
    TraceScope ts(RL_K_SIMT_BWD, s);
    k_simt_gemm<<<grid, SIMT_THREADS, 0, s>>>(
        static_cast<int64_t>(V), h, 0, 0, 1, hdr, LA_dz_cols{dz, V},
        LB_hid<T>{static_cast<const T*>(hidden), hd->ld_hidden, active_idx},
        ST_acc{grad_weight, h});
  }
  RLH_CHECK_LAUNCH();
  return RL_OK;
}

rl_status launch_simt_fwd(const rl_head* hd, const void* hidden, const void* weight,
                          const WsLayout& L, char* ws, cudaStream_t s) {
  return hd->dtype == RL_F32 ? simt_fwd_t<float>(hd, hidden, weight, L, ws, s)
                             : simt_fwd_t<__nv_bfloat16>(hd, hidden, weight, L, ws, s);
}
rl_status launch_simt_bwd(const rl_head* hd, const void* hidden, const void* weight,
                          void* grad_hidden, float* grad_weight, bool entropy_on,
                          const WsLayout& L, char* ws, cudaStream_t s) {
  return hd->dtype == RL_F32
             ? simt_bwd_t<float>(hd, hidden, weight, grad_hidden, grad_weight, entropy_on, L, ws,
                                 s)
             : simt_bwd_t<__nv_bfloat16>(hd, hidden, weight, grad_hidden, grad_weight, entropy_on,
                                         L, ws, s);
}

}  // namespace rlh
