// H2: GRPO group-relative advantage ("normalization must
// aggregate all responses for a query"; readings DESIGN.md §3
// #5-#8). One CTA per group; each thread accumulates its strided members in
// index order, then a fixed-order warp-shuffle + shared-memory reduction
// (deterministic, fp64). With given (all-reduced) statistics the scan is
// skipped and only the per-member normalisation runs.
#include "kernels.h"

namespace rlh {

constexpr int GRPO_THREADS = 256;

struct GStat {
  double n, s1, s2, mx, nmn;  // count, sum, sum of squares, max, -min
};

__device__ __forceinline__ GStat gstat_combine(GStat a, GStat b) {
  return {a.n + b.n, a.s1 + b.s1, a.s2 + b.s2, fmax(a.mx, b.mx), fmax(a.nmn, b.nmn)};
}

__device__ GStat block_reduce_gstat(GStat v) {
  __shared__ GStat sh[GRPO_THREADS / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    GStat w{__shfl_xor_sync(0xffffffffu, v.n, o), __shfl_xor_sync(0xffffffffu, v.s1, o),
            __shfl_xor_sync(0xffffffffu, v.s2, o), __shfl_xor_sync(0xffffffffu, v.mx, o),
            __shfl_xor_sync(0xffffffffu, v.nmn, o)};
    v = gstat_combine(v, w);
  }
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  GStat t = sh[0];
  for (int w = 1; w < GRPO_THREADS / 32; ++w) t = gstat_combine(t, sh[w]);
  __syncthreads();
  return t;
}

// blockIdx.x < G: group blockIdx.x. blockIdx.x == G: invalid-id sweep.
__global__ void __launch_bounds__(GRPO_THREADS)
k_grpo(const float* __restrict__ r, const int32_t* __restrict__ gos, int32_t S, int32_t G,
       const double* __restrict__ sum_in, const double* __restrict__ max_in, float eps,
       int32_t unbiased, float* __restrict__ adv, double* __restrict__ sum_out,
       double* __restrict__ max_out, int32_t* err) {
  const int g = blockIdx.x;
  if (g == G) {
    int bad = 0;
    for (int i = threadIdx.x; i < S; i += GRPO_THREADS) {
      const int32_t gi = gos[i];
      if (gi < 0 || gi >= G) {
        bad = 1;
        if (adv) adv[i] = 0.f;
      }
    }
    bad = __syncthreads_or(bad);
    if (threadIdx.x == 0 && bad && err) atomicOr(err, RL_DEVERR_GROUP);
    return;
  }
  GStat st;
  if (sum_in) {
    st = {sum_in[3 * g], sum_in[3 * g + 1], sum_in[3 * g + 2], max_in[2 * g], max_in[2 * g + 1]};
  } else {
    GStat v{0.0, 0.0, 0.0, -INFINITY, -INFINITY};
    for (int i = threadIdx.x; i < S; i += GRPO_THREADS) {
      if (gos[i] == g) {
        const double x = static_cast<double>(r[i]);
        v.n += 1.0;
        v.s1 += x;
        v.s2 += x * x;
        v.mx = fmax(v.mx, x);
        v.nmn = fmax(v.nmn, -x);
      }
    }
    st = block_reduce_gstat(v);
  }
  if (sum_out && threadIdx.x == 0) {
    sum_out[3 * g] = st.n;
    sum_out[3 * g + 1] = st.s1;
    sum_out[3 * g + 2] = st.s2;
    max_out[2 * g] = st.mx;
    max_out[2 * g + 1] = st.nmn;
  }
  if (!adv) return;
  // A = 0 exactly for singleton / zero-variance groups (reading #8).
  const bool degenerate = (st.n <= 1.0) || (st.mx == -st.nmn);
  const double mu = st.n > 0 ? st.s1 / st.n : 0.0;
  double var = st.s2 - st.n * mu * mu;
  var = var > 0.0 ? var : 0.0;
  var /= unbiased ? (st.n - 1.0) : st.n;
  const double denom = sqrt(var) + static_cast<double>(eps);
  for (int i = threadIdx.x; i < S; i += GRPO_THREADS) {
    if (gos[i] == g)
      adv[i] = degenerate ? 0.f : static_cast<float>((static_cast<double>(r[i]) - mu) / denom);
  }
}

rl_status launch_grpo(const float* rewards, const int32_t* gos, int32_t S, int32_t G,
                      const double* sum_in, const double* max_in, float eps, int32_t unbiased,
                      float* adv, double* sum_out, double* max_out, int32_t* err,
                      cudaStream_t s) {
  if (G <= 0 && S <= 0) return RL_OK;
  TraceScope ts(RL_K_GRPO, s);
  k_grpo<<<G + 1, GRPO_THREADS, 0, s>>>(rewards, gos, S, G, sum_in, max_in, eps, unbiased, adv,
                                       sum_out, max_out, err);
  RLH_CHECK_LAUNCH();
  return RL_OK;
}

}  // namespace rlh
