// H2: GRPO group-relative advantage ("normalization must
// aggregate all responses for a query"; readings DESIGN.md §3
// #5-#8). k_grpo_seg (below): one pass, segmented by group id with warp
// match/fold steps, fixed summation order (deterministic, fp64); k_grpo (one
// CTA per group, each scanning all sequences) only when the groups' shared-
// memory accumulators would not fit. With given (all-reduced) statistics the
// scan is skipped and only the per-member normalisation runs.
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

// Segmented form (default while the per-warp accumulators fit in shared
// memory, G <= GSEG_MAX_G): ONE pass over the sequences. Warp w owns the
// contiguous chunk [w S/8, (w+1) S/8) and walks it 32 sequences at a time:
// a warp-shuffle SEGMENTED inclusive scan over the runs of equal group id
// (5 shuffle rounds; a GRPO group's responses are adjacent in a packed batch,
// so a step holds 1-3 runs) leaves each run's (n, sum r, sum r^2, max, -min)
// in its last lane, which adds it into the warp's shared-memory accumulator
// of that group; tails of the same group in one step (ids not contiguous)
// are folded by the lowest such lane in lane order. Thread g then folds the
// warps' accumulators of group g in warp order and the normalisation pass
// writes A. 32 warps (a few serial steps each: the kernel is latency-bound)
// while 32 x G accumulators fit in shared memory (G <= 140), else 8 warps.
// O(S + warps G) work, fixed combination order (deterministic run to run),
// 12 B of HBM per sequence.
constexpr int GSEG_MAX_G = 512;          // 8 warps x 512 groups of accumulators
constexpr int GSEG_WIDE_MAX_G = 140;     // 32 warps (fewer serial steps) up to this G

__device__ __forceinline__ GStat gstat_shfl_up(const GStat& v, int d) {
  return {__shfl_up_sync(0xffffffffu, v.n, d), __shfl_up_sync(0xffffffffu, v.s1, d),
          __shfl_up_sync(0xffffffffu, v.s2, d), __shfl_up_sync(0xffffffffu, v.mx, d),
          __shfl_up_sync(0xffffffffu, v.nmn, d)};
}

template <int GSEG_WARPS>
__global__ void __launch_bounds__(GSEG_WARPS * 32)
k_grpo_seg(const float* __restrict__ r, const int32_t* __restrict__ gos, int32_t S, int32_t G,
           const double* __restrict__ sum_in, const double* __restrict__ max_in, float eps,
           int32_t unbiased, float* __restrict__ adv, double* __restrict__ sum_out,
           double* __restrict__ max_out, int32_t* err) {
  extern __shared__ double gsm[];
  GStat* acc = reinterpret_cast<GStat*>(gsm);                          // [GSEG_WARPS][G]
  GStat* stg = acc + static_cast<int64_t>(GSEG_WARPS) * G;             // [GSEG_WARPS][32]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int bad = 0;
  if (!sum_in) {
    for (int k = threadIdx.x; k < GSEG_WARPS * G; k += (GSEG_WARPS * 32))
      acc[k] = GStat{0.0, 0.0, 0.0, -INFINITY, -INFINITY};
    __syncthreads();
    const int per = ((S + GSEG_WARPS - 1) / GSEG_WARPS + 31) & ~31;
    const int i0 = w * per, i1 = min(S, i0 + per);
    GStat* my = acc + static_cast<int64_t>(w) * G;
    GStat* st = stg + w * 32;
    constexpr int U = 2;  // steps whose loads are issued together (code size: one cold CTA)
    for (int b0 = i0; b0 < i1; b0 += 32 * U) {
      int32_t gk[U];
      float rk[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int i = b0 + 32 * k + lane;
        gk[k] = i < i1 ? gos[i] : -1;
        rk[k] = i < i1 ? r[i] : 0.f;
      }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      if (b0 + 32 * k >= i1) break;      // warp-uniform
      const int i = b0 + 32 * k + lane;
      int key = -1 - lane;               // invalid / past the end: a run of its own
      GStat v{0.0, 0.0, 0.0, -INFINITY, -INFINITY};
      if (i < i1) {
        const int32_t g = gk[k];
        if (g >= 0 && g < G) {
          key = g;
          const double x = static_cast<double>(rk[k]);
          v = GStat{1.0, x, x * x, x, -x};
        } else {
          bad = 1;
        }
      }
      const int kprev = __shfl_up_sync(0xffffffffu, key, 1);
      const int knext = __shfl_down_sync(0xffffffffu, key, 1);
      int f = (lane == 0 || kprev != key) ? 1 : 0;      // run head
      const bool tail = lane == 31 || knext != key;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {                // segmented inclusive scan
        const GStat pv = gstat_shfl_up(v, d);
        const int pf = __shfl_up_sync(0xffffffffu, f, d);
        if (lane >= d) {
          if (!f) v = gstat_combine(pv, v);
          f |= pf;
        }
      }
      st[lane] = v;
      const int tkey = (tail && key >= 0) ? key : -1 - lane;
      const uint32_t peers = __match_any_sync(0xffffffffu, tkey);
      __syncwarp();
      if (tkey >= 0 && lane == __ffs(peers) - 1) {
        GStat t = my[key];
        for (uint32_t m = peers; m; m &= m - 1) t = gstat_combine(t, st[__ffs(m) - 1]);
        my[key] = t;
      }
      __syncwarp();
    }
    }
  } else {
    for (int i = threadIdx.x; i < S; i += (GSEG_WARPS * 32)) {
      const int32_t g = gos[i];
      if (g < 0 || g >= G) bad = 1;
    }
  }
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0 && bad && err) atomicOr(err, RL_DEVERR_GROUP);
  // per group: fold the warps in order; keep (mu, sigma + eps, degenerate) in slot g
  for (int g = threadIdx.x; g < G; g += (GSEG_WARPS * 32)) {
    GStat t;
    if (sum_in) {
      t = {sum_in[3 * g], sum_in[3 * g + 1], sum_in[3 * g + 2], max_in[2 * g], max_in[2 * g + 1]};
    } else {
      t = acc[g];
      for (int k = 1; k < GSEG_WARPS; ++k)
        t = gstat_combine(t, acc[static_cast<int64_t>(k) * G + g]);
    }
    if (sum_out) {
      sum_out[3 * g] = t.n;
      sum_out[3 * g + 1] = t.s1;
      sum_out[3 * g + 2] = t.s2;
      max_out[2 * g] = t.mx;
      max_out[2 * g + 1] = t.nmn;
    }
    // A = 0 exactly for singleton / zero-variance groups (reading #8).
    const bool degenerate = (t.n <= 1.0) || (t.mx == -t.nmn);
    const double mu = t.n > 0 ? t.s1 / t.n : 0.0;
    double var = t.s2 - t.n * mu * mu;
    var = var > 0.0 ? var : 0.0;
    var /= unbiased ? (t.n - 1.0) : t.n;
    acc[g] = GStat{mu, sqrt(var) + static_cast<double>(eps), degenerate ? 1.0 : 0.0, 0.0, 0.0};
  }
  if (!adv) return;
  __syncthreads();
  for (int i = threadIdx.x; i < S; i += (GSEG_WARPS * 32)) {
    const int32_t g = gos[i];
    float a = 0.f;
    if (g >= 0 && g < G) {
      const GStat t = acc[g];
      if (t.s2 == 0.0) a = static_cast<float>((static_cast<double>(r[i]) - t.n) / t.s1);
    }
    adv[i] = a;
  }
}

static size_t grpo_seg_smem(int32_t G, int warps) {
  return (static_cast<size_t>(warps) * G + warps * 32) * sizeof(GStat);
}

rl_status launch_grpo(const float* rewards, const int32_t* gos, int32_t S, int32_t G,
                      const double* sum_in, const double* max_in, float eps, int32_t unbiased,
                      float* adv, double* sum_out, double* max_out, int32_t* err,
                      cudaStream_t s) {
  if (G <= 0 && S <= 0) return RL_OK;
  TraceScope ts(RL_K_GRPO, s);
  if (G >= 1 && G <= GSEG_MAX_G) {
    static const cudaError_t attr8 = cudaFuncSetAttribute(
        k_grpo_seg<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
        static_cast<int>(grpo_seg_smem(GSEG_MAX_G, 8)));
    static const cudaError_t attr32 = cudaFuncSetAttribute(
        k_grpo_seg<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
        static_cast<int>(grpo_seg_smem(GSEG_WIDE_MAX_G, 32)));
    if (G <= GSEG_WIDE_MAX_G ? attr32 != cudaSuccess : attr8 != cudaSuccess) return RL_ERR_CUDA;
    if (G <= GSEG_WIDE_MAX_G)
      k_grpo_seg<32><<<1, 32 * 32, grpo_seg_smem(G, 32), s>>>(rewards, gos, S, G, sum_in, max_in,
                                                             eps, unbiased, adv, sum_out, max_out,
                                                             err);
    else
      k_grpo_seg<8><<<1, 8 * 32, grpo_seg_smem(G, 8), s>>>(rewards, gos, S, G, sum_in, max_in, eps,
                                                          unbiased, adv, sum_out, max_out, err);
  } else {
    // many groups: one CTA per group (each scans all S; G x S work)
    k_grpo<<<G + 1, GRPO_THREADS, 0, s>>>(rewards, gos, S, G, sum_in, max_in, eps, unbiased, adv,
                                         sum_out, max_out, err);
  }
  RLH_CHECK_LAUNCH();
  return RL_OK;
}

// NEXT-1, REINFORCE++-style batch normalisation (DESIGN.md §3 #33):
// x_s = r_s - mu_g(s) (group baseline, mu from the given group sums) or r_s;
// A_s = (x_s - mean_B x) / (std_B x + eps) over the valid sequences. One CTA:
// each thread accumulates its strided members in index order, then the fixed-
// order block reduction above (deterministic fp64). bin != NULL: the batch
// statistics (n, sum x, sum x^2, max x, -min x) were all-reduced by the
// caller; bout != NULL: write this call's local ones.
__device__ __forceinline__ bool bn_x(const float* r, const int32_t* gos, int32_t G, int32_t gb,
                                     const double* gsum, int i, double* x) {
  double v = static_cast<double>(r[i]);
  if (gos) {
    const int32_t g = gos[i];
    if (g < 0 || g >= G) return false;
    if (gb) {
      const double n = gsum[3 * g];
      v = n > 0.0 ? v - gsum[3 * g + 1] / n : 0.0;
    }
  }
  *x = v;
  return true;
}

__global__ void __launch_bounds__(GRPO_THREADS)
k_batch_adv(const float* __restrict__ r, const int32_t* __restrict__ gos, int32_t S, int32_t G,
            int32_t gb, const double* __restrict__ gsum, const double* __restrict__ bin,
            double* __restrict__ bout, float eps, int32_t unbiased, float* __restrict__ adv,
            int32_t* err) {
  GStat st;
  int bad = 0;
  if (!bin || bout) {
    GStat v{0.0, 0.0, 0.0, -INFINITY, -INFINITY};
    for (int i = threadIdx.x; i < S; i += GRPO_THREADS) {
      double x;
      if (!bn_x(r, gos, G, gb, gsum, i, &x)) {
        bad = 1;
        continue;
      }
      v.n += 1.0;
      v.s1 += x;
      v.s2 += x * x;
      v.mx = fmax(v.mx, x);
      v.nmn = fmax(v.nmn, -x);
    }
    st = block_reduce_gstat(v);
  }
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0 && bad && err) atomicOr(err, RL_DEVERR_GROUP);
  if (bout && threadIdx.x == 0) {
    bout[0] = st.n;
    bout[1] = st.s1;
    bout[2] = st.s2;
    bout[3] = st.mx;
    bout[4] = st.nmn;
  }
  if (!adv) return;
  if (bin) st = {bin[0], bin[1], bin[2], bin[3], bin[4]};
  const bool degenerate = (st.n <= 1.0) || (st.mx == -st.nmn);
  const double mu = st.n > 0 ? st.s1 / st.n : 0.0;
  double var = st.s2 - st.n * mu * mu;
  var = var > 0.0 ? var : 0.0;
  var /= unbiased ? (st.n - 1.0) : st.n;
  const double denom = sqrt(var) + static_cast<double>(eps);
  for (int i = threadIdx.x; i < S; i += GRPO_THREADS) {
    double x;
    const bool ok = bn_x(r, gos, G, gb, gsum, i, &x);
    adv[i] = (!ok || degenerate) ? 0.f : static_cast<float>((x - mu) / denom);
  }
}

rl_status launch_batch_adv(const float* rewards, const int32_t* gos, int32_t S, int32_t G,
                           int32_t group_baseline, const double* gsum, const double* bin,
                           double* bout, float eps, int32_t unbiased, float* adv, int32_t* err,
                           cudaStream_t s) {
  TraceScope ts(RL_K_GRPO, s);
  k_batch_adv<<<1, GRPO_THREADS, 0, s>>>(rewards, gos, S, G, group_baseline, gsum, bin, bout, eps,
                                         unbiased, adv, err);
  RLH_CHECK_LAUNCH();
  return RL_OK;
}

}  // namespace rlh
