// NEXT-2: mini-batch update control, stream-ordered and without host syncs.
//  * rl_minibatch_early_stop: "discard minibatches with too large importance
//    ratio" (DESIGN.md §3 #29). Reads the (all-reduced)
//    loss statistics on the device, writes the decision to a device flag and,
//    when set, zeroes the accumulated dW (the discarded update).
//  * rl_scale_by_inverse_count: x *= 1/N with N read on the device -- the
//    deferred token-mean normalisation of streaming (elastic-pipelining,
//    P:L433-436) micro-batches that ran with loss_scale = 1.
// Both are HBM-bound grid-stride kernels over 16-B vectors.
#include "kernels.h"

namespace rlh {

constexpr int UPD_THREADS = 256;

__global__ void k_early_stop_decide(const rl_loss_stats* __restrict__ st, float max_ratio,
                                    float max_mean_ratio, int32_t* __restrict__ flag) {
  int stop = 0;
  if (max_ratio > 0.f && st->ratio_max > max_ratio) stop = 1;
  if (max_mean_ratio > 0.f && st->tokens > 0 &&
      st->ratio_sum / static_cast<double>(st->tokens) > static_cast<double>(max_mean_ratio))
    stop = 1;
  *flag = stop;
}

// x[i] *= 1/N when scaling; when *zero_if (early stop) x[i] := 0, stored
// directly (not multiplied by 0: a discarded update may hold NaN/Inf).
__global__ void __launch_bounds__(UPD_THREADS)
k_scale(float* __restrict__ x, int64_t n, const int32_t* __restrict__ zero_if,
        const int64_t* __restrict__ count) {
  float s = 1.f;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * UPD_THREADS;
  if (zero_if) {
    if (*zero_if == 0) return;
    float4* x4 = reinterpret_cast<float4*>(x);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * UPD_THREADS + threadIdx.x; i < n / 4;
         i += stride)
      x4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t i = 4 * (n / 4) + static_cast<int64_t>(blockIdx.x) * UPD_THREADS + threadIdx.x;
         i < n; i += stride)
      x[i] = 0.f;
    return;
  } else {
    const long long c = *count;
    s = c > 0 ? static_cast<float>(1.0 / static_cast<double>(c)) : 0.f;
  }
  const int64_t n4 = n / 4;
  float4* x4 = reinterpret_cast<float4*>(x);
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * UPD_THREADS + threadIdx.x; i < n4;
       i += stride) {
    float4 v = x4[i];
    v.x *= s;
    v.y *= s;
    v.z *= s;
    v.w *= s;
    x4[i] = v;
  }
  for (int64_t i = 4 * n4 + static_cast<int64_t>(blockIdx.x) * UPD_THREADS + threadIdx.x; i < n;
       i += stride)
    x[i] *= s;
}

static rl_status launch_scale(float* x, int64_t n, const int32_t* zero_if, const int64_t* count,
                              cudaStream_t s) {
  if (n <= 0) return RL_OK;
  const int64_t blocks = std::min<int64_t>(ceil_div(n / 4 + 1, UPD_THREADS), 148 * 8);
  TraceScope ts(RL_K_MISC, s);
  k_scale<<<static_cast<unsigned>(blocks), UPD_THREADS, 0, s>>>(x, n, zero_if, count);
  RLH_CHECK_LAUNCH();
  return RL_OK;
}

}  // namespace rlh

using namespace rlh;

extern "C" {

rl_status rl_minibatch_early_stop(const rl_loss_stats* stats, float max_ratio,
                                  float max_mean_ratio, int32_t* stop_flag, float* grad_weight,
                                  int64_t n, rl_stream_t stream) {
  if (!stats || !stop_flag || n < 0 || (n > 0 && !grad_weight)) return RL_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(grad_weight) & 15) != 0) return RL_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  {
    TraceScope ts(RL_K_MISC, s);
    k_early_stop_decide<<<1, 1, 0, s>>>(stats, max_ratio, max_mean_ratio, stop_flag);
  }
  RLH_CHECK_LAUNCH();
  return launch_scale(grad_weight, n, stop_flag, nullptr, s);
}

rl_status rl_scale_by_inverse_count(float* x, int64_t n, const int64_t* count,
                                    rl_stream_t stream) {
  if (!count || n < 0 || (n > 0 && !x)) return RL_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(x) & 15) != 0) return RL_ERR_INVALID_ARG;
  return launch_scale(x, n, nullptr, count, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
