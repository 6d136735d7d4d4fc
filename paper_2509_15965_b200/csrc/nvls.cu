// Collectives over NVLink peer memory for the two exchange steps that follow
// a GEMM on the hot path: the vocab-parallel sum of
// dL/dH (below) and the owner side of the DP dW reduce-scatter
// (k_reduce_bcast_f32; the send side is the dW GEMM epilogue). The GEMM epilogue writes its fp32 result
// straight into a symmetric buffer (mapped on every rank); after a cross-rank
// barrier this kernel sums the P copies without NCCL and without staging:
//  * NVLS (NVLink SHARP, multicast object available): two-shot all-reduce --
//    rank p pulls its 1/P slice through the switch with
//    multimem.ld_reduce.add (the switch adds the P copies) and multicasts the
//    sum back to every rank with multimem.st;
//  * otherwise P2P: rank p loads its slice from the P peers in rank order
//    (deterministic), adds, and stores the sum to every peer.
// A second barrier (caller) makes the result visible before use.
#include "kernels.h"

namespace rlh {

constexpr int AR_THREADS = 512;
constexpr int AR_MAX_PEERS = 8;

struct PeerPtrs {
  float* p[AR_MAX_PEERS];
};

__global__ void __launch_bounds__(AR_THREADS)
k_nvls_allreduce_f32(float* mc, int64_t n4, int rank, int world) {
  const int64_t per = (n4 + world - 1) / world;
  const int64_t b = static_cast<int64_t>(rank) * per;
  const int64_t e = b + per < n4 ? b + per : n4;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * AR_THREADS;
  for (int64_t i = b + static_cast<int64_t>(blockIdx.x) * AR_THREADS + threadIdx.x; i < e;
       i += stride) {
    float* a = mc + 4 * i;
    uint32_t x, y, z, w;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(x), "=r"(y), "=r"(z), "=r"(w)
                 : "l"(a)
                 : "memory");
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(a), "r"(x),
                 "r"(y), "r"(z), "r"(w)
                 : "memory");
  }
}

__global__ void __launch_bounds__(AR_THREADS)
k_p2p_allreduce_f32(PeerPtrs peers, int64_t n4, int rank, int world) {
  const int64_t per = (n4 + world - 1) / world;
  const int64_t b = static_cast<int64_t>(rank) * per;
  const int64_t e = b + per < n4 ? b + per : n4;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * AR_THREADS;
  for (int64_t i = b + static_cast<int64_t>(blockIdx.x) * AR_THREADS + threadIdx.x; i < e;
       i += stride) {
    float4 s = reinterpret_cast<const float4*>(peers.p[0])[i];
    for (int q = 1; q < world; ++q) {  // fixed rank order: deterministic
      const float4 v = reinterpret_cast<const float4*>(peers.p[q])[i];
      s.x += v.x;
      s.y += v.y;
      s.z += v.z;
      s.w += v.w;
    }
    for (int q = 0; q < world; ++q) reinterpret_cast<float4*>(peers.p[q])[i] = s;
  }
}

// DP dW sum after the last dW GEMM (collective "nvls"): rank r
// owns float4s [b4, e4) of the [rows][cols] buffer. NVLS: multimem.ld_reduce
// pulls the element-wise sum of every rank's copy through the switch; the sum
// goes back to every copy (multimem.st, bcast = 1) or into this rank's own
// buffer only (bcast = 0: a sharded gradient). P2P: loads from every peer in
// rank order (deterministic), stores to every peer or to this rank only.
// RD_UNROLL independent loads per thread keep the NVLink requests in flight.
constexpr int RD_UNROLL = 4;
__global__ void __launch_bounds__(AR_THREADS)
k_nvls_rows_reduce_f32(float* mc, float* local, int64_t b4, int64_t e4, int bcast) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * AR_THREADS;
  for (int64_t i0 = b4 + static_cast<int64_t>(blockIdx.x) * AR_THREADS + threadIdx.x; i0 < e4;
       i0 += stride * RD_UNROLL) {
    uint32_t v[RD_UNROLL][4];
#pragma unroll
    for (int u = 0; u < RD_UNROLL; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < e4)
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[u][0]), "=r"(v[u][1]), "=r"(v[u][2]), "=r"(v[u][3])
                     : "l"(mc + 4 * i)
                     : "memory");
    }
#pragma unroll
    for (int u = 0; u < RD_UNROLL; ++u) {
      const int64_t i = i0 + u * stride;
      if (i >= e4) continue;
      if (bcast)
        asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + 4 * i),
                     "r"(v[u][0]), "r"(v[u][1]), "r"(v[u][2]), "r"(v[u][3])
                     : "memory");
      else
        reinterpret_cast<uint4*>(local)[i] = make_uint4(v[u][0], v[u][1], v[u][2], v[u][3]);
    }
  }
}

__global__ void __launch_bounds__(AR_THREADS)
k_p2p_rows_reduce_f32(PeerPtrs peers, int64_t b4, int64_t e4, int rank, int world, int bcast) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * AR_THREADS;
  for (int64_t i0 = b4 + static_cast<int64_t>(blockIdx.x) * AR_THREADS + threadIdx.x; i0 < e4;
       i0 += stride * RD_UNROLL) {
    float4 s[RD_UNROLL];
#pragma unroll
    for (int u = 0; u < RD_UNROLL; ++u) {
      const int64_t i = i0 + u * stride;
      s[u] = i < e4 ? reinterpret_cast<const float4*>(peers.p[0])[i] : make_float4(0, 0, 0, 0);
    }
    for (int q = 1; q < world; ++q) {  // fixed rank order: deterministic
#pragma unroll
      for (int u = 0; u < RD_UNROLL; ++u) {
        const int64_t i = i0 + u * stride;
        if (i >= e4) continue;
        const float4 x = reinterpret_cast<const float4*>(peers.p[q])[i];
        s[u].x += x.x;
        s[u].y += x.y;
        s[u].z += x.z;
        s[u].w += x.w;
      }
    }
#pragma unroll
    for (int u = 0; u < RD_UNROLL; ++u) {
      const int64_t i = i0 + u * stride;
      if (i >= e4) continue;
      if (bcast) {
        for (int q = 0; q < world; ++q) reinterpret_cast<float4*>(peers.p[q])[i] = s[u];
      } else {
        reinterpret_cast<float4*>(peers.p[rank])[i] = s[u];
      }
    }
  }
}

// Owner side of the DP dW reduce-scatter: sum the `world`
// staged copies of this rank's slab in rank order (deterministic) and store
// the sum into every rank's output -- multimem.st through the multicast
// address, or plain stores to each peer. i: float4 index within the slab.
__global__ void __launch_bounds__(AR_THREADS)
k_reduce_bcast_f32(const float* __restrict__ staging, int64_t slab4, int world, PeerPtrs out,
                   float* mc, int64_t off4, int64_t n4) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * AR_THREADS;
  const float4* st = reinterpret_cast<const float4*>(staging);
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * AR_THREADS + threadIdx.x; i < n4;
       i += stride) {
    float4 s = st[i];
    for (int q = 1; q < world; ++q) {
      const float4 v = st[q * slab4 + i];
      s.x += v.x;
      s.y += v.y;
      s.z += v.z;
      s.w += v.w;
    }
    if (mc) {
      asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(
                       mc + 4 * (off4 + i)),
                   "f"(s.x), "f"(s.y), "f"(s.z), "f"(s.w)
                   : "memory");
    } else {
      for (int q = 0; q < world; ++q)
        if (out.p[q]) reinterpret_cast<float4*>(out.p[q])[off4 + i] = s;
    }
  }
}

__global__ void __launch_bounds__(256)
k_f32_rows_to_bf16(const float* __restrict__ src, int64_t R, int h, __nv_bfloat16* dst,
                   int64_t ld) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (t >= R) return;
  const float2* s = reinterpret_cast<const float2*>(src + t * h);
  __nv_bfloat162* d = reinterpret_cast<__nv_bfloat162*>(dst + t * ld);
  for (int k = threadIdx.x & 31; k < h / 2; k += 32) d[k] = __float22bfloat162_rn(s[k]);
}

}  // namespace rlh

using namespace rlh;

extern "C" {

rl_status rl_allreduce_sum_f32(float* const* peer_ptrs, float* mc_ptr, int32_t rank,
                               int32_t world, int64_t n, rl_stream_t stream) {
  if (world < 1 || world > AR_MAX_PEERS || rank < 0 || rank >= world || n < 0 || (n & 3))
    return RL_ERR_INVALID_ARG;
  if (n == 0 || world == 1) return RL_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t n4 = n / 4;
  const int64_t per = (n4 + world - 1) / world;
  const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(per, AR_THREADS), 148 * 2));
  TraceScope ts(RL_K_MISC, s);
  if (mc_ptr) {
    if ((reinterpret_cast<uintptr_t>(mc_ptr) & 15) != 0) return RL_ERR_INVALID_ARG;
    k_nvls_allreduce_f32<<<blocks, AR_THREADS, 0, s>>>(mc_ptr, n4, rank, world);
  } else {
    if (!peer_ptrs) return RL_ERR_INVALID_ARG;
    PeerPtrs pp{};
    for (int q = 0; q < world; ++q) {
      if (!peer_ptrs[q] || (reinterpret_cast<uintptr_t>(peer_ptrs[q]) & 15) != 0)
        return RL_ERR_INVALID_ARG;
      pp.p[q] = peer_ptrs[q];
    }
    k_p2p_allreduce_f32<<<blocks, AR_THREADS, 0, s>>>(pp, n4, rank, world);
  }
  RLH_CHECK_LAUNCH();
  return RL_OK;
}

rl_status rl_reduce_bcast_rows_f32(const float* staging, float* const* out_peers, float* out_mc,
                                   int32_t rank, int32_t world, int64_t num_rows, int64_t cols,
                                   int64_t rows_per_rank, rl_stream_t stream) {
  if (world < 1 || world > AR_MAX_PEERS || rank < 0 || rank >= world || num_rows < 0 ||
      cols <= 0 || (cols & 3) || rows_per_rank <= 0 || rows_per_rank * world < num_rows ||
      !staging || (reinterpret_cast<uintptr_t>(staging) & 15) != 0)
    return RL_ERR_INVALID_ARG;
  PeerPtrs pp{};
  if (!out_mc) {
    if (!out_peers) return RL_ERR_INVALID_ARG;
    // NULL entries (other than this rank's) are skipped: the sum stays on the
    // owner (a sharded gradient, FSDP / ZeRO-2 style)
    if (!out_peers[rank]) return RL_ERR_INVALID_ARG;
    for (int q = 0; q < world; ++q) {
      if (out_peers[q] && (reinterpret_cast<uintptr_t>(out_peers[q]) & 15) != 0)
        return RL_ERR_INVALID_ARG;
      pp.p[q] = out_peers[q];
    }
  } else if ((reinterpret_cast<uintptr_t>(out_mc) & 15) != 0) {
    return RL_ERR_INVALID_ARG;
  }
  const int64_t r0 = std::min<int64_t>(static_cast<int64_t>(rank) * rows_per_rank, num_rows);
  const int64_t r1 = std::min(r0 + rows_per_rank, num_rows);
  if (r1 <= r0) return RL_OK;
  const int64_t n4 = (r1 - r0) * cols / 4;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(n4, AR_THREADS), 148 * 4));
  TraceScope ts(RL_K_MISC, s);
  k_reduce_bcast_f32<<<blocks, AR_THREADS, 0, s>>>(staging, rows_per_rank * cols / 4, world, pp,
                                                   out_mc, r0 * cols / 4, n4);
  RLH_CHECK_LAUNCH();
  return RL_OK;
}

rl_status rl_dw_reduce_rows_f32(float* const* peer_ptrs, float* mc_ptr, int32_t rank,
                                int32_t world, int64_t num_rows, int64_t cols,
                                int64_t rows_per_rank, int32_t broadcast, rl_stream_t stream) {
  if (world < 1 || world > AR_MAX_PEERS || rank < 0 || rank >= world || num_rows < 0 ||
      cols <= 0 || (cols & 3) || rows_per_rank <= 0 || rows_per_rank * world < num_rows ||
      !peer_ptrs)
    return RL_ERR_INVALID_ARG;
  PeerPtrs pp{};
  for (int q = 0; q < world; ++q) {
    if (!peer_ptrs[q] || (reinterpret_cast<uintptr_t>(peer_ptrs[q]) & 15) != 0)
      return RL_ERR_INVALID_ARG;
    pp.p[q] = peer_ptrs[q];
  }
  if (mc_ptr && (reinterpret_cast<uintptr_t>(mc_ptr) & 15) != 0) return RL_ERR_INVALID_ARG;
  if (world == 1) return RL_OK;
  const int64_t r0 = std::min<int64_t>(static_cast<int64_t>(rank) * rows_per_rank, num_rows);
  const int64_t r1 = std::min(r0 + rows_per_rank, num_rows);
  if (r1 <= r0) return RL_OK;
  const int64_t b4 = r0 * cols / 4, e4 = r1 * cols / 4;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int blocks = static_cast<int>(
      std::min<int64_t>(ceil_div(ceil_div(e4 - b4, RD_UNROLL), AR_THREADS), 148 * 4));
  TraceScope ts(RL_K_MISC, s);
  if (mc_ptr)
    k_nvls_rows_reduce_f32<<<blocks, AR_THREADS, 0, s>>>(mc_ptr, pp.p[rank], b4, e4,
                                                          broadcast ? 1 : 0);
  else
    k_p2p_rows_reduce_f32<<<blocks, AR_THREADS, 0, s>>>(pp, b4, e4, rank, world,
                                                         broadcast ? 1 : 0);
  RLH_CHECK_LAUNCH();
  return RL_OK;
}

rl_status rl_cast_rows_bf16(const float* src, int64_t num_rows, int32_t hidden, void* dst,
                            int64_t ld, rl_stream_t stream) {
  if (num_rows < 0 || hidden < 2 || (hidden & 1) || ld < hidden || (ld & 1) ||
      (num_rows > 0 && (!src || !dst)))
    return RL_ERR_INVALID_ARG;
  if (num_rows == 0) return RL_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  TraceScope ts(RL_K_MISC, s);
  k_f32_rows_to_bf16<<<static_cast<unsigned>(ceil_div(num_rows, 8)), 256, 0, s>>>(
      src, num_rows, hidden, static_cast<__nv_bfloat16*>(dst), ld);
  RLH_CHECK_LAUNCH();
  return RL_OK;
}

}  // extern "C"
