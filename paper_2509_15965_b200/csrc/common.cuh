// Shared host/device plumbing of librlhead: launch tracing, workspace layout,
// small device reductions. Nothing here is numerics of the method.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstddef>

#include "../../include/rlhead.h"

namespace rlh {

// ---------------------------------------------------------------- tracing ----
// Every kernel launch goes through TraceScope so that rl_launch_count() and the
// optional event tracer (rl_trace_begin/end) see it.
void trace_before(int kind, cudaStream_t s);
void trace_after(int kind, cudaStream_t s);
struct TraceScope {
  int kind;
  cudaStream_t s;
  TraceScope(int k, cudaStream_t st) : kind(k), s(st) { trace_before(kind, s); }
  ~TraceScope() { trace_after(kind, s); }
};

#define RLH_CHECK_LAUNCH()                                   \
  do {                                                       \
    cudaError_t e_ = cudaGetLastError();                     \
    if (e_ != cudaSuccess) return RL_ERR_CUDA;               \
  } while (0)

// ---------------------------------------------------------------- tiling ----
constexpr int TC_BM = 128;   // rows per tcgen05 tile (UMMA M)
constexpr int TC_BN = 256;   // columns per tile (UMMA N)
constexpr int TC_BK = 64;    // K per pipeline stage (one 128-B swizzle row)
constexpr int H1_TILE_ROWS = 1024;  // smallest H1 scan tile (status words per call)

// Vocabulary of the whole (possibly vocab-sharded) head; targets live in it.
inline int64_t vocab_total(const rl_head* hd) {
  return hd->vocab_total > 0 ? hd->vocab_total : hd->vocab;
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// Workspace carve-up. All offsets 256-B aligned. Sizes depend on the head,
// the row bound R and whether the backward runs.
struct WsLayout {
  int64_t R, Rp;          // rows, rows padded to TC_BM (+1 tile of slack)
  int64_t n_vt;           // vocab tiles (partials per row)
  int64_t Vp;             // vocab padded to TC_BN (dZ row stride)
  int64_t nblk_rows;      // H1_TILE_ROWS-row tiles of the bookkeeping scan (status words)
  int64_t nblk_loss;      // 32-row blocks of the merge/loss kernel
  size_t prep_total;      // bytes rl_batch_prepare needs (a prefix of the layout)
  size_t off_hdr, off_flags, off_blkcnt, off_blkoff, off_active, off_rowseq, off_tgt,
      off_seq, off_hc, off_pm, off_ps, off_pu, off_zy, off_lse, off_g, off_ge, off_ez, off_dz,
      off_st_d, off_st_f, off_st_i, off_keep, off_oidx2, off_st2, off_dz2, off_hc2, total;
};
bool ws_layout(const rl_head* hd, int64_t R, int want_bwd, WsLayout* L);

// Header words at ws + off_hdr.
struct WsHeader {
  int64_t n_active;   // active rows of this call
  int32_t bad_cu;     // malformed cu_seqlens
  uint32_t tile_ctr;  // H1 scan: tiles claimed in order (zeroed by k_validate)
  // dynamic tile scheduler of the tensor-core GEMMs, one {claimed, retired}
  // counter pair per GEMM kind; zeroed by k_validate and by the last CTA of
  // every launch that uses it
  uint32_t sched[8][2];
  int64_t n_bwd;      // rows with dL/dlogp != 0 (the backward's rows in skip mode)
  uint32_t tile_ctr2; // backward-row compaction: tiles claimed in order
  uint32_t pad2;
};

// ------------------------------------------ decoupled look-back scan ----
// Status word of a tile of a single-pass scan: flag in the top 2 bits.
constexpr unsigned long long ST_AGG = 1ull << 62;   // this tile's count only
constexpr unsigned long long ST_PFX = 2ull << 62;   // inclusive prefix through this tile
constexpr unsigned long long ST_VAL = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v);

// One warp: publish this tile's count `agg`, look back over the preceding
// tiles' status words 32 at a time (every predecessor is already running:
// tiles are claimed in order from a counter) until the nearest one with an
// inclusive prefix, publish this tile's inclusive prefix; returns the
// exclusive prefix (all lanes). status[] zeroed before the launch.
__device__ __forceinline__ long long decoupled_lookback(unsigned long long* status, int64_t tile,
                                                        long long agg, int lane) {
  long long excl = 0;
  if (tile == 0) {
    if (lane == 0) atomicExch(status, ST_PFX | static_cast<unsigned long long>(agg));
    return 0;
  }
  if (lane == 0) atomicExch(status + tile, ST_AGG | static_cast<unsigned long long>(agg));
  int64_t j = tile - 1;
  while (true) {
    const int64_t idx = j - lane;
    unsigned long long v = ST_PFX;  // before tile 0: prefix 0
    if (idx >= 0) {
      do {
        v = ld_volatile_u64(status + idx);
      } while ((v >> 62) == 0ull);
    }
    const uint32_t pm = __ballot_sync(0xffffffffu, (v >> 62) == 2ull);
    const int stop = pm ? __ffs(pm) - 1 : 31;  // nearest predecessor with a prefix
    long long x = lane <= stop ? static_cast<long long>(v & ST_VAL) : 0ll;
    x = warp_sum(x);
    excl += x;
    if (pm) break;
    j -= 32;
  }
  if (lane == 0) atomicExch(status + tile, ST_PFX | static_cast<unsigned long long>(excl + agg));
  return excl;
}

// ------------------------------------------------------ device reductions ----
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}

}  // namespace rlh
