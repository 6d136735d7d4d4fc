// H1: packed-batch bookkeeping (validation, row -> sequence map, active-row
// compaction in packed order) and the row gather feeding the tensor-core
// GEMMs. HBM-bound; coalesced loads, 16-B vectors for the row copies.
// Semantics: include/rlhead.h (rl_batch), DESIGN.md §5.
#include "kernels.h"

#include <cstdlib>

namespace rlh {

constexpr int PREP_THREADS = 256;
// rows per thread: 8 (2048-row tiles) for whole mini-batches, 4 (1024-row
// tiles) for micro-batches, so a 16k-row call still spreads over 16 SMs
// (RLHEAD_H1_ITEMS = 4 | 8 | 16 overrides, for A/B runs)
constexpr int PREP_ITEMS_BIG = 8, PREP_ITEMS_SMALL = 4;
static_assert(PREP_THREADS * PREP_ITEMS_SMALL == H1_TILE_ROWS, "workspace status words");

// Launch 1 of 2: validate cu_seqlens, reset the header (active count, tile
// claim counter, GEMM tile schedulers) and the scan's tile status words.
__global__ void __launch_bounds__(1024)
k_validate(const int32_t* __restrict__ cu, int32_t S, int64_t R, WsHeader* hdr,
           unsigned long long* __restrict__ status, int64_t ntiles,
           unsigned long long* __restrict__ status2, int64_t ntiles2, int32_t* err) {
  int bad = 0;
  for (int64_t i = threadIdx.x; i <= S; i += blockDim.x) {
    const int32_t c = cu[i];
    if (i == 0 && c != 0) bad = 1;
    if (i == S && static_cast<int64_t>(c) != R) bad = 1;
    if (i < S && cu[i + 1] < c) bad = 1;
    if (c < 0 || static_cast<int64_t>(c) > R) bad = 1;
  }
  for (int64_t i = threadIdx.x; i < ntiles; i += blockDim.x) status[i] = 0ull;
  if (status2)
    for (int64_t i = threadIdx.x; i < ntiles2; i += blockDim.x) status2[i] = 0ull;
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    hdr->bad_cu = bad;
    hdr->n_active = 0;
    hdr->tile_ctr = 0u;
    hdr->n_bwd = 0;
    hdr->tile_ctr2 = 0u;
    if (bad && err) atomicOr(err, RL_DEVERR_CU_SEQLENS);
  }
  if (threadIdx.x < 16) hdr->sched[threadIdx.x >> 1][threadIdx.x & 1] = 0u;
}

// First index i in [lo, n) with cu[i] > t (cu non-decreasing).
__device__ __forceinline__ int32_t upper_bound_i32(const int32_t* __restrict__ cu, int32_t lo,
                                                   int32_t n, int64_t t) {
  int32_t hi = n;
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    if (static_cast<int64_t>(__ldg(cu + mid)) <= t) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Launch 2 of 2 (single pass): per row the active flag (mask set, target in
// range, batch well formed) and its sequence; a block-wide ballot scan of the
// flags; the tile's global offset by decoupled look-back over the preceding
// tiles' status words (tiles claimed in order from a counter, so every
// predecessor is already running); then the compaction in packed order.
// Rows are lane-interleaved (row = tile * 4096 + it * 256 + thread): every
// load/store instruction of a warp touches 32 consecutive rows.
template <int PREP_ITEMS>
__global__ void __launch_bounds__(PREP_THREADS, PREP_ITEMS <= 8 ? 4 : 2)
k_flags_compact(const int32_t* __restrict__ cu, int32_t S, int64_t R,
                const int32_t* __restrict__ targets, const uint8_t* __restrict__ mask, int32_t V,
                WsHeader* hdr, unsigned long long* status, int64_t ntiles,
                uint8_t* __restrict__ act, int32_t* __restrict__ row_seq,
                int32_t* __restrict__ active_idx, int32_t* __restrict__ tgt_c,
                int32_t* __restrict__ seq_c, int64_t* n_active_user, int64_t* n_accum,
                float* zero0, float* zero1, float* zero2, int32_t* err) {
  __shared__ int32_t s_cnt[PREP_ITEMS][PREP_THREADS / 32];
  __shared__ long long s_tile_total, s_prefix;
  __shared__ int32_t s_tile;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = static_cast<int32_t>(atomicAdd(&hdr->tile_ctr, 1u));
  __syncthreads();
  const int64_t tile = s_tile;
  const int bad = hdr->bad_cu;
  constexpr int PREP_TILE = PREP_THREADS * PREP_ITEMS;
  const int64_t base = tile * PREP_TILE + tid;
  // all of this thread's loads first (16 + 16 independent loads in flight)
  uint8_t mk[PREP_ITEMS];
  int32_t tg[PREP_ITEMS];
#pragma unroll
  for (int it = 0; it < PREP_ITEMS; ++it) {
    const int64_t t = base + static_cast<int64_t>(it) * PREP_THREADS;
    mk[it] = t < R ? mask[t] : 0;
    tg[it] = t < R ? targets[t] : 0;
  }
  uint32_t abits = 0;  // bit it: row base + it * 256 is active
  int32_t seq[PREP_ITEMS];
  int terr = 0;
  // sequence of the first row by binary search, then a forward walk (rows grow
  // by 256 per item; long walks fall back to a binary search over the rest)
  int32_t s = (!bad && base < R) ? upper_bound_i32(cu, 0, S + 1, base) - 1 : 0;
#pragma unroll
  for (int it = 0; it < PREP_ITEMS; ++it) {
    const int64_t t = base + static_cast<int64_t>(it) * PREP_THREADS;
    seq[it] = -1;
    if (t < R) {
      uint8_t a = 0;
      if (!bad) {
        int steps = 0;
        while (s < S && static_cast<int64_t>(__ldg(cu + s + 1)) <= t) {
          if (++steps > 8) {
            s = upper_bound_i32(cu, s, S + 1, t) - 1;
            break;
          }
          ++s;
        }
        seq[it] = s;
        if (mk[it]) {
          const int32_t y = tg[it];
          if (y >= 0 && y < V) a = 1; else terr = 1;
        }
      }
      act[t] = a;
      if (row_seq) row_seq[t] = bad ? -1 : s;
      if (!a) {
        if (zero0) zero0[t] = 0.f;
        if (zero1) zero1[t] = 0.f;
        if (zero2) zero2[t] = 0.f;
      }
      abits |= static_cast<uint32_t>(a) << it;
    }
  }
  if (terr && err) atomicOr(err, RL_DEVERR_TARGET);
  // counts per (it, warp): the packed order of the tile is it-major, then warp, then lane
#pragma unroll
  for (int it = 0; it < PREP_ITEMS; ++it) {
    const uint32_t b = __ballot_sync(0xffffffffu, (abits >> it) & 1u);
    if (lane == 0) s_cnt[it][warp] = __popc(b);
  }
  __syncthreads();
  if (warp == 0) {
    // exclusive scan of the ITEMS x 8 (it, warp) counts: lane owns PER consecutive
    constexpr int PER = PREP_ITEMS * (PREP_THREADS / 32) / 32;
    int32_t* flat = &s_cnt[0][0];
    int32_t c4[PER], sum = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      c4[k] = flat[lane * PER + k];
      sum += c4[k];
    }
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    int run = incl - sum;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      flat[lane * PER + k] = run;
      run += c4[k];
    }
    const long long agg = __shfl_sync(0xffffffffu, incl, 31);
    const long long excl = decoupled_lookback(status, tile, agg, lane);
    if (lane == 0) {
      s_prefix = excl;
      s_tile_total = agg;
      if (tile == ntiles - 1) {  // every row's flag is counted: the batch total
        const long long total = excl + agg;
        hdr->n_active = total;
        if (n_active_user) *n_active_user = total;
        if (n_accum) *n_accum += total;
      }
    }
  }
  __syncthreads();
  const long long pfx = s_prefix;
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int it = 0; it < PREP_ITEMS; ++it) {
    const uint32_t b = __ballot_sync(0xffffffffu, (abits >> it) & 1u);
    if ((abits >> it) & 1u) {
      const long long o = pfx + s_cnt[it][warp] + __popc(b & lt);
      active_idx[o] = static_cast<int32_t>(base + static_cast<int64_t>(it) * PREP_THREADS);
      tgt_c[o] = tg[it];
      seq_c[o] = seq[it];
    }
  }
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

// Sequences with at least one active row (the seq-mean normaliser S).
__global__ void __launch_bounds__(PREP_THREADS)
k_seq_count(const int32_t* __restrict__ cu, int32_t S, const int32_t* __restrict__ active_idx,
            const WsHeader* __restrict__ hdr, int64_t* nseq_accum) {
  const int64_t T = hdr->n_active;
  const int s = blockIdx.x * PREP_THREADS + threadIdx.x;
  int nonempty = 0;
  if (s < S && !hdr->bad_cu)
    nonempty = lower_bound_rows(active_idx, T, cu[s + 1]) > lower_bound_rows(active_idx, T, cu[s]);
  const int c = __syncthreads_count(nonempty);
  if (threadIdx.x == 0 && c)
    atomicAdd(reinterpret_cast<unsigned long long*>(nseq_accum), static_cast<unsigned long long>(c));
}

rl_status launch_prepare(const rl_head* hd, const rl_batch* b, const WsLayout& L, char* ws,
                         int32_t* row_seq_user, int32_t* active_idx_user, int64_t* n_active_user,
                         int64_t* n_accum, int64_t* nseq_accum, float* zero0, float* zero1,
                         float* zero2, cudaStream_t s) {
  WsHeader* hdr = reinterpret_cast<WsHeader*>(ws + L.off_hdr);
  uint8_t* act = reinterpret_cast<uint8_t*>(ws + L.off_flags);
  unsigned long long* status = reinterpret_cast<unsigned long long*>(ws + L.off_blkoff);
  int32_t* active_idx =
      active_idx_user ? active_idx_user : reinterpret_cast<int32_t*>(ws + L.off_active);
  int32_t* tgt_c = reinterpret_cast<int32_t*>(ws + L.off_tgt);
  int32_t* seq_c = reinterpret_cast<int32_t*>(ws + L.off_seq);
  const int64_t R = b->num_rows;
  static const int items_env = [] {
    const char* e = std::getenv("RLHEAD_H1_ITEMS");
    return (e && *e) ? std::atoi(e) : 0;
  }();
  const int items = (items_env == 4 || items_env == 8 || items_env == 16)
                        ? items_env
                        : (R >= (int64_t(1) << 21) ? PREP_ITEMS_BIG : PREP_ITEMS_SMALL);
  const int64_t ntiles = ceil_div(R, PREP_THREADS * items);
  {
    TraceScope ts(RL_K_PREPARE, s);
    // the backward-row compaction's status words (loss calls on the tensor-
    // core path; absent when rl_batch_prepare's workspace prefix is all there is)
    const bool st2 = L.off_st2 < L.off_dz2 && L.off_st2 + 8 <= L.total;
    k_validate<<<1, 1024, 0, s>>>(
        b->cu_seqlens, b->num_seqs, R, hdr, status, ntiles,
        st2 ? reinterpret_cast<unsigned long long*>(ws + L.off_st2) : nullptr,
        st2 ? ceil_div(L.Rp, H1_TILE_ROWS) : 0, b->err_flags);
  }
  RLH_CHECK_LAUNCH();
  if (ntiles > 0) {
    TraceScope ts(RL_K_PREPARE, s);
    auto kern = items == 16 ? k_flags_compact<16>
                : items == 8  ? k_flags_compact<8>
                              : k_flags_compact<4>;
    kern<<<static_cast<unsigned>(ntiles), PREP_THREADS, 0, s>>>(
        b->cu_seqlens, b->num_seqs, R, b->targets, b->mask,
        static_cast<int32_t>(vocab_total(hd)), hdr, status, ntiles, act, row_seq_user,
        active_idx, tgt_c, seq_c, n_active_user, n_accum, zero0, zero1, zero2, b->err_flags);
  } else if (n_active_user || n_accum) {
    // no rows: the counts are 0 (n_accum unchanged); n_active_user := 0
    if (n_active_user && cudaMemsetAsync(n_active_user, 0, sizeof(int64_t), s) != cudaSuccess)
      return RL_ERR_CUDA;
  }
  RLH_CHECK_LAUNCH();
  if (nseq_accum && b->num_seqs > 0) {
    TraceScope ts(RL_K_PREPARE, s);
    k_seq_count<<<static_cast<unsigned>(ceil_div(b->num_seqs, PREP_THREADS)), PREP_THREADS, 0,
                  s>>>(b->cu_seqlens, b->num_seqs, active_idx, hdr, nseq_accum);
  }
  RLH_CHECK_LAUNCH();
  return RL_OK;
}

// ---------------------------------------------------------------- gather ----
__global__ void __launch_bounds__(256)
k_gather_bf16(const uint4* __restrict__ hidden, int64_t ld_vec, int32_t hvec,
              const int32_t* __restrict__ active_idx, const WsHeader* __restrict__ hdr,
              uint4* __restrict__ hc, int64_t rows_bound) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int64_t T = hdr->n_active;
  const int64_t Tp = (T + 2 * TC_BM - 1) / (2 * TC_BM) * (2 * TC_BM);  // CTA-pair tile
  if (r >= Tp || r >= rows_bound) return;
  uint4* dst = hc + r * hvec;
  if (r < T) {
    const uint4* src = hidden + static_cast<int64_t>(active_idx[r]) * ld_vec;
    int i = lane;
    for (; i + 96 < hvec; i += 128) {
      uint4 a = __ldg(src + i), b2 = __ldg(src + i + 32), c = __ldg(src + i + 64),
            d = __ldg(src + i + 96);
      dst[i] = a; dst[i + 32] = b2; dst[i + 64] = c; dst[i + 96] = d;
    }
    for (; i < hvec; i += 32) dst[i] = __ldg(src + i);
  } else {
    const uint4 z = make_uint4(0, 0, 0, 0);
    for (int i = lane; i < hvec; i += 32) dst[i] = z;
  }
}

rl_status launch_gather_bf16(const rl_head* hd, const void* hidden, const WsLayout& L, char* ws,
                             cudaStream_t s) {
  const WsHeader* hdr = reinterpret_cast<const WsHeader*>(ws + L.off_hdr);
  const int32_t* active_idx = reinterpret_cast<const int32_t*>(ws + L.off_active);
  uint4* hc = reinterpret_cast<uint4*>(ws + L.off_hc);
  const int64_t blocks = ceil_div(L.Rp, 8);
  if (blocks == 0) return RL_OK;
  TraceScope ts(RL_K_GATHER, s);
  k_gather_bf16<<<static_cast<unsigned>(blocks), 256, 0, s>>>(
      static_cast<const uint4*>(hidden), hd->ld_hidden / 8, hd->hidden / 8, active_idx, hdr, hc,
      L.Rp);
  RLH_CHECK_LAUNCH();
  return RL_OK;
}

// ------------------------------------------------------- zero inactive rows ----
__global__ void __launch_bounds__(256)
k_zero_inactive(char* __restrict__ out, int64_t ld_bytes, int64_t row_bytes, int64_t R,
                const uint8_t* __restrict__ act) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= R || (act && act[t])) return;
  char* row = out + t * ld_bytes;
  if ((row_bytes & 15) == 0 && (reinterpret_cast<uintptr_t>(row) & 15) == 0) {
    uint4* v = reinterpret_cast<uint4*>(row);
    const uint4 z = make_uint4(0, 0, 0, 0);
    for (int64_t i = lane; i < row_bytes / 16; i += 32) v[i] = z;
  } else {
    for (int64_t i = lane; i < row_bytes; i += 32) row[i] = 0;
  }
}

rl_status launch_zero_inactive(const rl_head* hd, void* grad_hidden, const WsLayout& L, char* ws,
                               cudaStream_t s, bool f32_rows, bool all_rows) {
  const uint8_t* act = all_rows ? nullptr : reinterpret_cast<const uint8_t*>(ws + L.off_flags);
  const int64_t esz = (hd->dtype == RL_BF16 && !f32_rows) ? 2 : 4;
  const int64_t ld = f32_rows ? hd->hidden : hd->ld_hidden;
  const int64_t blocks = ceil_div(L.R, 8);
  if (blocks == 0) return RL_OK;
  TraceScope ts(RL_K_MISC, s);
  k_zero_inactive<<<static_cast<unsigned>(blocks), 256, 0, s>>>(
      static_cast<char*>(grad_hidden), ld * esz, static_cast<int64_t>(hd->hidden) * esz,
      L.R, act);
  RLH_CHECK_LAUNCH();
  return RL_OK;
}

}  // namespace rlh
