// H1: packed-batch bookkeeping (validation, row -> sequence map, active-row
// compaction in packed order) and the row gather feeding the tensor-core
// GEMMs. HBM-bound; coalesced loads, 16-B vectors for the row copies.
// Semantics: include/rlhead.h (rl_batch), DESIGN.md §5.
#include "kernels.h"

namespace rlh {

constexpr int PREP_THREADS = 256;
constexpr int PREP_ROWS = 1024;  // rows per block (4 per thread)

__global__ void k_validate(const int32_t* __restrict__ cu, int32_t S, int64_t R,
                           WsHeader* hdr, int32_t* err) {
  int bad = 0;
  for (int64_t i = threadIdx.x; i <= S; i += blockDim.x) {
    const int32_t c = cu[i];
    if (i == 0 && c != 0) bad = 1;
    if (i == S && static_cast<int64_t>(c) != R) bad = 1;
    if (i < S && cu[i + 1] < c) bad = 1;
    if (c < 0 || static_cast<int64_t>(c) > R) bad = 1;
  }
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    hdr->bad_cu = bad;
    hdr->n_active = 0;
  }
  if (threadIdx.x < 16) {
    hdr->sched[threadIdx.x >> 1][threadIdx.x & 1] = 0u;
  }
  if (threadIdx.x == 0) {
    if (bad && err) atomicOr(err, RL_DEVERR_CU_SEQLENS);
  }
}

// First index i in [0, n) with cu[i] > t (cu non-decreasing).
__device__ __forceinline__ int32_t upper_bound_i32(const int32_t* __restrict__ cu, int32_t n,
                                                   int64_t t) {
  int32_t lo = 0, hi = n;
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    if (static_cast<int64_t>(__ldg(cu + mid)) <= t) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Rows per thread: ROWS_PT consecutive rows, so the row -> sequence map needs
// one binary search of cu_seqlens per thread, then a forward walk.
constexpr int ROWS_PT = PREP_ROWS / PREP_THREADS;

__global__ void __launch_bounds__(PREP_THREADS)
k_flags(const int32_t* __restrict__ cu, int32_t S, int64_t R, const int32_t* __restrict__ targets,
        const uint8_t* __restrict__ mask, int32_t V, const WsHeader* __restrict__ hdr,
        uint8_t* __restrict__ act, int32_t* __restrict__ row_seq, int32_t* __restrict__ blk_cnt,
        float* zero0, float* zero1, float* zero2, int32_t* err) {
  const int bad = hdr->bad_cu;
  int cnt = 0, terr = 0;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * PREP_ROWS + threadIdx.x * ROWS_PT;
  // last sequence s with cu[s] <= t0 (empty sequences skipped), as the binary
  // search below each row would give
  int32_t s = (!bad && t0 < R) ? upper_bound_i32(cu, S + 1, t0) - 1 : -1;
#pragma unroll
  for (int j = 0; j < ROWS_PT; ++j) {
    const int64_t t = t0 + j;
    if (t >= R) break;
    uint8_t a = 0;
    if (!bad) {
      while (s < S && static_cast<int64_t>(__ldg(cu + s + 1)) <= t) ++s;
      if (mask[t]) {
        const int32_t y = targets[t];
        if (y >= 0 && y < V) a = 1; else terr = 1;
      }
    }
    act[t] = a;
    row_seq[t] = bad ? -1 : s;
    cnt += a;
    if (!a) {
      if (zero0) zero0[t] = 0.f;
      if (zero1) zero1[t] = 0.f;
      if (zero2) zero2[t] = 0.f;
    }
  }
  if (terr && err) atomicOr(err, RL_DEVERR_TARGET);
  cnt = warp_sum(cnt);
  __shared__ int wsum[PREP_THREADS / 32];
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int w = 0; w < PREP_THREADS / 32; ++w) tot += wsum[w];
    blk_cnt[blockIdx.x] = tot;
  }
}

// Exclusive scan of the per-block counts (one block), total -> header and
// the optional user counters.
__global__ void __launch_bounds__(1024)
k_scan(const int32_t* __restrict__ blk_cnt, int64_t nblk, int64_t* __restrict__ blk_off,
       WsHeader* hdr, int64_t* n_active_user, int64_t* n_accum) {
  __shared__ int64_t part[1024];
  const int64_t per = (nblk + blockDim.x - 1) / blockDim.x;
  const int64_t b0 = threadIdx.x * per;
  const int64_t b1 = b0 + per < nblk ? b0 + per : nblk;
  int64_t sum = 0;
  for (int64_t b = b0; b < b1; ++b) sum += blk_cnt[b];
  part[threadIdx.x] = sum;
  __syncthreads();
  // Hillis-Steele inclusive scan over 1024 partial sums.
  for (int o = 1; o < 1024; o <<= 1) {
    int64_t v = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int64_t run = threadIdx.x ? part[threadIdx.x - 1] : 0;
  for (int64_t b = b0; b < b1; ++b) {
    blk_off[b] = run;
    run += blk_cnt[b];
  }
  if (threadIdx.x == blockDim.x - 1) {
    const int64_t total = part[blockDim.x - 1];
    hdr->n_active = total;
    if (n_active_user) *n_active_user = total;
    if (n_accum) *n_accum += total;
  }
}

__global__ void __launch_bounds__(PREP_THREADS)
k_compact(int64_t R, const uint8_t* __restrict__ act, const int32_t* __restrict__ row_seq,
          const int32_t* __restrict__ targets, const int64_t* __restrict__ blk_off,
          int32_t* __restrict__ active_idx, int32_t* __restrict__ tgt_c,
          int32_t* __restrict__ seq_c) {
  // Thread = ROWS_PT consecutive rows (packed order = thread order, then row):
  // exclusive offset = block offset + warps before + lanes before (shuffle scan).
  __shared__ int wcnt[PREP_THREADS / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * PREP_ROWS + threadIdx.x * ROWS_PT;
  uint32_t bits = 0;
#pragma unroll
  for (int j = 0; j < ROWS_PT; ++j)
    if (t0 + j < R && act[t0 + j]) bits |= 1u << j;
  const int c = __popc(bits);
  int incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wcnt[warp] = incl;
  __syncthreads();
  int woff = 0;
  for (int w = 0; w < warp; ++w) woff += wcnt[w];
  int64_t o = blk_off[blockIdx.x] + woff + (incl - c);
#pragma unroll
  for (int j = 0; j < ROWS_PT; ++j) {
    if (bits & (1u << j)) {
      const int64_t t = t0 + j;
      active_idx[o] = static_cast<int32_t>(t);
      tgt_c[o] = targets[t];
      seq_c[o] = row_seq[t];
      ++o;
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
  int32_t* blk_cnt = reinterpret_cast<int32_t*>(ws + L.off_blkcnt);
  int64_t* blk_off = reinterpret_cast<int64_t*>(ws + L.off_blkoff);
  int32_t* row_seq = row_seq_user ? row_seq_user : reinterpret_cast<int32_t*>(ws + L.off_rowseq);
  int32_t* active_idx =
      active_idx_user ? active_idx_user : reinterpret_cast<int32_t*>(ws + L.off_active);
  int32_t* tgt_c = reinterpret_cast<int32_t*>(ws + L.off_tgt);
  int32_t* seq_c = reinterpret_cast<int32_t*>(ws + L.off_seq);
  const int64_t R = b->num_rows;
  {
    TraceScope ts(RL_K_PREPARE, s);
    k_validate<<<1, 1024, 0, s>>>(b->cu_seqlens, b->num_seqs, R, hdr, b->err_flags);
  }
  RLH_CHECK_LAUNCH();
  const int64_t nblk = ceil_div(R, PREP_ROWS);
  if (nblk > 0) {
    TraceScope ts(RL_K_PREPARE, s);
    k_flags<<<static_cast<unsigned>(nblk), PREP_THREADS, 0, s>>>(
        b->cu_seqlens, b->num_seqs, R, b->targets, b->mask,
        static_cast<int32_t>(vocab_total(hd)), hdr, act, row_seq, blk_cnt,
        zero0, zero1, zero2, b->err_flags);
  }
  RLH_CHECK_LAUNCH();
  {
    TraceScope ts(RL_K_PREPARE, s);
    k_scan<<<1, 1024, 0, s>>>(blk_cnt, nblk, blk_off, hdr, n_active_user, n_accum);
  }
  RLH_CHECK_LAUNCH();
  if (nblk > 0) {
    TraceScope ts(RL_K_PREPARE, s);
    k_compact<<<static_cast<unsigned>(nblk), PREP_THREADS, 0, s>>>(R, act, row_seq, b->targets,
                                                                    blk_off, active_idx, tgt_c,
                                                                    seq_c);
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
  if (t >= R || act[t]) return;
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
                               cudaStream_t s, bool f32_rows) {
  const uint8_t* act = reinterpret_cast<const uint8_t*>(ws + L.off_flags);
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
