// C ABI of librlhead (include/rlhead.h): host-side validation, workspace
// layout, path selection (tcgen05 for bf16, CUDA cores for fp32) and the
// stream-ordered composition of the kernels. No allocation, no sync.
#include "kernels.h"

#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

namespace rlh {

// ---------------------------------------------------------------- tracing ----
static std::atomic<long long> g_launches{0};
static struct {
  std::mutex mu;
  bool on = false;
  std::vector<cudaEvent_t> ev;
  std::vector<int> kinds;
  int n = 0;
  bool pending = false;
} g_tr;

void trace_before(int kind, cudaStream_t s) {
  (void)kind;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (g_tr.on && 2 * (g_tr.n + 1) <= static_cast<int>(g_tr.ev.size())) {
    cudaEventRecord(g_tr.ev[2 * g_tr.n], s);
    g_tr.pending = true;
  }
}
void trace_after(int kind, cudaStream_t s) {
  if (g_tr.on && g_tr.pending) {
    cudaEventRecord(g_tr.ev[2 * g_tr.n + 1], s);
    g_tr.kinds.push_back(kind);
    g_tr.n++;
    g_tr.pending = false;
  }
}

static bool force_simt() {
  const char* e = std::getenv("RLHEAD_FORCE_SIMT");
  return e && e[0] == '1';
}
static bool use_tc(const rl_head* hd) { return hd->dtype == RL_BF16 && !force_simt(); }
static bool bwd_skip() {
  const char* e = std::getenv("RLHEAD_BWD_SKIP");
  return !(e && e[0] == '0');
}
static bool dz_fused() {
  const char* e = std::getenv("RLHEAD_DZ_FUSED");
  return e && e[0] == '1';
}
static bool dz_recompute() {
  const char* e = std::getenv("RLHEAD_DZ_RECOMPUTE");
  return e && e[0] == '1';
}

static size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

bool ws_layout(const rl_head* hd, int64_t R, int want_bwd, WsLayout* L) {
  const bool tc = use_tc(hd);
  const int64_t h = hd->hidden, V = hd->vocab;
  L->R = R;
  L->Rp = round_up(R > 0 ? R : 1, 2 * TC_BM);  // whole CTA-pair tiles
  L->n_vt = tc ? ceil_div(V, TC_BN) : 1;
  L->Vp = round_up(V, TC_BN);
  L->nblk_rows = ceil_div(R, H1_TILE_ROWS);
  L->nblk_loss = ceil_div(L->Rp, 32);  // k_merge: 32 rows per block
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = align256(o + bytes);
    return at;
  };
  L->off_hdr = take(sizeof(WsHeader));
  L->off_flags = take(static_cast<size_t>(R));
  L->off_blkcnt = take(static_cast<size_t>(L->nblk_rows) * 4);
  L->off_blkoff = take(static_cast<size_t>(L->nblk_rows) * 8);
  L->off_active = take(static_cast<size_t>(L->Rp) * 4);
  L->off_rowseq = take(static_cast<size_t>(R) * 4);
  L->off_tgt = take(static_cast<size_t>(L->Rp) * 4);
  L->off_seq = take(static_cast<size_t>(L->Rp) * 4);
  L->prep_total = o;  // everything rl_batch_prepare touches lies before this
  L->off_hc = take(tc ? static_cast<size_t>(L->Rp) * h * 2 : 0);
  L->off_pm = take(static_cast<size_t>(L->n_vt) * L->Rp * 4);
  L->off_ps = take(static_cast<size_t>(L->n_vt) * L->Rp * 4);
  L->off_pu = take(static_cast<size_t>(L->n_vt) * L->Rp * 4);
  L->off_zy = take(static_cast<size_t>(L->Rp) * 4);
  L->off_lse = take(static_cast<size_t>(L->Rp) * 4);
  L->off_g = take(static_cast<size_t>(L->Rp) * 4);
  L->off_ge = take(static_cast<size_t>(L->Rp) * 4);
  L->off_ez = take(static_cast<size_t>(L->Rp) * 4);
  L->off_dz = take(want_bwd ? (tc ? static_cast<size_t>(L->Rp) * L->Vp * 2
                                  : static_cast<size_t>(L->Rp) * V * 4)
                            : 0);
  L->off_st_d = take(static_cast<size_t>(L->nblk_loss) * 5 * 8);
  L->off_st_f = take(static_cast<size_t>(L->nblk_loss) * 4);
  L->off_st_i = take(static_cast<size_t>(L->nblk_loss) * 3 * 8);
  // backward-row compaction (q mode): rows with dL/dlogp != 0, their dZ and
  // Hc rows packed densely so dH / dW skip the rows whose gradient is exactly 0
  const bool bwd_tc = want_bwd && tc;
  L->off_keep = take(bwd_tc ? static_cast<size_t>(L->Rp) * 4 : 0);
  L->off_oidx2 = take(bwd_tc ? static_cast<size_t>(L->Rp) * 4 : 0);
  L->off_st2 = take(bwd_tc ? static_cast<size_t>(ceil_div(L->Rp, H1_TILE_ROWS)) * 8 : 0);
  L->off_dz2 = take(bwd_tc ? static_cast<size_t>(L->Rp) * L->Vp * 2 : 0);
  L->off_hc2 = take(bwd_tc ? static_cast<size_t>(L->Rp) * h * 2 : 0);
  L->total = o;
  return true;
}

static bool head_ok(const rl_head* hd) {
  if (!hd) return false;
  if (hd->hidden < 1 || hd->hidden > 65536 || hd->vocab < 1 || hd->vocab > (1 << 24)) return false;
  if (hd->ld_hidden < hd->hidden) return false;
  if (hd->dtype != RL_F32 && hd->dtype != RL_BF16) return false;
  if (!(hd->inv_temperature > 0.f) || !std::isfinite(hd->inv_temperature)) return false;
  if (hd->dtype == RL_F32 && hd->hidden > 12288) return false;  // SIMT smem row cache
  if (use_tc(hd) && (hd->hidden % 64 != 0 || hd->ld_hidden % 8 != 0)) return false;
  if (hd->vocab_total != 0) {  // vocab shard [offset, offset + vocab) of vocab_total
    if (hd->vocab_total < 0 || hd->vocab_total >= (int64_t(1) << 31) || hd->vocab_offset < 0 ||
        hd->vocab_offset + hd->vocab > hd->vocab_total)
      return false;
  }
  return true;
}

static bool batch_ok(const rl_batch* b) {
  if (!b) return false;
  if (b->num_rows < 0 || b->num_rows >= (int64_t(1) << 31) - 256) return false;
  if (b->num_seqs < 0 || !b->cu_seqlens) return false;
  if (b->num_rows > 0 && (!b->targets || !b->mask)) return false;
  return true;
}

static bool aligned(const void* p, size_t a) {
  return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0;
}

}  // namespace rlh

using namespace rlh;

extern "C" {

size_t rl_workspace_size(const rl_head* hd, int64_t num_rows, int32_t want_bwd) {
  if (!head_ok(hd) || num_rows < 0) return 0;
  if (want_bwd < 0 || want_bwd > 2) return 0;
  WsLayout L;
  ws_layout(hd, num_rows, want_bwd == 1, &L);
  return want_bwd == 2 ? L.prep_total : L.total;
}

rl_status rl_batch_prepare(const rl_head* hd, const rl_batch* b, int32_t* row_seq,
                           int32_t* active_idx, int64_t* n_active, int64_t* n_accum,
                           int64_t* nseq_accum, void* ws, size_t ws_bytes, rl_stream_t stream) {
  if (!head_ok(hd) || !batch_ok(b)) return RL_ERR_INVALID_ARG;
  WsLayout L;
  ws_layout(hd, b->num_rows, 0, &L);
  if (!ws || ws_bytes < L.prep_total) return RL_ERR_WORKSPACE;
  if (!aligned(ws, 256)) return RL_ERR_INVALID_ARG;
  return launch_prepare(hd, b, L, static_cast<char*>(ws), row_seq, active_idx, n_active, n_accum,
                        nseq_accum, nullptr, nullptr, nullptr,
                        reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"

// Forward (H1, H3, H4). parts_out == NULL: finish the softmax locally into
// logp/entropy/lse; else write this vocab shard's merged partials.
static rl_status fwd_impl(const rl_head* hd, const void* hidden, const void* weight,
                          const rl_batch* b, float* logp, float* entropy, float* lse,
                          float* parts_out, void* ws, size_t ws_bytes, rl_stream_t stream) {
  if (!head_ok(hd) || !batch_ok(b) || !weight || (!logp && !parts_out)) return RL_ERR_INVALID_ARG;
  if (b->num_rows > 0 && !hidden) return RL_ERR_INVALID_ARG;
  WsLayout L;
  ws_layout(hd, b->num_rows, 0, &L);
  if (!ws || ws_bytes < L.total) return RL_ERR_WORKSPACE;
  if (!aligned(ws, 256)) return RL_ERR_INVALID_ARG;
  const bool tc = use_tc(hd);
  if (tc && (!aligned(hidden, 16) || !aligned(weight, 16))) return RL_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(ws);
  rl_status st = launch_prepare(hd, b, L, w, nullptr, nullptr, nullptr, nullptr, nullptr, logp,
                                entropy, lse, s);
  if (st != RL_OK) return st;
  if (tc) {
    if ((st = launch_gather_bf16(hd, hidden, L, w, s)) != RL_OK) return st;
    if ((st = launch_tc_fwd(hd, weight, L, w, s)) != RL_OK) return st;
  } else {
    if ((st = launch_simt_fwd(hd, hidden, weight, L, w, s)) != RL_OK) return st;
  }
  MergeArgs a{};
  a.pm = reinterpret_cast<const float*>(w + L.off_pm);
  a.ps = reinterpret_cast<const float*>(w + L.off_ps);
  a.pu = reinterpret_cast<const float*>(w + L.off_pu);
  a.zy = reinterpret_cast<const float*>(w + L.off_zy);
  a.active_idx = reinterpret_cast<const int32_t*>(w + L.off_active);
  a.seq_c = reinterpret_cast<const int32_t*>(w + L.off_seq);
  if (parts_out) {
    a.parts_out = parts_out;
    a.ldo = b->num_rows;
    a.tgt_c = reinterpret_cast<const int32_t*>(w + L.off_tgt);
    a.y_off = hd->vocab_total > 0 ? hd->vocab_offset : 0;
    a.v_shard = hd->vocab;
  } else {
    a.logp = logp;
    a.entropy = entropy;
    a.lse = lse;
  }
  return launch_merge(L, w, a, s);
}

// MergeArgs reading P gathered shard partials parts_all [P][4][R].
static void gathered_parts(MergeArgs& a, const float* parts_all, int32_t nparts, int64_t R,
                           const WsLayout& L, char* w) {
  a.pm = parts_all;
  a.ps = parts_all + R;
  a.pu = parts_all + 2 * R;
  a.nparts = nparts;
  a.part_stride = 4 * R;
  a.zy = reinterpret_cast<const float*>(w + L.off_zy);  // filled by launch_zy_combine
  a.active_idx = reinterpret_cast<const int32_t*>(w + L.off_active);
  a.seq_c = reinterpret_cast<const int32_t*>(w + L.off_seq);
}

extern "C" {

rl_status rl_logprob_fwd(const rl_head* hd, const void* hidden, const void* weight,
                         const rl_batch* b, float* logp, float* entropy, float* lse, void* ws,
                         size_t ws_bytes, rl_stream_t stream) {
  if (!logp) return RL_ERR_INVALID_ARG;
  return fwd_impl(hd, hidden, weight, b, logp, entropy, lse, nullptr, ws, ws_bytes, stream);
}

rl_status rl_logprob_partials(const rl_head* hd, const void* hidden, const void* weight,
                              const rl_batch* b, float* parts, void* ws, size_t ws_bytes,
                              rl_stream_t stream) {
  if (!parts) return RL_ERR_INVALID_ARG;
  return fwd_impl(hd, hidden, weight, b, nullptr, nullptr, nullptr, parts, ws, ws_bytes, stream);
}

rl_status rl_logprob_merge(const rl_head* hd, const rl_batch* b, const float* parts_all,
                           int32_t nparts, float* logp, float* entropy, float* lse, void* ws,
                           size_t ws_bytes, rl_stream_t stream) {
  if (!head_ok(hd) || !batch_ok(b) || !logp || nparts < 1) return RL_ERR_INVALID_ARG;
  if (b->num_rows > 0 && !parts_all) return RL_ERR_INVALID_ARG;
  WsLayout L;
  ws_layout(hd, b->num_rows, 0, &L);
  if (!ws || ws_bytes < L.total) return RL_ERR_WORKSPACE;
  if (!aligned(ws, 256)) return RL_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(ws);
  rl_status st = launch_prepare(hd, b, L, w, nullptr, nullptr, nullptr, nullptr, nullptr, logp,
                                entropy, lse, s);
  if (st != RL_OK) return st;
  if ((st = launch_zy_combine(parts_all, nparts, b->num_rows, L, w, s)) != RL_OK) return st;
  MergeArgs a{};
  gathered_parts(a, parts_all, nparts, b->num_rows, L, w);
  a.logp = logp;
  a.entropy = entropy;
  a.lse = lse;
  return launch_merge(L, w, a, s);
}

rl_status rl_grpo_group_stats(const float* rewards, const int32_t* group_of_seq, int32_t num_seqs,
                              int32_t num_groups, double* sum_stats, double* max_stats,
                              int32_t* err_flags, rl_stream_t stream) {
  if (num_seqs < 0 || num_groups < 0 || !sum_stats || !max_stats) return RL_ERR_INVALID_ARG;
  if (num_seqs > 0 && (!rewards || !group_of_seq)) return RL_ERR_INVALID_ARG;
  return launch_grpo(rewards, group_of_seq, num_seqs, num_groups, nullptr, nullptr, 0.f, 1,
                     nullptr, sum_stats, max_stats, err_flags,
                     reinterpret_cast<cudaStream_t>(stream));
}

rl_status rl_grpo_advantage(const float* rewards, const int32_t* group_of_seq, int32_t num_seqs,
                            int32_t num_groups, const double* sum_stats, const double* max_stats,
                            float eps, int32_t unbiased, float* adv, int32_t* err_flags,
                            rl_stream_t stream) {
  if (num_seqs < 0 || num_groups < 0 || !(eps >= 0.f)) return RL_ERR_INVALID_ARG;
  if (num_seqs > 0 && (!rewards || !group_of_seq || !adv)) return RL_ERR_INVALID_ARG;
  if ((sum_stats == nullptr) != (max_stats == nullptr)) return RL_ERR_INVALID_ARG;
  return launch_grpo(rewards, group_of_seq, num_seqs, num_groups, sum_stats, max_stats, eps,
                     unbiased, adv, nullptr, nullptr, err_flags,
                     reinterpret_cast<cudaStream_t>(stream));
}

rl_status rl_read_device_error(const int32_t* err_flags, int32_t* host_code,
                               rl_stream_t stream) {
  if (!err_flags || !host_code) return RL_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (cudaMemcpyAsync(host_code, err_flags, sizeof(int32_t), cudaMemcpyDeviceToHost, s) !=
          cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return RL_ERR_CUDA;
  return RL_OK;
}

rl_status rl_batch_norm_advantage(const float* rewards, const int32_t* group_of_seq,
                                  int32_t num_seqs, int32_t num_groups, int32_t group_baseline,
                                  const double* group_sum_stats, const double* batch_stats_in,
                                  double* batch_stats_out, float eps, int32_t unbiased,
                                  float* adv, int32_t* err_flags, rl_stream_t stream) {
  if (num_seqs < 0 || num_groups < 0 || !(eps >= 0.f)) return RL_ERR_INVALID_ARG;
  if (group_baseline != 0 && group_baseline != 1) return RL_ERR_INVALID_ARG;
  if (group_baseline && (!group_of_seq || !group_sum_stats)) return RL_ERR_INVALID_ARG;
  if (!adv && !batch_stats_out) return RL_ERR_INVALID_ARG;
  if (num_seqs > 0 && !rewards) return RL_ERR_INVALID_ARG;
  return launch_batch_adv(rewards, group_of_seq, num_seqs, num_groups, group_baseline,
                          group_sum_stats, batch_stats_in, batch_stats_out, eps, unbiased, adv,
                          err_flags, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"

// Training-worker path (H1-H8). parts_all == NULL: the softmax is finished
// from this call's own forward GEMM; else (vocab-parallel) from the P
// gathered shard partials, and the backward covers this shard only.
static rl_status loss_impl(const rl_head* hd, const void* hidden, const void* weight,
                           const rl_batch* b, const float* parts_all, int32_t nparts,
                           const float* old_logp, const float* adv, const rl_loss_params* p,
                           float* logp, float* entropy, void* grad_hidden, float* grad_weight,
                           rl_loss_stats* stats, void* ws, size_t ws_bytes, rl_stream_t stream,
                           int gh_mode = 0, int phase = 3) {
  // phase bit 1: H1-H5 (forward, loss, dL/dlogp, stats); bit 2: H6-H8 (dZ, dH,
  // dW) from the state the forward left in ws (same arguments for both).
  const bool gh_f32 = gh_mode != 0, gh_mc = gh_mode == 2;
  if (!head_ok(hd) || !batch_ok(b) || !weight || !p || !logp || !grad_weight)
    return RL_ERR_INVALID_ARG;
  if (parts_all && nparts < 1) return RL_ERR_INVALID_ARG;
  if (b->num_rows > 0 && (!hidden || !old_logp || !grad_hidden)) return RL_ERR_INVALID_ARG;
  if (b->num_seqs > 0 && !adv) return RL_ERR_INVALID_ARG;
  if (!(p->clip_lo >= 0.f) || !(p->clip_lo < 1.f) || !(p->clip_hi >= 0.f) ||
      !(p->logratio_clamp > 0.f) || !std::isfinite(p->loss_scale))
    return RL_ERR_INVALID_ARG;
  if (!(p->dual_clip == 0.f || p->dual_clip > 1.f) || !(p->kl_coef >= 0.f) ||
      !(p->entropy_coef >= 0.f) || (p->seq_mean != 0 && p->seq_mean != 1) ||
      (p->adv_per_token != 0 && p->adv_per_token != 1))
    return RL_ERR_INVALID_ARG;
  if (p->adv_per_token && b->num_rows > 0 && !adv) return RL_ERR_INVALID_ARG;
  if (p->kl_coef > 0.f && b->num_rows > 0 && !p->ref_logp) return RL_ERR_INVALID_ARG;
  const rl_peer_group* rs = p->dw_reduce_scatter;
  if (rs) {
    if (rs->world < 1 || rs->world > 8 || rs->rank < 0 || rs->rank >= rs->world ||
        rs->rows_per_rank <= 0 || rs->rows_per_rank * rs->world < hd->vocab)
      return RL_ERR_INVALID_ARG;
    for (int q = 0; q < rs->world; ++q)
      if (!rs->peers[q] || !aligned(rs->peers[q], 16)) return RL_ERR_INVALID_ARG;
  }
  const bool entropy_on = p->entropy_coef > 0.f;
  WsLayout L;
  ws_layout(hd, b->num_rows, 1, &L);
  // q mode (default on the tensor-core path): the forward also stores the
  // tile-normalised softmax q, and dZ is built from it by one HBM pass instead
  // of recomputing the logits (the entropy bonus needs z itself, and the
  // vocab-parallel call has no forward GEMM: both keep the recompute).
  // RLHEAD_DZ_RECOMPUTE=1 forces the recompute GEMM.
  const bool q_mode = use_tc(hd) && !parts_all && !entropy_on && !dz_recompute();
  // skip mode (q mode, default): the backward GEMMs run only over the rows with
  // dL/dlogp != 0 -- GRPO groups whose rewards are all equal (A = 0), clipped
  // and padding rows have dZ = 0 and contribute exactly nothing to dH / dW.
  // RLHEAD_BWD_SKIP=0 keeps every active row.
  const bool skip_rows = q_mode && bwd_skip();
  // fused backward (RLHEAD_DZ_FUSED=1; token-mean GRPO without KL): the rows
  // of A = 0 sequences are moved behind the others before the forward, so the
  // backward covers a prefix of the compact rows in place (no packed copies)
  const bool fused_dz = skip_rows && dz_fused() && p->kl_coef == 0.f && !p->seq_mean &&
                        !p->adv_per_token;
  const int bwd_rows = fused_dz ? BWD_PREFIX : skip_rows ? BWD_PACKED : BWD_DENSE;
  if (!ws || ws_bytes < L.total) return RL_ERR_WORKSPACE;
  if (!aligned(ws, 256)) return RL_ERR_INVALID_ARG;
  const bool tc = use_tc(hd);
  // fp32 dL/dH rows [R, hidden]: native for fp32 heads (ld must be hidden),
  // the tensor-core path's EPI_ROWS fp32 store for bf16 heads.
  if (gh_f32 && (hd->dtype == RL_BF16 ? !tc : hd->ld_hidden != hd->hidden))
    return RL_ERR_INVALID_ARG;
  if (gh_mc && !tc) return RL_ERR_INVALID_ARG;
  if (rs && !tc) return RL_ERR_INVALID_ARG;
  if (tc && (!aligned(hidden, 16) || !aligned(weight, 16) || !aligned(grad_hidden, 16) ||
             !aligned(grad_weight, 16)))
    return RL_ERR_INVALID_ARG;
  if (phase < 1 || phase > 3) return RL_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(ws);
  rl_status st = RL_OK;
  // grad_hidden rows of inactive rows := 0 (from H1's active flags). Not in
  // multicast mode: the caller pre-zeroed every copy; plain stores to a
  // multicast address are not allowed, and inactive rows receive no adds.
  const bool zero_gh = (phase & 2) && !gh_mc;
  if (phase == 2) {  // backward only: the forward's state is in ws
    if (zero_gh &&
        (st = launch_zero_inactive(hd, grad_hidden, L, w, s, gh_f32, skip_rows)) != RL_OK)
      return st;
    if (q_mode && (st = launch_dz_from_q(hd, L, w, s, bwd_rows)) != RL_OK) return st;
    if (tc)
      return launch_tc_bwd(hd, weight, gh_f32 ? nullptr : grad_hidden,
                           gh_f32 ? static_cast<float*>(grad_hidden) : nullptr, gh_mc,
                           grad_weight, rs, entropy_on, L, w, s, q_mode, bwd_rows);
    return launch_simt_bwd(hd, hidden, weight, grad_hidden, grad_weight, entropy_on, L, w, s);
  }
  st = launch_prepare(hd, b, L, w, nullptr, nullptr, nullptr, nullptr, nullptr, logp, entropy,
                      nullptr, s);
  if (st != RL_OK) return st;
  if (fused_dz && (st = launch_partition_rows(L, w, adv, s)) != RL_OK) return st;
  if (zero_gh &&
      (st = launch_zero_inactive(hd, grad_hidden, L, w, s, gh_f32, skip_rows)) != RL_OK)
    return st;
  if (tc && (st = launch_gather_bf16(hd, hidden, L, w, s)) != RL_OK) return st;
  MergeArgs a{};
  if (parts_all) {
    if ((st = launch_zy_combine(parts_all, nparts, b->num_rows, L, w, s)) != RL_OK) return st;
    gathered_parts(a, parts_all, nparts, b->num_rows, L, w);
  } else {
    if (tc) {
      // with no KL term, A = 0 means dL/dlogp = 0: those rows' q is never read
      const bool adv_gate = skip_rows && p->kl_coef == 0.f;
      if ((st = launch_tc_fwd(hd, weight, L, w, s, q_mode, adv_gate ? adv : nullptr,
                              p->adv_per_token != 0)) != RL_OK)
        return st;
    } else {
      if ((st = launch_simt_fwd(hd, hidden, weight, L, w, s)) != RL_OK) return st;
    }
    a.pm = reinterpret_cast<const float*>(w + L.off_pm);
    a.ps = reinterpret_cast<const float*>(w + L.off_ps);
    a.pu = reinterpret_cast<const float*>(w + L.off_pu);
    a.zy = reinterpret_cast<const float*>(w + L.off_zy);
    a.active_idx = reinterpret_cast<const int32_t*>(w + L.off_active);
    a.seq_c = reinterpret_cast<const int32_t*>(w + L.off_seq);
  }
  a.logp = logp;
  a.entropy = entropy;
  a.lse = nullptr;
  a.old_logp = old_logp;
  a.adv = adv;
  a.clip_lo = p->clip_lo;
  a.clip_hi = p->clip_hi;
  a.clamp_c = p->logratio_clamp;
  a.loss_scale = p->loss_scale;
  a.n_global = p->n_tokens_global;
  a.dual_clip = p->dual_clip;
  a.kl_coef = p->kl_coef;
  a.entropy_coef = p->entropy_coef;
  a.seq_mean = p->seq_mean;
  a.adv_per_token = p->adv_per_token;
  a.ref_logp = p->kl_coef > 0.f ? p->ref_logp : nullptr;
  a.n_seqs_global = p->n_seqs_global;
  a.cu_seqlens = b->cu_seqlens;
  a.g_c = reinterpret_cast<float*>(w + L.off_g);
  a.lse_c = reinterpret_cast<float*>(w + L.off_lse);
  a.ge_c = entropy_on ? reinterpret_cast<float*>(w + L.off_ge) : nullptr;
  a.ez_c = entropy_on ? reinterpret_cast<float*>(w + L.off_ez) : nullptr;
  a.st_d = reinterpret_cast<double*>(w + L.off_st_d);
  a.st_f = reinterpret_cast<float*>(w + L.off_st_f);
  a.st_i = reinterpret_cast<long long*>(w + L.off_st_i);
  if ((st = launch_merge(L, w, a, s)) != RL_OK) return st;
  if ((st = launch_stats_reduce(L, w, stats, s)) != RL_OK) return st;
  if (!(phase & 2)) return RL_OK;
  if (q_mode && (st = launch_dz_from_q(hd, L, w, s, bwd_rows)) != RL_OK) return st;
  if (tc)
    return launch_tc_bwd(hd, weight, gh_f32 ? nullptr : grad_hidden,
                         gh_f32 ? static_cast<float*>(grad_hidden) : nullptr, gh_mc,
                         grad_weight, rs, entropy_on, L, w, s, q_mode, bwd_rows);
  return launch_simt_bwd(hd, hidden, weight, grad_hidden, grad_weight, entropy_on, L, w, s);
}

extern "C" {

rl_status rl_policy_loss_fwd_bwd(const rl_head* hd, const void* hidden, const void* weight,
                                 const rl_batch* b, const float* old_logp, const float* adv,
                                 const rl_loss_params* p, float* logp, float* entropy,
                                 void* grad_hidden, float* grad_weight, rl_loss_stats* stats,
                                 void* ws, size_t ws_bytes, rl_stream_t stream) {
  return loss_impl(hd, hidden, weight, b, nullptr, 0, old_logp, adv, p, logp, entropy,
                   grad_hidden, grad_weight, stats, ws, ws_bytes, stream);
}

rl_status rl_policy_loss_fwd(const rl_head* hd, const void* hidden, const void* weight,
                             const rl_batch* b, const float* old_logp, const float* adv,
                             const rl_loss_params* p, float* logp, float* entropy,
                             void* grad_hidden, float* grad_weight, rl_loss_stats* stats,
                             void* ws, size_t ws_bytes, rl_stream_t stream) {
  return loss_impl(hd, hidden, weight, b, nullptr, 0, old_logp, adv, p, logp, entropy,
                   grad_hidden, grad_weight, stats, ws, ws_bytes, stream, 0, 1);
}

rl_status rl_policy_loss_bwd(const rl_head* hd, const void* hidden, const void* weight,
                             const rl_batch* b, const float* old_logp, const float* adv,
                             const rl_loss_params* p, float* logp, float* entropy,
                             void* grad_hidden, float* grad_weight, rl_loss_stats* stats,
                             void* ws, size_t ws_bytes, rl_stream_t stream) {
  return loss_impl(hd, hidden, weight, b, nullptr, 0, old_logp, adv, p, logp, entropy,
                   grad_hidden, grad_weight, stats, ws, ws_bytes, stream, 0, 2);
}

rl_status rl_policy_loss_fwd_bwd_vp(const rl_head* hd, const void* hidden, const void* weight,
                                    const rl_batch* b, const float* parts_all, int32_t nparts,
                                    const float* old_logp, const float* adv,
                                    const rl_loss_params* p, float* logp, float* entropy,
                                    void* grad_hidden, int32_t grad_hidden_fp32,
                                    float* grad_weight, rl_loss_stats* stats, void* ws,
                                    size_t ws_bytes, rl_stream_t stream) {
  if (b && b->num_rows > 0 && !parts_all) return RL_ERR_INVALID_ARG;
  if (nparts < 1 || grad_hidden_fp32 < 0 || grad_hidden_fp32 > 2) return RL_ERR_INVALID_ARG;
  return loss_impl(hd, hidden, weight, b, parts_all, nparts, old_logp, adv, p, logp, entropy,
                   grad_hidden, grad_weight, stats, ws, ws_bytes, stream, grad_hidden_fp32);
}

rl_status rl_loss_stats_reduce(const rl_loss_stats* gathered, int32_t nranks,
                               rl_loss_stats* out, rl_stream_t stream) {
  if (!gathered || !out || nranks < 1) return RL_ERR_INVALID_ARG;
  return launch_stats_ranks(gathered, nranks, out, reinterpret_cast<cudaStream_t>(stream));
}

const char* rl_status_string(rl_status s) {
  switch (s) {
    case RL_OK: return "RL_OK";
    case RL_ERR_INVALID_ARG: return "RL_ERR_INVALID_ARG";
    case RL_ERR_UNSUPPORTED: return "RL_ERR_UNSUPPORTED";
    case RL_ERR_WORKSPACE: return "RL_ERR_WORKSPACE";
    case RL_ERR_CUDA: return "RL_ERR_CUDA";
  }
  return "RL_ERR_UNKNOWN";
}

const char* rl_build_info(void) {
  return "librlhead sm_100a (tcgen05/TMEM/TMA bf16 head; fp32 CUDA-core head), CUDA "
#ifdef __CUDACC_VER_MAJOR__
      "nvcc"
#endif
      ;
}

int64_t rl_launch_count(void) { return g_launches.load(); }

rl_status rl_trace_begin(int32_t capacity_launches) {
  if (capacity_launches < 1 || capacity_launches > (1 << 20)) return RL_ERR_INVALID_ARG;
  const int32_t capacity_events = 2 * capacity_launches;
  std::lock_guard<std::mutex> lk(g_tr.mu);
  if (static_cast<int>(g_tr.ev.size()) < capacity_events) {
    const size_t old = g_tr.ev.size();
    g_tr.ev.resize(capacity_events);
    for (size_t i = old; i < g_tr.ev.size(); ++i)
      if (cudaEventCreate(&g_tr.ev[i]) != cudaSuccess) return RL_ERR_CUDA;
  }
  g_tr.kinds.clear();
  g_tr.n = 0;
  g_tr.pending = false;
  g_tr.on = true;
  return RL_OK;
}

int32_t rl_trace_end(int32_t* kinds) {
  std::lock_guard<std::mutex> lk(g_tr.mu);
  g_tr.on = false;
  if (kinds)
    for (int i = 0; i < g_tr.n; ++i) kinds[i] = g_tr.kinds[i];
  return g_tr.n;
}

// Durations (ms) of the launches traced by the last rl_trace_begin/end pair;
// waits for the recorded events. Returns the number written.
int32_t rl_trace_durations(float* ms, int32_t cap) {
  std::lock_guard<std::mutex> lk(g_tr.mu);
  const int n = g_tr.n < cap ? g_tr.n : cap;
  for (int i = 0; i < n; ++i) {
    cudaEventSynchronize(g_tr.ev[2 * i + 1]);
    float t = 0.f;
    cudaEventElapsedTime(&t, g_tr.ev[2 * i], g_tr.ev[2 * i + 1]);
    ms[i] = t;
  }
  return n;
}

}  // extern "C"
