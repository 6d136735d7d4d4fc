// Internal launchers of librlhead (host side). Each returns RL_OK or
// RL_ERR_CUDA and launches through TraceScope.
#pragma once
#include "common.cuh"

namespace rlh {

// H1 bookkeeping: validate cu_seqlens, per-row flags/row_seq, block scan,
// compaction into active_idx/tgt_c/seq_c (all in ws unless user pointers
// given). Zeroes zero0..2 [R] (fp32, may be NULL) on inactive rows.
rl_status launch_prepare(const rl_head* hd, const rl_batch* b, const WsLayout& L, char* ws,
                         int32_t* row_seq_user, int32_t* active_idx_user, int64_t* n_active_user,
                         int64_t* n_accum, int64_t* nseq_accum, float* zero0, float* zero1,
                         float* zero2, cudaStream_t s);
// Compact bf16 rows Hc[r] = hidden[active_idx[r]], zero rows up to the tile.
rl_status launch_gather_bf16(const rl_head* hd, const void* hidden, const WsLayout& L, char* ws,
                             cudaStream_t s);
// grad_hidden rows of inactive rows := 0.
// all_rows: zero every row (skip mode: dH writes only the rows with g != 0).
rl_status launch_zero_inactive(const rl_head* hd, void* grad_hidden, const WsLayout& L, char* ws,
                               cudaStream_t s, bool f32_rows = false, bool all_rows = false);

// H2 GRPO.
rl_status launch_grpo(const float* rewards, const int32_t* gos, int32_t S, int32_t G,
                      const double* sum_in, const double* max_in, float eps, int32_t unbiased,
                      float* adv, double* sum_out, double* max_out, int32_t* err,
                      cudaStream_t s);
rl_status launch_batch_adv(const float* rewards, const int32_t* gos, int32_t S, int32_t G,
                           int32_t group_baseline, const double* gsum, const double* bin,
                           double* bout, float eps, int32_t unbiased, float* adv, int32_t* err,
                           cudaStream_t s);

// H4 merge of the split-V partials (+ H5 loss when old_logp != NULL).
struct MergeArgs {
  // partial n of compact row r: part_stride > 0: [n * part_stride + r] (the
  // gathered vocab-parallel parts); part_stride == 0: this call's own split-V
  // partials, row-blocked [((r >> 5) * nparts + n) * 32 + (r & 31)]
  const float *pm, *ps, *pu, *zy;
  int64_t nparts, part_stride;
  const int32_t *active_idx, *seq_c;
  float *logp, *entropy, *lse;          // row space, may be NULL
  // vocab-parallel phase 1: write this shard's merged (m, s, u, zy-or-0) to
  // parts_out[k * ldo + r] instead of logp/entropy/lse
  float* parts_out;
  int64_t ldo;
  const int32_t* tgt_c;
  int64_t y_off, v_shard;
  // loss
  const float* old_logp;                // row space; NULL = fwd only
  const float* adv;                     // per sequence
  float clip_lo, clip_hi, clamp_c;
  double loss_scale;
  const int64_t* n_global;
  // NEXT-1 variants
  float dual_clip, kl_coef, entropy_coef;
  int32_t seq_mean;
  int32_t adv_per_token;                // adv indexed by row (PPO) instead of sequence
  const float* ref_logp;                // row space
  const int64_t* n_seqs_global;
  const int32_t* cu_seqlens;            // for n_s (seq_mean)
  float *g_c, *lse_c;                   // compact, for the backward
  float *ge_c, *ez_c;                   // compact: w c_ent and E_p[z] (entropy bonus)
  double* st_d;                         // [nblk][5] loss, ratio, entropy, kl, objective
  float* st_f;                          // [nblk] ratio max
  long long* st_i;                      // [nblk][3] clip_lo, clip_hi, tokens
};
rl_status launch_merge(const WsLayout& L, char* ws, const MergeArgs& a, cudaStream_t s);
// zy[r] = sum_p parts_all[p][3][r] (exactly one shard holds the target).
rl_status launch_zy_combine(const float* parts_all, int64_t nparts, int64_t ldr,
                            const WsLayout& L, char* ws, cudaStream_t s);
rl_status launch_stats_reduce(const WsLayout& L, char* ws, rl_loss_stats* stats, cudaStream_t s);
rl_status launch_stats_ranks(const rl_loss_stats* gathered, int32_t n, rl_loss_stats* out,
                             cudaStream_t s);

// CUDA-core path (fp32 exact; also bf16 for cross-checks).
rl_status launch_simt_fwd(const rl_head* hd, const void* hidden, const void* weight,
                          const WsLayout& L, char* ws, cudaStream_t s);
rl_status launch_simt_bwd(const rl_head* hd, const void* hidden, const void* weight,
                          void* grad_hidden, float* grad_weight, bool entropy_on,
                          const WsLayout& L, char* ws, cudaStream_t s);

// Tensor-core path (bf16, tcgen05/TMEM/TMA).
// q_out: the epilogue also stores q = e^{z - m_tile} (bf16, 0 at the target)
// into the dZ buffer for launch_dz_from_q.
// q_adv (with q_out): advantages per sequence (per packed row if
// q_adv_per_row); a warp's 32 rows that all have A = 0 store no q (skip mode
// never reads them back). NULL: store every box.
rl_status launch_tc_fwd(const rl_head* hd, const void* weight, const WsLayout& L, char* ws,
                        cudaStream_t s, bool q_out = false, const float* q_adv = nullptr,
                        bool q_adv_per_row = false);
// dZ = tau^-1 g (onehot - p) in place over the q tiles of launch_tc_fwd(q_out):
// p = q e^{m_tile - lse} off the target, 1 - p_y = -expm1(z_y - lse) at it.
// Which rows the backward GEMMs (and the dZ pass) cover:
//  BWD_DENSE  every active row, dZ in place, Hc as gathered (hdr->n_active);
//  BWD_PACKED the rows with dL/dlogp != 0, packed by k_keep_compact into the
//             dz2 / hc2 buffers (hdr->n_bwd; rows with g = 0 add exactly nothing);
//  BWD_PREFIX the prefix [0, hdr->n_bwd) of the compact rows after
//             launch_partition_rows (A != 0 rows first): dZ in place, Hc as is.
enum { BWD_DENSE = 0, BWD_PACKED = 1, BWD_PREFIX = 2 };
rl_status launch_dz_from_q(const rl_head* hd, const WsLayout& L, char* ws, cudaStream_t s,
                           int bwd_rows = BWD_DENSE);
// Fused-backward mode: reorder the compact rows (A != 0 first, A = 0 tail);
// hdr->n_bwd = the prefix length. Run after H1, before the gather.
rl_status launch_partition_rows(const WsLayout& L, char* ws, const float* adv, cudaStream_t s);
// grad_hidden_f32 != NULL: dL/dH as fp32 rows [R, hidden] there instead of
// bf16 rows into grad_hidden; gh_multicast: grad_hidden_f32 is an NVLS
// multicast address and the rows are added into every rank's copy.
rl_status launch_tc_bwd(const rl_head* hd, const void* weight, void* grad_hidden,
                        float* grad_hidden_f32, bool gh_multicast, float* grad_weight,
                        const rl_peer_group* dw_rs, bool entropy_on, const WsLayout& L, char* ws,
                        cudaStream_t s, bool dz_ready = false, int bwd_rows = BWD_DENSE);

int num_sms();

}  // namespace rlh
