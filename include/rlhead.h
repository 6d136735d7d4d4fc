/*
 * rlhead.h -- C ABI of the B200 (sm_100a) GRPO policy-loss head.
 *
 * The token-level policy-loss head that RLinf's inference worker (old/ref
 * log-probs) and training worker (policy update,
 * P:L181) run on every micro-batch: LM-head projection
 * Z = tau^-1 H W^T, online log-sum-exp over the vocabulary, target gather
 * (log-prob, entropy), GRPO group-relative advantages (P:L178-179,
 * P:L388-391), the masked clipped-ratio surrogate with token-level averaging
 * and its backward dL/dH, dL/dW. Formulas: DESIGN.md §2 (O.1);
 * readings of what the paper leaves open: DESIGN.md §3.
 *
 * Conventions for every call:
 *   - Pointers are DEVICE pointers unless the comment says "host".
 *   - Calls are asynchronous and stream-ordered on `stream` (a cudaStream_t;
 *     NULL = legacy default stream). No call allocates device memory,
 *     synchronises the stream or keeps state between calls; all scratch lives
 *     in the caller's workspace `ws` (size from rl_workspace_size).
 *   - The caller owns every buffer. Outputs are overwritten unless marked
 *     "accumulated (+=)".
 *   - Host-side argument errors return RL_ERR_* with NOTHING launched.
 *   - Data errors found on the device (bad cu_seqlens, target or group id)
 *     are OR-ed into the optional device word `err_flags` (RL_DEVERR_*) and
 *     the offending rows/sequences are treated as inactive; no host sync.
 *   - Re-entrant: concurrent calls on different streams are legal when their
 *     outputs and workspaces are disjoint. The workspace also holds the
 *     tensor-core GEMMs' tile-scheduler counters; every launch
 *     leaves them at zero (and the bookkeeping pass zeroes them), so a
 *     workspace carries no state from one call to the next, but one
 *     workspace must never be used by two calls in flight at once.
 */
#ifndef RLHEAD_H
#define RLHEAD_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define RL_API __attribute__((visibility("default")))
#else
#define RL_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *rl_stream_t; /* == cudaStream_t */

typedef enum {
  RL_OK = 0,
  RL_ERR_INVALID_ARG = 1, /* null/negative/misaligned argument, nothing launched */
  RL_ERR_UNSUPPORTED = 2, /* valid but unsupported shape/dtype on this build/device */
  RL_ERR_WORKSPACE = 3,   /* ws NULL or ws_bytes < rl_workspace_size(...) */
  RL_ERR_CUDA = 4         /* a CUDA runtime/driver call failed */
} rl_status;

typedef enum { RL_F32 = 0, RL_BF16 = 1 } rl_dtype;

/* Device error word bits (err_flags). */
#define RL_DEVERR_CU_SEQLENS 1 /* cu[0]!=0, decreasing, or cu[S]!=num_rows: ALL rows inactive */
#define RL_DEVERR_TARGET 2     /* mask!=0 row with target outside [0,V): that row inactive */
#define RL_DEVERR_GROUP 4      /* group id outside [0,num_groups): that sequence gets A=0 */

/* Packed ragged micro-batch (BASELINE.json north_star: "packed variable-
 * length sequences with a response mask and group ids").
 * Row t belongs to sequence s iff cu_seqlens[s] <= t < cu_seqlens[s+1].
 * Row t is ACTIVE iff the batch is well formed, mask[t] != 0 and
 * 0 <= targets[t] < vocab. Active rows are processed in packed order. */
typedef struct {
  int64_t num_rows;          /* R >= 0: packed rows incl. prompt rows          */
  int32_t num_seqs;          /* S >= 0                                          */
  const int32_t *cu_seqlens; /* [S+1]                                           */
  const int32_t *targets;    /* [R] token id predicted by row t (pre-shifted)   */
  const uint8_t *mask;       /* [R] != 0: response token that carries the loss  */
  int32_t *err_flags;        /* optional device int32, RL_DEVERR_* OR-ed in     */
} rl_batch;

/* The LM head (host struct). hidden is [num_rows, ld_hidden] row-major of
 * `dtype`; weight is W[vocab, hidden] row-major (nn.Linear layout), same
 * dtype, densely packed (row stride = hidden). logits = inv_temperature*H W^T.
 * RL_BF16 runs the tcgen05/TMEM/TMA tensor-core path and needs hidden % 64
 * == 0 and ld_hidden % 8 == 0; RL_F32 runs the exact-fp32 CUDA-core path.
 * Vocab-parallel head (NEXT-3, tensor parallelism as the paper's actor TP,
 * P:L783): `weight` holds rows [vocab_offset, vocab_offset + vocab) of a
 * vocab_total-row head; targets stay GLOBAL ids in [0, vocab_total).
 * vocab_total = 0 means unsharded (vocab_total = vocab, offset 0). */
typedef struct {
  int32_t hidden;        /* h  (1..65536)                                      */
  int32_t vocab;         /* V  (1..2^24): rows of `weight` on this rank         */
  rl_dtype dtype;        /* RL_F32 | RL_BF16                                   */
  int64_t ld_hidden;     /* row stride of hidden / grad_hidden in elements >= h */
  float inv_temperature; /* tau^-1 > 0 (1 = plain softmax)                     */
  int64_t vocab_offset;  /* first global vocab id held by `weight` (sharded)   */
  int64_t vocab_total;   /* full vocabulary (0 = unsharded)                    */
} rl_head;

/* Workspace bytes for a call on up to `num_rows` packed rows: want_bwd = 0
 * for rl_logprob_fwd / the vocab-parallel calls, 1 for rl_policy_loss_fwd_bwd
 * (+ _fwd / _bwd / _vp), 2 for rl_batch_prepare alone (bookkeeping only,
 * ~21 B/row). The backward's share on the tensor-core path is dominated by two
 * bf16 [rows, V] buffers (the forward's q / dZ, and the dZ of the rows with a
 * gradient packed densely): ~4 V B per row, ~10 GB at 16k rows and V = 152k.
 * 0 if the head or want_bwd is invalid. */
RL_API size_t rl_workspace_size(const rl_head *hd, int64_t num_rows, int32_t want_bwd);

/* H1 bookkeeping alone (it also runs inside the two head calls).
 * row_seq [R] (out, may be NULL): sequence of row t, -1 on a malformed batch.
 * active_idx [R] (out, may be NULL): active rows in packed order; entries
 *   at and beyond n_active are left unspecified.
 * n_active (device int64, out, may be NULL): number of active rows.
 * n_accum (device int64, ACCUMULATED +=, may be NULL): for the loss
 *   normaliser N summed over micro-batches/ranks (DESIGN.md §3 #13).
 * nseq_accum (device int64, ACCUMULATED +=, may be NULL): sequences with at
 *   least one active row -- the normaliser S of seq-mean aggregation. */
RL_API rl_status rl_batch_prepare(const rl_head *hd, const rl_batch *b, int32_t *row_seq,
                           int32_t *active_idx, int64_t *n_active, int64_t *n_accum,
                           int64_t *nseq_accum, void *ws, size_t ws_bytes,
                           rl_stream_t stream);

/* Inference-worker call: per-row log-prob of the
 * target, entropy (nats) and log-sum-exp of tau^-1 H W^T over the full V.
 * logp/entropy/lse are [R] fp32 (entropy, lse may be NULL); 0 on inactive
 * rows. Full logits never reach HBM. */
RL_API rl_status rl_logprob_fwd(const rl_head *hd, const void *hidden, const void *weight,
                         const rl_batch *b, float *logp, float *entropy, float *lse,
                         void *ws, size_t ws_bytes, rl_stream_t stream);

/* GRPO group statistics (normalisation aggregates all responses
 * of a query). Over sequences with a valid group id:
 *   sum_stats[g] = (n_g, sum r, sum r^2)   fp64 [num_groups][3], out
 *   max_stats[g] = (max r, -min r)         fp64 [num_groups][2], out
 * Empty groups give (0,0,0) and (-inf,-inf). Split groups across DP ranks
 * all-reduce these (SUM / MAX) before rl_grpo_advantage. */
RL_API rl_status rl_grpo_group_stats(const float *rewards, const int32_t *group_of_seq,
                              int32_t num_seqs, int32_t num_groups, double *sum_stats,
                              double *max_stats, int32_t *err_flags, rl_stream_t stream);

/* GRPO advantage per sequence (formula DESIGN.md §3 #5-#8):
 *   A_s = (r_s - mu_g) / (sigma_g + eps),  sigma over n-1 (unbiased != 0) or n,
 *   A_s = 0 exactly when n_g <= 1 or max_g r == min_g r, or the group id is
 *   invalid (RL_DEVERR_GROUP).
 * sum_stats/max_stats: NULL = compute the group statistics from this call's
 * rewards (all members local); else use the given (all-reduced) ones.
 * adv [num_seqs] fp32 out. */
RL_API rl_status rl_grpo_advantage(const float *rewards, const int32_t *group_of_seq,
                            int32_t num_seqs, int32_t num_groups, const double *sum_stats,
                            const double *max_stats, float eps, int32_t unbiased, float *adv,
                            int32_t *err_flags, rl_stream_t stream);

/* Debug helper (the only call that synchronises): copy the device error word
 * err_flags (RL_DEVERR_* bits, OR-ed by the calls that were given it) into
 * *host_code after everything queued on `stream` has finished. */
RL_API rl_status rl_read_device_error(const int32_t *err_flags, int32_t *host_code,
                                      rl_stream_t stream);

/* REINFORCE++-style batch-normalised advantage (NEXT-1; P:L654 names
 * REINFORCE++, no formula; DESIGN.md §3 #33):
 *   x_s = r_s - mu_g(s)  if group_baseline (mu_g = n_g^-1 sum r from
 *                         group_sum_stats, as rl_grpo_group_stats writes it,
 *                         all-reduced if groups are split), else x_s = r_s;
 *   A_s = (x_s - mean_B x) / (std_B x + eps) over the batch's sequences with a
 *         valid group id (std over n-1 if unbiased else n); A_s = 0 exactly
 *         when n <= 1 or max x == min x, and for invalid ids (RL_DEVERR_GROUP;
 *         group_of_seq may be NULL without baseline: every sequence valid).
 * Batch statistics fp64 [5] = (n, sum x, sum x^2, max x, -min x):
 *   batch_stats_out != NULL: this call's local statistics are written there
 *     (multi-rank: call with adv = NULL, all-reduce SUM [0:3] / MAX [3:5],
 *     then call again with batch_stats_in);
 *   batch_stats_in != NULL: A uses these instead of the local ones.
 * adv [num_seqs] fp32 out (may be NULL when only statistics are wanted). */
RL_API rl_status rl_batch_norm_advantage(const float *rewards, const int32_t *group_of_seq,
                                         int32_t num_seqs, int32_t num_groups,
                                         int32_t group_baseline, const double *group_sum_stats,
                                         const double *batch_stats_in, double *batch_stats_out,
                                         float eps, int32_t unbiased, float *adv,
                                         int32_t *err_flags, rl_stream_t stream);

/* Loss parameters (host struct; DESIGN.md §3 #12-#15, NEXT-1 variants
 * #25-#28). Per active token t of sequence s with weight w_t:
 *   L += w_t (l_t + kl_coef * k3_t - entropy_coef * H_t)
 *   l_t  = max(-A r, -A clip(r, 1-clip_lo, 1+clip_hi)), and for A < 0 with
 *          dual_clip > 1: min(l_t, -A dual_clip)  (gradient 0 if r > dual_clip)
 *   k3_t = e^q - q - 1, q = clamp(ref_logp_t - logp_t, -c, c)
 *   w_t  = 1/N (token mean)  or, if seq_mean != 0,
 *          1/(S n_s) with n_s the active tokens of s (seq-mean-token-mean).
 * 1/N (1/S) comes from n_tokens_global (n_seqs_global) when given, else
 * loss_scale is used in its place (streaming mode). */
typedef struct {
  float clip_lo;                  /* eps_lo: ratio clipped below at 1 - eps_lo (0.2) */
  float clip_hi;                  /* eps_hi: ratio clipped above at 1 + eps_hi (0.2) */
  float logratio_clamp;           /* c: d = logp - old clamped to [-c, c] (20)       */
  double loss_scale;              /* used when the device normaliser is NULL         */
  const int64_t *n_tokens_global; /* device: N (all micro-batches, all ranks);
                                     scale = 1/N (0 if N == 0)                      */
  float dual_clip;                /* 0 = off, else > 1                               */
  float kl_coef;                  /* beta >= 0; > 0 needs ref_logp                   */
  float entropy_coef;             /* c_ent >= 0 (entropy bonus)                      */
  int32_t seq_mean;               /* 0 token mean, 1 seq-mean-token-mean             */
  const float *ref_logp;          /* [R] device: reference-policy log-probs          */
  const int64_t *n_seqs_global;   /* device: S (seq_mean); see rl_batch_prepare      */
  int32_t adv_per_token;          /* 0: adv is [S] per sequence (GRPO); 1: adv is [R]
                                     per row (PPO/GAE, NEXT-4)                        */
  const struct rl_peer_group *dw_reduce_scatter; /* NULL: grad_weight += locally.
                                     Else (the LAST micro-batch of a mini-batch on
                                     every DP rank; bf16 tensor-core path): partial +
                                     this micro-batch go to the owners' staging
                                     buffers instead, see rl_peer_group                */
} rl_loss_params;

/* DP reduction of dW fused into the last micro-batch's dW GEMM (C3 of
 * SURVEY §8(e)). Vocab rows are owned in slabs:
 * owner(j) = min(j / rows_per_rank, world - 1), rows_per_rank * world >= V.
 * Every rank has a staging buffer float [world][rows_per_rank][h] that all
 * ranks have mapped (symmetric memory; peers[q] = rank q's). With
 * params->dw_reduce_scatter set, the dW epilogue stores, for every finished
 * tile, (this rank's accumulated grad_weight partial + the tile) into slot
 * [rank][j - owner*rows_per_rank] of the OWNER's staging buffer over NVLink
 * (plain stores; a rank whose micro-batch has no active row still sends its
 * partial), so the reduce-scatter runs tile by tile under the GEMM. The
 * local grad_weight is read, not updated. After the call returned on every
 * rank and a cross-rank barrier, rl_reduce_bcast_rows_f32 on every rank sums
 * its slab's `world` slots in rank order (deterministic) and broadcasts the
 * sum into every rank's dW buffer (all-reduce). bf16 tensor-core path only. */
typedef struct rl_peer_group {
  int32_t rank;                   /* this rank in the group                          */
  int32_t world;                  /* 1..8                                            */
  int64_t rows_per_rank;          /* > 0, rows_per_rank * world >= vocab             */
  float *peers[8];                /* device: every rank's staging buffer             */
  int32_t no_partial;             /* 1: grad_weight holds no partial yet (this is the
                                     rank's only micro-batch of the mini-batch): the
                                     epilogue sends the tile alone, grad_weight is
                                     not read. 0: partial + tile                      */
} rl_peer_group;

/* Loss statistics, device resident, ACCUMULATED (+=) by every call. The
 * caller zeroes it at the start of a mini-batch. Raw sums over active rows:
 * loss_sum = sum l_t, kl_sum = sum k3_t, objective = sum w_t(l_t + beta k3_t
 * - c_ent H_t) (this call's share of L). clip_hi_count = #{A>0, r>1+eps_hi},
 * clip_lo_count = #{A<0, r<1-eps_lo}; ratio_max feeds the minibatch
 * early-stop. */
typedef struct {
  double loss_sum;
  double ratio_sum;
  double entropy_sum;
  double kl_sum;
  double objective;
  float ratio_max;
  int32_t reserved;
  int64_t clip_lo_count;
  int64_t clip_hi_count;
  int64_t tokens;
} rl_loss_stats;

/* Training-worker call: forward + backward of the masked clipped-ratio
 * token-mean loss on one micro-batch (micro-batch = fwd/bwd unit).
 *   old_logp [R] fp32, adv [S] fp32 (one per sequence, broadcast to its rows),
 *   logp [R] / entropy [R] fp32 out (entropy may be NULL), 0 on inactive rows,
 *   grad_hidden [R, ld_hidden] out, dtype of hidden, 0 on inactive rows,
 *   grad_weight [V, h] fp32 ACCUMULATED (+=): zero it once per mini-batch,
 *   stats (device, may be NULL) ACCUMULATED.
 * g_t = dL/dlogp_t = w_t(-A r [unclipped][|d| <= c] + beta (1 - e^q));
 * dZ = tau^-1 (g (onehot - p) + w c_ent p (z - E_p z)); dH = dZ W;
 * dW += dZ^T H. Logits are recomputed in the backward instead of stored. */
RL_API rl_status rl_policy_loss_fwd_bwd(const rl_head *hd, const void *hidden, const void *weight,
                                 const rl_batch *b, const float *old_logp, const float *adv,
                                 const rl_loss_params *p, float *logp, float *entropy,
                                 void *grad_hidden, float *grad_weight, rl_loss_stats *stats,
                                 void *ws, size_t ws_bytes, rl_stream_t stream);

/* rl_loss_stats_reduce: *out := the combination of nranks rl_loss_stats
 * gathered from the DP ranks (device array gathered[nranks], e.g. one NCCL
 * all-gather of the 72-B struct): the fp64/int64 fields summed in rank
 * order (deterministic), ratio_max the maximum. Replaces three all-reduces
 * (SUM fp64, MAX fp32, SUM int64) by one all-gather.
 * out may not alias gathered. RL_ERR_INVALID_ARG: null pointer or
 * nranks < 1 (nothing launched). */
RL_API rl_status rl_loss_stats_reduce(const rl_loss_stats *gathered, int32_t nranks,
                                      rl_loss_stats *out, rl_stream_t stream);

/* Split form of rl_policy_loss_fwd_bwd, for pipelining micro-batches (same
 * arguments for both calls, same ws, stream-ordered fwd before bwd):
 * rl_policy_loss_fwd runs H1-H5 -- bookkeeping, projection with the online
 * LSE (and, on the tensor-core path, the tile-normalised softmax q into ws),
 * loss, dL/dlogp, stats -- writing logp/entropy/stats and leaving the
 * backward's state in ws; rl_policy_loss_bwd runs H6-H8 from that state --
 * dZ (from q, or by recomputing the logits), dL/dH, dW += -- writing
 * grad_hidden and accumulating grad_weight. fwd + bwd on one stream is
 * bit-identical to rl_policy_loss_fwd_bwd. Between the two calls ws belongs
 * to this micro-batch; another micro-batch may run in another workspace on
 * another stream (e.g. bwd(i)'s memory-bound dZ pass beside fwd(i+1)'s GEMM).
 * Errors as rl_policy_loss_fwd_bwd (both calls validate every argument). */
RL_API rl_status rl_policy_loss_fwd(const rl_head *hd, const void *hidden, const void *weight,
                                    const rl_batch *b, const float *old_logp, const float *adv,
                                    const rl_loss_params *p, float *logp, float *entropy,
                                    void *grad_hidden, float *grad_weight, rl_loss_stats *stats,
                                    void *ws, size_t ws_bytes, rl_stream_t stream);
RL_API rl_status rl_policy_loss_bwd(const rl_head *hd, const void *hidden, const void *weight,
                                    const rl_batch *b, const float *old_logp, const float *adv,
                                    const rl_loss_params *p, float *logp, float *entropy,
                                    void *grad_hidden, float *grad_weight, rl_loss_stats *stats,
                                    void *ws, size_t ws_bytes, rl_stream_t stream);

/* ---- mini-batch update control (NEXT-2) ---------------------------------
 * rl_minibatch_early_stop: "discard minibatches with too large importance
 * ratio" (DESIGN.md §3 #29). From the (all-reduced) device stats:
 * stop = (max_ratio > 0 && ratio_max > max_ratio) ||
 *        (max_mean_ratio > 0 && tokens > 0 && ratio_sum / tokens > max_mean_ratio);
 * *stop_flag (device int32) = stop; if stop, grad_weight[0..n) := 0.
 * rl_scale_by_inverse_count: x[0..n) *= 1/count (0 if count == 0), count a
 * device int64 -- the deferred 1/N of micro-batches run with loss_scale = 1
 * before N was known (elastic pipelining). x 16-B aligned. */
RL_API rl_status rl_minibatch_early_stop(const rl_loss_stats *stats, float max_ratio,
                                         float max_mean_ratio, int32_t *stop_flag,
                                         float *grad_weight, int64_t n, rl_stream_t stream);
RL_API rl_status rl_scale_by_inverse_count(float *x, int64_t n, const int64_t *count,
                                           rl_stream_t stream);

/* ---- PPO pieces (NEXT-4; DESIGN.md §3 #30-#32) --------------------------
 * rl_gae: generalised advantage estimation over packed trajectories
 * (embodied PPO; the RLHF critic). Trajectory s owns steps
 * [cu_steps[s], cu_steps[s+1]); per step t: rewards, values, dones (uint8,
 * may be NULL = none); bootstrap[s] (may be NULL = 0) is V after the last step.
 *   delta_t = r_t + gamma (1-done_t) V_{t+1} - V_t
 *   A_t = delta_t + gamma lam (1-done_t) A_{t+1};  returns_t = A_t + V_t.
 * fp64 recurrence, fp32 outputs. */
RL_API rl_status rl_gae(const float *rewards, const float *values, const uint8_t *dones,
                        const float *bootstrap, const int32_t *cu_steps, int32_t num_traj,
                        float gamma, float lam, float *adv, float *returns, rl_stream_t stream);

/* Value head v_t = <w_v, h_t> + b_v on the rows with mask != 0 and the PPO
 * clipped value loss L_v = scale * sum_t 0.5 max((v-R)^2, (clip(v, v_old-eps,
 * v_old+eps)-R)^2), scale = 1/N (n_tokens_global) or loss_scale.
 *   values [R] out (0 on other rows); grad_hidden [R, ld] ACCUMULATED (+=,
 *   add the value head's dL/dh to the policy's); grad_w [h] fp32 and grad_b
 *   [1] fp32 (may be NULL) ACCUMULATED; stats (may be NULL) accumulate
 *   loss_sum, objective, clip_hi_count (= clipped-branch tokens), tokens.
 * hidden and w_v share hd->dtype; ws from rl_value_workspace_size. */
typedef struct {
  float clip_eps;                 /* eps_v >= 0                                     */
  double loss_scale;              /* used when n_tokens_global is NULL              */
  const int64_t *n_tokens_global; /* device: N                                       */
} rl_value_params;
RL_API size_t rl_value_workspace_size(int32_t hidden, int64_t num_rows);
RL_API rl_status rl_value_loss_fwd_bwd(const rl_head *hd, const void *hidden, const void *w_v,
                                       float b_v, const rl_batch *b, const float *returns,
                                       const float *old_values, const rl_value_params *p,
                                       float *values, void *grad_hidden, float *grad_w,
                                       float *grad_b, rl_loss_stats *stats, void *ws,
                                       size_t ws_bytes, rl_stream_t stream);

/* ---- vocab-parallel head (NEXT-3) ----------------------
 * A vocab shard cannot finish the log-sum-exp alone. Phase 1 on every rank:
 *   rl_logprob_partials -> parts [4][num_rows] fp32 for THIS shard, in compact
 *   (active-row) order: (m, s = sum e^{z-m}, u = sum e^{z-m}(z-m), z_y or 0
 *   when the target is not in this shard); entries >= n_active unspecified.
 * The caller all-gathers parts over the TP group -> parts_all [P][4][num_rows]
 * (P shards, any order). Phase 2, on every rank:
 *   rl_logprob_merge            -> logp / entropy / lse (full vocabulary), or
 *   rl_policy_loss_fwd_bwd_vp   -> as rl_policy_loss_fwd_bwd, with the softmax
 *     over all shards; grad_hidden is this shard's PARTIAL dL/dH (the caller
 *     all-reduces SUM over the TP group), grad_weight this shard's rows of
 *     dL/dW (accumulated). logp/entropy/stats are identical on every rank of
 *     the TP group (do not sum stats over TP ranks). grad_hidden_fp32:
 *     0: grad_hidden in hd->dtype with row stride hd->ld_hidden (above);
 *     1: grad_hidden is float [num_rows][hidden] (row stride = hidden) -- the
 *        partial dL/dH in fp32, e.g. straight into a symmetric NVLink buffer
 *        for rl_allreduce_sum_f32; bf16 heads need the tensor-core path, fp32
 *        heads ld_hidden == hidden;
 *     2: as 1, but grad_hidden is the NVLS MULTICAST address of a symmetric
 *        fp32 buffer that the caller zeroed on every rank (then barriered):
 *        the dL/dH GEMM epilogue adds each tile into every rank's copy through
 *        the switch (multimem.red.add), so after the call on all ranks (and a
 *        barrier) every copy holds the TP sum -- the all-reduce fused into the
 *        GEMM. bf16 tensor-core path only.
 *     Other values / unsupported combinations: RL_ERR_INVALID_ARG. */
RL_API rl_status rl_logprob_partials(const rl_head *hd, const void *hidden, const void *weight,
                                     const rl_batch *b, float *parts, void *ws, size_t ws_bytes,
                                     rl_stream_t stream);
RL_API rl_status rl_logprob_merge(const rl_head *hd, const rl_batch *b, const float *parts_all,
                                  int32_t nparts, float *logp, float *entropy, float *lse,
                                  void *ws, size_t ws_bytes, rl_stream_t stream);
RL_API rl_status rl_policy_loss_fwd_bwd_vp(const rl_head *hd, const void *hidden,
                                           const void *weight, const rl_batch *b,
                                           const float *parts_all, int32_t nparts,
                                           const float *old_logp, const float *adv,
                                           const rl_loss_params *p, float *logp, float *entropy,
                                           void *grad_hidden, int32_t grad_hidden_fp32,
                                           float *grad_weight, rl_loss_stats *stats, void *ws,
                                           size_t ws_bytes, rl_stream_t stream);

/* ---- sum over NVLink peer memory ----------------------
 * The exchange step after a GEMM on the sharded path -- the vocab-parallel
 * SUM of the partial dL/dH (H7 summed over vocab shards: dL/dH = sum_p dZ_p
 * W_p) -- done by one kernel over a symmetric buffer that every rank of the
 * group has mapped, no NCCL. buf holds n floats on each rank; on return
 * (after the caller's next cross-rank barrier) every rank's buf holds the
 * element-wise sum over the `world` ranks.
 *   mc_ptr != NULL: the NVLS multicast address of buf (NVSwitch SHARP):
 *     rank r sums slice r through the switch (multimem.ld_reduce.add) and
 *     multicasts it back (multimem.st); peer_ptrs is ignored. Rounding order
 *     is the switch's.
 *   mc_ptr == NULL: peer_ptrs[q] (a HOST array of `world` device pointers,
 *     peer_ptrs[rank] = the local buf) are the P2P mappings; rank r loads
 *     slice r from every peer in rank order 0..world-1 (deterministic) and
 *     stores the sum to every peer.
 * The caller brackets the call with cross-rank barriers (all partials written
 * before; all slices stored after). n % 4 == 0, pointers 16-B aligned,
 * 1 <= world <= 8, else RL_ERR_INVALID_ARG; world == 1 is a no-op. */
RL_API rl_status rl_allreduce_sum_f32(float *const *peer_ptrs, float *mc_ptr, int32_t rank,
                                      int32_t world, int64_t n, rl_stream_t stream);
/* Owner side of the fused DP dW reduce-scatter (rl_peer_group): rank `rank`
 * owns rows [rank*rows_per_rank, min((rank+1)*rows_per_rank, num_rows)) of
 * the [num_rows][cols] fp32 dW; out[row] = sum over q = 0..world-1 (in this
 * order) of staging[q][row - rank*rows_per_rank] (staging = this rank's
 * [world][rows_per_rank][cols] buffer), stored into EVERY rank's output --
 * multimem.st through the multicast address out_mc when given, else plain
 * stores to out_peers (HOST array of world device pointers; entries other
 * than out_peers[rank] may be NULL and are skipped -- with only the own entry
 * set the call leaves a sharded gradient, each rank holding its summed rows,
 * as FSDP / ZeRO-2 gradient reduce-scatter does). Bracket with
 * cross-rank barriers. cols % 4 == 0, 16-B aligned pointers. */
RL_API rl_status rl_reduce_bcast_rows_f32(const float *staging, float *const *out_peers,
                                          float *out_mc, int32_t rank, int32_t world,
                                          int64_t num_rows, int64_t cols, int64_t rows_per_rank,
                                          rl_stream_t stream);
/* DP dW SUM after the last micro-batch's dW GEMM, without staging (C3 of SURVEY
 * §8(e), collective "nvls"). Every rank's [num_rows][cols] fp32
 * dW lives in a buffer that all ranks have mapped: peer_ptrs[q] (HOST array of
 * world device pointers, peer_ptrs[rank] = the local one). Rank `rank` owns
 * rows [rank*rows_per_rank, min((rank+1)*rows_per_rank, num_rows)) (the
 * owner(j) rule of rl_peer_group) and sums them over the ranks:
 *   mc_ptr != NULL: multimem.ld_reduce.add through the NVLS multicast address
 *     of the buffer (the switch adds the world copies; its rounding order);
 *   mc_ptr == NULL: loads from every peer in rank order 0..world-1
 *     (deterministic).
 * broadcast != 0: the sum is stored into every rank's buffer (multimem.st, or
 * P2P stores) -- every rank ends with the whole reduced dW. broadcast == 0:
 * only into this rank's own buffer (a sharded gradient as FSDP / ZeRO-2
 * reduce-scatter leaves it; the other rows keep this rank's own partial).
 * Bracket with cross-rank barriers (all dW GEMMs done before; all sums stored
 * after). cols % 4 == 0, 16-B aligned pointers, 1 <= world <= 8, else
 * RL_ERR_INVALID_ARG. */
RL_API rl_status rl_dw_reduce_rows_f32(float *const *peer_ptrs, float *mc_ptr, int32_t rank,
                                       int32_t world, int64_t num_rows, int64_t cols,
                                       int64_t rows_per_rank, int32_t broadcast,
                                       rl_stream_t stream);

/* dst[t][0:hidden] (bf16, row stride ld) = round-to-nearest(src[t][0:hidden])
 * (fp32, row stride hidden), t < num_rows; hidden even, ld >= hidden even. */
RL_API rl_status rl_cast_rows_bf16(const float *src, int64_t num_rows, int32_t hidden, void *dst,
                                   int64_t ld, rl_stream_t stream);

/* ---- introspection / tracing (P:L682-690 worker timers, device-side) ---- */
RL_API const char *rl_status_string(rl_status s);
RL_API const char *rl_build_info(void);
/* Number of kernels this library has launched since it was loaded. */
RL_API int64_t rl_launch_count(void);

/* Kernel kinds reported by the tracer. */
typedef enum {
  RL_K_PREPARE = 0, RL_K_GATHER = 1, RL_K_GEMM_LSE = 2, RL_K_MERGE = 3,
  RL_K_GEMM_DZ = 4, RL_K_GEMM_DH = 5, RL_K_GEMM_DW = 6, RL_K_GRPO = 7,
  RL_K_SIMT_FWD = 8, RL_K_SIMT_BWD = 9, RL_K_REDUCE = 10, RL_K_MISC = 11,
  RL_K_GEMM_DHDW = 12, /* fused dH + dW launch (two GEMMs of 2hV flop/token each) */
  RL_K_DZQ = 13,       /* dZ from the forward's q tiles (HBM pass replacing the recompute) */
  RL_K_NUM_KINDS = 14
} rl_kernel_kind;

/* Tracing (not thread-safe; for benchmarks, cf. the worker-group timers of
 * P:L682-690). While active, every launch is bracketed by cudaEventRecord on
 * its own stream (events owned by the library, created on first use).
 * rl_trace_end stops tracing, writes the kind of each traced launch into
 * kinds[0..n) (host, may be NULL) and returns n. rl_trace_durations then
 * waits for those events and writes each launch's device time in ms
 * (host array, up to cap entries). Launches beyond capacity_launches are
 * counted by rl_launch_count but not traced. */
RL_API rl_status rl_trace_begin(int32_t capacity_launches);
RL_API int32_t rl_trace_end(int32_t *kinds);
RL_API int32_t rl_trace_durations(float *ms, int32_t cap);

#ifdef __cplusplus
}
#endif
#endif /* RLHEAD_H */
