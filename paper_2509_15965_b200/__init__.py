"""B200-native (sm_100a) GRPO policy-loss head -- the data-parallel hot path of
RLinf's inference and training workers (arXiv 2509.15965).

The compute lives in ``librlhead.so`` (CUDA, include/rlhead.h); this package is
its thin ctypes binding (``rlhead``) plus the host-side data-parallel driver
(``dp``: micro-batch packing, LPT sharding, NCCL collectives).
"""
from .rlhead import (  # noqa: F401
    Batch, Head, LossParams, PeerGroup, Trace, Workspace, RLHeadError, new_stats, read_stats,
    rl_batch_prepare, rl_build_info, rl_grpo_advantage, rl_grpo_group_stats,
    rl_launch_count, rl_logprob_fwd, rl_policy_loss_fwd_bwd, rl_workspace_size,
    rl_logprob_partials, rl_logprob_merge, rl_policy_loss_fwd_bwd_vp,
    rl_minibatch_early_stop, rl_scale_by_inverse_count, rl_gae, rl_value_loss_fwd_bwd,
    rl_allreduce_sum_f32, rl_reduce_bcast_rows_f32, rl_dw_reduce_rows_f32, rl_cast_rows_bf16, rl_batch_norm_advantage,
    rl_read_device_error, rl_loss_stats_reduce, rl_policy_loss_fwd, rl_policy_loss_bwd,
    RL_DEVERR_CU_SEQLENS, RL_DEVERR_GROUP, RL_DEVERR_TARGET, KERNEL_KINDS, EXPORTED,
)
