"""ctypes binding of librlhead.so (include/rlhead.h): argument marshalling only.

Every function here has the C name and forwards torch tensors as raw device
pointers plus the current CUDA stream; all arithmetic runs in the library's
CUDA kernels. There is no CPU fallback: importing this module fails loudly
when librlhead.so is missing (build it with ``python
paper_2509_15965_b200/build.py`` or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "librlhead.so")
if not os.path.exists(_LIB_PATH):
    raise ImportError(f"librlhead.so not built at {_LIB_PATH}; run `python "
                      "paper_2509_15965_b200/build.py` (no CPU fallback exists)")
lib = C.CDLL(_LIB_PATH)

RL_OK, RL_ERR_INVALID_ARG, RL_ERR_UNSUPPORTED, RL_ERR_WORKSPACE, RL_ERR_CUDA = range(5)
RL_F32, RL_BF16 = 0, 1
RL_DEVERR_CU_SEQLENS, RL_DEVERR_TARGET, RL_DEVERR_GROUP = 1, 2, 4
KERNEL_KINDS = ["prepare", "gather", "gemm_lse", "merge", "gemm_dz", "gemm_dh", "gemm_dw",
                "grpo", "simt_fwd", "simt_bwd", "reduce", "misc", "gemm_dhdw", "dz_from_q"]
# tensor flops per token of each GEMM kind, in units of 2 h V
GEMM_FLOP_UNITS = {"gemm_lse": 1, "gemm_dz": 1, "gemm_dh": 1, "gemm_dw": 1, "gemm_dhdw": 2}


class rl_batch(C.Structure):
    _fields_ = [("num_rows", C.c_int64), ("num_seqs", C.c_int32), ("cu_seqlens", C.c_void_p),
                ("targets", C.c_void_p), ("mask", C.c_void_p), ("err_flags", C.c_void_p)]


class rl_head(C.Structure):
    _fields_ = [("hidden", C.c_int32), ("vocab", C.c_int32), ("dtype", C.c_int),
                ("ld_hidden", C.c_int64), ("inv_temperature", C.c_float),
                ("vocab_offset", C.c_int64), ("vocab_total", C.c_int64)]


class rl_peer_group(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("rows_per_rank", C.c_int64),
                ("peers", C.c_void_p * 8), ("no_partial", C.c_int32)]


class rl_loss_params(C.Structure):
    _fields_ = [("clip_lo", C.c_float), ("clip_hi", C.c_float), ("logratio_clamp", C.c_float),
                ("loss_scale", C.c_double), ("n_tokens_global", C.c_void_p),
                ("dual_clip", C.c_float), ("kl_coef", C.c_float), ("entropy_coef", C.c_float),
                ("seq_mean", C.c_int32), ("ref_logp", C.c_void_p), ("n_seqs_global", C.c_void_p),
                ("adv_per_token", C.c_int32), ("dw_reduce_scatter", C.POINTER(rl_peer_group))]


class rl_value_params(C.Structure):
    _fields_ = [("clip_eps", C.c_float), ("loss_scale", C.c_double),
                ("n_tokens_global", C.c_void_p)]


class rl_loss_stats(C.Structure):
    _fields_ = [("loss_sum", C.c_double), ("ratio_sum", C.c_double), ("entropy_sum", C.c_double),
                ("kl_sum", C.c_double), ("objective", C.c_double), ("ratio_max", C.c_float), ("reserved", C.c_int32), ("clip_lo_count", C.c_int64),
                ("clip_hi_count", C.c_int64), ("tokens", C.c_int64)]


STATS_BYTES = C.sizeof(rl_loss_stats)
_vp, _sz = C.c_void_p, C.c_size_t

lib.rl_workspace_size.restype = C.c_size_t
lib.rl_workspace_size.argtypes = [C.POINTER(rl_head), C.c_int64, C.c_int32]
lib.rl_batch_prepare.restype = C.c_int
lib.rl_batch_prepare.argtypes = [C.POINTER(rl_head), C.POINTER(rl_batch), _vp, _vp, _vp, _vp,
                                 _vp, _vp, _sz, _vp]
lib.rl_logprob_fwd.restype = C.c_int
lib.rl_logprob_fwd.argtypes = [C.POINTER(rl_head), _vp, _vp, C.POINTER(rl_batch), _vp, _vp, _vp,
                               _vp, _sz, _vp]
lib.rl_grpo_group_stats.restype = C.c_int
lib.rl_grpo_group_stats.argtypes = [_vp, _vp, C.c_int32, C.c_int32, _vp, _vp, _vp, _vp]
lib.rl_grpo_advantage.restype = C.c_int
lib.rl_grpo_advantage.argtypes = [_vp, _vp, C.c_int32, C.c_int32, _vp, _vp, C.c_float, C.c_int32,
                                  _vp, _vp, _vp]
lib.rl_batch_norm_advantage.restype = C.c_int
lib.rl_batch_norm_advantage.argtypes = [_vp, _vp, C.c_int32, C.c_int32, C.c_int32, _vp, _vp, _vp,
                                        C.c_float, C.c_int32, _vp, _vp, _vp]
lib.rl_read_device_error.restype = C.c_int
lib.rl_read_device_error.argtypes = [_vp, C.POINTER(C.c_int32), _vp]
lib.rl_policy_loss_fwd_bwd.restype = C.c_int
lib.rl_policy_loss_fwd_bwd.argtypes = [C.POINTER(rl_head), _vp, _vp, C.POINTER(rl_batch), _vp,
                                       _vp, C.POINTER(rl_loss_params), _vp, _vp, _vp, _vp, _vp,
                                       _vp, _sz, _vp]
for _fn in (lib.rl_policy_loss_fwd, lib.rl_policy_loss_bwd):
    _fn.restype = C.c_int
    _fn.argtypes = lib.rl_policy_loss_fwd_bwd.argtypes
lib.rl_logprob_partials.restype = C.c_int
lib.rl_logprob_partials.argtypes = [C.POINTER(rl_head), _vp, _vp, C.POINTER(rl_batch), _vp, _vp,
                                    _sz, _vp]
lib.rl_logprob_merge.restype = C.c_int
lib.rl_logprob_merge.argtypes = [C.POINTER(rl_head), C.POINTER(rl_batch), _vp, C.c_int32, _vp,
                                 _vp, _vp, _vp, _sz, _vp]
lib.rl_policy_loss_fwd_bwd_vp.restype = C.c_int
lib.rl_policy_loss_fwd_bwd_vp.argtypes = [C.POINTER(rl_head), _vp, _vp, C.POINTER(rl_batch), _vp,
                                          C.c_int32, _vp, _vp, C.POINTER(rl_loss_params), _vp,
                                          _vp, _vp, C.c_int32, _vp, _vp, _vp, _sz, _vp]
lib.rl_allreduce_sum_f32.restype = C.c_int
lib.rl_allreduce_sum_f32.argtypes = [C.POINTER(C.c_void_p), _vp, C.c_int32, C.c_int32, C.c_int64,
                                     _vp]
lib.rl_reduce_bcast_rows_f32.restype = C.c_int
lib.rl_reduce_bcast_rows_f32.argtypes = [_vp, C.POINTER(C.c_void_p), _vp, C.c_int32, C.c_int32,
                                         C.c_int64, C.c_int64, C.c_int64, _vp]
lib.rl_dw_reduce_rows_f32.restype = C.c_int
lib.rl_dw_reduce_rows_f32.argtypes = [C.POINTER(C.c_void_p), _vp, C.c_int32, C.c_int32,
                                      C.c_int64, C.c_int64, C.c_int64, C.c_int32, _vp]
lib.rl_cast_rows_bf16.restype = C.c_int
lib.rl_cast_rows_bf16.argtypes = [_vp, C.c_int64, C.c_int32, _vp, C.c_int64, _vp]
lib.rl_minibatch_early_stop.restype = C.c_int
lib.rl_minibatch_early_stop.argtypes = [_vp, C.c_float, C.c_float, _vp, _vp, C.c_int64, _vp]
lib.rl_scale_by_inverse_count.restype = C.c_int
lib.rl_scale_by_inverse_count.argtypes = [_vp, C.c_int64, _vp, _vp]
lib.rl_gae.restype = C.c_int
lib.rl_gae.argtypes = [_vp, _vp, _vp, _vp, _vp, C.c_int32, C.c_float, C.c_float, _vp, _vp, _vp]
lib.rl_value_workspace_size.restype = C.c_size_t
lib.rl_value_workspace_size.argtypes = [C.c_int32, C.c_int64]
lib.rl_value_loss_fwd_bwd.restype = C.c_int
lib.rl_value_loss_fwd_bwd.argtypes = [C.POINTER(rl_head), _vp, _vp, C.c_float, C.POINTER(rl_batch),
                                      _vp, _vp, C.POINTER(rl_value_params), _vp, _vp, _vp, _vp,
                                      _vp, _vp, _sz, _vp]
lib.rl_loss_stats_reduce.restype = C.c_int
lib.rl_loss_stats_reduce.argtypes = [_vp, C.c_int32, _vp, _vp]
lib.rl_status_string.restype = C.c_char_p
lib.rl_status_string.argtypes = [C.c_int]
lib.rl_build_info.restype = C.c_char_p
lib.rl_launch_count.restype = C.c_int64
lib.rl_trace_begin.restype = C.c_int
lib.rl_trace_begin.argtypes = [C.c_int32]
lib.rl_trace_end.restype = C.c_int32
lib.rl_trace_end.argtypes = [_vp]
lib.rl_trace_durations.restype = C.c_int32
lib.rl_trace_durations.argtypes = [_vp, C.c_int32]

EXPORTED = ["rl_workspace_size", "rl_batch_prepare", "rl_logprob_fwd", "rl_grpo_group_stats",
            "rl_grpo_advantage", "rl_policy_loss_fwd_bwd", "rl_status_string", "rl_build_info",
            "rl_launch_count", "rl_trace_begin", "rl_trace_end", "rl_trace_durations",
            "rl_logprob_partials", "rl_logprob_merge", "rl_policy_loss_fwd_bwd_vp",
            "rl_minibatch_early_stop", "rl_scale_by_inverse_count", "rl_gae",
            "rl_value_workspace_size", "rl_value_loss_fwd_bwd", "rl_allreduce_sum_f32",
            "rl_cast_rows_bf16", "rl_batch_norm_advantage", "rl_read_device_error",
            "rl_reduce_bcast_rows_f32", "rl_loss_stats_reduce", "rl_policy_loss_fwd",
            "rl_policy_loss_bwd", "rl_dw_reduce_rows_f32"]


class RLHeadError(RuntimeError):
    pass


def _check(st: int, what: str):
    if st != RL_OK:
        raise RLHeadError(f"{what}: {lib.rl_status_string(st).decode()}")


def _ptr(t):
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())


def _stream(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


# ------------------------------------------------------------ descriptors ----
@dataclass
class Head:
    """rl_head: hidden size h, vocab V, dtype ('bf16' | 'f32'), ld_hidden, 1/tau."""
    hidden: int
    vocab: int                 # rows of the weight passed with this head (a shard if sharded)
    dtype: str = "bf16"
    ld_hidden: int | None = None
    inv_temperature: float = 1.0
    vocab_offset: int = 0      # vocab-parallel shard: first global id of `vocab` rows
    vocab_total: int = 0       # 0 = unsharded

    def c(self) -> rl_head:
        return rl_head(self.hidden, self.vocab, RL_BF16 if self.dtype == "bf16" else RL_F32,
                       self.ld_hidden or self.hidden, self.inv_temperature, self.vocab_offset,
                       self.vocab_total)


@dataclass
class Batch:
    """rl_batch over device tensors: cu_seqlens int32[S+1], targets int32[R],
    mask uint8[R], optional err_flags int32[1]."""
    cu_seqlens: object
    targets: object
    mask: object
    err_flags: object = None
    num_rows: int | None = None

    def c(self) -> rl_batch:
        R = self.num_rows if self.num_rows is not None else int(self.mask.shape[0])
        return rl_batch(R, int(self.cu_seqlens.shape[0]) - 1, _ptr(self.cu_seqlens),
                        _ptr(self.targets), _ptr(self.mask), _ptr(self.err_flags))


@dataclass
class LossParams:
    """rl_loss_params (include/rlhead.h); defaults = GRPO/DAPO token-mean loss."""
    clip_lo: float = 0.2
    clip_hi: float = 0.2
    logratio_clamp: float = 20.0
    loss_scale: float = 1.0
    n_tokens_global: object = None  # device int64[1] tensor: scale = 1/N
    dual_clip: float = 0.0
    kl_coef: float = 0.0
    entropy_coef: float = 0.0
    seq_mean: bool = False
    ref_logp: object = None         # device fp32 [R] (needed when kl_coef > 0)
    n_seqs_global: object = None    # device int64[1]: S for seq_mean
    adv_per_token: bool = False     # adv [R] per row (PPO/GAE) instead of [S]
    dw_reduce_scatter: object = None  # PeerGroup: fused DP dW reduce-scatter (last micro-batch)

    def c(self) -> rl_loss_params:
        pg = self.dw_reduce_scatter.c() if self.dw_reduce_scatter is not None else None
        p = rl_loss_params(self.clip_lo, self.clip_hi, self.logratio_clamp, self.loss_scale,
                           _ptr(self.n_tokens_global), self.dual_clip, self.kl_coef,
                           self.entropy_coef, int(bool(self.seq_mean)), _ptr(self.ref_logp),
                           _ptr(self.n_seqs_global), int(bool(self.adv_per_token)),
                           C.pointer(pg) if pg is not None else None)
        p._keep = pg                # keep the pointed-to struct alive with the params
        return p


@dataclass
class PeerGroup:
    """rl_peer_group: every rank's dW staging buffer [world, rows_per_rank, h]
    (symmetric memory) and the row-slab ownership of the fused dW
    reduce-scatter (include/rlhead.h)."""
    rank: int
    world: int
    rows_per_rank: int
    peers: list                     # device addresses (ints) of every rank's staging buffer
    no_partial: bool = False        # grad_weight holds no partial yet (only micro-batch)

    def c(self) -> rl_peer_group:
        arr = (C.c_void_p * 8)(*([int(x) for x in self.peers] + [0] * (8 - len(self.peers))))
        return rl_peer_group(int(self.rank), int(self.world), int(self.rows_per_rank), arr,
                             1 if self.no_partial else 0)


class Workspace:
    """A growable device scratch buffer (256-B aligned torch allocation)."""

    def __init__(self, device="cuda"):
        self.device = device
        self.buf = None

    def get(self, nbytes: int):
        import torch
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
        return self.buf


def new_stats(device="cuda"):
    """A zeroed device rl_loss_stats (as a uint8 tensor of sizeof bytes)."""
    import torch
    return torch.zeros(STATS_BYTES, dtype=torch.uint8, device=device)


def read_stats(t) -> dict:
    raw = t.detach().to("cpu").numpy().tobytes()
    s = rl_loss_stats.from_buffer_copy(raw)
    return {k: getattr(s, k) for k, _ in rl_loss_stats._fields_ if k != "reserved"}


# --------------------------------------------------------------- C calls ----
def rl_workspace_size(head: Head, num_rows: int, want_bwd) -> int:
    """want_bwd: False/0 forward, True/1 loss fwd+bwd, 2 rl_batch_prepare only."""
    hd = head.c()
    n = lib.rl_workspace_size(C.byref(hd), int(num_rows), int(want_bwd))
    if n == 0:
        raise RLHeadError("rl_workspace_size: invalid head")
    return int(n)


def rl_batch_prepare(head: Head, batch: Batch, row_seq=None, active_idx=None, n_active=None,
                     n_accum=None, nseq_accum=None, ws: Workspace | None = None, stream=None):
    hd, b = head.c(), batch.c()
    ws = ws or Workspace()
    nb = rl_workspace_size(head, b.num_rows, 2)      # bookkeeping-only prefix
    buf = ws.get(nb)
    _check(lib.rl_batch_prepare(C.byref(hd), C.byref(b), _ptr(row_seq), _ptr(active_idx),
                                _ptr(n_active), _ptr(n_accum), _ptr(nseq_accum), _ptr(buf),
                                buf.numel(), _stream(stream)), "rl_batch_prepare")


def rl_logprob_fwd(head: Head, hidden, weight, batch: Batch, logp, entropy=None, lse=None,
                   ws: Workspace | None = None, stream=None):
    hd, b = head.c(), batch.c()
    ws = ws or Workspace()
    buf = ws.get(rl_workspace_size(head, b.num_rows, False))
    _check(lib.rl_logprob_fwd(C.byref(hd), _ptr(hidden), _ptr(weight), C.byref(b), _ptr(logp),
                              _ptr(entropy), _ptr(lse), _ptr(buf), buf.numel(), _stream(stream)),
           "rl_logprob_fwd")


def rl_grpo_group_stats(rewards, group_of_seq, num_groups: int, sum_stats, max_stats,
                        err_flags=None, stream=None):
    _check(lib.rl_grpo_group_stats(_ptr(rewards), _ptr(group_of_seq), int(rewards.shape[0]),
                                   int(num_groups), _ptr(sum_stats), _ptr(max_stats),
                                   _ptr(err_flags), _stream(stream)), "rl_grpo_group_stats")


def rl_grpo_advantage(rewards, group_of_seq, num_groups: int, adv, sum_stats=None, max_stats=None,
                      eps: float = 1e-6, unbiased: bool = True, err_flags=None, stream=None):
    _check(lib.rl_grpo_advantage(_ptr(rewards), _ptr(group_of_seq), int(rewards.shape[0]),
                                 int(num_groups), _ptr(sum_stats), _ptr(max_stats), float(eps),
                                 int(bool(unbiased)), _ptr(adv), _ptr(err_flags),
                                 _stream(stream)), "rl_grpo_advantage")


def rl_batch_norm_advantage(rewards, group_of_seq, num_groups: int, adv, group_baseline=True,
                            group_sum_stats=None, batch_stats_in=None, batch_stats_out=None,
                            eps: float = 1e-6, unbiased: bool = True, err_flags=None,
                            stream=None):
    """REINFORCE++-style batch-normalised advantage (NEXT-1). With the group
    baseline and no group_sum_stats given, the group sums are computed here
    (rl_grpo_group_stats into a scratch tensor) -- all members local."""
    import torch
    if group_baseline and group_sum_stats is None:
        G = max(int(num_groups), 1)
        group_sum_stats = torch.empty(G, 3, dtype=torch.float64, device=rewards.device)
        mx = torch.empty(G, 2, dtype=torch.float64, device=rewards.device)
        rl_grpo_group_stats(rewards, group_of_seq, num_groups, group_sum_stats, mx,
                            err_flags=err_flags, stream=stream)
    _check(lib.rl_batch_norm_advantage(_ptr(rewards), _ptr(group_of_seq), int(rewards.shape[0]),
                                       int(num_groups), int(bool(group_baseline)),
                                       _ptr(group_sum_stats), _ptr(batch_stats_in),
                                       _ptr(batch_stats_out), float(eps), int(bool(unbiased)),
                                       _ptr(adv), _ptr(err_flags), _stream(stream)),
           "rl_batch_norm_advantage")


def rl_read_device_error(err_flags, stream=None) -> int:
    """Debug helper: synchronise the stream and return the device error word."""
    v = C.c_int32(0)
    _check(lib.rl_read_device_error(_ptr(err_flags), C.byref(v), _stream(stream)),
           "rl_read_device_error")
    return int(v.value)


def rl_policy_loss_fwd_bwd(head: Head, hidden, weight, batch: Batch, old_logp, adv,
                           params: LossParams, logp, grad_hidden, grad_weight, entropy=None,
                           stats=None, ws: Workspace | None = None, stream=None):
    hd, b, p = head.c(), batch.c(), params.c()
    ws = ws or Workspace()
    buf = ws.get(rl_workspace_size(head, b.num_rows, True))
    _check(lib.rl_policy_loss_fwd_bwd(C.byref(hd), _ptr(hidden), _ptr(weight), C.byref(b),
                                      _ptr(old_logp), _ptr(adv), C.byref(p), _ptr(logp),
                                      _ptr(entropy), _ptr(grad_hidden), _ptr(grad_weight),
                                      _ptr(stats), _ptr(buf), buf.numel(), _stream(stream)),
           "rl_policy_loss_fwd_bwd")


def _loss_phase(fn, name, head, hidden, weight, batch, old_logp, adv, params, logp, grad_hidden,
                grad_weight, entropy=None, stats=None, ws=None, stream=None):
    hd, b, p = head.c(), batch.c(), params.c()
    ws = ws or Workspace()
    buf = ws.get(rl_workspace_size(head, b.num_rows, True))
    _check(fn(C.byref(hd), _ptr(hidden), _ptr(weight), C.byref(b), _ptr(old_logp), _ptr(adv),
              C.byref(p), _ptr(logp), _ptr(entropy), _ptr(grad_hidden), _ptr(grad_weight),
              _ptr(stats), _ptr(buf), buf.numel(), _stream(stream)), name)


def rl_policy_loss_fwd(head: Head, hidden, weight, batch: Batch, old_logp, adv,
                       params: LossParams, logp, grad_hidden, grad_weight, entropy=None,
                       stats=None, ws: Workspace | None = None, stream=None):
    """H1-H5 of rl_policy_loss_fwd_bwd (same arguments); the state stays in ws."""
    _loss_phase(lib.rl_policy_loss_fwd, "rl_policy_loss_fwd", head, hidden, weight, batch,
                old_logp, adv, params, logp, grad_hidden, grad_weight, entropy, stats, ws, stream)


def rl_policy_loss_bwd(head: Head, hidden, weight, batch: Batch, old_logp, adv,
                       params: LossParams, logp, grad_hidden, grad_weight, entropy=None,
                       stats=None, ws: Workspace | None = None, stream=None):
    """H6-H8 of rl_policy_loss_fwd_bwd from the forward's state in ws."""
    _loss_phase(lib.rl_policy_loss_bwd, "rl_policy_loss_bwd", head, hidden, weight, batch,
                old_logp, adv, params, logp, grad_hidden, grad_weight, entropy, stats, ws, stream)


def rl_logprob_partials(head: Head, hidden, weight, batch: Batch, parts,
                        ws: Workspace | None = None, stream=None):
    """Vocab-parallel phase 1: this shard's merged partials, parts fp32 [4, R]."""
    hd, b = head.c(), batch.c()
    ws = ws or Workspace()
    buf = ws.get(rl_workspace_size(head, b.num_rows, False))
    _check(lib.rl_logprob_partials(C.byref(hd), _ptr(hidden), _ptr(weight), C.byref(b),
                                   _ptr(parts), _ptr(buf), buf.numel(), _stream(stream)),
           "rl_logprob_partials")


def rl_logprob_merge(head: Head, batch: Batch, parts_all, logp, entropy=None, lse=None,
                     ws: Workspace | None = None, stream=None):
    """Vocab-parallel phase 2 (inference): parts_all fp32 [P, 4, R] -> logp etc."""
    hd, b = head.c(), batch.c()
    ws = ws or Workspace()
    buf = ws.get(rl_workspace_size(head, b.num_rows, False))
    _check(lib.rl_logprob_merge(C.byref(hd), C.byref(b), _ptr(parts_all), int(parts_all.shape[0]),
                                _ptr(logp), _ptr(entropy), _ptr(lse), _ptr(buf), buf.numel(),
                                _stream(stream)), "rl_logprob_merge")


def rl_policy_loss_fwd_bwd_vp(head: Head, hidden, weight, batch: Batch, parts_all, old_logp, adv,
                              params: LossParams, logp, grad_hidden, grad_weight, entropy=None,
                              stats=None, ws: Workspace | None = None, stream=None,
                              grad_hidden_mc: int = 0):
    """Vocab-parallel phase 2 (training): grad_hidden is this shard's partial
    dL/dH (all-reduce SUM over the TP group), grad_weight its rows of dL/dW.
    A float32 grad_hidden [R, hidden] selects the fp32 partial (for
    rl_allreduce_sum_f32 over a symmetric buffer); grad_hidden_mc != 0 is the
    multicast address of such a (zeroed) buffer: the epilogue adds into every
    rank's copy (grad_hidden is then ignored)."""
    import torch
    hd, b, p = head.c(), batch.c(), params.c()
    ws = ws or Workspace()
    buf = ws.get(rl_workspace_size(head, b.num_rows, True))
    gh_f32 = int(grad_hidden is not None and grad_hidden.dtype == torch.float32
                 and head.dtype == "bf16")
    if grad_hidden_mc:
        gh_f32, grad_hidden = 2, None
    _check(lib.rl_policy_loss_fwd_bwd_vp(C.byref(hd), _ptr(hidden), _ptr(weight), C.byref(b),
                                         _ptr(parts_all), int(parts_all.shape[0]), _ptr(old_logp),
                                         _ptr(adv), C.byref(p), _ptr(logp), _ptr(entropy),
                                         C.c_void_p(int(grad_hidden_mc)) if grad_hidden_mc
                                         else _ptr(grad_hidden), gh_f32, _ptr(grad_weight),
                                         _ptr(stats),
                                         _ptr(buf), buf.numel(), _stream(stream)),
           "rl_policy_loss_fwd_bwd_vp")


def rl_allreduce_sum_f32(buf, rank: int, world: int, peer_ptrs=None, mc_ptr: int = 0,
                         stream=None):
    """Sum buf (fp32, n % 4 == 0) over `world` ranks through NVLink peer memory:
    NVLS multicast when mc_ptr != 0, else P2P over peer_ptrs (device addresses
    of every rank's buf). The caller barriers before and after (symm_mem)."""
    n = int(buf.numel())
    arr = None
    if not mc_ptr:
        arr = (C.c_void_p * world)(*[int(x) for x in peer_ptrs])
    _check(lib.rl_allreduce_sum_f32(arr, C.c_void_p(int(mc_ptr)) if mc_ptr else None, int(rank),
                                    int(world), n, _stream(stream)), "rl_allreduce_sum_f32")


def rl_reduce_bcast_rows_f32(staging, out, rank: int, world: int, rows_per_rank: int,
                             out_peer_ptrs=None, mc_ptr: int = 0, stream=None):
    """Owner side of the fused DP dW reduce-scatter: sum this rank's `world`
    staged slab copies (staging [world, rows_per_rank, cols]) in rank order and
    store the sum into every rank's out [rows, cols] (multicast when mc_ptr,
    else P2P stores to out_peer_ptrs)."""
    rows, cols = out.shape
    arr = None
    if not mc_ptr:
        arr = (C.c_void_p * world)(*[int(x) for x in out_peer_ptrs])
    _check(lib.rl_reduce_bcast_rows_f32(_ptr(staging), arr,
                                        C.c_void_p(int(mc_ptr)) if mc_ptr else None, int(rank),
                                        int(world), int(rows), int(cols), int(rows_per_rank),
                                        _stream(stream)), "rl_reduce_bcast_rows_f32")


def rl_dw_reduce_rows_f32(out, rank: int, world: int, rows_per_rank: int, peer_ptrs,
                          mc_ptr: int = 0, broadcast: bool = True, stream=None):
    """DP dW sum after the last dW GEMM (no staging): this rank's owned rows of
    out [rows, cols] (mapped by every rank: peer_ptrs) summed over the ranks --
    through the NVLS multicast address when mc_ptr, else P2P in rank order --
    and stored into every rank's copy (broadcast) or this rank's only."""
    rows, cols = out.shape
    arr = (C.c_void_p * world)(*[int(x) for x in peer_ptrs])
    _check(lib.rl_dw_reduce_rows_f32(arr, C.c_void_p(int(mc_ptr)) if mc_ptr else None,
                                     int(rank), int(world), int(rows), int(cols),
                                     int(rows_per_rank), 1 if broadcast else 0, _stream(stream)),
           "rl_dw_reduce_rows_f32")


def rl_cast_rows_bf16(src, dst, stream=None):
    """dst[t, :h] = bf16(src[t, :h]) (src fp32 contiguous [R, h]; dst row stride any)."""
    R, h = src.shape
    _check(lib.rl_cast_rows_bf16(_ptr(src), int(R), int(h), _ptr(dst), int(dst.stride(0)),
                                 _stream(stream)), "rl_cast_rows_bf16")


def rl_minibatch_early_stop(stats, stop_flag, grad_weight, max_ratio: float = 0.0,
                            max_mean_ratio: float = 0.0, stream=None):
    """device-side decision into stop_flag (int32[1]); zeroes grad_weight if set."""
    n = 0 if grad_weight is None else int(grad_weight.numel())
    _check(lib.rl_minibatch_early_stop(_ptr(stats), float(max_ratio), float(max_mean_ratio),
                                       _ptr(stop_flag), _ptr(grad_weight), n, _stream(stream)),
           "rl_minibatch_early_stop")


def rl_scale_by_inverse_count(x, count, stream=None):
    """x *= 1/count (device int64[1]); deferred normalisation of streaming mode."""
    _check(lib.rl_scale_by_inverse_count(_ptr(x), int(x.numel()), _ptr(count), _stream(stream)),
           "rl_scale_by_inverse_count")


def rl_gae(rewards, values, cu_steps, gamma: float, lam: float, adv, returns, dones=None,
           bootstrap=None, stream=None):
    """GAE over packed trajectories (NEXT-4)."""
    _check(lib.rl_gae(_ptr(rewards), _ptr(values), _ptr(dones), _ptr(bootstrap), _ptr(cu_steps),
                      int(cu_steps.shape[0]) - 1, float(gamma), float(lam), _ptr(adv),
                      _ptr(returns), _stream(stream)), "rl_gae")


def rl_value_loss_fwd_bwd(head: Head, hidden, w_v, b_v: float, batch: Batch, returns, old_values,
                          values, grad_hidden, grad_w, grad_b=None, clip_eps: float = 0.2,
                          n_tokens_global=None, loss_scale: float = 1.0, stats=None,
                          ws: Workspace | None = None, stream=None):
    """Value head + clipped value loss (NEXT-4); grad_hidden/grad_w/grad_b accumulate."""
    hd, b = head.c(), batch.c()
    p = rl_value_params(float(clip_eps), float(loss_scale), _ptr(n_tokens_global))
    ws = ws or Workspace()
    buf = ws.get(int(lib.rl_value_workspace_size(hd.hidden, b.num_rows)))
    _check(lib.rl_value_loss_fwd_bwd(C.byref(hd), _ptr(hidden), _ptr(w_v), float(b_v), C.byref(b),
                                     _ptr(returns), _ptr(old_values), C.byref(p), _ptr(values),
                                     _ptr(grad_hidden), _ptr(grad_w), _ptr(grad_b), _ptr(stats),
                                     _ptr(buf), buf.numel(), _stream(stream)),
           "rl_value_loss_fwd_bwd")


def rl_loss_stats_reduce(gathered, out, stream=None):
    """out := rank-order combination of gathered [nranks * STATS_BYTES] (uint8)
    rl_loss_stats (sums; max of ratio_max)."""
    n = int(gathered.numel()) // STATS_BYTES
    _check(lib.rl_loss_stats_reduce(_ptr(gathered), n, _ptr(out), _stream(stream)),
           "rl_loss_stats_reduce")


def rl_launch_count() -> int:
    return int(lib.rl_launch_count())


def rl_build_info() -> str:
    return lib.rl_build_info().decode()


class Trace:
    """Context manager around rl_trace_begin/end: per-launch device times."""

    def __init__(self, capacity: int = 1 << 16):
        self.capacity = capacity
        self.kinds = None
        self.ms = None

    def start(self):
        _check(lib.rl_trace_begin(self.capacity), "rl_trace_begin")
        return self

    def stop(self):
        kinds = np.zeros(self.capacity, dtype=np.int32)
        n = lib.rl_trace_end(kinds.ctypes.data_as(C.c_void_p))
        ms = np.zeros(max(n, 1), dtype=np.float32)
        lib.rl_trace_durations(ms.ctypes.data_as(C.c_void_p), n)
        self.kinds, self.ms = kinds[:n], ms[:n]
        return self

    def __enter__(self):
        return self.start()

    def __exit__(self, *exc):
        self.stop()
        return False

    def by_kind(self) -> dict:
        out = {}
        for k, t in zip(self.kinds, self.ms):
            name = KERNEL_KINDS[k]
            c, s = out.get(name, (0, 0.0))
            out[name] = (c + 1, s + float(t))
        return out
