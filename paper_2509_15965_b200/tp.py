"""Vocab-parallel (tensor-parallel) head driver, NEXT-3.

The paper trains its actors with tensor parallelism 2/4/8 (tab:math-eval-
config). For the LM head that means sharding the vocabulary: rank p of
the TP group holds W[off_p : off_p + V_p] (V_p a multiple of the 256-column
GEMM tile). One micro-batch then needs exactly two exchanges:

  1. all-gather of the per-row shard partials (m, s, u, z_y): 16 B per active
     row per rank, so every rank can finish the softmax over the full V;
  2. all-reduce (SUM) of dL/dH, the sum over shards of dZ_p W_p.

dW_p stays on its rank (each rank owns its rows of the head). All arithmetic
is in librlhead; this module only moves buffers through torch.distributed.
"""
from __future__ import annotations

from dataclasses import dataclass

from . import rlhead as R


def vocab_shards(vocab: int, parts: int, align: int = 256):
    """[(offset, size)] covering [0, vocab): sizes multiples of `align` except
    possibly the last, as equal as that allows."""
    per = -(-vocab // parts)
    per = -(-per // align) * align
    out, off = [], 0
    for _ in range(parts):
        size = max(0, min(per, vocab - off))
        out.append((off, size))
        off += size
    assert off == vocab and all(s > 0 for _, s in out), "too many shards for this vocab"
    return out


@dataclass
class VocabParallelHead:
    hidden: int
    vocab_total: int
    offset: int
    size: int
    dtype: str = "bf16"
    group: object = None          # torch.distributed process group (TP group)

    def head(self) -> R.Head:
        return R.Head(self.hidden, self.size, self.dtype, vocab_offset=self.offset,
                      vocab_total=self.vocab_total)

    def _gather_parts(self, parts_local):
        import torch
        import torch.distributed as dist
        P = dist.get_world_size(self.group) if dist.is_initialized() else 1
        if P == 1:
            return parts_local.unsqueeze(0)
        out = torch.empty((P,) + tuple(parts_local.shape), dtype=parts_local.dtype,
                          device=parts_local.device)
        dist.all_gather_into_tensor(out, parts_local.contiguous(), group=self.group)
        return out

    def logprob(self, hidden, weight_shard, batch: R.Batch, logp, entropy=None, lse=None, ws=None):
        import torch
        Rn = batch.c().num_rows
        parts = torch.empty(4, max(Rn, 1), dtype=torch.float32, device=hidden.device)
        R.rl_logprob_partials(self.head(), hidden, weight_shard, batch, parts, ws=ws)
        parts_all = self._gather_parts(parts)
        R.rl_logprob_merge(self.head(), batch, parts_all, logp, entropy, lse, ws=ws)
        return parts_all

    def loss_fwd_bwd(self, hidden, weight_shard, batch: R.Batch, old_logp, adv,
                     params: R.LossParams, logp, grad_hidden, grad_weight_shard, entropy=None,
                     stats=None, ws=None):
        import torch
        import torch.distributed as dist
        Rn = batch.c().num_rows
        parts = torch.empty(4, max(Rn, 1), dtype=torch.float32, device=hidden.device)
        R.rl_logprob_partials(self.head(), hidden, weight_shard, batch, parts, ws=ws)
        parts_all = self._gather_parts(parts)
        R.rl_policy_loss_fwd_bwd_vp(self.head(), hidden, weight_shard, batch, parts_all,
                                    old_logp, adv, params, logp, grad_hidden, grad_weight_shard,
                                    entropy=entropy, stats=stats, ws=ws)
        if dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.all_reduce(grad_hidden, group=self.group)   # sum_p dZ_p W_p
        return parts_all
