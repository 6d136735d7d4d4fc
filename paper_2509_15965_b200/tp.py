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

Exchange 2 follows the dL/dH GEMM, so besides NCCL (`collective="nccl"`) it
can run over NVLink peer memory on a torch symmetric-memory
buffer that every TP rank has mapped:
  "fused": the dL/dH GEMM epilogue adds each fp32 tile into every rank's copy
           through the NVSwitch (multimem.red) -- the all-reduce happens tile
           by tile inside the GEMM; needs NVLS multicast;
  "nvls":  epilogue stores fp32 locally, then one two-shot multimem
           ld_reduce/st kernel (rl_allreduce_sum_f32);
  "p2p":   same, summing over P2P loads in rank order (deterministic).
Then rl_cast_rows_bf16 writes the bf16 rows into grad_hidden.
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
    collective: str = "nccl"      # dL/dH sum: "nccl" | "fused" | "nvls" | "p2p" | "auto"

    def __post_init__(self):
        self._symm = None         # (tensor, handle, numel)

    def _world(self):
        import torch.distributed as dist
        return dist.get_world_size(self.group) if dist.is_initialized() else 1

    def _symm_buffer(self, numel, device):
        """fp32 symmetric buffer of >= numel elements mapped on every TP rank
        (collective: all ranks call it with the same numel)."""
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        if self._symm is None or self._symm[2] < numel:
            import torch
            n = max(numel, 1 << 20)
            t = symm_mem.empty(n, dtype=torch.float32, device=device)
            grp = self.group if self.group is not None else dist.group.WORLD
            hdl = symm_mem.rendezvous(t, grp)
            self._symm = (t, hdl, n)
        return self._symm

    def resolved_collective(self, device) -> str:
        if self.collective != "auto":
            return self.collective
        if self._world() == 1:
            return "nccl"
        _, hdl, _ = self._symm_buffer(1, device)
        # measured on 2 B200 (profiles/r1/tp_symm_tp2.json): nvls ~ NCCL time,
        # fused slower at 16k rows; all three sum in fp32 (NCCL sums bf16)
        return "nvls" if hdl.multicast_ptr else "p2p"

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
        mode = self.resolved_collective(hidden.device) if self._world() > 1 else "nccl"
        if mode == "nccl":
            R.rl_policy_loss_fwd_bwd_vp(self.head(), hidden, weight_shard, batch, parts_all,
                                        old_logp, adv, params, logp, grad_hidden,
                                        grad_weight_shard, entropy=entropy, stats=stats, ws=ws)
            if dist.is_initialized() and dist.get_world_size(self.group) > 1:
                dist.all_reduce(grad_hidden, group=self.group)   # sum_p dZ_p W_p
            return parts_all
        # symmetric-memory modes: sum_p dZ_p W_p over NVLink peer memory
        h = self.hidden
        n = Rn * h
        t, hdl, _ = self._symm_buffer(n, hidden.device)
        gh32 = t[:n].view(Rn, h)
        if mode == "fused":
            if not hdl.multicast_ptr:
                raise R.RLHeadError("collective='fused' needs NVLS multicast support")
            gh32.zero_()
            hdl.barrier(channel=0)        # every copy zeroed before any rank adds
            R.rl_policy_loss_fwd_bwd_vp(self.head(), hidden, weight_shard, batch, parts_all,
                                        old_logp, adv, params, logp, None, grad_weight_shard,
                                        entropy=entropy, stats=stats, ws=ws,
                                        grad_hidden_mc=hdl.multicast_ptr)
            hdl.barrier(channel=0)        # all ranks' adds landed
        else:
            R.rl_policy_loss_fwd_bwd_vp(self.head(), hidden, weight_shard, batch, parts_all,
                                        old_logp, adv, params, logp, gh32, grad_weight_shard,
                                        entropy=entropy, stats=stats, ws=ws)
            hdl.barrier(channel=0)        # every rank's partial written
            if mode == "nvls":
                if not hdl.multicast_ptr:
                    raise R.RLHeadError("collective='nvls' needs NVLS multicast support")
                R.rl_allreduce_sum_f32(gh32, hdl.rank, hdl.world_size, mc_ptr=hdl.multicast_ptr)
            elif mode == "p2p":
                R.rl_allreduce_sum_f32(gh32, hdl.rank, hdl.world_size,
                                       peer_ptrs=list(hdl.buffer_ptrs))
            else:
                raise ValueError(f"unknown collective {mode!r}")
            hdl.barrier(channel=0)        # every slice stored on every rank
        if Rn:
            if self.dtype == "bf16":
                R.rl_cast_rows_bf16(gh32, grad_hidden)
            else:
                grad_hidden.copy_(gh32)
        return parts_all
