#!/usr/bin/env python
"""DP dW reduction across real GPUs: the same mini-batch step
with collective="nccl" (dW all-reduce) and collective="symm" (reduce-scatter
fused into the last dW GEMM epilogue + NVLink all-gather); compares dW and the
stats, times both (CUDA events, max over ranks).

    torchrun --nproc-per-node 2 scripts/dp_check.py [--config qwen1.5b --max-mb 3]

--empty-last: rank 1's last micro-batch is fully masked (its dW GEMM has K = 0
and must still send its partial). Prints one JSON line on rank 0."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="qwen1.5b")
    ap.add_argument("--mb-rows", type=int, default=16384)
    ap.add_argument("--max-mb", type=int, default=3)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--empty-last", action="store_true")
    ap.add_argument("--modes", default="nccl,symm",
                    help="comma list of nccl|symm|nvls[:shard][-split] | "
                         "stream-nccl|stream-symm[-nolast]; :shard = owned dW rows only; "
                         "-split = sequence-level sharding with all-reduced group statistics "
                         "(compare with --max-mb 0); stream-* = StreamingPolicyLoss (deferred "
                         "1/N), -nolast = no last=True feed (partial sent by finish())")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_2509_15965_b200 as rl
    from paper_2509_15965_b200.dp import (PolicyLossStep, StreamingPolicyLoss, device_batch,
                                          shard_layout, shard_rows)
    from workload import CONFIGS, make_layout, make_tensors_torch, sub_layout
    rank, world, local = (int(os.environ.get(k, d)) for k, d in
                          (("RANK", 0), ("WORLD_SIZE", 1), ("LOCAL_RANK", 0)))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    cfg = CONFIGS[a.config]
    layout = make_layout(cfg, 0)
    _, W = make_tensors_torch(cfg, 0, seed=1, device=dev, hidden=False)
    head = rl.Head(cfg.hidden, cfg.vocab, cfg.dtype)
    # hidden rows are a function of the GLOBAL row (seeded per sequence-independent
    # chunks of the whole batch) so different shardings see the same data
    Hg, _ = make_tensors_torch(cfg, layout.num_rows, seed=5, device=dev, weight=False)
    cache = {}

    def rank_data(split):
        if split in cache:
            return cache[split]
        seqs, _ = shard_layout(layout, rank, world, split_groups=split)
        mine, rows = sub_layout(layout, seqs)
        if a.empty_last and rank == 1:
            db0 = device_batch(mine, a.mb_rows, device=dev)
            n = min(len(db0.mbs), a.max_mb) if a.max_mb else len(db0.mbs)
            _, _, r0, r1, _ = db0.mbs[n - 1]
            mine.mask[r0:r1] = 0
        if a.max_mb:  # keep the sequences of the first max_mb micro-batches only
            db0 = device_batch(mine, a.mb_rows, device=dev, global_groups=split)
            s_end = db0.mbs[min(a.max_mb, len(db0.mbs)) - 1][1]
            mine, sub_rows = sub_layout(mine, np.arange(s_end))
            rows = rows[sub_rows]
        db = device_batch(mine, a.mb_rows, device=dev, global_groups=split)
        H = Hg[torch.as_tensor(rows, device=dev)] if len(rows) else Hg[:1]
        # old log-probs = the policy's own (ratio 1): every unmasked token carries
        # gradient (old = 0 would clamp d = logp - old and zero the gradients)
        old = torch.zeros(max(mine.num_rows, 1), device=dev)
        ws = rl.Workspace(dev)
        for (_, _, r0, r1, cu_mb) in db.mbs:
            rl.rl_logprob_fwd(head, H[r0:r1], W, rl.Batch(cu_mb, db.targets[r0:r1],
                                                          db.mask[r0:r1], num_rows=r1 - r0),
                              old[r0:r1], ws=ws)
        gh = torch.empty(max(mine.num_rows, 1), cfg.hidden, dtype=H.dtype, device=dev)
        cache[split] = (db, H, old, gh)
        return cache[split]

    out = {}
    res = {}
    modes = a.modes.split(",")

    class Streamed:
        """StreamingPolicyLoss driven like PolicyLossStep.run (stream-<coll>[-nolast])."""

        def __init__(self, db, coll, use_last):
            self.db, self.use_last = db, use_last
            self.s = StreamingPolicyLoss(head, W, collective=coll)
            self.adv = torch.empty(max(db.cu.shape[0] - 1, 1), device=dev)
            self.logp = torch.empty(max(db.num_rows, 1), device=dev)
            self.grad_w, self.stats = self.s.grad_w, self.s.stats

        def run(self, H, old, gh):
            db, st = self.db, self.s
            rl.rl_grpo_advantage(db.rewards, db.gos, db.num_groups, self.adv)
            st.begin()
            for i, (s0, s1, r0, r1, cu_mb) in enumerate(db.mbs):
                b = rl.Batch(cu_mb, db.targets[r0:r1], db.mask[r0:r1], num_rows=r1 - r0)
                st.feed(H[r0:r1], b, old[r0:r1], self.adv[s0:s1], self.logp[r0:r1], gh[r0:r1],
                        last=self.use_last and i == len(db.mbs) - 1)
            st.finish()

    for mode in modes:
        split = mode.endswith("-split")
        db, H, old, gh = rank_data(split)
        if mode.startswith("stream-"):
            parts = mode.split("-")
            step = Streamed(db, parts[1], "nolast" not in parts)
        else:   # <collective>[:shard]: shard = owned dW rows only (FSDP gradient)
            coll, _, out_kind = mode.split("-")[0].partition(":")
            step = PolicyLossStep(head, W, db, collective=coll, split_groups=split,
                                  dw_output=out_kind or "full")
        step.run(H, old, gh)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            step.run(H, old, gh)
        e1.record()
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1) / a.reps], dtype=torch.float64, device=dev)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        gws = [torch.empty_like(step.grad_w) for _ in range(world)]
        dist.all_gather(gws, step.grad_w.contiguous())
        if ":shard" in mode:             # rank q's owned rows of its own buffer
            full = torch.cat([g[slice(*shard_rows(g.shape[0], world, q))]
                              for q, g in enumerate(gws)])
            res[mode] = (full, rl.read_stats(step.stats), gws)
            out[mode] = {"ms_per_step": round(float(ms.item()), 3), "ranks_identical_dW": True}
            continue
        res[mode] = (step.grad_w.clone(), rl.read_stats(step.stats), gws)
        out[mode] = {"ms_per_step": round(float(ms.item()), 3),
                     "ranks_identical_dW": all(torch.equal(g, gws[0]) for g in gws)}
    g_n, s_n, _ = res[modes[0]]
    nrm = float(g_n.double().norm())
    for mode in modes[1:]:
        g_s, s_s, _ = res[mode]
        out[mode]["rel_dW_vs_" + modes[0]] = float((g_s.double() - g_n.double()).norm()) / max(
            nrm, 1e-300)
        out[mode]["tokens"] = s_s["tokens"]
        out[mode]["loss_sum"] = s_s["loss_sum"]
    out[modes[0]]["tokens"] = s_n["tokens"]
    out[modes[0]]["loss_sum"] = s_n["loss_sum"]
    if rank == 0:
        print(json.dumps({"world": world, "config": a.config, "empty_last": a.empty_last,
                          "norm_dW": nrm, "modes": out}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
