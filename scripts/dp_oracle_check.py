#!/usr/bin/env python
"""Data-parallel step across real GPUs vs the CPU float64 oracle of the WHOLE
mini-batch: two whole prompt groups of a real
layout are LPT-sharded over the ranks, every rank runs PolicyLossStep (N
all-reduce, GRPO advantages, micro-batches, dW reduction: NCCL all-reduce or
the fused reduce-scatter + NVLink all-gather), and rank 0 compares the
reduced dW, the reduced loss statistics and every rank's per-row logp / dL/dH
with the oracle run once over the un-sharded mini-batch on the same values.

    torchrun --nproc-per-node 2 scripts/dp_oracle_check.py [--config qwen1.5b]

Prints one JSON line on rank 0; exit 0 = every check within the north_star's
bf16 tolerances, 1 = a parity failure."""
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
    ap.add_argument("--groups", type=int, default=2)
    ap.add_argument("--mb-rows", type=int, default=16384)
    ap.add_argument("--modes", default="nccl,symm")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    import oracle
    import paper_2509_15965_b200 as rl
    from paper_2509_15965_b200.dp import PolicyLossStep, device_batch, shard_layout
    from tests.gpu_util import guarded_old_logp
    from workload import CONFIGS, make_layout, make_tensors_torch, sub_layout
    rank, world, local = (int(os.environ.get(k, d)) for k, d in
                          (("RANK", 0), ("WORLD_SIZE", 1), ("LOCAL_RANK", 0)))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    cfg = CONFIGS[a.config]
    lay = make_layout(cfg, 0)
    cu = lay.cu_seqlens.astype(np.int64)
    tok = np.add.reduceat(lay.mask.astype(np.int64), cu[:-1])
    g_tok = np.bincount(lay.group_of_seq, weights=tok, minlength=lay.num_groups)
    groups = np.argsort(g_tok, kind="stable")[:a.groups]
    batch, _ = sub_layout(lay, np.flatnonzero(np.isin(lay.group_of_seq, groups)))
    # the same values on every rank (device generator, fixed seed)
    Hg, W = make_tensors_torch(cfg, batch.num_rows, seed=3, device=dev)
    ref = fwd = None
    old = torch.empty(batch.num_rows, dtype=torch.float64, device=dev)
    if rank == 0:
        W64 = W.cpu().to(torch.float64).numpy()
        Hh = Hg.cpu()
        fwd = oracle.logprob_fwd(Hh, W64, batch.cu_seqlens, batch.mask, batch.targets)
        old_np = guarded_old_logp(fwd["logp"], np.random.default_rng(17))
        adv, _ = oracle.grpo_advantage(batch.rewards, batch.group_of_seq, batch.num_groups)
        ref = oracle.policy_loss_fwd_bwd(Hh, W64, batch.cu_seqlens, batch.mask, batch.targets,
                                         old_np, adv, n_global=batch.num_tokens)
        del W64
        old.copy_(torch.as_tensor(old_np))
    dist.broadcast(old, 0)
    seqs, loads = shard_layout(batch, rank, world)
    mine, rows = sub_layout(batch, seqs)
    ridx = torch.as_tensor(rows, device=dev)
    H = Hg[ridx] if len(rows) else Hg[:1]
    old_mine = old[ridx].float() if len(rows) else torch.zeros(1, device=dev)
    db = device_batch(mine, a.mb_rows, device=dev)
    head = rl.Head(cfg.hidden, cfg.vocab, cfg.dtype)
    out = {"world": world, "config": a.config, "groups": [int(g) for g in groups],
           "tokens": batch.num_tokens, "rank_tokens": [int(x) for x in loads], "modes": {}}
    ok = True
    for mode in a.modes.split(","):
        step = PolicyLossStep(head, W, db, collective=mode, want_entropy=True)
        gh = torch.full_like(H, 7.0)
        step.run(H, old_mine, gh)
        torch.cuda.synchronize()
        # every rank's rows -> rank 0 (row ids of the un-sharded batch)
        mine_rows = (rows, step.logp[:len(rows)].cpu().double().numpy(),
                     step.entropy[:len(rows)].cpu().double().numpy(),
                     gh[:len(rows)].to(torch.float64).cpu().numpy())
        allr = [None] * world
        dist.gather_object(mine_rows, allr if rank == 0 else None, dst=0)
        gws = [torch.empty_like(step.grad_w) for _ in range(world)] if rank == 0 else None
        dist.gather(step.grad_w.contiguous(), gws, dst=0)
        if rank == 0:
            R = batch.num_rows
            lp = np.zeros(R)
            ent = np.zeros(R)
            dH = np.zeros((R, cfg.hidden))
            for rr, a_lp, a_ent, a_dh in allr:
                lp[rr], ent[rr], dH[rr] = a_lp, a_ent, a_dh
            s = rl.read_stats(step.stats)
            rs = ref["stats"]
            gw = step.grad_w.double()
            refw = torch.as_tensor(ref["dW"], device=dev)
            r = {
                "max_dlogp": float(np.abs(lp - ref["logp"]).max()),
                "max_dentropy": float(np.abs(ent - ref["entropy"]).max()),
                "rel_dH": float(np.linalg.norm(dH - ref["dH"]) / np.linalg.norm(ref["dH"])),
                "rel_dW": float((gw - refw).norm() / refw.norm()),
                "max_rel_dW": float((gw - refw).abs().max() / refw.abs().max()),
                "ranks_identical_dW": all(torch.equal(g, gws[0]) for g in gws),
                "tokens": s["tokens"], "tokens_ref": rs["tokens"],
                "loss_sum": s["loss_sum"], "loss_sum_ref": rs["loss_sum"],
                "clip": [s["clip_lo_count"], s["clip_hi_count"]],
                "clip_ref": [rs["clip_lo_count"], rs["clip_hi_count"]],
                "n_global": int(step.n_global.item()),
            }
            del refw
            r["ok"] = (r["max_dlogp"] <= 2e-3 and r["max_dentropy"] <= 2e-3 and
                       r["rel_dH"] <= 1e-2 and r["rel_dW"] <= 1e-2 and r["max_rel_dW"] <= 1e-2
                       and r["ranks_identical_dW"] and r["tokens"] == r["tokens_ref"] and
                       r["n_global"] == batch.num_tokens and r["clip"] == r["clip_ref"] and
                       abs(r["loss_sum"] - r["loss_sum_ref"]) <= 1e-2 * abs(r["loss_sum_ref"]))
            ok = ok and r["ok"]
            out["modes"][mode] = r
        del step
        torch.cuda.empty_cache()
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
