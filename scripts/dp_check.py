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

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="qwen1.5b")
    ap.add_argument("--mb-rows", type=int, default=16384)
    ap.add_argument("--max-mb", type=int, default=3)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--empty-last", action="store_true")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_2509_15965_b200 as rl
    from paper_2509_15965_b200.dp import PolicyLossStep, device_batch, shard_layout
    from workload import CONFIGS, make_layout, make_tensors_torch, sub_layout
    rank, world, local = (int(os.environ.get(k, d)) for k, d in
                          (("RANK", 0), ("WORLD_SIZE", 1), ("LOCAL_RANK", 0)))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    cfg = CONFIGS[a.config]
    layout = make_layout(cfg, 0)
    seqs, _ = shard_layout(layout, rank, world)
    mine, _ = sub_layout(layout, seqs)
    if a.empty_last and rank == 1:
        db0 = device_batch(mine, a.mb_rows, device=dev)
        n = min(len(db0.mbs), a.max_mb)
        _, _, r0, r1, _ = db0.mbs[n - 1]
        mine.mask[r0:r1] = 0
    db = device_batch(mine, a.mb_rows, device=dev)
    db.mbs = db.mbs[:a.max_mb]
    _, W = make_tensors_torch(cfg, 0, seed=1, device=dev, hidden=False)
    H, _ = make_tensors_torch(cfg, mine.num_rows, seed=100 + rank, device=dev, weight=False)
    head = rl.Head(cfg.hidden, cfg.vocab, cfg.dtype)
    # old log-probs = the policy's own (ratio 1): every unmasked token carries
    # gradient (old = 0 would clamp d = logp - old and zero the gradients)
    old = torch.zeros(max(mine.num_rows, 1), device=dev)
    ws = rl.Workspace(dev)
    for (_, _, r0, r1, cu_mb) in db.mbs:
        rl.rl_logprob_fwd(head, H[r0:r1], W, rl.Batch(cu_mb, db.targets[r0:r1], db.mask[r0:r1],
                                                      num_rows=r1 - r0), old[r0:r1], ws=ws)
    del ws
    gh = torch.empty(mine.num_rows, cfg.hidden, dtype=H.dtype, device=dev)
    out = {}
    res = {}
    for mode in ("nccl", "symm"):
        step = PolicyLossStep(head, W, db, collective=mode)
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
        res[mode] = (step.grad_w.clone(), rl.read_stats(step.stats), gws)
        out[mode] = {"ms_per_step": round(float(ms.item()), 3),
                     "ranks_identical_dW": all(torch.equal(g, gws[0]) for g in gws)}
    g_n, s_n, _ = res["nccl"]
    g_s, s_s, _ = res["symm"]
    nrm = float(g_n.double().norm())
    rel = float((g_s.double() - g_n.double()).norm()) / max(nrm, 1e-300)
    if rank == 0:
        print(json.dumps({"world": world, "config": a.config, "micro_batches": len(db.mbs),
                          "empty_last": a.empty_last, "rel_dW_symm_vs_nccl": rel,
                          "norm_dW": nrm,
                          "tokens": s_n["tokens"], "tokens_symm": s_s["tokens"],
                          "loss_sum_nccl": s_n["loss_sum"], "loss_sum_symm": s_s["loss_sum"],
                          "modes": out}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
