#!/usr/bin/env python
"""Vocab-parallel head across real GPUs (NEXT-3): every rank holds one vocab
shard of the head; rank 0 also runs the unsharded head on its GPU and compares.

    torchrun --nproc-per-node 2 scripts/tp_check.py [--config qwen7b --rows 16384]

Prints one JSON line: max |dlogp| vs unsharded, relative dH / dW differences,
and the TP micro-batch time (CUDA events, max over ranks)."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="qwen7b")
    ap.add_argument("--rows", type=int, default=16384)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--collectives", default="nccl,p2p,nvls,fused",
                    help="dL/dH sum modes to run (tp.VocabParallelHead.collective)")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_2509_15965_b200 as rl
    from paper_2509_15965_b200.dp import pack_micro_batches
    from paper_2509_15965_b200.tp import VocabParallelHead, vocab_shards
    from workload import CONFIGS, make_layout, make_tensors_torch, sub_layout
    rank, world, local = (int(os.environ.get(k, d)) for k, d in
                          (("RANK", 0), ("WORLD_SIZE", 1), ("LOCAL_RANK", 0)))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    cfg = CONFIGS[a.config]
    lay = make_layout(cfg, 0)
    cu = lay.cu_seqlens.astype(np.int64)
    s0, s1 = pack_micro_batches(cu[1:] - cu[:-1], a.rows)[0]
    mb, _ = sub_layout(lay, np.arange(s0, s1))
    H, W = make_tensors_torch(cfg, mb.num_rows, seed=5, device=dev)   # same on every rank
    off, size = vocab_shards(cfg.vocab, world)[rank]
    Ws = W[off:off + size].contiguous()
    b = rl.Batch(torch.as_tensor(mb.cu_seqlens, device=dev), torch.as_tensor(mb.targets, device=dev),
                 torch.as_tensor(mb.mask, device=dev))
    Rn = mb.num_rows
    old = torch.zeros(Rn, device=dev)
    adv = torch.linspace(-1, 1, mb.num_seqs, device=dev)
    p = rl.LossParams(n_tokens_global=torch.tensor([mb.num_tokens], device=dev))
    ws = rl.Workspace(dev)
    ref = None
    if rank == 0:
        head = rl.Head(cfg.hidden, cfg.vocab, cfg.dtype)
        lp1 = torch.empty(Rn, device=dev)
        gh1 = torch.empty_like(H)
        gw1 = torch.zeros(cfg.vocab, cfg.hidden, device=dev)
        rl.rl_policy_loss_fwd_bwd(head, H, W, b, old, adv, p, lp1, gh1, gw1, ws=ws)
        torch.cuda.synchronize()
        ref = (lp1, gh1, gw1)
    rel = lambda x, y: float((x.double() - y.double()).norm() / y.double().norm())  # noqa: E731
    results = {}
    gh_first = None
    for mode in [m for m in a.collectives.split(",") if m]:
        vp = VocabParallelHead(cfg.hidden, cfg.vocab, off, size, cfg.dtype, collective=mode)
        if mode in ("nvls", "fused") and world > 1 and not vp._symm_buffer(1, dev)[1].multicast_ptr:
            results[mode] = {"skipped": "no NVLS multicast"}
            continue
        logp = torch.empty(Rn, device=dev)
        gh = torch.empty_like(H)
        gw = torch.zeros(size, cfg.hidden, device=dev)
        vp.loss_fwd_bwd(H, Ws, b, old, adv, p, logp, gh, gw, ws=ws)   # warm-up
        gw.zero_()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            vp.loss_fwd_bwd(H, Ws, b, old, adv, p, logp, gh, gw, ws=ws)
        e1.record()
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1) / a.reps], device=dev, dtype=torch.float64)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        gw /= a.reps
        # every rank holds the same summed dL/dH
        ghs = [torch.empty_like(gh) for _ in range(world)]
        dist.all_gather(ghs, gh)
        shards = [torch.empty(s_, cfg.hidden, device=dev) for _, s_ in vocab_shards(cfg.vocab, world)]
        dist.all_gather(shards, gw)
        if rank == 0:
            lp1, gh1, gw1 = ref
            gh_first = gh if gh_first is None else gh_first
            results[mode] = {
                "max_dlogp": float((logp - lp1).abs().max()),
                "rel_dH": rel(gh, gh1), "rel_dW": rel(torch.cat(shards), gw1),
                "ranks_identical_dH": all(torch.equal(g, ghs[0]) for g in ghs),
                "rel_dH_vs_first_mode": rel(gh, gh_first),
                "ms_per_microbatch": round(float(ms.item()), 3),
                "tokens_per_s": round(mb.num_tokens / (float(ms.item()) / 1e3), 1)}
    if rank == 0:
        print(json.dumps({"tp": world, "config": a.config, "tokens": mb.num_tokens,
                          "rows": Rn, "modes": results}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
