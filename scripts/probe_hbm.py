#!/usr/bin/env python
"""HBM-bound kernels of the head, timed live (library CUDA-event tracer):

* H1 bookkeeping (k_validate + k_flags_compact) once over a config's WHOLE
  packed mini-batch (6.18M rows at qwen7b);
* H2 GRPO advantage (k_grpo_seg) over the mini-batch's S sequences;
* H1 + gather + merge/loss + zero-inactive inside one 16k-row micro-batch of
  rl_policy_loss_fwd_bwd (the launch configuration bench.py times).

Bytes are algorithmic (what each kernel must read and write), GB/s against
MEASURED_PEAKS.json. Wrap in ncu for DRAM bytes per kernel:

    python scripts/probe_hbm.py --reps 5
    ncu --set full -k regex:"k_flags_compact|k_validate|k_grpo_seg|k_merge|k_gather" \\
        python scripts/probe_hbm.py --reps 1
"""
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
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--mb-rows", type=int, default=16384)
    a = ap.parse_args()
    import torch

    import paper_2509_15965_b200 as rl
    from paper_2509_15965_b200.dp import pack_micro_batches
    from workload import CONFIGS, make_layout, make_tensors_torch, sub_layout
    try:
        hbm = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        hbm = 6650.0
    cfg = CONFIGS[a.config]
    lay = make_layout(cfg, 0)
    dev = "cuda"
    R = lay.num_rows
    S = lay.num_seqs
    head = rl.Head(cfg.hidden, cfg.vocab, cfg.dtype)
    out = {"config": a.config, "hbm_peak_gbs": hbm}

    def timed(fn, reps):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    # H1 over the whole mini-batch
    b = rl.Batch(torch.as_tensor(lay.cu_seqlens, device=dev),
                 torch.as_tensor(lay.targets, device=dev), torch.as_tensor(lay.mask, device=dev))
    row_seq = torch.empty(R, dtype=torch.int32, device=dev)
    act = torch.empty(R, dtype=torch.int32, device=dev)
    na = torch.zeros(1, dtype=torch.int64, device=dev)
    ws = rl.Workspace(dev)
    ms = timed(lambda: rl.rl_batch_prepare(head, b, row_seq=row_seq, active_idx=act, n_active=na,
                                           ws=ws), a.reps)
    T = int(na.item())
    alg = R * (1 + 4 + 4) + 4 * (S + 1) + 4 * T          # mask, targets in; row_seq, active out
    moved = alg + R * 1 + 8 * T                           # + act flags, compact targets/seqs
    out["h1_whole_batch"] = {"rows": R, "tokens": T, "launches": 2, "ms": round(ms, 4),
                             "bytes_alg": alg, "bytes_moved": moved,
                             "gbs_alg": round(alg / ms / 1e6, 1),
                             "gbs_moved": round(moved / ms / 1e6, 1),
                             "frac_hbm_moved": round(moved / ms / 1e6 / hbm, 4)}
    # H2 over the mini-batch's sequences
    gos = torch.as_tensor(lay.group_of_seq, device=dev)
    rw = torch.as_tensor(lay.rewards, device=dev)
    adv = torch.empty(S, device=dev)
    ms = timed(lambda: rl.rl_grpo_advantage(rw, gos, lay.num_groups, adv), a.reps)
    nb = 12 * S
    out["h2_grpo"] = {"seqs": S, "groups": lay.num_groups, "ms": round(ms, 4), "bytes": nb,
                      "gbs": round(nb / ms / 1e6, 2),
                      "note": "latency-bound: 12 B per sequence, one CTA"}
    # one bench micro-batch: per-kind live times of the HBM kernels
    cu = lay.cu_seqlens.astype(np.int64)
    s0, s1 = pack_micro_batches(cu[1:] - cu[:-1], a.mb_rows)[0]
    mb, _ = sub_layout(lay, np.arange(s0, s1))
    H, W = make_tensors_torch(cfg, mb.num_rows, seed=0, device=dev)
    bm = rl.Batch(torch.as_tensor(mb.cu_seqlens, device=dev),
                  torch.as_tensor(mb.targets, device=dev), torch.as_tensor(mb.mask, device=dev))
    Rm, Tm = mb.num_rows, mb.num_tokens
    old = torch.zeros(Rm, device=dev)
    rl.rl_logprob_fwd(head, H, W, bm, old, ws=ws)
    advm = torch.linspace(-1, 1, mb.num_seqs, device=dev)
    p = rl.LossParams(n_tokens_global=torch.tensor([lay.num_tokens], device=dev))
    logp = torch.empty(Rm, device=dev)
    gh = torch.empty_like(H)
    gw = torch.zeros(cfg.vocab, cfg.hidden, device=dev)
    rl.rl_policy_loss_fwd_bwd(head, H, W, bm, old, advm, p, logp, gh, gw, ws=ws)
    torch.cuda.synchronize()
    tr = rl.Trace(4096).start()
    for _ in range(a.reps):
        rl.rl_policy_loss_fwd_bwd(head, H, W, bm, old, advm, p, logp, gh, gw, ws=ws)
    torch.cuda.synchronize()
    kinds = tr.stop().by_kind()
    n_vt = -(-cfg.vocab // 256)
    per = {"merge": (12 * n_vt + 30) * Tm,
           "gather": 4 * cfg.hidden * Tm,
           "prepare": Rm * (1 + 4 + 1) + 12 * Tm}
    mbo = {"rows": Rm, "tokens": Tm}
    for k, (c, t) in kinds.items():
        ms = t / c
        e = {"launches_per_call": c // a.reps, "ms_per_launch": round(ms, 4)}
        if k in per:
            nbytes = per[k] * (a.reps / c)
            e["bytes_per_launch"] = int(nbytes)
            e["gbs"] = round(nbytes / ms / 1e6, 1)
            e["frac_hbm"] = round(nbytes / ms / 1e6 / hbm, 4)
        mbo[k] = e
    out["micro_batch"] = mbo
    print(json.dumps(out))


if __name__ == "__main__":
    main()
