#!/usr/bin/env python
"""Quick GEMM probe: one micro-batch of a config through rl_policy_loss_fwd_bwd
`--reps` times, per-kernel-kind device times (library CUDA-event tracer).
Cheap to set up (only the micro-batch's rows are generated), so it is the
command to wrap in ncu for kernel experiments:

    python scripts/probe.py --config qwen7b --reps 3
    ncu --metrics ... -k regex:k_tc_gemm python scripts/probe.py --reps 1
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
    ap.add_argument("--rows", type=int, default=65536)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--mb-index", type=int, default=10,
                    help="which micro-batch of the layout (the first ones belong to the "
                         "forced A = 0 groups, whose rows the backward skips)")
    ap.add_argument("--fwd-only", action="store_true")
    ap.add_argument("--cublas", action="store_true", help="also time torch.matmul of the shapes")
    ap.add_argument("--sustain", type=float, default=0.0, help="seconds of warm-up load")
    a = ap.parse_args()
    import torch

    import paper_2509_15965_b200 as rl
    from paper_2509_15965_b200.dp import pack_micro_batches
    from workload import CONFIGS, make_layout, make_tensors_torch, sub_layout
    cfg = CONFIGS[a.config]
    lay = make_layout(cfg, 0)
    cu = lay.cu_seqlens.astype(np.int64)
    mbs = pack_micro_batches(cu[1:] - cu[:-1], a.rows)
    s0, s1 = mbs[min(a.mb_index, len(mbs) - 1)]
    mb, _ = sub_layout(lay, np.arange(s0, s1))
    dev = "cuda"
    H, W = make_tensors_torch(cfg, mb.num_rows, seed=0, device=dev)
    head = rl.Head(cfg.hidden, cfg.vocab, cfg.dtype)
    b = rl.Batch(torch.as_tensor(mb.cu_seqlens, device=dev), torch.as_tensor(mb.targets, device=dev),
                 torch.as_tensor(mb.mask, device=dev))
    R = mb.num_rows
    # ratios near 1 (old = own log-probs + 0.01) and |A| = 1: every active row
    # carries a gradient, so the backward GEMMs see all rows (no skip)
    old = torch.empty(R, device=dev)
    rl.rl_logprob_fwd(head, H, W, b, old)
    old += 0.01
    adv = torch.where(torch.arange(mb.num_seqs, device=dev) % 2 == 0, 1.0, -1.0)
    p = rl.LossParams(n_tokens_global=torch.tensor([lay.num_tokens], device=dev))
    logp = torch.empty(R, device=dev)
    gh = torch.empty_like(H)
    gw = torch.zeros(cfg.vocab, cfg.hidden, device=dev)
    ws = rl.Workspace(dev)
    tr = rl.Trace(4096)

    def once():
        if a.fwd_only:
            rl.rl_logprob_fwd(head, H, W, b, logp, ws=ws)
        else:
            rl.rl_policy_loss_fwd_bwd(head, H, W, b, old, adv, p, logp, gh, gw, ws=ws)

    once()
    torch.cuda.synchronize()
    import time
    t_end = time.time() + a.sustain
    while time.time() < t_end:         # reach the power-capped steady state
        once()
        torch.cuda.synchronize()
    tok = int(mb.mask.sum())
    out = {"config": a.config, "tokens": tok, "reps": a.reps, "micro_batch": int(a.mb_index)}
    shapes = {}
    if a.cublas:
        # library reference: cuBLAS (torch.matmul) for the same GEMM shapes,
        # outputs materialised (what an unfused head would do); timed
        # interleaved with ours so both see the same power/clock state.
        Hc = H[torch.as_tensor(np.flatnonzero(mb.mask), device=dev)].contiguous()
        # real-valued operands (uninitialised memory can be zeros, which draw
        # less power and clock higher): dZ ~ the magnitude of a softmax gradient
        gz = torch.Generator(device=dev).manual_seed(9)
        dZ = (torch.randn(tok, cfg.vocab, generator=gz, device=dev) * 1e-6).to(H.dtype)
        shapes = {"cublas_fwd_HWt": (Hc, W.t()),
                  "cublas_dH_ZW": (dZ, W),
                  "cublas_dW_ZtH": (dZ.t(), Hc)}
    cub = {k: 0.0 for k in shapes}
    tr.start()
    for _ in range(a.reps):
        once()
        for k, (x, y) in shapes.items():
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            z = torch.matmul(x, y)
            e1.record()
            torch.cuda.synchronize()
            cub[k] += e0.elapsed_time(e1)
            del z
    torch.cuda.synchronize()
    tr.stop()
    for k, t in cub.items():
        ms = t / a.reps
        out[k] = {"ms": round(ms, 3),
                  "tflops": round(2.0 * cfg.hidden * cfg.vocab * tok / (ms / 1e3) / 1e12, 1)}
    for k, (c, t) in tr.by_kind().items():
        ms = t / c
        entry = {"ms": round(ms, 3)}
        if k.startswith("gemm"):
            units = rl.rlhead.GEMM_FLOP_UNITS.get(k, 1)
            entry["tflops"] = round(units * 2.0 * cfg.hidden * cfg.vocab * tok / (ms / 1e3) / 1e12,
                                    1)
        out[k] = entry
    print(json.dumps(out))


if __name__ == "__main__":
    main()
