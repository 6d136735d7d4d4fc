#!/usr/bin/env python
"""H1 bookkeeping probe: rl_batch_prepare once over a config's whole packed
mini-batch (6.18M rows at qwen7b), `--reps` times, device time per call and
algorithmic GB/s. Wrap in ncu for per-kernel times and DRAM bytes:

    python scripts/probe_h1.py --reps 5
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        -k regex:"k_validate|k_flags|k_scan|k_compact|k_seq" python scripts/probe_h1.py --reps 1
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="qwen7b")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import torch

    import paper_2509_15965_b200 as rl
    from workload import CONFIGS, make_layout
    cfg = CONFIGS[a.config]
    lay = make_layout(cfg, 0)
    dev = "cuda"
    R = lay.num_rows
    S = lay.cu_seqlens.shape[0] - 1
    b = rl.Batch(torch.as_tensor(lay.cu_seqlens, device=dev), torch.as_tensor(lay.targets, device=dev),
                 torch.as_tensor(lay.mask, device=dev))
    head = rl.Head(cfg.hidden, cfg.vocab, cfg.dtype)
    row_seq = torch.empty(R, dtype=torch.int32, device=dev)
    act = torch.empty(R, dtype=torch.int32, device=dev)
    na = torch.zeros(1, dtype=torch.int64, device=dev)
    ws = rl.Workspace(dev)
    rl.rl_batch_prepare(head, b, row_seq=row_seq, active_idx=act, n_active=na, ws=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        rl.rl_batch_prepare(head, b, row_seq=row_seq, active_idx=act, n_active=na, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    T = int(na.item())
    nbytes = R * (4 + 1 + 4) + 4 * (S + 1) + 4 * T
    print(json.dumps({"config": a.config, "rows": R, "tokens": T, "ms": round(ms, 4),
                      "bytes": nbytes, "gbs": round(nbytes / (ms / 1e3) / 1e9, 1)}))


if __name__ == "__main__":
    main()
