"""Shared helpers of the GPU parity tests: move a workload to the device, run
the CUDA path through the C ABI, run the oracle on the same values, compare."""
from __future__ import annotations

import numpy as np


def dev_tensors(lay, device="cuda"):
    import torch
    return dict(
        cu=torch.as_tensor(lay.cu_seqlens, dtype=torch.int32, device=device),
        targets=torch.as_tensor(lay.targets, dtype=torch.int32, device=device),
        mask=torch.as_tensor(lay.mask, dtype=torch.uint8, device=device),
        gos=torch.as_tensor(lay.group_of_seq, dtype=torch.int32, device=device),
        rewards=torch.as_tensor(lay.rewards, dtype=torch.float32, device=device),
        err=torch.zeros(1, dtype=torch.int32, device=device),
    )


def guarded_old_logp(logp64, rng, clip_lo=0.2, clip_hi=0.2, band=1e-2, sigma=0.2):
    """old = logp - ln r*, r* ~ lognormal, rejected within `band` of 1 +- eps
    (keeps fp32-vs-fp64 clip decisions identical)."""
    n = logp64.shape[0]
    out = np.empty(n)
    for i in range(n):
        while True:
            x = float(np.exp(rng.normal(0.0, sigma)))
            if min(abs(x - (1 - clip_lo)), abs(x - (1 + clip_hi))) > band:
                break
        out[i] = logp64[i] - np.log(x)
    return out


def rel_fro(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def max_rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.abs(b).max()
    return float(np.abs(a - b).max() / (den if den > 0 else 1.0))
