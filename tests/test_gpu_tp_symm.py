"""Vocab-parallel head across 2 real GPUs: every dL/dH
sum mode -- NCCL, P2P over symmetric memory, NVLS two-shot, and the fused
multimem.red GEMM epilogue -- against the unsharded head on rank 0. Skipped
on boxes with fewer than 2 GPUs."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_tp2_all_collectives():
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29533",
           os.path.join(ROOT, "scripts", "tp_check.py"), "--config", "qwen1.5b", "--rows", "4096",
           "--reps", "2"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = [x for x in out.stdout.splitlines() if x.startswith("{")][-1]
    res = json.loads(line)["modes"]
    for mode, r in res.items():
        if "skipped" in r:
            assert mode in ("nvls", "fused"), (mode, r)
            continue
        assert r["max_dlogp"] <= 2e-3, (mode, r)
        assert r["rel_dH"] <= 1e-2 and r["rel_dW"] <= 1e-2, (mode, r)
        assert r["ranks_identical_dH"], (mode, r)
