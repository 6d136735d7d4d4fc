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


def _dp_check(args):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29534",
           os.path.join(ROOT, "scripts", "dp_check.py")] + args
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    return json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])


@pytest.mark.parametrize("empty_last", [False, True])
def test_dp2_fused_dw_reduce_scatter(empty_last):
    """the DP step with the dW reduce-scatter fused into the
    last micro-batch's dW GEMM epilogue + NVLink all-gather gives the NCCL
    all-reduce's dW on every rank (P = 2: the same two fp32 terms, bit-equal;
    1e-6 allowed), also when one rank's last micro-batch has no active row."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    res = _dp_check(["--config", "qwen1.5b", "--max-mb", "2", "--mb-rows", "8192", "--reps", "1"]
                    + (["--empty-last"] if empty_last else []))
    m = res["modes"]
    assert res["norm_dW"] > 0 and m["symm"]["rel_dW_vs_nccl"] <= 1e-6, res
    assert m["symm"]["tokens"] == m["nccl"]["tokens"]
    assert all(v["ranks_identical_dW"] for v in m.values()), res


def test_dp2_split_groups():
    """Split-group sharding (sequences, not whole groups, are
    LPT-assigned; group statistics all-reduced by global id): the whole-batch
    dW and token count equal the group-sharded step's (same global rows)."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    res = _dp_check(["--config", "qwen1.5b", "--max-mb", "0", "--mb-rows", "65536", "--reps", "1",
                     "--modes", "nccl,nccl-split,symm-split"])
    m = res["modes"]
    assert res["norm_dW"] > 0
    for k in ("nccl-split", "symm-split"):
        assert m[k]["rel_dW_vs_nccl"] <= 1e-5, res
        assert m[k]["tokens"] == m["nccl"]["tokens"], res
        assert abs(m[k]["loss_sum"] - m["nccl"]["loss_sum"]) <= 1e-6 * abs(m["nccl"]["loss_sum"]) + 1e-6
    assert all(v["ranks_identical_dW"] for v in m.values()), res
