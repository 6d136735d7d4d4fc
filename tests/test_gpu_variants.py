"""The tensor-core GEMM variants (1-CTA tiles, 2-CTA 256-wide tiles, 2-CTA
512-wide dH/dW tiles) all pass the bf16 parity tests. The variant is fixed per
process (read once from the environment), so each runs in a subprocess."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [{"RLHEAD_CTA_GROUP": "1"},
                                 {"RLHEAD_CTA_GROUP": "2", "RLHEAD_WIDE": "0"},
                                 {"RLHEAD_CTA_GROUP": "2", "RLHEAD_WIDE": "1",
                                  "RLHEAD_FUSED_BWD": "1"},
                                 {"RLHEAD_CTA_GROUP": "2", "RLHEAD_WIDE": "1",
                                  "RLHEAD_GROUP_M": "16", "RLHEAD_GROUP_M_BWD": "4"},
                                 {"RLHEAD_DW_RED": "0"},
                                 {"RLHEAD_DW_RED": "1", "RLHEAD_FUSED_BWD": "1"},
                                 {"RLHEAD_DW_RED": "2"},
                                 {"RLHEAD_L2_DW": "21", "RLHEAD_L2_DH": "21"},
                                 {"RLHEAD_DW_SERP": "1", "RLHEAD_DW_RED": "2"},
                                 {"RLHEAD_NONPERSIST_DW": "1", "RLHEAD_NONPERSIST_DH": "1"},
                                 {"RLHEAD_DYN_SCHED": "1"},
                                 {"RLHEAD_DYN_SCHED": "1", "RLHEAD_FUSED_BWD": "1",
                                  "RLHEAD_CTA_GROUP": "2"},
                                 {"RLHEAD_DYN_SCHED": "1", "RLHEAD_CTA_GROUP": "1"},
                                 {"RLHEAD_DZ_TMA": "1", "RLHEAD_CTA_GROUP": "1"},
                                 {"RLHEAD_DZ_TMA": "1", "RLHEAD_DW_RED": "2",
                                  "RLHEAD_DYN_SCHED": "1"},
                                 {"RLHEAD_DZ_RECOMPUTE": "1"},
                                 {"RLHEAD_DZ_RECOMPUTE": "1", "RLHEAD_FUSED_BWD": "1"},
                                 {"RLHEAD_DZ_FUSED": "1"}],
                         ids=["cta1", "cta2-narrow", "cta2-wide-fused", "cta2-unfused-raster",
                              "dw-load-store", "dw-red-fused", "dw-tma-reduce", "l2-hints",
                              "dw-serpentine", "non-persistent",
                              "dyn-sched", "dyn-sched-fused", "dyn-sched-cta1",
                              "dz-tma-cta1", "tma-all-dyn", "dz-recompute",
                              "dz-recompute-fused", "dz-fused-prefix"])
def test_variant_parity(env):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        "tests/test_gpu_parity.py", "-k", "bf16 or qwen15b or determinism"],
                       cwd=ROOT, env={**os.environ, **env}, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_dw_accumulate_paths_bit_identical(rl):
    """dW += dZ^T Hc through the three epilogue accumulate paths (load+add+
    store, red.global.add, TMA bulk reduce-add of smem boxes) adds the same
    fp32 tile to the same fp32 value once per element per launch: the results
    must be bit-identical, over a ragged V (not a multiple of the 256-row
    tile) and h (not a multiple of the 512-column tile), starting from a
    non-zero accumulator and over two launches."""
    import numpy as np
    import torch
    from tests.gpu_util import dev_tensors
    from workload import custom_layout
    rng = np.random.default_rng(11)
    V, h = 3000, 576
    lay = custom_layout(rng.integers(0, 30, 24), rng.integers(1, 200, 24), np.arange(24) // 4,
                        rng.choice([-5.0, 5.0], 24), vocab=V, num_groups=6)
    d = dev_tensors(lay)
    g = torch.Generator(device="cuda").manual_seed(5)
    H = torch.randn(lay.num_rows, h, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(V, h, device="cuda", generator=g) * (4 / h ** 0.5)).to(torch.bfloat16)
    gw0 = torch.randn(V, h, device="cuda", generator=g) * 1e-3
    head = rl.Head(h, V, "bf16")
    old = torch.empty(lay.num_rows, device="cuda")      # ratio = 1: every token has a gradient
    rl.rl_logprob_fwd(head, H, W, rl.Batch(d["cu"], d["targets"], d["mask"], d["err"]), old)
    adv = torch.linspace(-1, 1, lay.num_seqs, device="cuda")
    out = {}
    prev = os.environ.get("RLHEAD_DW_RED")
    try:
        for mode in ("0", "1", "2"):
            os.environ["RLHEAD_DW_RED"] = mode
            gw = gw0.clone()
            for _ in range(2):
                logp = torch.empty(lay.num_rows, device="cuda")
                gh = torch.empty_like(H)
                b = rl.Batch(d["cu"], d["targets"], d["mask"], d["err"])
                rl.rl_policy_loss_fwd_bwd(head, H, W, b, old, adv, rl.LossParams(), logp, gh, gw)
            torch.cuda.synchronize()
            out[mode] = gw.cpu()
    finally:
        if prev is None:
            os.environ.pop("RLHEAD_DW_RED", None)
        else:
            os.environ["RLHEAD_DW_RED"] = prev
    assert not torch.equal(out["1"], gw0.cpu())
    assert torch.equal(out["0"], out["1"])
    assert torch.equal(out["2"], out["1"])


def test_schedule_and_store_paths_bit_identical(rl):
    """The dynamic tile scheduler (RLHEAD_DYN_SCHED=1) only changes which CTA
    pair runs a tile and when, and the TMA dZ stores (RLHEAD_DZ_TMA=1) only
    how the same bf16 values reach HBM: logp, entropy, dH and dW must be
    bit-identical to the static schedule with per-row stores, over a multi-
    wave problem (1.5k forward tiles on 74 pairs, V not a multiple of 32), and
    the scheduler counters must reset between launches (repeated calls on one
    workspace give the same result)."""
    import numpy as np
    import torch
    from tests.gpu_util import dev_tensors
    from workload import custom_layout
    rng = np.random.default_rng(12)
    V, h = 32061, 512
    lay = custom_layout(rng.integers(0, 40, 32), rng.integers(1, 180, 32), np.arange(32) // 8,
                        rng.choice([-5.0, 5.0], 32), vocab=V, num_groups=4)
    d = dev_tensors(lay)
    g = torch.Generator(device="cuda").manual_seed(6)
    H = torch.randn(lay.num_rows, h, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(V, h, device="cuda", generator=g) * (4 / h ** 0.5)).to(torch.bfloat16)
    head = rl.Head(h, V, "bf16")
    old = torch.empty(lay.num_rows, device="cuda")
    rl.rl_logprob_fwd(head, H, W, rl.Batch(d["cu"], d["targets"], d["mask"], d["err"]), old)
    old += 0.05
    adv = torch.linspace(-1, 1, lay.num_seqs, device="cuda")
    ws = rl.Workspace("cuda")
    variants = [{"RLHEAD_DYN_SCHED": "0", "RLHEAD_DZ_TMA": "0", "RLHEAD_DW_RED": "1"},
                {"RLHEAD_DYN_SCHED": "1", "RLHEAD_DZ_TMA": "0", "RLHEAD_DW_RED": "1"},
                {"RLHEAD_DYN_SCHED": "1", "RLHEAD_DZ_TMA": "0", "RLHEAD_DW_RED": "1"},
                {"RLHEAD_DYN_SCHED": "0", "RLHEAD_DZ_TMA": "1", "RLHEAD_DW_RED": "2"},
                {"RLHEAD_DYN_SCHED": "1", "RLHEAD_DZ_TMA": "1", "RLHEAD_DW_RED": "2"}]
    res = []
    saved = {k: os.environ.get(k) for k in variants[0]}
    try:
        for env in variants:
            os.environ.update(env)
            logp = torch.empty(lay.num_rows, device="cuda")
            ent = torch.empty(lay.num_rows, device="cuda")
            gh = torch.empty_like(H)
            gw = torch.zeros(V, h, device="cuda")
            b = rl.Batch(d["cu"], d["targets"], d["mask"], d["err"])
            rl.rl_policy_loss_fwd_bwd(head, H, W, b, old, adv, rl.LossParams(), logp, gh, gw,
                                      entropy=ent, ws=ws)
            torch.cuda.synchronize()
            res.append([x.cpu() for x in (logp, ent, gh, gw)])
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    for env, other in zip(variants[1:], res[1:]):
        for name, a, b in zip(("logp", "entropy", "dH", "dW"), res[0], other):
            assert torch.equal(a, b), (env, name)
    assert float(res[0][3].abs().max()) > 0


def test_fused_backward_bit_identical(rl):
    """The fused dH + dW launch (RLHEAD_FUSED_BWD=1: one persistent tile
    space, dH tiles first, so the dH launch's partial last wave fills with dW
    tiles) runs every tile exactly as the two separate launches do -- same K
    order (serpentine dW waves counted from the first dW tile), same TMA
    reduce-add of the dW boxes -- so dH and dW must be bit-identical, over a
    problem with several dH and dW waves and a ragged V."""
    import numpy as np
    import torch
    from tests.gpu_util import dev_tensors
    from workload import custom_layout
    rng = np.random.default_rng(13)
    V, h = 40007, 1024
    lay = custom_layout(rng.integers(0, 40, 40), rng.integers(200, 900, 40), np.arange(40) // 8,
                        rng.choice([-5.0, 5.0], 40), vocab=V, num_groups=5)
    d = dev_tensors(lay)
    g = torch.Generator(device="cuda").manual_seed(7)
    H = torch.randn(lay.num_rows, h, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(V, h, device="cuda", generator=g) * (4 / h ** 0.5)).to(torch.bfloat16)
    head = rl.Head(h, V, "bf16")
    old = torch.empty(lay.num_rows, device="cuda")
    rl.rl_logprob_fwd(head, H, W, rl.Batch(d["cu"], d["targets"], d["mask"], d["err"]), old)
    adv = torch.linspace(-1, 1, lay.num_seqs, device="cuda")
    res = {}
    prev = os.environ.get("RLHEAD_FUSED_BWD")
    try:
        for mode in ("0", "1"):
            os.environ["RLHEAD_FUSED_BWD"] = mode
            gw = torch.full((V, h), 0.25, device="cuda")
            gh = torch.empty_like(H)
            logp = torch.empty(lay.num_rows, device="cuda")
            tr = rl.Trace(64).start()
            rl.rl_policy_loss_fwd_bwd(head, H, W, rl.Batch(d["cu"], d["targets"], d["mask"]),
                                      old, adv, rl.LossParams(), logp, gh, gw)
            torch.cuda.synchronize()
            kinds = tr.stop().by_kind()
            res[mode] = (gh.cpu(), gw.cpu(), kinds)
    finally:
        if prev is None:
            os.environ.pop("RLHEAD_FUSED_BWD", None)
        else:
            os.environ["RLHEAD_FUSED_BWD"] = prev
    assert "gemm_dhdw" in res["1"][2] and "gemm_dh" not in res["1"][2]
    assert "gemm_dh" in res["0"][2] and "gemm_dw" in res["0"][2]
    assert torch.equal(res["0"][0], res["1"][0])
    assert torch.equal(res["0"][1], res["1"][1])
    assert float((res["0"][1] - 0.25).abs().max()) > 0
