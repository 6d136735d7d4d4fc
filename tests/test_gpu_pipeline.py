"""The split loss API (rl_policy_loss_fwd + rl_policy_loss_bwd) and the
two-stream micro-batch pipeline built on it (PolicyLossStep(pipeline=True):
fwd(i+1) on the main stream beside bwd(i) on an auxiliary stream, two
workspaces) compute exactly what the serial rl_policy_loss_fwd_bwd loop does:
the same kernels on the same values in the same per-stream order, so logp,
dL/dH, dW and the loss statistics must be bit-identical."""
import numpy as np
import pytest

from workload import CONFIGS, HeadConfig, make_layout, make_tensors_torch

pytestmark = pytest.mark.gpu

SMALL_BF16 = HeadConfig("small-bf16", 256, 3000, 8, 4, 300, "bf16", "reasoning")


@pytest.mark.parametrize("cfg,mb_rows", [(SMALL_BF16, 600), (CONFIGS["openvla"], 4096)],
                         ids=["small", "openvla-head"])
def test_pipeline_bit_identical(rl, cfg, mb_rows):
    import torch
    from paper_2509_15965_b200.dp import PolicyLossStep, device_batch
    from workload import sub_layout
    lay = make_layout(cfg, seed=3)
    if cfg.name == "openvla":
        lay, _ = sub_layout(lay, np.arange(48))         # 6 groups, 21.5k rows
    dev = "cuda"
    H, W = make_tensors_torch(cfg, lay.num_rows, seed=3, device=dev)
    head = rl.Head(cfg.hidden, cfg.vocab, cfg.dtype)
    db = device_batch(lay, mb_rows, device=dev)
    assert len(db.mbs) >= 3
    old = torch.empty(lay.num_rows, device=dev)
    for (_, _, r0, r1, cu_mb) in db.mbs:
        rl.rl_logprob_fwd(head, H[r0:r1], W, rl.Batch(cu_mb, db.targets[r0:r1], db.mask[r0:r1],
                                                      num_rows=r1 - r0), old[r0:r1])
    old += 0.03
    out = {}
    for pipe in (False, True):
        step = PolicyLossStep(head, W, db, pipeline=pipe)
        gh = torch.full_like(H, 9.0)
        for _ in range(2):                              # repeated steps reuse the buffers
            step.run(H, old, gh)
        torch.cuda.synchronize()
        out[pipe] = (step.logp.cpu(), gh.cpu(), step.grad_w.cpu(), rl.read_stats(step.stats))
    for a, b in zip(out[False][:3], out[True][:3]):
        assert torch.equal(a, b)
    assert out[False][3] == out[True][3]
    assert float(out[True][2].abs().max()) > 0


def test_split_api_equals_fused_call(rl):
    import torch
    from tests.gpu_util import dev_tensors
    cfg = SMALL_BF16
    lay = make_layout(cfg, seed=4)
    H, W = make_tensors_torch(cfg, lay.num_rows, seed=4, device="cuda")
    d = dev_tensors(lay)
    head = rl.Head(cfg.hidden, cfg.vocab, cfg.dtype)
    b = rl.Batch(d["cu"], d["targets"], d["mask"])
    old = torch.empty(lay.num_rows, device="cuda")
    rl.rl_logprob_fwd(head, H, W, b, old)
    old -= 0.02
    adv = torch.linspace(-1, 1, lay.num_seqs, device="cuda")
    res = []
    for split in (False, True):
        logp = torch.empty(lay.num_rows, device="cuda")
        gh = torch.empty_like(H)
        gw = torch.zeros(cfg.vocab, cfg.hidden, device="cuda")
        st = rl.new_stats()
        args = (head, H, W, b, old, adv, rl.LossParams(), logp, gh, gw)
        if split:
            rl.rl_policy_loss_fwd(*args, stats=st)
            rl.rl_policy_loss_bwd(*args, stats=st)
        else:
            rl.rl_policy_loss_fwd_bwd(*args, stats=st)
        torch.cuda.synchronize()
        res.append((logp.cpu(), gh.cpu(), gw.cpu(), rl.read_stats(st)))
    for a, c in zip(res[0][:3], res[1][:3]):
        assert torch.equal(a, c)
    assert res[0][3] == res[1][3]
