"""NEXT-2 on the GPU: the micro-batch streaming interface (deferred 1/N)
reproduces the known-N step, and the minibatch early stop decides
exactly as the oracle rule on the same statistics and discards dW."""
import numpy as np
import pytest

import oracle
from tests.gpu_util import dev_tensors, rel_fro
from workload import HeadConfig, make_layout, make_tensors_host

pytestmark = pytest.mark.gpu

SMALL_BF16 = HeadConfig("small-bf16", 192, 1000, 6, 4, 96, "bf16", "reasoning")


def test_streaming_equals_known_n(rl):
    import torch
    from paper_2509_15965_b200.dp import (PolicyLossStep, StreamingPolicyLoss, device_batch,
                                          pack_micro_batches)
    cfg = SMALL_BF16
    lay = make_layout(cfg, seed=41)
    H, W = make_tensors_host(cfg, lay.num_rows, seed=41)
    dev = "cuda"
    Hd, Wd = H.to(dev), W.to(dev)
    head = rl.Head(cfg.hidden, cfg.vocab, cfg.dtype)
    db = device_batch(lay, 2048, device=dev)
    assert len(db.mbs) >= 3
    old = torch.zeros(lay.num_rows, device=dev)
    step = PolicyLossStep(head, Wd, db)
    gh = torch.empty_like(Hd)
    step.run(Hd, old, gh)
    s = StreamingPolicyLoss(head, Wd)
    s.begin()
    logp = torch.empty(lay.num_rows, device=dev)
    gh2 = torch.empty_like(Hd)
    for (s0, s1, r0, r1, cu_mb) in db.mbs:         # micro-batches arriving one by one
        b = rl.Batch(cu_mb, db.targets[r0:r1], db.mask[r0:r1], num_rows=r1 - r0)
        s.feed(Hd[r0:r1], b, old[r0:r1], step.adv[s0:s1], logp[r0:r1], gh2[r0:r1])
    s.finish()
    torch.cuda.synchronize()
    assert int(s.n_tokens.item()) == lay.num_tokens and int(s.stop_flag.item()) == 0
    # dZ is rounded to bf16 in both runs but at different scales (g vs g/N), so
    # the two dW differ by at most two bf16 roundings: 2 * 2^-9 relative.
    assert rel_fro(s.grad_w.cpu().numpy(), step.grad_w.cpu().numpy()) <= 2 * 2 ** -9
    a, b = rl.read_stats(s.stats), rl.read_stats(step.stats)
    assert a["loss_sum"] == pytest.approx(b["loss_sum"], rel=1e-6)
    # the unscaled dL/dH of each micro-batch times 1/N is the known-N dL/dH
    gh2_scaled = gh2.double() / lay.num_tokens
    assert rel_fro(gh2_scaled.cpu().numpy(), gh.double().cpu().numpy()) <= 1e-2


@pytest.mark.parametrize("max_ratio,max_mean", [(1.5, 0.0), (0.0, 1.01), (100.0, 0.0),
                                                (0.0, 0.0)])
def test_early_stop_matches_rule(rl, max_ratio, max_mean):
    import torch
    stats = {"loss_sum": 1.0, "ratio_sum": 105.0, "entropy_sum": 0.0, "kl_sum": 0.0,
             "objective": 0.0, "ratio_max": 2.25, "clip_lo_count": 0, "clip_hi_count": 0,
             "tokens": 100}
    from paper_2509_15965_b200 import rlhead as R
    raw = bytes(R.rl_loss_stats(stats["loss_sum"], stats["ratio_sum"], stats["entropy_sum"], 0.0,
                                0.0, stats["ratio_max"], 0, 0, 0, stats["tokens"]))
    st = torch.frombuffer(bytearray(raw), dtype=torch.uint8).clone().cuda()
    flag = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    gw = torch.ones(1000, 7, device="cuda")
    gw[3, 2] = float("nan")                 # a discarded update may hold NaN/Inf
    gw[999, 6] = float("inf")
    rl.rl_minibatch_early_stop(st, flag, gw, max_ratio, max_mean)
    torch.cuda.synchronize()
    want = oracle.head.minibatch_early_stop(stats, max_ratio, max_mean)
    assert int(flag.item()) == int(want)
    if want:                                # grad_weight := 0 exactly (header contract)
        assert bool((gw == 0).all())
    else:
        assert torch.isnan(gw[3, 2]) and float(gw[0].abs().max()) == 1.0


def test_scale_by_inverse_count(rl):
    import torch
    x = torch.arange(1, 1003, dtype=torch.float32, device="cuda")
    for n in (7, 0):
        y = x.clone()
        rl.rl_scale_by_inverse_count(y, torch.tensor([n], device="cuda"))
        torch.cuda.synchronize()
        ref = oracle.head.scale_by_inverse_count(x.cpu().numpy(), n)
        # fp32: 1/N rounded once, the product rounded once -> 2 ulp relative
        np.testing.assert_allclose(y.cpu().numpy(), ref, rtol=2 * 2 ** -23)


def test_streaming_vs_oracle(rl):
    """The streaming interface (micro-batches fed before N is known, deferred
    1/N) against the CPU float64 oracle of the whole global batch:
    dW, the statistics and every micro-batch's logp within the bf16 tolerances."""
    import torch
    from paper_2509_15965_b200.dp import StreamingPolicyLoss, device_batch
    cfg = SMALL_BF16
    lay = make_layout(cfg, seed=43)
    H, W = make_tensors_host(cfg, lay.num_rows, seed=43)
    adv, _ = oracle.grpo_advantage(lay.rewards, lay.group_of_seq, lay.num_groups)
    fwd = oracle.logprob_fwd(H, W, lay.cu_seqlens, lay.mask, lay.targets)
    from tests.gpu_util import guarded_old_logp
    old = guarded_old_logp(fwd["logp"], np.random.default_rng(43))
    ref = oracle.policy_loss_fwd_bwd(H, W, lay.cu_seqlens, lay.mask, lay.targets, old, adv,
                                     n_global=lay.num_tokens)
    dev = "cuda"
    Hd, Wd = H.to(dev), W.to(dev)
    head = rl.Head(cfg.hidden, cfg.vocab, cfg.dtype)
    db = device_batch(lay, 2048, device=dev)
    assert len(db.mbs) >= 3
    old_t = torch.as_tensor(old, dtype=torch.float32, device=dev)
    adv_t = torch.as_tensor(adv, dtype=torch.float32, device=dev)
    s = StreamingPolicyLoss(head, Wd)
    s.begin()
    logp = torch.empty(lay.num_rows, device=dev)
    gh = torch.empty_like(Hd)
    for (s0, s1, r0, r1, cu_mb) in db.mbs:
        b = rl.Batch(cu_mb, db.targets[r0:r1], db.mask[r0:r1], num_rows=r1 - r0)
        s.feed(Hd[r0:r1], b, old_t[r0:r1], adv_t[s0:s1], logp[r0:r1], gh[r0:r1])
    s.finish()
    torch.cuda.synchronize()
    st = rl.read_stats(s.stats)
    assert st["tokens"] == ref["stats"]["tokens"]
    assert st["loss_sum"] == pytest.approx(ref["stats"]["loss_sum"], rel=1e-2)
    assert np.abs(logp.cpu().double().numpy() - ref["logp"]).max() <= 2e-3
    gw = s.grad_w.cpu().double().numpy()
    assert rel_fro(gw, ref["dW"]) <= 1e-2
    # dL/dH of the streamed micro-batches is unscaled (loss_scale = 1): x 1/N
    assert rel_fro(gh.cpu().double().numpy() / lay.num_tokens, ref["dH"]) <= 1e-2
