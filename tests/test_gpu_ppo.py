"""NEXT-4 on the CUDA path vs the oracle (oracle/ppo.py): GAE over packed
trajectories, the value head with the clipped value loss (fp32 and bf16), and
the policy loss with per-token (GAE) advantages."""
import numpy as np
import pytest

import oracle
from oracle import ppo
from tests.gpu_util import dev_tensors, guarded_old_logp, rel_fro
from workload import HeadConfig, custom_layout, make_layout, make_tensors_host

pytestmark = pytest.mark.gpu


def test_gae_parity(rl):
    import torch
    rng = np.random.default_rng(0)
    lens = np.concatenate([np.full(64, 64), rng.integers(1, 300, 40)])   # OpenVLA-like + ragged
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    n = int(cu[-1])
    r = rng.choice([0.0, 1.0], size=n, p=[0.9, 0.1]).astype(np.float32)
    v = rng.normal(0, 0.5, size=n).astype(np.float32)
    d = (rng.random(n) < 0.02).astype(np.uint8)
    boot = rng.normal(size=len(lens)).astype(np.float32)
    dev = "cuda"
    for gamma, lam, use_d, use_b in [(0.99, 0.95, True, True), (1.0, 1.0, False, False),
                                      (0.9, 0.0, True, False)]:
        adv = torch.empty(n, device=dev)
        ret = torch.empty(n, device=dev)
        rl.rl_gae(torch.as_tensor(r, device=dev), torch.as_tensor(v, device=dev),
                  torch.as_tensor(cu, device=dev), gamma, lam, adv, ret,
                  dones=torch.as_tensor(d, device=dev) if use_d else None,
                  bootstrap=torch.as_tensor(boot, device=dev) if use_b else None)
        torch.cuda.synchronize()
        ra, rr = ppo.gae(r, v, d if use_d else np.zeros_like(d),
                         boot if use_b else np.zeros_like(boot), cu, gamma, lam)
        np.testing.assert_allclose(adv.cpu().double().numpy(), ra, rtol=1e-6, atol=1e-6)
        np.testing.assert_allclose(ret.cpu().double().numpy(), rr, rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("dtype,tol_v,tol_g", [("f32", 1e-5, 1e-5), ("bf16", 2e-3, 1e-2)])
def test_value_loss_parity(rl, dtype, tol_v, tol_g):
    import torch
    cfg = HeadConfig("v", 256, 8, 4, 4, 64, dtype, "reasoning")
    lay = make_layout(cfg, seed=5)
    H, _ = make_tensors_host(cfg, lay.num_rows, seed=5)
    rng = np.random.default_rng(6)
    w = torch.as_tensor(rng.normal(0, 1 / 16, size=cfg.hidden), dtype=H.dtype)
    bv = 0.25
    v_or = ppo.value_fwd(H, w, bv, lay.cu_seqlens, lay.mask)
    # old values / returns with the clip decision away from its boundaries
    old = v_or + rng.choice([-1, 1], lay.num_rows) * rng.choice([0.05, 0.5], lay.num_rows)
    ret = v_or + rng.normal(0, 0.4, lay.num_rows)
    N = lay.num_tokens + 5
    ref = ppo.value_loss_fwd_bwd(H, w, bv, lay.cu_seqlens, lay.mask, ret, old, 0.2, n_global=N)
    d = dev_tensors(lay)
    dev = "cuda"
    Hd = H.to(dev)
    values = torch.full((lay.num_rows,), 9.0, device=dev)
    gh = torch.zeros_like(Hd)
    gw = torch.zeros(cfg.hidden, device=dev)
    gb = torch.zeros(1, device=dev)
    st = rl.new_stats()
    rl.rl_value_loss_fwd_bwd(rl.Head(cfg.hidden, 1, dtype), Hd, w.to(dev), bv,
                             rl.Batch(d["cu"], d["targets"], d["mask"]),
                             torch.as_tensor(ret, dtype=torch.float32, device=dev),
                             torch.as_tensor(old, dtype=torch.float32, device=dev), values, gh,
                             gw, gb, clip_eps=0.2,
                             n_tokens_global=torch.tensor([N], device=dev), stats=st)
    torch.cuda.synchronize()
    np.testing.assert_allclose(values.cpu().double().numpy(), ref["values"], atol=tol_v, rtol=0)
    s = rl.read_stats(st)
    assert s["tokens"] == lay.num_tokens and s["clip_hi_count"] == ref["clip_count"]
    assert s["objective"] == pytest.approx(ref["loss"], rel=tol_g)
    assert rel_fro(gh.cpu().double().numpy(), ref["dH"]) <= tol_g
    assert rel_fro(gw.cpu().double().numpy(), ref["dw"]) <= tol_g
    assert float(gb.item()) == pytest.approx(ref["db"], rel=tol_g, abs=1e-7)


def test_policy_loss_per_token_advantages(rl):
    """PPO: GAE advantages per token (e.g. a step's advantage on its 7 action
    tokens) through the same fused head."""
    import torch
    cfg = HeadConfig("small-bf16", 192, 1000, 6, 4, 96, "bf16", "reasoning")
    lay = make_layout(cfg, seed=51)
    H, W = make_tensors_host(cfg, lay.num_rows, seed=51)
    rng = np.random.default_rng(7)
    adv = rng.normal(size=lay.num_rows).astype(np.float32)
    lp = oracle.logprob_fwd(H, W, lay.cu_seqlens, lay.mask, lay.targets)["logp"]
    old = guarded_old_logp(lp, rng)
    ref = oracle.policy_loss_fwd_bwd(H, W, lay.cu_seqlens, lay.mask, lay.targets, old, adv,
                                     adv_per_token=True)
    d = dev_tensors(lay)
    dev = "cuda"
    Hd, Wd = H.to(dev), W.to(dev)
    logp = torch.empty(lay.num_rows, device=dev)
    gh = torch.empty_like(Hd)
    gw = torch.zeros(cfg.vocab, cfg.hidden, device=dev)
    p = rl.LossParams(adv_per_token=True,
                      n_tokens_global=torch.tensor([lay.num_tokens], device=dev))
    rl.rl_policy_loss_fwd_bwd(rl.Head(cfg.hidden, cfg.vocab), Hd, Wd,
                              rl.Batch(d["cu"], d["targets"], d["mask"]),
                              torch.as_tensor(old, dtype=torch.float32, device=dev),
                              torch.as_tensor(adv, device=dev), p, logp, gh, gw)
    torch.cuda.synchronize()
    assert rel_fro(gh.cpu().double().numpy(), ref["dH"]) <= 1e-2
    assert rel_fro(gw.cpu().double().numpy(), ref["dW"]) <= 1e-2
