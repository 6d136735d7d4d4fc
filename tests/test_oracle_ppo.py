"""Pins of the PPO oracle pieces (NEXT-4; DESIGN.md §3 #30-#32): GAE against
its explicit-sum form and the lambda = 0 / lambda = 1 closed forms, episode
resets; the clipped value loss against torch autograd of its definition."""
import numpy as np
import pytest

from oracle import ppo


def _traj(seed=0, S=5):
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, 12, size=S)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    n = int(cu[-1])
    r = rng.normal(size=n)
    v = rng.normal(size=n)
    d = (rng.random(n) < 0.15).astype(np.uint8)
    boot = rng.normal(size=S)
    return cu, r, v, d, boot


@pytest.mark.parametrize("gamma,lam", [(0.99, 0.95), (1.0, 1.0), (0.9, 0.0), (0.5, 0.7)])
def test_gae_explicit_sum(gamma, lam):
    """A_t = sum_l (gamma lam)^l delta_{t+l}, truncated at the first done."""
    cu, r, v, d, boot = _traj(1)
    adv, ret = ppo.gae(r, v, d, boot, cu, gamma, lam)
    for s in range(len(cu) - 1):
        a, b = cu[s], cu[s + 1]
        for t in range(a, b):
            total, coef = 0.0, 1.0
            for k in range(t, b):
                nv = boot[s] if k == b - 1 else v[k + 1]
                delta = r[k] + gamma * (0.0 if d[k] else 1.0) * nv - v[k]
                total += coef * delta
                if d[k]:
                    break
                coef *= gamma * lam
            assert adv[t] == pytest.approx(total, abs=1e-12)
    np.testing.assert_allclose(ret, adv + v, atol=0)


def test_gae_closed_forms():
    cu, r, v, d, boot = _traj(2)
    d[:] = 0
    g = 0.97
    a1, _ = ppo.gae(r, v, d, boot, cu, g, 1.0)        # lambda = 1: MC return - V
    for s in range(len(cu) - 1):
        a, b = cu[s], cu[s + 1]
        for t in range(a, b):
            mc = sum(g ** (k - t) * r[k] for k in range(t, b)) + g ** (b - t) * boot[s]
            assert a1[t] == pytest.approx(mc - v[t], abs=1e-12)
    a0, _ = ppo.gae(r, v, d, boot, cu, g, 0.0)        # lambda = 0: one-step TD error
    nv = np.concatenate([v[1:], [0]])
    for s in range(len(cu) - 1):
        nv[cu[s + 1] - 1] = boot[s]
    np.testing.assert_allclose(a0, r + g * nv - v, atol=1e-12)
    d[cu[1] - 1] = 1                                    # a done ignores the bootstrap
    a2, _ = ppo.gae(r, v, d, boot, cu, g, 0.9)
    assert a2[cu[1] - 1] == pytest.approx(r[cu[1] - 1] - v[cu[1] - 1], abs=1e-15)


def test_value_loss_autograd():
    import torch
    rng = np.random.default_rng(3)
    R, h = 30, 7
    H = rng.normal(size=(R, h))
    w = rng.normal(size=h)
    bv = 0.3
    mask = (rng.random(R) < 0.7).astype(np.uint8)
    cu = np.array([0, 13, R], np.int32)
    v = H @ w + bv
    old = v + rng.choice([-1, 1], R) * rng.uniform(0.0, 0.6, R)   # some beyond eps = 0.2
    ret = v + rng.normal(0, 0.5, R)
    eps = 0.2
    # keep |v - (old +- eps)| away from 0 so the clip decision is unambiguous
    out = ppo.value_loss_fwd_bwd(H, w, bv, cu, mask, ret, old, eps)
    Ht = torch.tensor(H, requires_grad=True)
    wt = torch.tensor(w, requires_grad=True)
    bt = torch.tensor(bv, dtype=torch.float64, requires_grad=True)
    vt = Ht @ wt + bt
    oldt, rett = torch.tensor(old), torch.tensor(ret)
    vc = torch.minimum(torch.maximum(vt, oldt - eps), oldt + eps)
    per = 0.5 * torch.maximum((vt - rett) ** 2, (vc - rett) ** 2)
    m = torch.tensor(mask, dtype=torch.float64)
    L = (per * m).sum() / mask.sum()
    L.backward()
    assert out["loss"] == pytest.approx(L.item(), abs=1e-14)
    np.testing.assert_allclose(out["dH"], Ht.grad.numpy(), atol=1e-14)
    np.testing.assert_allclose(out["dw"], wt.grad.numpy(), atol=1e-14)
    assert out["db"] == pytest.approx(bt.grad.item(), abs=1e-14)
    assert (out["dH"][mask == 0] == 0).all()


def test_value_loss_no_clip_closed_form():
    rng = np.random.default_rng(4)
    H = rng.normal(size=(9, 4))
    w = rng.normal(size=4)
    cu, mask = np.array([0, 9], np.int32), np.ones(9, np.uint8)
    v = H @ w
    ret = rng.normal(size=9)
    out = ppo.value_loss_fwd_bwd(H, w, 0.0, cu, mask, ret, v, 0.2)   # old = v: clip inactive
    assert out["loss"] == pytest.approx(0.5 * np.mean((v - ret) ** 2), abs=1e-14)
    assert out["clip_count"] == 0
