"""Pins of the oracle's NEXT-1 loss variants (dual clip, KL-k3 to a reference
policy, entropy bonus, seq-mean-token-mean aggregation; DESIGN.md §3 #25-#28):
torch float64 autograd of the definitional objective, closed forms."""
import math

import numpy as np
import pytest

import oracle
from oracle.head import _kl_k3, _surrogate


def _problem(seed=0, R=26, h=6, V=13):
    rng = np.random.default_rng(seed)
    H = rng.normal(0, 1, size=(R, h))
    W = rng.normal(0, 1, size=(V, h))
    y = rng.integers(0, V, size=R).astype(np.int32)
    mask = np.ones(R, np.uint8)
    mask[[2, 9, 20]] = 0
    cu = np.array([0, 8, 17, R], np.int32)
    adv = np.array([1.1, -0.8, -0.3])
    return H, W, y, cu, mask, adv


def _guard(x, bounds, band=1e-3):
    return all(abs(x - b) > band for b in bounds)


def _inputs(H, W, y, cu, mask, tau, p, rng):
    lp = oracle.logprob_fwd(H, W, cu, mask, y, inv_temperature=tau)["logp"]
    old, ref = np.empty_like(lp), np.empty_like(lp)
    for t in range(len(lp)):
        while True:
            r = math.exp(rng.normal(0, 0.5))
            if _guard(r, [1 - p.clip_lo, 1 + p.clip_hi, p.dual_clip]):
                break
        old[t] = lp[t] - math.log(r)
        ref[t] = lp[t] + rng.normal(0, 0.3)
    return old, ref


def _torch_objective(H, W, y, cu, mask, old, ref, adv, tau, p, N=None, S=None):
    import torch
    Ht = torch.tensor(H, requires_grad=True)
    Wt = torch.tensor(W, requires_grad=True)
    seq = np.searchsorted(cu, np.arange(len(y)), side="right") - 1
    Z = (Ht @ Wt.T) * tau
    logsm = torch.log_softmax(Z, dim=1)
    logp = logsm[torch.arange(len(y)), torch.tensor(y).long()]
    Hent = -(logsm.exp() * logsm).sum(1)
    c = p.logratio_clamp
    r = torch.exp(torch.clamp(logp - torch.tensor(old), -c, c))
    A = torch.tensor(adv[seq])
    surr = torch.maximum(-A * r, -A * torch.clamp(r, 1 - p.clip_lo, 1 + p.clip_hi))
    if p.dual_clip > 0:
        surr = torch.where(A < 0, torch.minimum(surr, -A * p.dual_clip), surr)
    q = torch.clamp(torch.tensor(ref) - logp, -c, c)
    k3 = torch.exp(q) - q - 1
    obj = surr + p.kl_coef * k3 - p.entropy_coef * Hent
    m = torch.tensor(mask, dtype=torch.float64)
    if p.seq_mean:
        ns = np.bincount(seq[mask == 1], minlength=len(adv)).astype(np.float64)
        S = S if S is not None else int((ns > 0).sum())
        w = torch.tensor(1.0 / (S * np.maximum(ns[seq], 1)))
    else:
        w = torch.full((len(y),), 1.0 / (N if N is not None else int(mask.sum())),
                       dtype=torch.float64)
    L = (m * w * obj).sum()
    L.backward()
    return L.item(), Ht.grad.numpy(), Wt.grad.numpy()


@pytest.mark.parametrize("seq_mean", [False, True])
@pytest.mark.parametrize("tau", [1.0, 1.3])
def test_all_variants_vs_autograd(seq_mean, tau):
    H, W, y, cu, mask, adv = _problem(seed=3)
    p = oracle.LossParams(clip_lo=0.2, clip_hi=0.28, dual_clip=3.0, kl_coef=0.05,
                          entropy_coef=0.01, seq_mean=seq_mean)
    old, ref = _inputs(H, W, y, cu, mask, tau, p, np.random.default_rng(1))
    out = oracle.policy_loss_fwd_bwd(H, W, cu, mask, y, old, adv, p, inv_temperature=tau,
                                     ref_logp=ref)
    L, dH, dW = _torch_objective(H, W, y, cu, mask, old, ref, adv, tau, p)
    assert out["loss"] == pytest.approx(L, abs=1e-14)
    np.testing.assert_allclose(out["dH"], dH, atol=1e-14)
    np.testing.assert_allclose(out["dW"], dW, atol=1e-14)


def test_kl_at_reference_is_zero():
    """ref = own logp -> k3 = 0 and zero gradient: identical to kl_coef = 0."""
    H, W, y, cu, mask, adv = _problem(seed=5)
    lp = oracle.logprob_fwd(H, W, cu, mask, y)["logp"]
    old = lp - 0.05
    a = oracle.policy_loss_fwd_bwd(H, W, cu, mask, y, old, adv)
    b = oracle.policy_loss_fwd_bwd(H, W, cu, mask, y, old, adv, oracle.LossParams(kl_coef=0.7),
                                   ref_logp=lp)
    assert b["stats"]["kl_sum"] == pytest.approx(0.0, abs=1e-15)
    np.testing.assert_allclose(a["dW"], b["dW"], atol=1e-16)
    k, dk = _kl_k3(-1.0, -1.5, 20.0)
    assert k == pytest.approx(math.exp(-0.5) + 0.5 - 1) and dk == pytest.approx(1 - math.exp(-0.5))


def test_seq_mean_ratio_one_closed_form():
    """r = 1: L = -(1/S) sum_s A_s over sequences with tokens (seq-mean-token-mean)."""
    H, W, y, cu, mask, adv = _problem(seed=6)
    lp = oracle.logprob_fwd(H, W, cu, mask, y)["logp"]
    out = oracle.policy_loss_fwd_bwd(H, W, cu, mask, y, lp, adv,
                                     oracle.LossParams(seq_mean=True))
    assert out["loss"] == pytest.approx(-adv.mean(), abs=1e-14)


def test_dual_clip_quadrants():
    p = oracle.LossParams(dual_clip=3.0)
    _, l, g, _, _ = _surrogate(math.log(5.0), 0.0, -2.0, p)    # capped
    assert l == pytest.approx(6.0) and g == 0.0
    _, l, g, _, _ = _surrogate(math.log(2.0), 0.0, -2.0, p)    # below the cap
    assert l == pytest.approx(4.0) and g == pytest.approx(4.0)
    _, l, g, _, _ = _surrogate(math.log(5.0), 0.0, 2.0, p)     # A > 0 unaffected
    assert l == pytest.approx(-2.0 * 1.2) and g == 0.0


def test_entropy_bonus_uniform_has_no_gradient():
    """Zero logits: H = ln V is at its maximum -> the bonus adds no gradient."""
    V, h = 11, 4
    H = np.zeros((3, h))
    W = np.random.default_rng(0).normal(size=(V, h))
    cu, mask, y = np.array([0, 3], np.int32), np.ones(3, np.uint8), np.array([1, 2, 3], np.int32)
    old = oracle.logprob_fwd(H, W, cu, mask, y)["logp"]
    a = oracle.policy_loss_fwd_bwd(H, W, cu, mask, y, old, np.array([0.5]))
    b = oracle.policy_loss_fwd_bwd(H, W, cu, mask, y, old, np.array([0.5]),
                                   oracle.LossParams(entropy_coef=0.3))
    np.testing.assert_allclose(a["dH"], b["dH"], atol=1e-15)
    assert b["loss"] == pytest.approx(a["loss"] - 0.3 * math.log(V), abs=1e-14)


def test_streaming_deferred_scale_equals_token_mean():
    """P:L433-436 elastic pipelining: micro-batches with loss_scale = 1 then
    x 1/N at the end == the token mean computed with N known upfront."""
    H, W, y, cu, mask, adv = _problem(seed=9)
    lp = oracle.logprob_fwd(H, W, cu, mask, y)["logp"]
    old = lp + 0.03
    N = int(mask.sum())
    whole = oracle.policy_loss_fwd_bwd(H, W, cu, mask, y, old, adv)
    acc = np.zeros_like(whole["dW"])
    for s0, s1 in [(0, 2), (2, 3)]:
        r0, r1 = cu[s0], cu[s1]
        part = oracle.policy_loss_fwd_bwd(H[r0:r1], W, cu[s0:s1 + 1] - r0, mask[r0:r1], y[r0:r1],
                                          old[r0:r1], adv[s0:s1], oracle.LossParams(loss_scale=1.0))
        acc += part["dW"]
    np.testing.assert_allclose(oracle.head.scale_by_inverse_count(acc, N), whole["dW"], atol=1e-16)
    assert (oracle.head.scale_by_inverse_count(acc, 0) == 0).all()


def test_minibatch_early_stop_rule():
    """discard on too large importance ratio (max or token mean)."""
    st = dict(ratio_max=3.5, ratio_sum=120.0, tokens=100)
    es = oracle.head.minibatch_early_stop
    assert es(st, max_ratio=3.0) and not es(st, max_ratio=4.0)
    assert es(st, max_mean_ratio=1.1) and not es(st, max_mean_ratio=1.25)
    assert not es(st) and not es(dict(st, tokens=0), max_mean_ratio=1.0)
    assert not es(st, max_ratio=3.5)                 # strictly larger discards


# ---- REINFORCE++-style batch-normalised advantage (DESIGN.md §3 #33) -------
@pytest.mark.parametrize("Gn,G,k", [(1, 16, 5), (4, 8, 3), (8, 16, 1), (3, 4, 2)])
def test_batch_adv_identical_groups_closed_form(Gn, G, k):
    """Gn identical groups of G responses, k correct (+-5). With the
    group baseline x_correct = 10(G-k)/G, x_wrong = -10k/G, mean_B x = 0 and
    the unbiased batch variance is 100 Gn k(G-k)/G / (Gn G - 1), so
    A_correct = sqrt((G-k)(Gn G-1) / (G k Gn)), A_wrong = -k/(G-k) A_correct
    (Gn = 1 reduces to GRPO's unbiased P6). Without the baseline the batch is
    one pool of Gn*k correct of Gn*G: P6 with G -> Gn G."""
    r = np.array(([5.0] * k + [-5.0] * (G - k)) * Gn, dtype=np.float32)
    gos = np.repeat(np.arange(Gn), G).astype(np.int32)
    A, err = oracle.batch_norm_advantage(r, gos, Gn, group_baseline=True, eps=0.0)
    assert err == 0
    ac = math.sqrt((G - k) * (Gn * G - 1) / (G * k * Gn))
    np.testing.assert_allclose(A[r > 0], ac, rtol=1e-12)
    np.testing.assert_allclose(A[r < 0], -k / (G - k) * ac, rtol=1e-12)
    if Gn == 1:
        Ag, _ = oracle.grpo_advantage(r, gos, 1, eps=0.0)
        np.testing.assert_allclose(A, Ag, rtol=1e-12)
    n = Gn * G
    A, _ = oracle.batch_norm_advantage(r, gos, Gn, group_baseline=False, eps=0.0, unbiased=False)
    kk = Gn * k
    np.testing.assert_allclose(A[r > 0], math.sqrt((n - kk) / kk), rtol=1e-12)
    np.testing.assert_allclose(A[r < 0], -math.sqrt(kk / (n - kk)), rtol=1e-12)


def test_batch_adv_invariants():
    """sum_B A = 0, sum_B A^2 = n-1 (unbiased) / n (population), eps = 0; the
    group baseline makes A invariant to shifting one group's rewards, the
    no-baseline form is not; both are invariant to a global affine map."""
    rng = np.random.default_rng(8)
    r = rng.normal(size=40)
    gos = rng.integers(0, 5, size=40).astype(np.int32)
    for gb in (True, False):
        for unbiased, want in [(True, 39.0), (False, 40.0)]:
            A, _ = oracle.batch_norm_advantage(r, gos, 5, group_baseline=gb, eps=0.0,
                                               unbiased=unbiased)
            assert abs(A.sum()) < 1e-12
            assert (A ** 2).sum() == pytest.approx(want, rel=1e-12)
        A0, _ = oracle.batch_norm_advantage(r, gos, 5, group_baseline=gb, eps=0.0)
        A1, _ = oracle.batch_norm_advantage(3.0 * r - 2.0, gos, 5, group_baseline=gb, eps=0.0)
        np.testing.assert_allclose(A1, A0, rtol=1e-10, atol=1e-12)
        r2 = r.copy()
        r2[gos == 2] += 7.0
        A2, _ = oracle.batch_norm_advantage(r2, gos, 5, group_baseline=gb, eps=0.0)
        assert np.allclose(A2, A0, rtol=1e-10, atol=1e-12) == gb


def test_batch_adv_degenerate_and_invalid():
    """A = 0 exactly: every group zero-variance under the baseline (all x = 0),
    a single valid sequence, an all-equal batch without baseline. Invalid group
    ids get A = 0, raise ERR_GROUP and are left out of the batch statistics."""
    r = np.array([0.7] * 7 + [5, 5, 5], dtype=np.float32)
    gos = np.array([0] * 7 + [1] * 3, dtype=np.int32)
    A, err = oracle.batch_norm_advantage(r, gos, 2, group_baseline=True)
    assert err == 0 and (A == 0.0).all()
    A, _ = oracle.batch_norm_advantage(np.array([3.0], np.float32), np.array([0], np.int32), 1)
    assert (A == 0.0).all()
    A, _ = oracle.batch_norm_advantage(np.full(6, 2.5, np.float32), np.zeros(6, np.int32), 1,
                                       group_baseline=False)
    assert (A == 0.0).all()
    r = np.array([5, -5, 5, -5, 100.0], dtype=np.float32)
    gos = np.array([0, 0, 1, 1, 9], dtype=np.int32)
    A, err = oracle.batch_norm_advantage(r, gos, 2, group_baseline=False, eps=0.0, unbiased=False)
    assert err == oracle.ERR_GROUP and A[4] == 0.0
    np.testing.assert_allclose(A[:4], [1, -1, 1, -1], rtol=1e-12)
