"""Pins of the CPU float64 oracle against things other than itself.

PAPER.md prints no value for this path, so the oracle is pinned by
(DESIGN.md §6): brute-force arbitrary-precision softmax, closed forms
(zero logits, GRPO +-5 groups from P:L833, ratio = 1, clip quadrants),
invariants, an independent float64 autograd of the *definitional* loss and
central finite differences. Each pin is chosen so that a plausible slip (a
dropped term, a sign, a wrong index or a transposed operand) fails it.
"""
import math

import mpmath
import numpy as np
import pytest

import oracle
from oracle.head import _surrogate
from workload import custom_layout

pytestmark = pytest.mark.filterwarnings("ignore::RuntimeWarning")


def _rand_problem(R=10, h=6, V=11, seed=0, scale=1.0):
    rng = np.random.default_rng(seed)
    H = rng.normal(0, 1, size=(R, h))
    W = rng.normal(0, scale, size=(V, h))
    y = rng.integers(0, V, size=R).astype(np.int32)
    return H, W, y


def _flat_batch(R, mask=None):
    cu = np.array([0, R], dtype=np.int32)
    m = np.ones(R, dtype=np.uint8) if mask is None else np.asarray(mask, dtype=np.uint8)
    return cu, m


# ----------------------------------------------------------------- H3/H4 ----
def test_p1_bruteforce_mpmath_softmax():
    """P1: 50-digit brute force of log-softmax and entropy, V <= 16. Entropy is
    computed as -sum p log p (not the oracle's lse - E_p[z])."""
    mpmath.mp.dps = 50
    for seed, V, tau in [(0, 7, 1.0), (1, 16, 1.0), (2, 11, 1 / 0.7)]:
        H, W, y = _rand_problem(R=5, h=4, V=V, seed=seed, scale=2.0)
        cu, m = _flat_batch(5)
        out = oracle.logprob_fwd(H, W, cu, m, y, inv_temperature=tau)
        for t in range(5):
            z = [mpmath.mpf(tau) * mpmath.fsum(mpmath.mpf(H[t, k]) * mpmath.mpf(W[j, k])
                                                for k in range(4)) for j in range(V)]
            lse = mpmath.log(mpmath.fsum(mpmath.exp(zj) for zj in z))
            p = [mpmath.exp(zj - lse) for zj in z]
            ent = -mpmath.fsum(pj * mpmath.log(pj) for pj in p)
            assert abs(out["logp"][t] - float(z[y[t]] - lse)) < 1e-13
            assert abs(out["lse"][t] - float(lse)) < 1e-13
            assert abs(out["entropy"][t] - float(ent)) < 1e-13


def test_p2_library_logsoftmax():
    """P2: torch float64 log_softmax / scipy logsumexp at a mid-size shape."""
    import torch
    from scipy.special import logsumexp
    H, W, y = _rand_problem(R=40, h=16, V=333, seed=3, scale=1.5)
    cu, m = _flat_batch(40)
    out = oracle.logprob_fwd(H, W, cu, m, y)
    Z = torch.from_numpy(H) @ torch.from_numpy(W).T
    ref = torch.log_softmax(Z, dim=1)[torch.arange(40), torch.from_numpy(y).long()].numpy()
    np.testing.assert_allclose(out["logp"], ref, atol=1e-12, rtol=0)
    np.testing.assert_allclose(out["lse"], logsumexp(Z.numpy(), axis=1), atol=1e-12, rtol=0)


@pytest.mark.parametrize("V", [11, 1000, 32064])
def test_p3_zero_logits_closed_form(V):
    """P3: zero hidden -> uniform softmax: logp = -ln V, entropy = lse = ln V."""
    H = np.zeros((3, 8))
    W = np.random.default_rng(0).normal(size=(V, 8))
    cu, m = _flat_batch(3)
    out = oracle.logprob_fwd(H, W, cu, m, np.array([0, V // 2, V - 1], dtype=np.int32))
    assert np.allclose(out["logp"], -math.log(V), atol=1e-12, rtol=0)
    assert np.allclose(out["entropy"], math.log(V), atol=1e-12, rtol=0)
    assert np.allclose(out["lse"], math.log(V), atol=1e-12, rtol=0)
    if V == 11:
        assert out["logp"][0] == pytest.approx(-2.3978952727983707, abs=1e-15)


def test_p4_dominant_logit_limit():
    """P4: z_y - z_other = 60 -> logp -> 0^- and entropy -> 0^+."""
    V, h = 50, 4
    W = np.zeros((V, h))
    W[7, 0] = 60.0
    H = np.zeros((1, h))
    H[0, 0] = 1.0
    cu, m = _flat_batch(1)
    out = oracle.logprob_fwd(H, W, cu, m, np.array([7], dtype=np.int32))
    assert -1e-20 < out["logp"][0] <= 0.0
    assert 0.0 <= out["entropy"][0] < 1e-20
    out = oracle.logprob_fwd(H, W, cu, m, np.array([3], dtype=np.int32))
    assert out["logp"][0] == pytest.approx(-60.0, abs=1e-12)


def test_p5_invariants():
    """P5: logp <= 0, 0 <= entropy <= ln V, lse >= max z."""
    H, W, y = _rand_problem(R=64, h=12, V=97, seed=5, scale=3.0)
    cu, m = _flat_batch(64)
    out = oracle.logprob_fwd(H, W, cu, m, y)
    assert (out["logp"] <= 0).all()
    assert (out["entropy"] >= -1e-12).all() and (out["entropy"] <= math.log(97) + 1e-12).all()
    assert (out["lse"] >= (H @ W.T).max(axis=1) - 1e-12).all()


def test_temperature_scales_logits():
    """tau^-1 multiplies the logits: fwd(H, W, tau) == fwd(H * tau^-1, W, 1)."""
    H, W, y = _rand_problem(R=9, h=5, V=13, seed=8)
    cu, m = _flat_batch(9)
    a = oracle.logprob_fwd(H, W, cu, m, y, inv_temperature=1.7)
    b = oracle.logprob_fwd(H * 1.7, W, cu, m, y, inv_temperature=1.0)
    np.testing.assert_allclose(a["logp"], b["logp"], atol=1e-12)


# -------------------------------------------------------------------- H1 ----
def test_bookkeeping_matches_searchsorted_and_mask():
    rng = np.random.default_rng(1)
    lay = custom_layout(rng.integers(0, 5, 20), rng.integers(0, 9, 20),
                        np.arange(20) // 4, np.ones(20), vocab=50, num_groups=5)
    bk = oracle.bookkeeping(lay.cu_seqlens, lay.mask, lay.targets, 50)
    t = np.arange(lay.num_rows)
    assert (bk["row_seq"] == np.searchsorted(lay.cu_seqlens, t, side="right") - 1).all()
    assert (bk["active_idx"] == np.flatnonzero(lay.mask)).all()
    assert bk["n_active"] == lay.num_tokens and bk["err"] == 0


@pytest.mark.parametrize("cu,R", [([1, 3, 5], 5), ([0, 4, 3, 6], 6), ([0, 2, 4], 5)])
def test_bookkeeping_bad_cu_seqlens(cu, R):
    bk = oracle.bookkeeping(np.array(cu), np.ones(R, np.uint8), np.zeros(R, np.int32), 10)
    assert bk["err"] == oracle.ERR_CU_SEQLENS and bk["n_active"] == 0
    assert (bk["row_seq"] == -1).all()


def test_bookkeeping_bad_target_and_empty():
    targets = np.array([0, 10, -1, 3, 9], dtype=np.int32)
    mask = np.array([1, 1, 1, 0, 1], dtype=np.uint8)
    cu = np.array([0, 0, 2, 2, 5], dtype=np.int32)          # empty sequences 0 and 2
    bk = oracle.bookkeeping(cu, mask, targets, 10)
    assert bk["err"] == oracle.ERR_TARGET
    assert list(bk["active_idx"]) == [0, 4]
    assert list(bk["row_seq"]) == [1, 1, 3, 3, 3]
    # masked-out rows never raise, whatever their target
    bk = oracle.bookkeeping(cu, np.array([1, 0, 0, 0, 1], np.uint8), targets, 10)
    assert bk["err"] == 0
    bk = oracle.bookkeeping(np.array([0], np.int32), np.zeros(0, np.uint8), np.zeros(0, np.int32), 10)
    assert bk["err"] == 0 and bk["n_active"] == 0


# -------------------------------------------------------------------- H2 ----
@pytest.mark.parametrize("G,k", [(16, 5), (8, 1), (8, 7), (32, 16), (4, 1)])
def test_p6_grpo_pm5_closed_form(G, k):
    """P6: rewards +-5, k of G correct. Population std gives
    A_correct = sqrt((G-k)/k), A_wrong = -sqrt(k/(G-k)); unbiased multiplies
    both by sqrt((G-1)/G)."""
    r = np.array([5.0] * k + [-5.0] * (G - k), dtype=np.float32)
    gos = np.zeros(G, np.int32)
    for unbiased, f in [(False, 1.0), (True, math.sqrt((G - 1) / G))]:
        A, err = oracle.grpo_advantage(r, gos, 1, eps=1e-6, unbiased=unbiased)
        assert err == 0
        np.testing.assert_allclose(A[:k], f * math.sqrt((G - k) / k), rtol=1e-6)
        np.testing.assert_allclose(A[k:], -f * math.sqrt(k / (G - k)), rtol=1e-6)
    if (G, k) == (16, 5):
        A, _ = oracle.grpo_advantage(r, gos, 1, eps=0.0, unbiased=True)
        assert A[0] == pytest.approx(1.4361406616345074, rel=1e-14)
        A, _ = oracle.grpo_advantage(r, gos, 1, eps=0.0, unbiased=False)
        assert A[0] == pytest.approx(1.4832396974191326, rel=1e-14)


def test_p7_group_sums():
    """P7: sum_g A = 0 and sum_g A^2 = G-1 (unbiased, eps = 0) / G (population)."""
    rng = np.random.default_rng(2)
    r = rng.normal(size=48).astype(np.float32)
    gos = np.repeat(np.arange(4), 12).astype(np.int32)
    rng.shuffle(gos)
    for unbiased, want in [(True, 11.0), (False, 12.0)]:
        A, _ = oracle.grpo_advantage(r, gos, 4, eps=0.0, unbiased=unbiased)
        for g in range(4):
            assert abs(A[gos == g].sum()) < 1e-12
            assert (A[gos == g] ** 2).sum() == pytest.approx(want, rel=1e-12)


def test_p8_zero_variance_and_singletons_exact_zero():
    """P8: A = 0 bit-exactly for all-equal groups and n = 1 groups; includes the
    fp32 hazard of seven 0.7s whose naive deviation is 6e-8 (reading #8)."""
    r = np.array([0.7] * 7 + [5, 5, 5] + [3.0] + [1, 2], dtype=np.float32)
    gos = np.array([0] * 7 + [1] * 3 + [2] + [3, 3], dtype=np.int32)
    A, _ = oracle.grpo_advantage(r, gos, 5)
    assert (A[:11] == 0.0).all()
    assert A[11] < 0 < A[12]
    s, mx, _ = oracle.grpo_group_stats(r, gos, 5)
    assert s[4, 0] == 0 and mx[4, 0] == -np.inf       # empty group


def test_p9_affine_invariance():
    """P9: A(a r + b) = A(r) for a > 0 (eps = 0)."""
    rng = np.random.default_rng(4)
    r = rng.normal(size=24)
    gos = np.repeat(np.arange(3), 8).astype(np.int32)
    A1, _ = oracle.grpo_advantage(r, gos, 3, eps=0.0)
    A2, _ = oracle.grpo_advantage(3.5 * r - 2.0, gos, 3, eps=0.0)
    np.testing.assert_allclose(A1, A2, atol=1e-12)


def test_group_stats_split_merge_and_from_stats():
    """Split-group path: stats of two shards added (sum) /
    maxed equal the whole; advantages from merged stats equal the two-pass
    definition."""
    rng = np.random.default_rng(6)
    r = rng.choice([-5.0, 5.0], size=64).astype(np.float32)
    gos = np.repeat(np.arange(8), 8).astype(np.int32)
    s_all, m_all, _ = oracle.grpo_group_stats(r, gos, 8)
    s_a, m_a, _ = oracle.grpo_group_stats(r[:29], gos[:29], 8)
    s_b, m_b, _ = oracle.grpo_group_stats(r[29:], gos[29:], 8)
    np.testing.assert_array_equal(s_a + s_b, s_all)
    np.testing.assert_array_equal(np.maximum(m_a, m_b), m_all)
    A_def, _ = oracle.grpo_advantage(r, gos, 8)
    A_st = oracle.grpo_advantage_from_stats(r, gos, s_a + s_b, np.maximum(m_a, m_b))
    np.testing.assert_allclose(A_def, A_st, atol=1e-12)


def test_invalid_group_ids():
    r = np.array([1.0, 2.0, 3.0, 9.0], np.float32)
    gos = np.array([0, 0, 5, -1], np.int32)
    A, err = oracle.grpo_advantage(r, gos, 2)
    assert err == oracle.ERR_GROUP and A[2] == 0 and A[3] == 0 and A[0] < 0 < A[1]


# ------------------------------------------------------------- H5-H8 --------
def _loss_problem(seed=0, R=24, h=6, V=13, masked=(3, 4, 17)):
    H, W, y = _rand_problem(R=R, h=h, V=V, seed=seed, scale=1.0)
    mask = np.ones(R, np.uint8)
    mask[list(masked)] = 0
    cu = np.array([0, 7, 15, R], np.int32)
    adv = np.array([1.3, -0.7, 0.4])
    return H, W, y, cu, mask, adv


def _guarded_old(H, W, cu, mask, y, rng, tau=1.0, p=None):
    """old_logp = logp - ln r*, r* away from the clip boundaries (O.6)."""
    p = p or oracle.LossParams()
    lp = oracle.logprob_fwd(H, W, cu, mask, y, inv_temperature=tau)["logp"]
    rs = []
    while len(rs) < len(lp):
        x = float(np.exp(rng.normal(0, 0.2)))
        if min(abs(x - (1 - p.clip_lo)), abs(x - (1 + p.clip_hi))) > 1e-3:
            rs.append(x)
    return lp - np.log(np.array(rs))


def test_p10_ratio_one_closed_form():
    """P10: old = own logp -> r = 1: L = -(sum_t m_t A_t)/N, g_t = -m_t A_t / N."""
    H, W, y, cu, mask, adv = _loss_problem()
    lp = oracle.logprob_fwd(H, W, cu, mask, y)["logp"]
    out = oracle.policy_loss_fwd_bwd(H, W, cu, mask, y, lp, adv)
    seq = np.searchsorted(cu, np.arange(len(y)), side="right") - 1
    N = int(mask.sum())
    At = adv[seq] * mask
    assert out["loss"] == pytest.approx(-At.sum() / N, abs=1e-14)
    np.testing.assert_allclose(out["g"], -At / N, atol=1e-15)
    assert out["stats"]["ratio_sum"] == pytest.approx(N, abs=1e-12)
    assert out["stats"]["clip_lo_count"] == 0 and out["stats"]["clip_hi_count"] == 0


def test_p11_clip_quadrants_and_boundaries():
    """P11: the four clip quadrants and boundary inclusion (reading #14)."""
    p = oracle.LossParams(clip_lo=0.2, clip_hi=0.2)
    cases = [  # (A, r) -> (loss, dL/dlogp)
        (1.0, 1.3, -1.2, 0.0), (-1.0, 0.7, 0.8, 0.0),
        (1.0, 0.7, -0.7, -0.7), (-1.0, 1.3, 1.3, 1.3),
        (2.0, 1.1, -2.2, -2.2), (-2.0, 0.9, 1.8, 1.8), (0.0, 5.0, 0.0, 0.0),
    ]
    for A, r, want_l, want_g in cases:
        rr, loss, g, _, _ = _surrogate(math.log(r), 0.0, A, p)
        assert loss == pytest.approx(want_l, abs=1e-12)
        assert g == pytest.approx(want_g, abs=1e-12)
    # exact boundaries: find d with exp(d) == 1 + eps (and 1 - eps) in float64
    for target, A in [(1.0 + 0.2, 1.0), (1.0 - 0.2, -1.0)]:
        d = math.log(target)
        for _ in range(64):
            if math.exp(d) == target:
                break
            d = math.nextafter(d, math.inf if math.exp(d) < target else -math.inf)
        assert math.exp(d) == target
        _, loss, g, clo, chi = _surrogate(d, 0.0, A, p)
        assert g == pytest.approx(-A * target) and not clo and not chi
    # the log-ratio clamp: gradient 0 beyond c, inclusive at c
    _, _, g, _, _ = _surrogate(20.5, 0.0, -1.0, p)
    assert g == 0.0
    _, _, g, _, _ = _surrogate(-20.0, 0.0, 1.0, p)
    assert g == pytest.approx(-math.exp(-20.0))


def test_p11_counts_in_full_loss():
    H, W, y, cu, mask, adv = _loss_problem(seed=2)
    lp = oracle.logprob_fwd(H, W, cu, mask, y)["logp"]
    seq = np.searchsorted(cu, np.arange(len(y)), side="right") - 1
    r_star = np.where(np.arange(len(y)) % 2 == 0, 1.5, 0.5)
    out = oracle.policy_loss_fwd_bwd(H, W, cu, mask, y, lp - np.log(r_star), adv)
    A = adv[seq]
    m = mask.astype(bool)
    assert out["stats"]["clip_hi_count"] == int(((A > 0) & (r_star > 1.2) & m).sum())
    assert out["stats"]["clip_lo_count"] == int(((A < 0) & (r_star < 0.8) & m).sum())
    assert out["stats"]["ratio_max"] == pytest.approx(1.5)


def _torch_definitional_loss(H, W, y, cu, mask, old, adv, tau, p, N):
    """The loss written directly from its definition, differentiated by torch."""
    import torch
    Ht = torch.tensor(H, dtype=torch.float64, requires_grad=True)
    Wt = torch.tensor(W, dtype=torch.float64, requires_grad=True)
    seq = np.searchsorted(cu, np.arange(len(y)), side="right") - 1
    Z = (Ht @ Wt.T) * tau
    logp = torch.log_softmax(Z, dim=1)[torch.arange(len(y)), torch.tensor(y).long()]
    d = logp - torch.tensor(old)
    r = torch.exp(torch.clamp(d, -p.logratio_clamp, p.logratio_clamp))
    A = torch.tensor(adv[seq])
    surr = torch.maximum(-A * r, -A * torch.clamp(r, 1 - p.clip_lo, 1 + p.clip_hi))
    L = (surr * torch.tensor(mask, dtype=torch.float64)).sum() / N
    L.backward()
    return L.item(), Ht.grad.numpy(), Wt.grad.numpy()


@pytest.mark.parametrize("tau", [1.0, 1 / 0.7])
def test_p12_autograd_of_definition(tau):
    """P12: torch float64 autograd of the definitional loss equals the oracle's
    analytic dH / dW (different method: reverse-mode AD through log_softmax)."""
    H, W, y, cu, mask, adv = _loss_problem(seed=7)
    rng = np.random.default_rng(0)
    p = oracle.LossParams(clip_lo=0.2, clip_hi=0.28)
    old = _guarded_old(H, W, cu, mask, y, rng, tau, p)
    N = 40
    out = oracle.policy_loss_fwd_bwd(H, W, cu, mask, y, old, adv, p, n_global=N, inv_temperature=tau)
    L, dH, dW = _torch_definitional_loss(H, W, y, cu, mask, old, adv, tau, p, N)
    assert out["loss"] == pytest.approx(L, abs=1e-14)
    np.testing.assert_allclose(out["dH"], dH, atol=1e-14)
    np.testing.assert_allclose(out["dW"], dW, atol=1e-14)


def test_p13_finite_differences():
    """P13: central differences of the oracle's own forward loss."""
    H, W, y, cu, mask, adv = _loss_problem(seed=9)
    rng = np.random.default_rng(1)
    old = _guarded_old(H, W, cu, mask, y, rng)
    out = oracle.policy_loss_fwd_bwd(H, W, cu, mask, y, old, adv)
    eps = 1e-6

    def L(Hx, Wx):
        return oracle.policy_loss_fwd_bwd(Hx, Wx, cu, mask, y, old, adv, want_grads=False,
                                          n_global=out["n_active"])["loss"]
    for (t, k) in [(0, 0), (5, 3), (20, 5)]:
        Hp, Hm = H.copy(), H.copy()
        Hp[t, k] += eps
        Hm[t, k] -= eps
        fd = (L(Hp, W) - L(Hm, W)) / (2 * eps)
        assert fd == pytest.approx(out["dH"][t, k], rel=1e-6, abs=1e-10)
    for (j, k) in [(0, 1), (y[2], 4), (12, 0)]:
        Wp, Wm = W.copy(), W.copy()
        Wp[j, k] += eps
        Wm[j, k] -= eps
        fd = (L(H, Wp) - L(H, Wm)) / (2 * eps)
        assert fd == pytest.approx(out["dW"][j, k], rel=1e-6, abs=1e-10)


def test_p14_p15_p16_invariants():
    """P14 sum_j dW_j = 0; P15 dH_t = tau^-1 g_t (W[y_t] - E_p[W]); P16 masked
    rows: dH = 0 exactly, and their hidden/targets do not affect L, dW."""
    tau = 1.25
    H, W, y, cu, mask, adv = _loss_problem(seed=11)
    rng = np.random.default_rng(2)
    old = _guarded_old(H, W, cu, mask, y, rng, tau)
    out = oracle.policy_loss_fwd_bwd(H, W, cu, mask, y, old, adv, inv_temperature=tau)
    assert np.abs(out["dW"].sum(axis=0)).max() < 1e-15
    Z = H @ W.T * tau
    P = np.exp(Z - Z.max(1, keepdims=True))
    P /= P.sum(1, keepdims=True)
    want = tau * out["g"][:, None] * (W[y] - P @ W)
    np.testing.assert_allclose(out["dH"], want, atol=1e-15)
    assert (out["dH"][mask == 0] == 0).all()
    H2, y2 = H.copy(), y.copy()
    H2[mask == 0] = 99.0
    y2[mask == 0] = (y2[mask == 0] + 5) % 13
    out2 = oracle.policy_loss_fwd_bwd(H2, W, cu, mask, y2, old, adv, inv_temperature=tau)
    assert out2["loss"] == out["loss"]
    np.testing.assert_array_equal(out2["dW"], out["dW"])


def test_p17_micro_batch_linearity():
    """P17: the whole batch equals the sum of its micro-batches at fixed N
    (micro-batch = fwd/bwd unit, global batch = update unit)."""
    H, W, y, cu, mask, adv = _loss_problem(seed=13)
    rng = np.random.default_rng(3)
    old = _guarded_old(H, W, cu, mask, y, rng)
    N = int(mask.sum())
    whole = oracle.policy_loss_fwd_bwd(H, W, cu, mask, y, old, adv, n_global=N)
    parts = []
    for s0, s1 in [(0, 1), (1, 3)]:
        r0, r1 = cu[s0], cu[s1]
        parts.append(oracle.policy_loss_fwd_bwd(H[r0:r1], W, cu[s0:s1 + 1] - r0, mask[r0:r1],
                                                y[r0:r1], old[r0:r1], adv[s0:s1], n_global=N))
    np.testing.assert_allclose(parts[0]["dW"] + parts[1]["dW"], whole["dW"], atol=1e-15)
    assert parts[0]["loss"] + parts[1]["loss"] == pytest.approx(whole["loss"], abs=1e-15)
    np.testing.assert_allclose(np.concatenate([parts[0]["dH"], parts[1]["dH"]]), whole["dH"], atol=0)


def test_p18_sequence_permutation():
    """P18: permuting sequences (with their advantages) permutes per-row outputs
    and leaves L and dW unchanged."""
    H, W, y, cu, mask, adv = _loss_problem(seed=15)
    rng = np.random.default_rng(4)
    old = _guarded_old(H, W, cu, mask, y, rng)
    a = oracle.policy_loss_fwd_bwd(H, W, cu, mask, y, old, adv)
    perm = [2, 0, 1]
    rows = np.concatenate([np.arange(cu[s], cu[s + 1]) for s in perm])
    lens = np.diff(cu)[perm]
    cu2 = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    b = oracle.policy_loss_fwd_bwd(H[rows], W, cu2, mask[rows], y[rows], old[rows], adv[perm])
    assert b["loss"] == pytest.approx(a["loss"], abs=1e-15)
    np.testing.assert_allclose(b["dW"], a["dW"], atol=1e-15)
    np.testing.assert_allclose(b["logp"], a["logp"][rows], atol=0)
    np.testing.assert_allclose(b["dH"], a["dH"][rows], atol=0)


def test_loss_scale_streaming_mode():
    """loss_scale replaces 1/N (streaming mode rescales later): dW scales linearly."""
    H, W, y, cu, mask, adv = _loss_problem(seed=17)
    rng = np.random.default_rng(5)
    old = _guarded_old(H, W, cu, mask, y, rng)
    a = oracle.policy_loss_fwd_bwd(H, W, cu, mask, y, old, adv)
    b = oracle.policy_loss_fwd_bwd(H, W, cu, mask, y, old, adv,
                                   oracle.LossParams(loss_scale=1.0))
    np.testing.assert_allclose(b["dW"] / a["n_active"], a["dW"], atol=1e-15)


# ------------------------------------------------------------- NEXT-3 -------
@pytest.mark.parametrize("cuts", [[0, 1000], [0, 333, 666, 1000], [0, 1, 999, 1000],
                                  [0, 512, 1000]])
def test_vocab_partition_merge_equals_full_softmax(cuts):
    """Vocab-parallel pin: merging shard partials over ANY partition of the
    vocabulary equals the unsharded log-softmax (associativity of logsumexp;
    the merge is written in a different form from the oracle's forward)."""
    rng = np.random.default_rng(len(cuts))
    R, h, V = 30, 8, 1000
    H = rng.normal(size=(R, h))
    W = rng.normal(scale=1.5, size=(V, h))
    y = rng.integers(0, V, size=R).astype(np.int32)
    cu, m = _flat_batch(R)
    full = oracle.logprob_fwd(H, W, cu, m, y, inv_temperature=1.3)
    parts = [oracle.head.logprob_shard_partials(H, W[a:b], a, V, cu, m, y, inv_temperature=1.3)
             for a, b in zip(cuts[:-1], cuts[1:])]
    mg = oracle.head.merge_shard_partials(np.stack(parts))
    np.testing.assert_allclose(mg["logp"], full["logp"], atol=1e-12)
    np.testing.assert_allclose(mg["entropy"], full["entropy"], atol=1e-12)
    np.testing.assert_allclose(mg["lse"], full["lse"], atol=1e-12)


def test_vocab_shard_partials_mpmath():
    """One shard's (m, s, u, zy) against 50-digit brute force."""
    mpmath.mp.dps = 50
    H, W, y = _rand_problem(R=3, h=4, V=9, seed=11, scale=2.0)
    y[:] = [2, 7, 5]
    cu, m = _flat_batch(3)
    p = oracle.head.logprob_shard_partials(H, W[4:9], 4, 9, cu, m, y)
    for t in range(3):
        z = [mpmath.fsum(mpmath.mpf(H[t, k]) * mpmath.mpf(W[j, k]) for k in range(4))
             for j in range(4, 9)]
        mx = max(z)
        s = mpmath.fsum(mpmath.exp(zj - mx) for zj in z)
        u = mpmath.fsum(mpmath.exp(zj - mx) * (zj - mx) for zj in z)
        assert p[0, t] == pytest.approx(float(mx), abs=1e-13)
        assert p[1, t] == pytest.approx(float(s), rel=1e-13)
        assert p[2, t] == pytest.approx(float(u), rel=1e-12, abs=1e-13)
        assert p[3, t] == (0.0 if y[t] < 4 else pytest.approx(float(z[y[t] - 4]), abs=1e-13))
