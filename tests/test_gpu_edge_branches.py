"""The surrogate's edge branches on the CUDA path vs the oracle (H5; P:L830
"discard minibatches with too large importance ratio" is exactly the regime
of large ratios): constructed rows whose log-ratio d = logp - old sits

  * beyond the log-ratio clamp (|d| = 25 > c = 20: r = e^{+-20}, no gradient;
    reading #15),
  * just inside it (|d| = 20 - margin: the gradient flows, r ~ 4.9e8),
  * beyond / inside the dual-clip cap c_dual = 3 for A < 0 (reading #25),
  * just beyond / inside the clip bounds 1 +- eps for both signs of A
    (reading #14),
  * with A = 0 (zero-variance group: no gradient, zero loss).

Each case is its own call (so a case's loss_sum is not swamped by the
e^20-sized rows of another). The checks: loss_sum (rel 1e-2), ratio_max
(rel 1e-2), clip counts (exact), every dH row zero exactly where the
oracle's is (g = 0) and within rel 1e-2 of the oracle's row otherwise.
The exact boundaries themselves are decided by floating point (fp32 on the
GPU, fp64 in the oracle) and are pinned on the oracle only (P11); here each
case keeps a margin of 1e-2 (bf16) / 1e-4 (fp32) in d from the boundary so
both sides take the same branch.
"""
import math

import numpy as np
import pytest

import oracle
from tests.gpu_util import dev_tensors
from workload import HeadConfig, custom_layout, make_tensors_host

pytestmark = pytest.mark.gpu

SMALL_BF16 = HeadConfig("edge-bf16", 192, 1000, 1, 1, 1, "bf16", "reasoning")
SMALL_F32 = HeadConfig("edge-f32", 64, 1000, 1, 1, 1, "f32", "reasoning")

C_DUAL = 3.0


def _cases(m):
    """(name, A, d) per case; m = margin in d."""
    L = math.log
    return [
        ("clamp-hi-Apos", 1.5, 25.0),            # r = e^20 clipped high, g = 0
        ("clamp-hi-Aneg", -1.5, 25.0),           # l = -A e^20, g = 0 only via the clamp gate
        ("inside-clamp-hi-Aneg", -1.5, 20.0 - m),  # gradient flows at r ~ 4.9e8
        ("clamp-lo-Apos", 1.5, -25.0),           # l = -A e^-20, g = 0 only via the clamp gate
        ("inside-clamp-lo-Apos", 1.5, -20.0 + m),
        ("dual-beyond", -1.5, L(C_DUAL) + 10 * m),   # l = -A c_dual, g = 0
        ("dual-inside", -1.5, L(C_DUAL) - 10 * m),   # l = -A r, g flows
        ("clip-hi-beyond", 1.5, L(1.2) + m),     # l = -A 1.2, g = 0
        ("clip-hi-inside", 1.5, L(1.2) - m),
        ("clip-lo-beyond", -1.5, L(0.8) - m),    # l = -A 0.8, g = 0
        ("clip-lo-inside", -1.5, L(0.8) + m),
        ("ratio-above-Aneg", -1.5, L(1.2) + m),  # unclipped side: g flows
        ("ratio-below-Apos", 1.5, L(0.8) - m),   # unclipped side: g flows
        ("A-zero", 0.0, 0.3),
    ]


def _check_case(rl, cfg, name, A, d, dual):
    import torch
    # 3 sequences of 7 prompt rows (mask 0) + 9 response rows, one advantage each
    lay = custom_layout([7, 7, 7], [9, 9, 9], [0, 0, 0], np.zeros(3), vocab=cfg.vocab,
                        num_groups=1, seed=sum(map(ord, name)))
    H, W = make_tensors_host(cfg, lay.num_rows, seed=5)
    fwd = oracle.logprob_fwd(H, W, lay.cu_seqlens, lay.mask, lay.targets)
    old = fwd["logp"] - d                      # d = logp - old, exactly in fp64
    adv = np.full(3, A)
    p_or = oracle.LossParams(dual_clip=C_DUAL if dual else 0.0)
    N = lay.num_tokens
    ref = oracle.policy_loss_fwd_bwd(H, W, lay.cu_seqlens, lay.mask, lay.targets, old, adv, p_or,
                                     n_global=N)
    dv = dev_tensors(lay)
    head = rl.Head(cfg.hidden, cfg.vocab, cfg.dtype)
    Hd, Wd = H.cuda(), W.cuda()
    logp = torch.empty(lay.num_rows, device="cuda")
    gh = torch.full_like(Hd, 3.0)
    gw = torch.zeros(cfg.vocab, cfg.hidden, device="cuda")
    st = rl.new_stats()
    p = rl.LossParams(dual_clip=C_DUAL if dual else 0.0,
                      n_tokens_global=torch.tensor([N], device="cuda"))
    rl.rl_policy_loss_fwd_bwd(head, Hd, Wd, rl.Batch(dv["cu"], dv["targets"], dv["mask"]),
                              torch.as_tensor(old, dtype=torch.float32, device="cuda"),
                              torch.as_tensor(adv, dtype=torch.float32, device="cuda"), p,
                              logp, gh, gw, stats=st)
    torch.cuda.synchronize()
    s = rl.read_stats(st)
    rs = ref["stats"]
    assert s["tokens"] == rs["tokens"] == N
    assert s["clip_hi_count"] == rs["clip_hi_count"], name
    assert s["clip_lo_count"] == rs["clip_lo_count"], name
    if rs["loss_sum"] == 0:
        assert s["loss_sum"] == 0, name
    else:
        assert s["loss_sum"] == pytest.approx(rs["loss_sum"], rel=1e-2), name
    assert s["ratio_max"] == pytest.approx(rs["ratio_max"], rel=1e-2), name
    dH = gh.cpu().double().numpy()
    act = lay.mask.astype(bool)
    assert (dH[~act] == 0).all()
    zero = np.all(ref["dH"] == 0, axis=1)
    np.testing.assert_array_equal(np.all(dH == 0, axis=1), zero, err_msg=name)
    for t in np.flatnonzero(~zero):
        err = np.linalg.norm(dH[t] - ref["dH"][t]) / np.linalg.norm(ref["dH"][t])
        assert err <= 1e-2, (name, t, err)
    gwn = gw.cpu().double().numpy()
    if np.all(ref["dW"] == 0):
        assert (gwn == 0).all(), name
    else:
        err = np.linalg.norm(gwn - ref["dW"]) / np.linalg.norm(ref["dW"])
        assert err <= 1e-2, (name, err)
    return ref


@pytest.mark.parametrize("cfg,margin", [(SMALL_BF16, 1e-2), (SMALL_F32, 1e-4)],
                         ids=["bf16-tc", "fp32-simt"])
@pytest.mark.parametrize("dual", [False, True], ids=["no-dual", "dual-clip"])
def test_surrogate_edge_branches(rl, cfg, margin, dual):
    grads = {}
    for name, A, d in _cases(margin):
        if name.startswith("dual") and not dual:
            continue
        ref = _check_case(rl, cfg, name, A, d, dual)
        grads[name] = bool(np.any(ref["g"] != 0))
    # the cases cover both outcomes of every gate (sanity of the construction)
    expect_zero = {"clamp-hi-Apos", "clamp-hi-Aneg", "clamp-lo-Apos", "clip-hi-beyond",
                   "clip-lo-beyond", "A-zero", "dual-beyond"}
    if dual:
        expect_zero.add("inside-clamp-hi-Aneg")    # r ~ 4.9e8 > c_dual
    for name, has_g in grads.items():
        assert has_g == (name not in expect_zero), name
