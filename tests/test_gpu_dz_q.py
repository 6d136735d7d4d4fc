"""H6 without the logits recompute (`k_dz_from_q`): the forward
epilogue stores q = e^{z - m_tile} (bf16, 0 at the target) and one HBM pass
turns it into dZ = tau^-1 g (onehot - q e^{m_tile - lse}), with the target
column from the fp32 target logit (1 - p_y = -expm1(z_y - lse)).

Checked against the CPU float64 oracle on rows from flat to very confident
softmaxes (p_y up to ~0.9999, where onehot - p cancels and the target column
must not come from q), per row (dH) and as a whole (dW), and against the
recompute path (RLHEAD_DZ_RECOMPUTE=1) -- both within the bf16 gradient
tolerance of the oracle, the q path no worse than 2x the recompute path's
error (it rounds q and dZ, two bf16 roundings instead of one)."""
import os

import numpy as np
import pytest

import oracle
from tests.gpu_util import dev_tensors, guarded_old_logp, max_rel, rel_fro
from workload import custom_layout

pytestmark = pytest.mark.gpu


def _case(seed, V=2000, h=256, tau=1.0):
    import torch
    rng = np.random.default_rng(seed)
    S = 12
    lay = custom_layout(rng.integers(0, 8, S), rng.integers(20, 120, S), np.arange(S) // 4,
                        rng.choice([-5.0, 5.0], S), vocab=V, num_groups=3, seed=seed)
    g = torch.Generator().manual_seed(seed)
    W = (torch.randn(V, h, generator=g) * (4 / h ** 0.5)).to(torch.bfloat16)
    H = torch.randn(lay.num_rows, h, generator=g)
    # confidence sweep: row t gets (beta_t / 16) W[y_t] added, raising its target
    # logit by ~beta_t (|W_y|^2 ~ 16): from flat (beta 0) to p_y > 0.999
    beta = torch.as_tensor(rng.choice([0.0, 0.0, 8.0, 14.0, 20.0, 26.0], lay.num_rows),
                           dtype=torch.float32)
    H = (H + (beta[:, None] / 16.0) *
         W.float()[torch.as_tensor(lay.targets.astype(np.int64))]).to(torch.bfloat16)
    return lay, H, W, tau


def _run(rl, lay, H, W, tau, old, adv, recompute):
    import torch
    d = dev_tensors(lay)
    head = rl.Head(H.shape[1], W.shape[0], "bf16", inv_temperature=1.0 / tau)
    prev = os.environ.get("RLHEAD_DZ_RECOMPUTE")
    os.environ["RLHEAD_DZ_RECOMPUTE"] = "1" if recompute else "0"
    try:
        logp = torch.empty(lay.num_rows, device="cuda")
        gh = torch.full((lay.num_rows, H.shape[1]), 5.0, dtype=torch.bfloat16, device="cuda")
        gw = torch.zeros(W.shape[0], W.shape[1], device="cuda")
        tr = rl.Trace(64).start()
        rl.rl_policy_loss_fwd_bwd(head, H.cuda(), W.cuda(), rl.Batch(d["cu"], d["targets"],
                                                                     d["mask"]),
                                  torch.as_tensor(old, dtype=torch.float32, device="cuda"),
                                  torch.as_tensor(adv, dtype=torch.float32, device="cuda"),
                                  rl.LossParams(n_tokens_global=torch.tensor(
                                      [lay.num_tokens], device="cuda")), logp, gh, gw)
        torch.cuda.synchronize()
        kinds = tr.stop().by_kind()
    finally:
        if prev is None:
            os.environ.pop("RLHEAD_DZ_RECOMPUTE", None)
        else:
            os.environ["RLHEAD_DZ_RECOMPUTE"] = prev
    return (logp.cpu().double().numpy(), gh.cpu().double().numpy(), gw.cpu().double().numpy(),
            kinds)


@pytest.mark.parametrize("seed,tau", [(1, 1.0), (2, 0.7)])
def test_dz_from_q_vs_oracle(rl, seed, tau):
    lay, H, W, tau = _case(seed, tau=tau)
    inv_t = 1.0 / tau
    fwd = oracle.logprob_fwd(H, W, lay.cu_seqlens, lay.mask, lay.targets,
                             inv_temperature=np.float32(inv_t))
    act = lay.mask.astype(bool)
    one_minus_py = -np.expm1(fwd["logp"])
    assert (one_minus_py[act] < 1e-2).sum() >= 10                 # confident rows present
    old = guarded_old_logp(fwd["logp"], np.random.default_rng(seed))
    adv, _ = oracle.grpo_advantage(lay.rewards, lay.group_of_seq, lay.num_groups)
    adv = adv.astype(np.float32)
    ref = oracle.policy_loss_fwd_bwd(H, W, lay.cu_seqlens, lay.mask, lay.targets, old, adv,
                                     n_global=lay.num_tokens, inv_temperature=np.float32(inv_t))
    lp_q, dH_q, dW_q, k_q = _run(rl, lay, H, W, tau, old, adv, recompute=False)
    lp_r, dH_r, dW_r, k_r = _run(rl, lay, H, W, tau, old, adv, recompute=True)
    assert "dz_from_q" in k_q and "gemm_dz" not in k_q          # the path under test ran
    assert "gemm_dz" in k_r and "dz_from_q" not in k_r
    # same forward GEMM; the q epilogue sums the tile in two passes (max, then
    # e^{z - m}) where the other rescales online: fp32 rounding differences only
    np.testing.assert_allclose(lp_q, lp_r, rtol=0, atol=1e-5)
    assert np.abs(lp_q - ref["logp"]).max() <= 2e-3
    for dH, dW in ((dH_q, dW_q), (dH_r, dW_r)):
        assert rel_fro(dH, ref["dH"]) <= 1e-2 and max_rel(dH, ref["dH"]) <= 1e-2
        assert rel_fro(dW, ref["dW"]) <= 1e-2 and max_rel(dW, ref["dW"]) <= 1e-2
    # per row, including confident ones (onehot - p cancels as p_y -> 1): rows
    # with 1 - p_y > 1e-4 (below that the fp32 lse itself, in either path,
    # carries a relative error of ~6e-8 / (1 - p_y) into 1 - p_y)
    nz = np.linalg.norm(ref["dH"], axis=1) > 0
    chk = nz & (one_minus_py > 1e-4)
    assert (chk & (one_minus_py < 1e-2)).sum() >= 5
    err_q = np.linalg.norm(dH_q - ref["dH"], axis=1)[chk] / np.linalg.norm(ref["dH"], axis=1)[chk]
    err_r = np.linalg.norm(dH_r - ref["dH"], axis=1)[chk] / np.linalg.norm(ref["dH"], axis=1)[chk]
    # a single bf16 row of dZ already carries ~1% relative error on its worst
    # rows in BOTH paths (measured: recompute 0.8-1.06%); the north_star's
    # 1e-2 is on the gradient as a whole (checked above). Per row: the q path
    # (two bf16 roundings) stays within 2x the recompute path, typical rows
    # well below the tolerance, and the confident rows are not singled out.
    conf = (one_minus_py[chk] < 1e-2)
    assert err_q.max() <= 2 * err_r.max() + 1e-3, (err_q.max(), err_r.max())
    assert np.median(err_q) <= 5e-3, np.median(err_q)
    assert err_q[conf].max() <= 2 * err_r[conf].max() + 1e-3, (err_q[conf].max(),
                                                               err_r[conf].max())
    assert rel_fro(dW_q, ref["dW"]) <= 2 * max(rel_fro(dW_r, ref["dW"]), 1e-3)
    assert (dH_q[lay.mask == 0] == 0).all()
    assert np.all(np.linalg.norm(ref["dH"], axis=1)[~nz] == 0)
    assert np.all(dH_q[~nz] == 0)


def _env_run(rl, env, fn):
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def test_backward_row_skip(rl):
    """Skip mode (default): the backward GEMMs run only over rows with
    dL/dlogp != 0 (GRPO groups with A = 0 here). dL/dH is bit-identical to the
    dense backward (each output row is the same dot products), dW equal to
    fp32 reassociation (the zero rows no longer share k-blocks), and both
    match the oracle; with a KL term (beta > 0) the A = 0 rows keep a gradient
    and must be kept."""
    import torch
    from workload import make_layout, make_tensors_torch, HeadConfig
    cfg = HeadConfig("skip-bf16", 256, 3000, 10, 4, 200, "bf16", "reasoning")
    lay = make_layout(cfg, seed=5)
    adv, _ = oracle.grpo_advantage(lay.rewards, lay.group_of_seq, lay.num_groups)
    assert (adv == 0).sum() >= 8 and (adv != 0).sum() >= 8     # forced A = 0 groups present
    H, W = make_tensors_torch(cfg, lay.num_rows, seed=5)
    fwd = oracle.logprob_fwd(H, W, lay.cu_seqlens, lay.mask, lay.targets)
    old = guarded_old_logp(fwd["logp"], np.random.default_rng(5))
    ref_lp = (fwd["logp"] + np.random.default_rng(6).normal(0, 0.3, lay.num_rows)).astype(np.float32)
    d = dev_tensors(lay)
    head = rl.Head(cfg.hidden, cfg.vocab, "bf16")
    for kl in (0.0, 0.05):
        def run():
            logp = torch.empty(lay.num_rows, device="cuda")
            gh = torch.full((lay.num_rows, cfg.hidden), 3.0, dtype=torch.bfloat16, device="cuda")
            gw = torch.zeros(cfg.vocab, cfg.hidden, device="cuda")
            p = rl.LossParams(kl_coef=kl, ref_logp=torch.as_tensor(ref_lp, device="cuda"),
                              n_tokens_global=torch.tensor([lay.num_tokens], device="cuda"))
            tr = rl.Trace(64).start()
            rl.rl_policy_loss_fwd_bwd(head, H.cuda(), W.cuda(),
                                      rl.Batch(d["cu"], d["targets"], d["mask"]),
                                      torch.as_tensor(old, dtype=torch.float32, device="cuda"),
                                      torch.as_tensor(adv, dtype=torch.float32, device="cuda"),
                                      p, logp, gh, gw)
            torch.cuda.synchronize()
            tr.stop()
            return gh.cpu(), gw.cpu().double()
        gh_s, gw_s = _env_run(rl, {"RLHEAD_BWD_SKIP": "1", "RLHEAD_DZ_FUSED": "0"}, run)
        gh_d, gw_d = _env_run(rl, {"RLHEAD_BWD_SKIP": "0", "RLHEAD_DZ_FUSED": "0"}, run)
        # A != 0 rows moved ahead of the A = 0 rows before the forward (fused mode)
        gh_f, gw_f = _env_run(rl, {"RLHEAD_BWD_SKIP": "1", "RLHEAD_DZ_FUSED": "1"}, run)
        assert torch.equal(gh_s, gh_d), kl
        assert torch.equal(gh_f, gh_d), kl
        assert float((gw_s - gw_d).norm() / gw_d.norm()) <= 1e-5, kl
        assert float((gw_f - gw_d).norm() / gw_d.norm()) <= 1e-5, kl
        ref = oracle.policy_loss_fwd_bwd(H, W, lay.cu_seqlens, lay.mask, lay.targets, old, adv,
                                         oracle.LossParams(kl_coef=kl), n_global=lay.num_tokens,
                                         ref_logp=ref_lp.astype(np.float64))
        dH = gh_s.double().numpy()
        assert rel_fro(dH, ref["dH"]) <= 1e-2 and max_rel(dH, ref["dH"]) <= 1e-2
        assert rel_fro(gw_s.numpy(), ref["dW"]) <= 1e-2
        zero = np.all(ref["dH"] == 0, axis=1)
        assert np.all(dH[zero] == 0)
        if kl == 0.0:
            assert zero[lay.mask.astype(bool)].sum() >= 50   # A = 0 rows really skipped
