"""CUDA path (librlhead.so through the C ABI) vs the CPU float64 oracle on the
same seeded inputs. Tolerances (BASELINE.json north_star):
bit-exact bookkeeping; |dlogp| <= 2e-3 (bf16) / 1e-5 (fp32); relative 1e-2 on
loss and gradients for bf16 (1e-5 fp32)."""
import os

import numpy as np
import pytest

import oracle
from tests.gpu_util import dev_tensors, guarded_old_logp, max_rel, rel_fro
from workload import CONFIGS, HeadConfig, custom_layout, make_layout, make_tensors_host, sub_layout

pytestmark = pytest.mark.gpu

SMALL_BF16 = HeadConfig("small-bf16", 192, 1000, 6, 4, 96, "bf16", "reasoning")
QWEN15_HEAD = CONFIGS["qwen1.5b"]


def _run_fwd(rl, head, H, W, d, lay):
    import torch
    R = lay.num_rows
    logp = torch.full((R,), 7.0, device="cuda")
    ent = torch.full((R,), 7.0, device="cuda")
    lse = torch.full((R,), 7.0, device="cuda")
    b = rl.Batch(d["cu"], d["targets"], d["mask"], d["err"])
    rl.rl_logprob_fwd(head, H, W, b, logp, ent, lse)
    torch.cuda.synchronize()
    return logp.cpu().double().numpy(), ent.cpu().double().numpy(), lse.cpu().double().numpy()


def _run_loss(rl, head, H, W, d, lay, old, adv, params=None, n_global=None):
    import torch
    R = lay.num_rows
    logp = torch.full((R,), 7.0, device="cuda")
    ent = torch.full((R,), 7.0, device="cuda")
    gh = torch.full_like(H, 3.0)
    gw = torch.zeros(W.shape[0], W.shape[1], dtype=torch.float32, device="cuda")
    st = rl.new_stats()
    p = params or rl.LossParams()
    if n_global is not None:
        p.n_tokens_global = torch.tensor([n_global], dtype=torch.int64, device="cuda")
    b = rl.Batch(d["cu"], d["targets"], d["mask"], d["err"])
    rl.rl_policy_loss_fwd_bwd(head, H, W, b, torch.as_tensor(old, dtype=torch.float32, device="cuda"),
                              torch.as_tensor(adv, dtype=torch.float32, device="cuda"), p,
                              logp, gh, gw, entropy=ent, stats=st)
    torch.cuda.synchronize()
    return dict(logp=logp.cpu().double().numpy(), entropy=ent.cpu().double().numpy(),
                dH=gh.cpu().double().numpy(), dW=gw.cpu().double().numpy(),
                stats=rl.read_stats(st), err=int(d["err"].item()))


# ------------------------------------------------------------ H1 bit-exact ----
def _layouts():
    rng = np.random.default_rng(3)
    yield "tiny", make_layout(CONFIGS["tiny"], seed=0)
    yield "ragged", custom_layout(rng.integers(0, 40, 64), rng.integers(0, 300, 64),
                                  np.arange(64) // 8, np.ones(64), vocab=1000, num_groups=8)
    yield "empty-seqs", custom_layout([3, 0, 0, 5, 0], [0, 0, 7, 0, 1], [0, 0, 1, 1, 1],
                                      np.ones(5), vocab=50, num_groups=2)
    lay = custom_layout(rng.integers(1, 9, 40), rng.integers(1, 2000, 40), np.arange(40) // 4,
                        np.ones(40), vocab=1000, num_groups=10)
    lay.targets[::97] = 1000     # out-of-range targets -> ERR_TARGET on masked rows
    lay.targets[5::211] = -3
    yield "bad-targets", lay
    lay2 = custom_layout([2, 3], [4, 5], [0, 0], np.ones(2), vocab=10, num_groups=1)
    lay2.cu_seqlens[1] = 99     # non-monotone cu_seqlens
    yield "bad-cu", lay2


@pytest.mark.parametrize("name,lay", list(_layouts()), ids=[n for n, _ in _layouts()])
def test_bookkeeping_bit_exact(rl, name, lay):
    import torch
    d = dev_tensors(lay)
    R = lay.num_rows
    head = rl.Head(64, lay.vocab, "bf16")
    row_seq = torch.full((R,), -7, dtype=torch.int32, device="cuda")
    act = torch.full((max(R, 1),), -7, dtype=torch.int32, device="cuda")
    n = torch.zeros(1, dtype=torch.int64, device="cuda")
    acc = torch.full((1,), 5, dtype=torch.int64, device="cuda")
    rl.rl_batch_prepare(head, rl.Batch(d["cu"], d["targets"], d["mask"], d["err"]), row_seq, act,
                        n, acc)
    torch.cuda.synchronize()
    ref = oracle.bookkeeping(lay.cu_seqlens, lay.mask, lay.targets, lay.vocab)
    assert int(n.item()) == ref["n_active"]
    assert int(acc.item()) == 5 + ref["n_active"]
    assert int(d["err"].item()) == ref["err"]
    np.testing.assert_array_equal(row_seq.cpu().numpy(), ref["row_seq"])
    np.testing.assert_array_equal(act.cpu().numpy()[:ref["n_active"]], ref["active_idx"])


# ------------------------------------------------------------------- H2 ----
def test_grpo_advantage_parity(rl):
    import torch
    rng = np.random.default_rng(0)
    G = 37
    gos = rng.integers(0, G, 700).astype(np.int32)
    r = rng.choice([-5.0, 5.0], 700).astype(np.float32)
    r[gos == 3] = 5.0                              # zero-variance group
    r[gos == 4] = rng.normal(size=(gos == 4).sum()).astype(np.float32)
    gos[[10, 20]] = [G + 2, -1]                    # invalid ids
    single = np.flatnonzero(gos == 5)
    gos[single[1:]] = 6                            # singleton group 5
    rt = torch.as_tensor(r, device="cuda")
    gt = torch.as_tensor(gos, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    for unbiased in (True, False):
        adv = torch.full((700,), 9.0, device="cuda")
        rl.rl_grpo_advantage(rt, gt, G, adv, eps=1e-6, unbiased=unbiased, err_flags=err)
        torch.cuda.synchronize()
        ref, rerr = oracle.grpo_advantage(r, gos, G, eps=1e-6, unbiased=unbiased)
        a = adv.cpu().double().numpy()
        np.testing.assert_allclose(a, ref, rtol=1e-5, atol=1e-5)
        assert (a[ref == 0] == 0).all()            # exact zeros: A = 0 rule
        assert int(err.item()) == rerr == oracle.ERR_GROUP
    # split-group path: stats of two shards, SUM/MAX-merged, then advantage
    s = torch.zeros(G, 3, dtype=torch.float64, device="cuda")
    m = torch.zeros(G, 2, dtype=torch.float64, device="cuda")
    s2, m2 = torch.zeros_like(s), torch.zeros_like(m)
    rl.rl_grpo_group_stats(rt[:300], gt[:300], G, s, m)
    rl.rl_grpo_group_stats(rt[300:], gt[300:], G, s2, m2)
    adv = torch.zeros(700, device="cuda")
    rl.rl_grpo_advantage(rt, gt, G, adv, sum_stats=s + s2, max_stats=torch.maximum(m, m2))
    torch.cuda.synchronize()
    ref_s, ref_m, _ = oracle.grpo_group_stats(r, gos, G)
    np.testing.assert_allclose((s + s2).cpu().numpy(), ref_s, rtol=1e-12, atol=1e-9)
    np.testing.assert_array_equal(torch.maximum(m, m2).cpu().numpy(), ref_m)
    ref, _ = oracle.grpo_advantage(r, gos, G)
    np.testing.assert_allclose(adv.cpu().double().numpy(), ref, rtol=1e-5, atol=1e-5)


# --------------------------------------------------------- fp32 tiny config ----
def test_tiny_fp32_forward(rl):
    cfg = CONFIGS["tiny"]
    lay = make_layout(cfg, seed=0)
    H, W = make_tensors_host(cfg, lay.num_rows, seed=0)
    d = dev_tensors(lay)
    head = rl.Head(cfg.hidden, cfg.vocab, "f32")
    lp, ent, lse = _run_fwd(rl, head, H.cuda(), W.cuda(), d, lay)
    ref = oracle.logprob_fwd(H, W, lay.cu_seqlens, lay.mask, lay.targets)
    np.testing.assert_allclose(lp, ref["logp"], atol=1e-5, rtol=0)
    np.testing.assert_allclose(ent, ref["entropy"], atol=1e-5, rtol=0)
    np.testing.assert_allclose(lse, ref["lse"], atol=1e-5, rtol=0)
    assert (lp[lay.mask == 0] == 0).all() and (lse[lay.mask == 0] == 0).all()
    # the committed oracle fixture (tests/golden/make_golden.py) agrees too
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "tiny_oracle.npz"))
    np.testing.assert_allclose(lp, g["logp"], atol=1e-5, rtol=0)


def test_tiny_fp32_loss_fwd_bwd(rl):
    cfg = CONFIGS["tiny"]
    lay = make_layout(cfg, seed=0)
    H, W = make_tensors_host(cfg, lay.num_rows, seed=0)
    d = dev_tensors(lay)
    head = rl.Head(cfg.hidden, cfg.vocab, "f32")
    adv, _ = oracle.grpo_advantage(lay.rewards, lay.group_of_seq, lay.num_groups)
    ref_f = oracle.logprob_fwd(H, W, lay.cu_seqlens, lay.mask, lay.targets)
    old = guarded_old_logp(ref_f["logp"], np.random.default_rng(1), band=1e-3)
    N = lay.num_tokens
    out = _run_loss(rl, head, H.cuda(), W.cuda(), d, lay, old, adv.astype(np.float32), n_global=N)
    ref = oracle.policy_loss_fwd_bwd(H, W, lay.cu_seqlens, lay.mask, lay.targets, old,
                                     adv.astype(np.float32), n_global=N)
    np.testing.assert_allclose(out["logp"], ref["logp"], atol=1e-5, rtol=0)
    # the 1e-5 logp budget propagates through r = e^{logp-old}:
    # |dl_t| <= |A_t| r_t * 1e-5, so |dL_sum| <= 1e-5 * sum_t |A_t| r_t, and
    # the gradients (linear in g_t = -A r / N) get a 2e-5 relative budget.
    seq = np.searchsorted(lay.cu_seqlens, np.arange(lay.num_rows), side="right") - 1
    act = lay.mask.astype(bool)
    budget = 1e-5 * np.sum(np.abs(adv[seq][act]) * np.exp(ref["logp"][act] - old[act]))
    assert abs(out["stats"]["loss_sum"] - ref["loss_sum"]) <= budget + 1e-7
    assert out["stats"]["tokens"] == N
    assert rel_fro(out["dH"], ref["dH"]) <= 2e-5
    assert rel_fro(out["dW"], ref["dW"]) <= 2e-5
    assert (out["dH"][lay.mask == 0] == 0).all()


# ----------------------------------------------------------- bf16 tcgen05 ----
def _bf16_case(cfg, seed, rows=None):
    lay = make_layout(cfg, seed=seed)
    if rows is not None:
        lay, _ = sub_layout(lay, np.arange(rows))
    H, W = make_tensors_host(cfg, lay.num_rows, seed=seed)
    return lay, H, W


@pytest.mark.parametrize("cfg", [SMALL_BF16], ids=["h192-V1000"])
def test_bf16_forward_tc(rl, cfg):
    lay, H, W = _bf16_case(cfg, seed=2)
    d = dev_tensors(lay)
    head = rl.Head(cfg.hidden, cfg.vocab, "bf16")
    lp, ent, lse = _run_fwd(rl, head, H.cuda(), W.cuda(), d, lay)
    ref = oracle.logprob_fwd(H, W, lay.cu_seqlens, lay.mask, lay.targets)
    assert np.abs(lp - ref["logp"]).max() <= 2e-3
    assert np.abs(ent - ref["entropy"]).max() <= 2e-3
    assert np.abs(lse - ref["lse"]).max() <= 2e-3
    assert (lp[lay.mask == 0] == 0).all()


def test_bf16_loss_fwd_bwd_tc(rl):
    cfg = SMALL_BF16
    lay, H, W = _bf16_case(cfg, seed=4)
    d = dev_tensors(lay)
    head = rl.Head(cfg.hidden, cfg.vocab, "bf16")
    adv, _ = oracle.grpo_advantage(lay.rewards, lay.group_of_seq, lay.num_groups)
    adv = adv.astype(np.float32)
    ref_f = oracle.logprob_fwd(H, W, lay.cu_seqlens, lay.mask, lay.targets)
    old = guarded_old_logp(ref_f["logp"], np.random.default_rng(5))
    N = lay.num_tokens + 17   # a global N larger than this micro-batch
    out = _run_loss(rl, head, H.cuda(), W.cuda(), d, lay, old, adv, n_global=N)
    ref = oracle.policy_loss_fwd_bwd(H, W, lay.cu_seqlens, lay.mask, lay.targets, old, adv,
                                     n_global=N)
    assert np.abs(out["logp"] - ref["logp"]).max() <= 2e-3
    assert out["stats"]["loss_sum"] == pytest.approx(ref["loss_sum"], rel=1e-2)
    assert out["stats"]["clip_hi_count"] == ref["stats"]["clip_hi_count"]
    assert out["stats"]["clip_lo_count"] == ref["stats"]["clip_lo_count"]
    assert rel_fro(out["dH"], ref["dH"]) <= 1e-2 and max_rel(out["dH"], ref["dH"]) <= 1e-2
    assert rel_fro(out["dW"], ref["dW"]) <= 1e-2 and max_rel(out["dW"], ref["dW"]) <= 1e-2
    assert (out["dH"][lay.mask == 0] == 0).all()


def test_bf16_simt_crosscheck(rl):
    """The CUDA-core path on bf16 inputs agrees with the oracle too (checks the
    shared merge/loss kernels independently of tcgen05)."""
    cfg = SMALL_BF16
    lay, H, W = _bf16_case(cfg, seed=6)
    d = dev_tensors(lay)
    head = rl.Head(cfg.hidden, cfg.vocab, "bf16")
    os.environ["RLHEAD_FORCE_SIMT"] = "1"
    try:
        lp, _, _ = _run_fwd(rl, head, H.cuda(), W.cuda(), d, lay)
    finally:
        os.environ.pop("RLHEAD_FORCE_SIMT")
    ref = oracle.logprob_fwd(H, W, lay.cu_seqlens, lay.mask, lay.targets)
    assert np.abs(lp - ref["logp"]).max() <= 2e-3


def test_qwen15b_head_subbatch(rl):
    """Qwen-1.5B head shape (h=1536, V=151936, BJ:L8): two whole sequences."""
    cfg = QWEN15_HEAD
    lay = make_layout(cfg, seed=0)
    order = np.argsort(lay.resp_len)
    lay, _ = sub_layout(lay, order[:2])           # two shortest responses (+ prompts)
    H, W = make_tensors_host(cfg, lay.num_rows, seed=0)
    d = dev_tensors(lay)
    head = rl.Head(cfg.hidden, cfg.vocab, "bf16")
    adv = np.array([1.25, -0.5], dtype=np.float32)
    ref_f = oracle.logprob_fwd(H, W, lay.cu_seqlens, lay.mask, lay.targets)
    old = guarded_old_logp(ref_f["logp"], np.random.default_rng(7))
    out = _run_loss(rl, head, H.cuda(), W.cuda(), d, lay, old, adv, n_global=lay.num_tokens)
    ref = oracle.policy_loss_fwd_bwd(H, W, lay.cu_seqlens, lay.mask, lay.targets, old, adv)
    assert np.abs(out["logp"] - ref["logp"]).max() <= 2e-3
    assert np.abs(out["entropy"] - ref["entropy"]).max() <= 2e-3
    assert out["stats"]["loss_sum"] == pytest.approx(ref["loss_sum"], rel=1e-2)
    assert rel_fro(out["dH"], ref["dH"]) <= 1e-2
    assert rel_fro(out["dW"], ref["dW"]) <= 1e-2 and max_rel(out["dW"], ref["dW"]) <= 1e-2


def test_determinism_and_invariants(rl):
    """Bit-identical re-runs; sum_j dW_j ~ 0 (P14); empty batch is a no-op."""
    import torch
    cfg = SMALL_BF16
    lay, H, W = _bf16_case(cfg, seed=8)
    d = dev_tensors(lay)
    head = rl.Head(cfg.hidden, cfg.vocab, "bf16")
    adv = np.linspace(-1, 1, lay.num_seqs).astype(np.float32)
    old = np.zeros(lay.num_rows)
    a = _run_loss(rl, head, H.cuda(), W.cuda(), d, lay, old, adv)
    b = _run_loss(rl, head, H.cuda(), W.cuda(), d, lay, old, adv)
    np.testing.assert_array_equal(a["dH"], b["dH"])
    np.testing.assert_array_equal(a["dW"], b["dW"])
    assert a["stats"] == b["stats"]
    colsum = np.abs(a["dW"].sum(axis=0)).max()
    assert colsum <= 1e-2 * np.abs(a["dW"]).max()
    # empty micro-batch
    e = custom_layout([], [], [], [], vocab=cfg.vocab, num_groups=1)
    de = dev_tensors(e)
    gw = torch.zeros(cfg.vocab, cfg.hidden, device="cuda")
    st = rl.new_stats()
    rl.rl_policy_loss_fwd_bwd(head, torch.zeros(1, cfg.hidden, dtype=torch.bfloat16, device="cuda"),
                              W.cuda(), rl.Batch(de["cu"], de["targets"], de["mask"]),
                              torch.zeros(1, device="cuda"), torch.zeros(1, device="cuda"),
                              rl.LossParams(), torch.zeros(1, device="cuda"),
                              torch.zeros(1, cfg.hidden, dtype=torch.bfloat16, device="cuda"), gw,
                              stats=st)
    torch.cuda.synchronize()
    assert gw.abs().max().item() == 0 and rl.read_stats(st)["tokens"] == 0


def test_strided_hidden_rows(rl):
    """ld_hidden > hidden (rows of a wider buffer, e.g. a fused trunk output):
    the same logp / dL/dH / dW bit for bit as contiguous rows, dL/dH written
    with the same row stride, and the columns past `hidden` never touched."""
    import torch
    cfg = SMALL_BF16
    lay, H, W = _bf16_case(cfg, seed=12)
    d = dev_tensors(lay)
    R, h, ld = lay.num_rows, cfg.hidden, cfg.hidden + 64
    adv = np.linspace(-1, 1, lay.num_seqs).astype(np.float32)
    adv[0] = 0.0                                      # a row set without gradient
    old = torch.zeros(R, device="cuda")
    rl.rl_logprob_fwd(rl.Head(h, cfg.vocab, "bf16"), H.cuda(), W.cuda(),
                      rl.Batch(d["cu"], d["targets"], d["mask"]), old)
    old += 0.02
    res = []
    for stride in (h, ld):
        buf = torch.full((R, stride), 5.0, dtype=torch.bfloat16, device="cuda")
        buf[:, :h] = H.cuda()
        gbuf = torch.full((R, stride), -3.0, dtype=torch.bfloat16, device="cuda")
        head = rl.Head(h, cfg.vocab, "bf16", ld_hidden=stride)
        logp = torch.empty(R, device="cuda")
        gw = torch.zeros(cfg.vocab, h, device="cuda")
        rl.rl_policy_loss_fwd_bwd(head, buf, W.cuda(), rl.Batch(d["cu"], d["targets"], d["mask"]),
                                  old, torch.as_tensor(adv, device="cuda"), rl.LossParams(), logp,
                                  gbuf, gw)
        torch.cuda.synchronize()
        if stride > h:
            assert bool((gbuf[:, h:] == -3.0).all())     # padding columns untouched
        res.append((logp.cpu(), gbuf[:, :h].cpu(), gw.cpu()))
    for a, b in zip(res[0], res[1]):
        assert torch.equal(a, b)
