"""Parity at BASELINE.json's full head sizes, in the launch configuration
bench.py times (PolicyLossStep with 16,384-row micro-batches: the same
driver, kernels, tile shapes and dW accumulation path).

* test_fullsize_oracle_subbatch: a sub-batch of WHOLE sequences of the real
  layout run through the bench's driver and through
  the CPU float64 oracle on the same values: every row's logp and entropy
  (<= 2e-3), loss_sum / ratio_sum / entropy_sum (rel 1e-2), tokens and both
  clip counts (exact; the guard band keeps fp32 and fp64 on the same side
  of 1 +- eps), advantages (1e-5), dH and dW (rel_fro and max_rel <= 1e-2).
  At the 7B/32B heads the dW GEMM has K ~ 4k rows (16 k-blocks of 256) and
  56 waves, so odd (serpentine, K walked backwards) waves are covered.
  Token-level mean over the sub-batch's N, micro-batch = fwd/bwd
  unit.
* test_fullsize_sampled_rows: the first 16k-row micro-batch of each real
  layout, sampled rows' logp / entropy / dL/dH vs the oracle, plus the P14
  column-sum bound on dW and exact zeros on masked rows.
* test_fullsize_dw_linearity: dW of a micro-batch == dW of its halves.
"""
import numpy as np
import pytest

import oracle
from paper_2509_15965_b200.dp import pack_micro_batches
from tests.gpu_util import guarded_old_logp, max_rel, rel_fro
from workload import CONFIGS, make_layout, make_tensors_torch, ratio_noise, sub_layout

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

MB_ROWS = 16384          # bench.py --mb-rows default


def _seq_tokens(lay):
    cu = lay.cu_seqlens.astype(np.int64)
    return np.add.reduceat(lay.mask.astype(np.int64), cu[:-1])


def _whole_seq_subbatch(lay, target):
    """Whole sequences of the real layout with >= `target` response tokens:
    the two shortest of the forced all-correct group 0 (zero variance ->
    A = 0 exactly, rows with no gradient) plus the shortest sequences of the
    mixed-reward group that reaches `target` with the fewest tokens."""
    tok = _seq_tokens(lay)
    gos = lay.group_of_seq
    g0 = np.flatnonzero(gos == 0)
    sel = list(g0[np.argsort(tok[g0], kind="stable")][:2])
    t0 = int(tok[sel].sum())
    best = None
    for g in range(2, lay.num_groups):
        m = np.flatnonzero(gos == g)
        acc, s = [], t0
        for i in m[np.argsort(tok[m], kind="stable")]:
            acc.append(int(i))
            s += int(tok[i])
            if s >= target and len(set(lay.rewards[acc].tolist())) == 2:
                break
        if s >= target and len(set(lay.rewards[acc].tolist())) == 2 and \
                (best is None or s < best[0]):
            best = (s, acc)
    return np.array(sorted(sel + best[1]))


def _smallest_groups(lay, k):
    tok = _seq_tokens(lay)
    g_tok = np.bincount(lay.group_of_seq, weights=tok, minlength=lay.num_groups)
    groups = np.argsort(g_tok, kind="stable")[:k]
    return np.flatnonzero(np.isin(lay.group_of_seq, groups))


def _subbatch(name):
    cfg = CONFIGS[name]
    lay = make_layout(cfg, seed=0)
    if name == "qwen1.5b":
        seqs = _smallest_groups(lay, 2)          # two whole prompt groups
    elif name == "openvla":
        seqs = np.flatnonzero(lay.group_of_seq == 5)   # one whole group of 8 envs
    else:
        seqs = _whole_seq_subbatch(lay, 4096)
    sub, _ = sub_layout(lay, seqs)
    return cfg, sub


def _chunked_cmp(gpu, ref, chunk=8192):
    """(rel_fro, max_rel) of a device fp32/bf16 matrix vs a float64 host
    matrix, streamed in row chunks (the 32B dW is 3.1 GB fp32 / 6.2 GB fp64)."""
    import torch
    num = den = 0.0
    dmax = rmax = 0.0
    for r0 in range(0, ref.shape[0], chunk):
        a = gpu[r0:r0 + chunk].to(torch.float64).cpu().numpy()
        b = ref[r0:r0 + chunk]
        d = a - b
        num += float(np.sum(d * d))
        den += float(np.sum(b * b))
        dmax = max(dmax, float(np.abs(d).max()))
        rmax = max(rmax, float(np.abs(b).max()))
    return (num / den) ** 0.5 if den > 0 else num ** 0.5, dmax / rmax if rmax > 0 else dmax


_ORACLE_CACHE = {}


def _oracle_case(name):
    """(cfg, sub-layout, H, W on cuda, old, oracle result) -- the oracle runs
    once per config (minutes of float64 work at the 32B head)."""
    import torch
    if name in _ORACLE_CACHE:
        return _ORACLE_CACHE[name]
    cfg, sub = _subbatch(name)
    H, W = make_tensors_torch(cfg, sub.num_rows, seed=3, device="cuda")
    Hh, Wh = H.cpu(), W.cpu()
    W64 = Wh.to(torch.float64).numpy()           # exact values of the bf16 weight
    fwd = oracle.logprob_fwd(Hh, W64, sub.cu_seqlens, sub.mask, sub.targets)
    # old = logp - ln r*, r* guard-banded 1e-2 away from 1 +- eps:
    # ~18% of the tokens lie beyond a clip bound, none near one.
    old = guarded_old_logp(fwd["logp"], np.random.default_rng(17))
    adv, err = oracle.grpo_advantage(sub.rewards, sub.group_of_seq, sub.num_groups)
    assert err == 0
    ref = oracle.policy_loss_fwd_bwd(Hh, W64, sub.cu_seqlens, sub.mask, sub.targets, old, adv,
                                     n_global=sub.num_tokens)
    del W64
    _ORACLE_CACHE[name] = (cfg, sub, H, W, old, adv, ref)
    return _ORACLE_CACHE[name]


@pytest.mark.parametrize("name,mb_rows", [("qwen1.5b", MB_ROWS), ("qwen1.5b", 3000),
                                          ("openvla", MB_ROWS), ("qwen7b", MB_ROWS),
                                          ("qwen32b", MB_ROWS)],
                         ids=["qwen1.5b", "qwen1.5b-multi-mb", "openvla", "qwen7b", "qwen32b"])
def test_fullsize_oracle_subbatch(rl, name, mb_rows):
    import torch
    from paper_2509_15965_b200.dp import PolicyLossStep, device_batch
    cfg, sub, H, W, old, adv_ref, ref = _oracle_case(name)
    if not (name == "qwen1.5b" and mb_rows == MB_ROWS):   # reused by the multi-mb case only
        _ORACLE_CACHE.pop(name)
    dev = H.device
    db = device_batch(sub, mb_rows, device=dev)
    if mb_rows < MB_ROWS:
        assert len(db.mbs) >= 3          # dW accumulated over several calls
    head = rl.Head(cfg.hidden, cfg.vocab, cfg.dtype)
    step = PolicyLossStep(head, W, db, want_entropy=True)
    gh = torch.full_like(H, 7.0)
    old_t = torch.as_tensor(old, dtype=torch.float32, device=dev)
    step.run(H, old_t, gh)
    torch.cuda.synchronize()
    R = sub.num_rows
    act = sub.mask.astype(bool)
    # advantages (H2) and N (H1)
    np.testing.assert_allclose(step.adv[:sub.num_seqs].cpu().double().numpy(), adv_ref,
                               rtol=1e-5, atol=1e-5)
    assert int(step.n_global.item()) == sub.num_tokens == ref["stats"]["tokens"]
    # per-row logp / entropy (H3, H4), every row; masked rows exactly 0
    lp = step.logp[:R].cpu().double().numpy()
    ent = step.entropy[:R].cpu().double().numpy()
    assert np.abs(lp - ref["logp"]).max() <= 2e-3
    assert np.abs(ent - ref["entropy"]).max() <= 2e-3
    assert (lp[~act] == 0).all() and (ent[~act] == 0).all()
    # loss statistics (H5)
    s = rl.read_stats(step.stats)
    rs = ref["stats"]
    assert s["tokens"] == rs["tokens"]
    assert s["clip_hi_count"] == rs["clip_hi_count"] > 0
    assert s["clip_lo_count"] == rs["clip_lo_count"] > 0
    assert s["loss_sum"] == pytest.approx(rs["loss_sum"], rel=1e-2)
    assert s["ratio_sum"] == pytest.approx(rs["ratio_sum"], rel=1e-2)
    assert s["entropy_sum"] == pytest.approx(rs["entropy_sum"], rel=1e-2)
    assert s["ratio_max"] == pytest.approx(rs["ratio_max"], rel=1e-2)
    # dL/dH (H6, H7): every row; masked rows and A = 0 rows exactly 0
    dH = gh.to(torch.float64).cpu().numpy()
    assert rel_fro(dH, ref["dH"]) <= 1e-2 and max_rel(dH, ref["dH"]) <= 1e-2
    assert (dH[~act] == 0).all()
    zero_rows = act & np.all(ref["dH"] == 0, axis=1)
    assert zero_rows.any() and (dH[zero_rows] == 0).all()
    # dL/dW (H8)
    fro, mrel = _chunked_cmp(step.grad_w, ref["dW"])
    assert fro <= 1e-2 and mrel <= 1e-2, (fro, mrel)


def _first_micro_batch(cfg, seed=0):
    lay = make_layout(cfg, seed=seed)
    cu = lay.cu_seqlens.astype(np.int64)
    s0, s1 = pack_micro_batches(cu[1:] - cu[:-1], MB_ROWS)[0]
    mb, _ = sub_layout(lay, np.arange(s0, s1))
    return lay, mb


@pytest.mark.parametrize("name", ["qwen1.5b", "openvla", "qwen7b", "qwen32b"])
def test_fullsize_sampled_rows(rl, name):
    import torch
    cfg = CONFIGS[name]
    lay, mb = _first_micro_batch(cfg)
    dev = "cuda"
    H, W = make_tensors_torch(cfg, mb.num_rows, seed=1, device=dev)
    head = rl.Head(cfg.hidden, cfg.vocab, "bf16")
    cu = torch.as_tensor(mb.cu_seqlens, device=dev)
    tg = torch.as_tensor(mb.targets, device=dev)
    mk = torch.as_tensor(mb.mask, device=dev)
    R = mb.num_rows
    # old = own logp + delta (the bench's construction); adv from the GRPO kernel
    old = torch.empty(R, device=dev)
    rl.rl_logprob_fwd(head, H, W, rl.Batch(cu, tg, mk), old)
    old += torch.as_tensor(ratio_noise(R, 11), dtype=torch.float32, device=dev)
    rw = torch.as_tensor(mb.rewards, device=dev)
    gos_np = np.unique(mb.group_of_seq, return_inverse=True)[1].astype(np.int32)
    adv = torch.empty(mb.num_seqs, device=dev)
    rl.rl_grpo_advantage(rw, torch.as_tensor(gos_np, device=dev), int(gos_np.max()) + 1, adv)
    N = lay.num_tokens                             # the whole mini-batch's N
    p = rl.LossParams(n_tokens_global=torch.tensor([N], device=dev))
    logp = torch.empty(R, device=dev)
    ent = torch.empty(R, device=dev)
    gh = torch.full_like(H, 1.0)
    gw = torch.zeros(cfg.vocab, cfg.hidden, device=dev)
    st = rl.new_stats()
    rl.rl_policy_loss_fwd_bwd(head, H, W, rl.Batch(cu, tg, mk), old, adv, p, logp, gh, gw,
                              entropy=ent, stats=st)
    torch.cuda.synchronize()
    s = rl.read_stats(st)
    assert s["tokens"] == mb.num_tokens
    # masked rows: exact zeros
    inact = torch.as_tensor(mb.mask == 0, device=dev)
    assert gh[inact].abs().max().item() == 0 if inact.any() else True
    assert logp[inact].abs().max().item() == 0 if inact.any() else True
    # P14 at full size: sum_j dW_j = sum_t (sum_j dZ_tj) h_t is 0 exactly; with
    # dZ rounded to bf16 each row sum is bounded by 2^-8 * sum_j |dZ_tj|
    # = 2^-8 * 2|g_t|(1 - p_y) <= 2^-7 |g_t|, so |colsum_k| <= 2^-7 sum_t |g_t h_tk|
    # (g_t from this run's logp; a consistency bound, not an oracle value).
    act_t = torch.as_tensor(mb.mask.astype(bool), device=dev)
    seq_t = torch.as_tensor(np.searchsorted(mb.cu_seqlens, np.arange(R), side="right") - 1,
                            device=dev)
    r_t = torch.exp(torch.clamp(logp - old, -20, 20))
    g_bound = (adv[seq_t].abs() * r_t / N * act_t).double()
    colsum = gw.double().sum(0).abs()
    bound = 2.0 ** -7 * (g_bound[:, None] * H.double().abs()).sum(0) * 1.05 + 1e-12
    assert bool((colsum <= bound).all()), float((colsum / bound).max())
    # sampled rows vs oracle (exact fp64 on the device tensors' values)
    rng = np.random.default_rng(0)
    act = np.flatnonzero(mb.mask)
    rows = np.sort(rng.choice(act, size=min(96, len(act)), replace=False))
    Hs = H[torch.as_tensor(rows, device=dev)].cpu()
    cu1 = np.arange(len(rows) + 1, dtype=np.int32)  # one row per sequence
    seq = np.searchsorted(mb.cu_seqlens, rows, side="right") - 1
    old_s = old.cpu().double().numpy()[rows]
    adv_s = adv.cpu().double().numpy()[seq]
    ref = oracle.policy_loss_fwd_bwd(Hs, W.cpu(), cu1, np.ones(len(rows), np.uint8),
                                     mb.targets[rows], old_s, adv_s, n_global=N)
    lp = logp.cpu().double().numpy()[rows]
    assert np.abs(lp - ref["logp"]).max() <= 2e-3
    assert np.abs(ent.cpu().double().numpy()[rows] - ref["entropy"]).max() <= 2e-3
    # rows whose clip decision is not within 1e-3 of a boundary (fp32 vs fp64)
    r = np.exp(ref["logp"] - old_s)
    safe = np.minimum(np.abs(r - 0.8), np.abs(r - 1.2)) > 1e-3
    dH = gh[torch.as_tensor(rows, device=dev)].cpu().double().numpy()
    assert rel_fro(dH[safe], ref["dH"][safe]) <= 1e-2
    assert max_rel(dH[safe], ref["dH"][safe]) <= 1e-2


@pytest.mark.parametrize("name", ["qwen7b"])
def test_fullsize_dw_linearity(rl, name):
    """dW of one 16k-row micro-batch == dW of its two halves accumulated by two
    calls (the micro-batch streaming contract), to fp32 rounding."""
    import torch
    cfg = CONFIGS[name]
    lay, mb = _first_micro_batch(cfg)
    dev = "cuda"
    H, W = make_tensors_torch(cfg, mb.num_rows, seed=2, device=dev)
    head = rl.Head(cfg.hidden, cfg.vocab, "bf16")
    old = torch.zeros(mb.num_rows, device=dev)
    adv = torch.linspace(-1, 1, mb.num_seqs, device=dev)
    p = rl.LossParams(n_tokens_global=torch.tensor([lay.num_tokens], device=dev))

    def run(seqs, gw):
        sub, rows = sub_layout(mb, seqs)
        ridx = torch.as_tensor(rows, device=dev)
        b = rl.Batch(torch.as_tensor(sub.cu_seqlens, device=dev),
                     torch.as_tensor(sub.targets, device=dev), torch.as_tensor(sub.mask, device=dev))
        rl.rl_policy_loss_fwd_bwd(head, H[ridx].contiguous(), W, b, old[ridx],
                                  adv[torch.as_tensor(seqs, device=dev)].contiguous(), p,
                                  torch.empty(len(rows), device=dev),
                                  torch.empty(len(rows), cfg.hidden, dtype=H.dtype, device=dev), gw)

    S = mb.num_seqs
    assert S >= 2
    g1 = torch.zeros(cfg.vocab, cfg.hidden, device=dev)
    run(np.arange(S), g1)
    g2 = torch.zeros_like(g1)
    run(np.arange(S // 2), g2)
    run(np.arange(S // 2, S), g2)
    torch.cuda.synchronize()
    err = (torch.linalg.vector_norm((g2 - g1).double()) /
           torch.linalg.vector_norm(g1.double())).item()
    assert err <= 1e-5
