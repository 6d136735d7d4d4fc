"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (one 65,536-row micro-batch of the real layout through
rl_policy_loss_fwd_bwd), on outputs the oracle can compute one by one:
sampled rows' logp / entropy / dL/dH, plus properties that hold at any size
(P14 column sums of dW, micro-batch linearity of dW, masked rows exactly 0)."""
import numpy as np
import pytest

import oracle
from paper_2509_15965_b200.dp import pack_micro_batches
from tests.gpu_util import max_rel, rel_fro
from workload import CONFIGS, make_layout, make_tensors_torch, ratio_noise, sub_layout

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

MB_ROWS = 65536


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
    """dW of one 65k-row micro-batch == dW of its two halves accumulated by two
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
    g1 = torch.zeros(cfg.vocab, cfg.hidden, device=dev)
    run(np.arange(S), g1)
    g2 = torch.zeros_like(g1)
    run(np.arange(S // 2), g2)
    run(np.arange(S // 2, S), g2)
    torch.cuda.synchronize()
    err = (torch.linalg.vector_norm((g2 - g1).double()) /
           torch.linalg.vector_norm(g1.double())).item()
    assert err <= 1e-5
