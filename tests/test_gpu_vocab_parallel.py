"""Vocab-parallel head (NEXT-3) on one GPU: the TP group is emulated by
calling each shard in turn and stacking their partials (what the all-gather
does), then checking against the unsharded oracle: logp/entropy/lse of the
merged softmax, the sum of the shards' dH partials (what the all-reduce does)
and the concatenation of the shards' dW rows."""
import numpy as np
import pytest

import oracle
from tests.gpu_util import dev_tensors, guarded_old_logp, max_rel, rel_fro
from workload import CONFIGS, HeadConfig, make_layout, make_tensors_host

pytestmark = pytest.mark.gpu

SMALL_BF16 = HeadConfig("small-bf16", 192, 1000, 6, 4, 96, "bf16", "reasoning")


@pytest.mark.parametrize("cfg,cuts,tol", [(SMALL_BF16, [0, 300, 1000], 2e-3),
                                          (SMALL_BF16, [0, 256, 512, 777, 1000], 2e-3),
                                          (CONFIGS["tiny"], [0, 333, 666, 1000], 1e-5)],
                         ids=["bf16-2way", "bf16-4way", "fp32-3way"])
def test_vocab_parallel_emulated(rl, cfg, cuts, tol):
    import torch
    lay = make_layout(cfg, seed=31)
    H, W = make_tensors_host(cfg, lay.num_rows, seed=31)
    d = dev_tensors(lay)
    dev = "cuda"
    R, V = lay.num_rows, cfg.vocab
    Hd = H.to(dev)
    batch = rl.Batch(d["cu"], d["targets"], d["mask"])
    heads = [rl.Head(cfg.hidden, b - a, cfg.dtype, vocab_offset=a, vocab_total=V)
             for a, b in zip(cuts[:-1], cuts[1:])]
    shards = [W[a:b].contiguous().to(dev) for a, b in zip(cuts[:-1], cuts[1:])]
    P = len(heads)
    parts = torch.zeros(P, 4, R, device=dev)
    for i in range(P):
        rl.rl_logprob_partials(heads[i], Hd, shards[i], batch, parts[i])
    logp = torch.empty(R, device=dev)
    ent = torch.empty(R, device=dev)
    lse = torch.empty(R, device=dev)
    rl.rl_logprob_merge(heads[0], batch, parts, logp, ent, lse)
    torch.cuda.synchronize()
    ref = oracle.logprob_fwd(H, W, lay.cu_seqlens, lay.mask, lay.targets)
    for k, v in (("logp", logp), ("entropy", ent), ("lse", lse)):
        assert np.abs(v.cpu().double().numpy() - ref[k]).max() <= tol, k
    # shard partials themselves vs the oracle's shard partials
    T = lay.num_tokens
    for i, (a, b) in enumerate(zip(cuts[:-1], cuts[1:])):
        po = oracle.head.logprob_shard_partials(H, W[a:b], a, V, lay.cu_seqlens, lay.mask,
                                                lay.targets)
        pg = parts[i, :, :T].cpu().double().numpy()
        assert np.abs(pg[0] - po[0]).max() <= tol and np.abs(pg[3] - po[3]).max() <= tol
        np.testing.assert_allclose(pg[1], po[1], rtol=max(tol, 1e-5))
    # training: each shard's backward with the gathered partials
    adv, _ = oracle.grpo_advantage(lay.rewards, lay.group_of_seq, lay.num_groups)
    adv = adv.astype(np.float32)
    old = guarded_old_logp(ref["logp"], np.random.default_rng(3),
                           band=1e-2 if cfg.dtype == "bf16" else 1e-3)
    N = T
    p = rl.LossParams(n_tokens_global=torch.tensor([N], device=dev))
    old_d = torch.as_tensor(old, dtype=torch.float32, device=dev)
    adv_d = torch.as_tensor(adv, device=dev)
    dH_sum = torch.zeros(R, cfg.hidden, dtype=torch.float64, device=dev)
    dW_rows = []
    logps = []
    for i in range(P):
        lp_i = torch.empty(R, device=dev)
        gh = torch.empty_like(Hd)
        gw = torch.zeros(shards[i].shape[0], cfg.hidden, device=dev)
        st = rl.new_stats()
        rl.rl_policy_loss_fwd_bwd_vp(heads[i], Hd, shards[i], batch, parts, old_d, adv_d, p, lp_i,
                                     gh, gw, stats=st)
        dH_sum += gh.double()
        dW_rows.append(gw)
        logps.append(lp_i)
    torch.cuda.synchronize()
    for lp_i in logps[1:]:            # identical softmax on every rank of the TP group
        assert torch.equal(lp_i, logps[0])
    refl = oracle.policy_loss_fwd_bwd(H, W, lay.cu_seqlens, lay.mask, lay.targets, old, adv,
                                      n_global=N)
    g_tol = 1e-2 if cfg.dtype == "bf16" else 5e-5
    dH = dH_sum.cpu().numpy()
    dW = torch.cat(dW_rows).cpu().double().numpy()
    assert rel_fro(dH, refl["dH"]) <= g_tol
    assert rel_fro(dW, refl["dW"]) <= g_tol and max_rel(dW, refl["dW"]) <= max(g_tol, 1e-4)


def test_vocab_parallel_fp32_partials_and_p2p_sum(rl):
    """DESIGN.md §7.3 on one GPU: (a) the fp32 partial dL/dH (grad_hidden_fp32 = 1)
    is the accumulator the bf16 path rounds -- bf16(fp32 rows) equals the bf16
    rows bit for bit; (b) rl_allreduce_sum_f32 in P2P mode, driven once per
    emulated rank over P buffers, leaves on every buffer the rank-order sum
    ((s0 + s1) + s2 ... in fp32) bit-exactly; (c) that sum matches the oracle's
    dL/dH and rl_cast_rows_bf16 rounds it to nearest-even like torch."""
    import torch
    cfg = SMALL_BF16
    cuts = [0, 256, 512, 777, 1000]
    lay = make_layout(cfg, seed=37)
    H, W = make_tensors_host(cfg, lay.num_rows, seed=37)
    d = dev_tensors(lay)
    dev = "cuda"
    R, V, h = lay.num_rows, cfg.vocab, cfg.hidden
    Hd = H.to(dev)
    batch = rl.Batch(d["cu"], d["targets"], d["mask"])
    heads = [rl.Head(h, b - a, "bf16", vocab_offset=a, vocab_total=V)
             for a, b in zip(cuts[:-1], cuts[1:])]
    shards = [W[a:b].contiguous().to(dev) for a, b in zip(cuts[:-1], cuts[1:])]
    P = len(heads)
    parts = torch.zeros(P, 4, R, device=dev)
    for i in range(P):
        rl.rl_logprob_partials(heads[i], Hd, shards[i], batch, parts[i])
    ref_f = oracle.logprob_fwd(H, W, lay.cu_seqlens, lay.mask, lay.targets)
    adv, _ = oracle.grpo_advantage(lay.rewards, lay.group_of_seq, lay.num_groups)
    adv = adv.astype(np.float32)
    old = guarded_old_logp(ref_f["logp"], np.random.default_rng(4), band=1e-2)
    N = lay.num_tokens
    p = rl.LossParams(n_tokens_global=torch.tensor([N], device=dev))
    old_d = torch.as_tensor(old, dtype=torch.float32, device=dev)
    adv_d = torch.as_tensor(adv, device=dev)
    bufs = []
    for i in range(P):
        lp = torch.empty(R, device=dev)
        gh16 = torch.empty_like(Hd)
        gh32 = torch.full((R, h), 7.0, device=dev)          # inactive rows must be zeroed
        gw = torch.zeros(shards[i].shape[0], h, device=dev)
        rl.rl_policy_loss_fwd_bwd_vp(heads[i], Hd, shards[i], batch, parts, old_d, adv_d, p, lp,
                                     gh16, gw)
        gw2 = torch.zeros_like(gw)
        rl.rl_policy_loss_fwd_bwd_vp(heads[i], Hd, shards[i], batch, parts, old_d, adv_d, p, lp,
                                     gh32, gw2)
        torch.cuda.synchronize()
        assert torch.equal(gh32.to(torch.bfloat16), gh16)                       # (a)
        assert torch.equal(gw, gw2)
        bufs.append(gh32)
    expect = bufs[0].clone()
    for q in range(1, P):
        expect = expect + bufs[q]
    ptrs = [b.data_ptr() for b in bufs]
    for r in range(P):                                # each emulated rank sums its slice
        rl.rl_allreduce_sum_f32(bufs[r], r, P, peer_ptrs=ptrs)
    torch.cuda.synchronize()
    for b in bufs:                                                              # (b)
        assert torch.equal(b, expect)
    refl = oracle.policy_loss_fwd_bwd(H, W, lay.cu_seqlens, lay.mask, lay.targets, old, adv,
                                      n_global=N)
    assert rel_fro(expect.cpu().double().numpy(), refl["dH"]) <= 1e-2                # (c)
    out = torch.full((R, h + 64), 3.0, dtype=torch.bfloat16, device=dev)[:, :h]
    rl.rl_cast_rows_bf16(expect, out)
    torch.cuda.synchronize()
    assert torch.equal(out, expect.to(torch.bfloat16))


def test_allreduce_sum_f32_args(rl):
    import torch
    x = torch.ones(8, device="cuda")
    rl.rl_allreduce_sum_f32(x, 0, 1, peer_ptrs=[x.data_ptr()])   # world 1: no-op
    torch.cuda.synchronize()
    assert torch.equal(x, torch.ones(8, device="cuda"))
    with pytest.raises(rl.RLHeadError):
        rl.rl_allreduce_sum_f32(torch.ones(6, device="cuda"), 0, 2, peer_ptrs=[x.data_ptr()] * 2)
    with pytest.raises(rl.RLHeadError):
        rl.rl_allreduce_sum_f32(x, 2, 2, peer_ptrs=[x.data_ptr()] * 2)
