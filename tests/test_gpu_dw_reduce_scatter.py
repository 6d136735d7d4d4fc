"""Fused DP dW reduce-scatter on ONE GPU, two ranks
emulated: each "rank" runs its two micro-batches, the last one with
rl_loss_params.dw_reduce_scatter pointing at two staging buffers; then each
rank's rl_reduce_bcast_rows_f32 writes its slab's rank-order sum into both
outputs (P2P path). Bit-exact expectations: the staged value is the same
fp32 (partial + tile) the local epilogue would have accumulated, and the
owner sums the slots as T_0 + T_1 -- so both outputs equal T_0 + T_1 of the
plain (non-fused) runs bit for bit, also when one rank's last micro-batch
has no active row (K = 0)."""
import numpy as np
import pytest

from workload import HeadConfig, make_layout, make_tensors_host, sub_layout

pytestmark = pytest.mark.gpu

CFG = HeadConfig("rs-bf16", 256, 1500, 8, 4, 200, "bf16", "reasoning")


def _rank_batches(rl, lay, dev, empty_last):
    import torch
    S = lay.num_seqs
    out = []
    for q, seqs in enumerate((np.arange(0, S // 2), np.arange(S // 2, S))):
        sub, _ = sub_layout(lay, seqs)
        h = len(seqs) // 2
        mbs = []
        for k, part in enumerate((np.arange(0, h), np.arange(h, len(seqs)))):
            mb, _ = sub_layout(sub, part)
            if empty_last and q == 1 and k == 1:
                mb.mask[:] = 0
            mbs.append(mb)
        out.append(mbs)
    return out


@pytest.mark.parametrize("bulk", ["0", "1"])
@pytest.mark.parametrize("empty_last", [False, True])
def test_fused_dw_reduce_scatter_two_ranks_one_gpu(rl, empty_last, bulk, monkeypatch):
    """bulk = 1: the epilogue ships each lane's 128-B row piece with a 1-D
    bulk copy from shared memory (RLHEAD_RS_BULK=1) -- same bits."""
    import torch
    monkeypatch.setenv("RLHEAD_RS_BULK", bulk)
    dev = "cuda"
    lay = make_layout(CFG, seed=71)
    V, h = CFG.vocab, CFG.hidden
    ranks = _rank_batches(rl, lay, dev, empty_last)
    _, W = make_tensors_host(CFG, 1, seed=71)
    Wd = W.to(dev)
    head = rl.Head(h, V, "bf16")
    rows = -(-V // 2)
    stg = [torch.full((2 * rows, h), float("nan"), device=dev) for _ in range(2)]
    outs = [torch.full((V, h), float("nan"), device=dev) for _ in range(2)]
    pg = [rl.PeerGroup(q, 2, rows, [t.data_ptr() for t in stg]) for q in range(2)]
    totals, partials = [], []
    for q, mbs in enumerate(ranks):
        feeds = []
        for k, mb in enumerate(mbs):
            H, _ = make_tensors_host(CFG, max(mb.num_rows, 1), seed=100 * q + k)
            feeds.append((mb, H[:mb.num_rows].to(dev)))
        N = sum(mb.num_tokens for mb in mbs)

        def run(mb, Hd, gw, p):
            adv = torch.linspace(-1, 1, mb.num_seqs, device=dev)
            b = rl.Batch(torch.as_tensor(mb.cu_seqlens, device=dev),
                         torch.as_tensor(mb.targets, device=dev),
                         torch.as_tensor(mb.mask, device=dev))
            lp = torch.empty(max(mb.num_rows, 1), device=dev)
            rl.rl_logprob_fwd(head, Hd, Wd, b, lp)
            old = lp - 0.05
            rl.rl_policy_loss_fwd_bwd(head, Hd, Wd, b, old, adv, p, torch.empty_like(lp),
                                      torch.empty_like(Hd), gw)

        nt = torch.tensor([max(N, 1)], device=dev)
        gw = torch.zeros(V, h, device=dev)
        for mb, Hd in feeds:                              # plain: T_q
            run(mb, Hd, gw, rl.LossParams(n_tokens_global=nt))
        totals.append(gw)
        gw2 = torch.zeros(V, h, device=dev)               # fused: last mb -> staging
        run(*feeds[0], gw2, rl.LossParams(n_tokens_global=nt))
        part = gw2.clone()
        run(*feeds[1], gw2, rl.LossParams(n_tokens_global=nt, dw_reduce_scatter=pg[q]))
        torch.cuda.synchronize()
        assert torch.equal(gw2, part)                     # local buffer only read
        partials.append(part)
    for q in range(2):
        rl.rl_reduce_bcast_rows_f32(stg[q], outs[q], q, 2, rows,
                                    out_peer_ptrs=[o.data_ptr() for o in outs])
    torch.cuda.synchronize()
    expect = totals[0] + totals[1]
    assert torch.equal(outs[0], expect) and torch.equal(outs[1], expect)
    assert float(expect.abs().max()) > 0


@pytest.mark.parametrize("bulk", ["0", "1"])
def test_fused_dw_reduce_scatter_no_partial(rl, bulk, monkeypatch):
    """rl_peer_group.no_partial = 1 (the rank's only micro-batch): the epilogue
    sends the tile alone and never reads grad_weight -- here filled with NaN,
    which would poison the sum if it were read. Owners' sums equal T_0 + T_1 of
    the plain single-micro-batch runs bit for bit."""
    import torch
    monkeypatch.setenv("RLHEAD_RS_BULK", bulk)
    dev = "cuda"
    lay = make_layout(CFG, seed=73)
    V, h = CFG.vocab, CFG.hidden
    S = lay.num_seqs
    _, W = make_tensors_host(CFG, 1, seed=73)
    Wd = W.to(dev)
    head = rl.Head(h, V, "bf16")
    rows = -(-V // 2)
    stg = [torch.full((2 * rows, h), float("nan"), device=dev) for _ in range(2)]
    outs = [torch.full((V, h), float("nan"), device=dev) for _ in range(2)]
    pg = [rl.PeerGroup(q, 2, rows, [t.data_ptr() for t in stg], no_partial=True)
          for q in range(2)]
    totals = []
    for q, seqs in enumerate((np.arange(0, S // 2), np.arange(S // 2, S))):
        mb, _ = sub_layout(lay, seqs)
        H, _ = make_tensors_host(CFG, max(mb.num_rows, 1), seed=300 + q)
        Hd = H[:mb.num_rows].to(dev)
        adv = torch.linspace(-1, 1, mb.num_seqs, device=dev)
        b = rl.Batch(torch.as_tensor(mb.cu_seqlens, device=dev),
                     torch.as_tensor(mb.targets, device=dev), torch.as_tensor(mb.mask, device=dev))
        lp = torch.empty(max(mb.num_rows, 1), device=dev)
        rl.rl_logprob_fwd(head, Hd, Wd, b, lp)
        old = lp - 0.05
        nt = torch.tensor([max(mb.num_tokens, 1)], device=dev)
        gw = torch.zeros(V, h, device=dev)
        rl.rl_policy_loss_fwd_bwd(head, Hd, Wd, b, old, adv, rl.LossParams(n_tokens_global=nt),
                                  torch.empty_like(lp), torch.empty_like(Hd), gw)
        totals.append(gw)
        gw_nan = torch.full((V, h), float("nan"), device=dev)
        rl.rl_policy_loss_fwd_bwd(head, Hd, Wd, b, old, adv,
                                  rl.LossParams(n_tokens_global=nt, dw_reduce_scatter=pg[q]),
                                  torch.empty_like(lp), torch.empty_like(Hd), gw_nan)
    for q in range(2):
        rl.rl_reduce_bcast_rows_f32(stg[q], outs[q], q, 2, rows,
                                    out_peer_ptrs=[o.data_ptr() for o in outs])
    torch.cuda.synchronize()
    expect = totals[0] + totals[1]
    assert torch.equal(outs[0], expect) and torch.equal(outs[1], expect)
    assert float(expect.abs().max()) > 0
