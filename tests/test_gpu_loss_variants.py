"""NEXT-1 loss variants on the CUDA path vs the oracle (DESIGN.md §3 #25-#28):
dual clip, KL-k3 to a reference policy, entropy bonus (extra dZ epilogue
term), seq-mean-token-mean aggregation (S from rl_batch_prepare)."""
import numpy as np
import pytest

import oracle
from tests.gpu_util import dev_tensors, guarded_old_logp, max_rel, rel_fro
from workload import CONFIGS, HeadConfig, make_layout, make_tensors_host

pytestmark = pytest.mark.gpu

SMALL_BF16 = HeadConfig("small-bf16", 192, 1000, 6, 4, 96, "bf16", "reasoning")


def _run(rl, cfg, seq_mean, seed, tol_g, tol_lp):
    import torch
    lay = make_layout(cfg, seed=seed)
    H, W = make_tensors_host(cfg, lay.num_rows, seed=seed)
    d = dev_tensors(lay)
    head = rl.Head(cfg.hidden, cfg.vocab, cfg.dtype)
    adv, _ = oracle.grpo_advantage(lay.rewards, lay.group_of_seq, lay.num_groups)
    adv = adv.astype(np.float32)
    rng = np.random.default_rng(seed + 1)
    lp = oracle.logprob_fwd(H, W, lay.cu_seqlens, lay.mask, lay.targets)["logp"]
    old = guarded_old_logp(lp, rng, clip_lo=0.2, clip_hi=0.28,
                           band=1e-2 if cfg.dtype == "bf16" else 1e-3)
    ref = (lp + rng.normal(0, 0.3, size=lp.shape)).astype(np.float32)
    p_or = oracle.LossParams(clip_lo=0.2, clip_hi=0.28, dual_clip=3.0, kl_coef=0.05,
                             entropy_coef=0.01, seq_mean=seq_mean)
    N, S = lay.num_tokens + 11, lay.num_seqs + 3      # global normalisers > this batch
    ref_out = oracle.policy_loss_fwd_bwd(H, W, lay.cu_seqlens, lay.mask, lay.targets, old, adv,
                                         p_or, n_global=N, n_seqs_global=S,
                                         ref_logp=ref.astype(np.float64))
    dev = "cuda"
    p = rl.LossParams(clip_lo=0.2, clip_hi=0.28, dual_clip=3.0, kl_coef=0.05, entropy_coef=0.01,
                      seq_mean=seq_mean, ref_logp=torch.as_tensor(ref, device=dev),
                      n_tokens_global=torch.tensor([N], device=dev),
                      n_seqs_global=torch.tensor([S], device=dev))
    R = lay.num_rows
    Hd, Wd = H.to(dev), W.to(dev)
    logp = torch.empty(R, device=dev)
    gh = torch.full_like(Hd, 2.0)
    gw = torch.zeros(cfg.vocab, cfg.hidden, device=dev)
    st = rl.new_stats()
    rl.rl_policy_loss_fwd_bwd(head, Hd, Wd, rl.Batch(d["cu"], d["targets"], d["mask"]),
                              torch.as_tensor(old, dtype=torch.float32, device=dev),
                              torch.as_tensor(adv, device=dev), p, logp, gh, gw, stats=st)
    torch.cuda.synchronize()
    s = rl.read_stats(st)
    assert np.abs(logp.cpu().double().numpy() - ref_out["logp"]).max() <= tol_lp
    assert s["objective"] == pytest.approx(ref_out["stats"]["objective"], rel=tol_g, abs=1e-9)
    assert s["kl_sum"] == pytest.approx(ref_out["stats"]["kl_sum"], rel=tol_g, abs=1e-6)
    dH = gh.cpu().double().numpy()
    dW = gw.cpu().double().numpy()
    assert rel_fro(dH, ref_out["dH"]) <= tol_g and rel_fro(dW, ref_out["dW"]) <= tol_g
    assert max_rel(dW, ref_out["dW"]) <= max(tol_g, 1e-2 if cfg.dtype == "bf16" else 1e-4)
    return lay


@pytest.mark.parametrize("seq_mean", [False, True], ids=["token-mean", "seq-mean"])
def test_variants_bf16_tc(rl, seq_mean):
    _run(rl, SMALL_BF16, seq_mean, seed=21, tol_g=1e-2, tol_lp=2e-3)


@pytest.mark.parametrize("seq_mean", [False, True], ids=["token-mean", "seq-mean"])
def test_variants_fp32_simt(rl, seq_mean):
    # fp32 budget: 1e-5 logp -> ~2e-5 relative on the gradients
    _run(rl, CONFIGS["tiny"], seq_mean, seed=22, tol_g=5e-5, tol_lp=1e-5)


def test_nseq_count_bit_exact(rl):
    import torch
    from workload import custom_layout
    lay = custom_layout([3, 0, 2, 5, 1], [0, 0, 4, 7, 0], [0, 0, 1, 1, 1], np.ones(5), vocab=50,
                        num_groups=2)
    d = dev_tensors(lay)
    n = torch.zeros(1, dtype=torch.int64, device="cuda")
    s = torch.full((1,), 10, dtype=torch.int64, device="cuda")
    rl.rl_batch_prepare(rl.Head(64, 50), rl.Batch(d["cu"], d["targets"], d["mask"]), n_accum=n,
                        nseq_accum=s)
    torch.cuda.synchronize()
    bk = oracle.bookkeeping(lay.cu_seqlens, lay.mask, lay.targets, 50)
    nonempty = len(set(bk["row_seq"][bk["active"]].tolist()))
    assert int(n.item()) == bk["n_active"] and int(s.item()) == 10 + nonempty == 12
