"""Seeded sweep of small shapes through the CUDA path vs the oracle: hidden
sizes that are one or several 64-wide K blocks, vocabularies that are below,
at and just above the 256-column tile (and V = 1), ragged layouts with empty
sequences, fully masked sequences and fully masked batches."""
import numpy as np
import pytest

import oracle
from tests.gpu_util import dev_tensors, guarded_old_logp, max_rel, rel_fro
from workload import HeadConfig, custom_layout, make_tensors_host

pytestmark = pytest.mark.gpu

CASES = [  # (hidden, vocab, dtype, seed)
    (64, 1, "bf16", 0), (64, 7, "bf16", 1), (128, 255, "bf16", 2), (64, 256, "bf16", 3),
    (192, 257, "bf16", 4), (320, 1000, "bf16", 5), (64, 4099, "bf16", 6), (512, 513, "bf16", 7),
    (16, 33, "f32", 8), (100, 300, "f32", 9), (64, 1, "f32", 10),
]


def _layout(V, seed):
    rng = np.random.default_rng(seed)
    S = int(rng.integers(1, 12))
    plen = rng.integers(0, 40, S)
    rlen = rng.integers(0, 300, S)
    rlen[rng.random(S) < 0.2] = 0                  # sequences without response rows
    lay = custom_layout(plen, rlen, np.arange(S) // 2, rng.choice([-5.0, 5.0], S), vocab=V,
                        num_groups=(S + 1) // 2, seed=seed)
    if seed % 4 == 3:
        lay.mask[:] = 0                            # a fully masked micro-batch
    return lay


@pytest.mark.parametrize("h,V,dtype,seed", CASES, ids=[f"h{c[0]}-V{c[1]}-{c[2]}" for c in CASES])
def test_sweep(rl, h, V, dtype, seed):
    import torch
    lay = _layout(V, seed)
    cfg = HeadConfig("sweep", h, V, 1, 1, 1, dtype, "tiny")
    H, W = make_tensors_host(cfg, max(lay.num_rows, 1), seed=seed)
    H = H[:lay.num_rows]
    adv, _ = oracle.grpo_advantage(lay.rewards, lay.group_of_seq, lay.num_groups)
    adv = adv.astype(np.float32)
    lp = oracle.logprob_fwd(H, W, lay.cu_seqlens, lay.mask, lay.targets)["logp"]
    old = guarded_old_logp(lp, np.random.default_rng(seed), band=1e-2)
    N = max(lay.num_tokens, 1)
    ref = oracle.policy_loss_fwd_bwd(H, W, lay.cu_seqlens, lay.mask, lay.targets, old, adv,
                                     n_global=N)
    d = dev_tensors(lay)
    dev = "cuda"
    R = lay.num_rows
    Hd = H.to(dev) if R else torch.zeros(1, h, dtype=H.dtype, device=dev)
    logp = torch.full((max(R, 1),), 5.0, device=dev)
    gh = torch.full_like(Hd, 3.0)
    gw = torch.zeros(V, h, device=dev)
    st = rl.new_stats()
    rl.rl_policy_loss_fwd_bwd(rl.Head(h, V, dtype), Hd, W.to(dev),
                              rl.Batch(d["cu"], d["targets"], d["mask"], num_rows=R),
                              torch.as_tensor(old, dtype=torch.float32, device=dev),
                              torch.as_tensor(adv, device=dev),
                              rl.LossParams(n_tokens_global=torch.tensor([N], device=dev)),
                              logp, gh, gw, stats=st)
    torch.cuda.synchronize()
    tol_lp, tol_g = (2e-3, 1e-2) if dtype == "bf16" else (1e-5, 2e-5)
    s = rl.read_stats(st)
    assert s["tokens"] == lay.num_tokens
    if R:
        assert np.abs(logp.cpu().double().numpy()[:R] - ref["logp"]).max() <= tol_lp
        dH = gh.cpu().double().numpy()
        assert (dH[lay.mask == 0] == 0).all()
        if np.abs(ref["dH"]).max() > 0:
            assert rel_fro(dH, ref["dH"]) <= tol_g
    dW = gw.cpu().double().numpy()
    if np.abs(ref["dW"]).max() > 0:
        assert rel_fro(dW, ref["dW"]) <= tol_g and max_rel(dW, ref["dW"]) <= max(tol_g, 1e-4)
    else:
        # exact zero in the oracle (V = 1: p = 1, dZ = g(1 - p) = 0); the kernel's
        # p = 2^((z - lse) log2 e) is 1 to fp32 rounding, so dW is zero relative
        # to the scale sum_t |g_t| max|h| it would otherwise have
        scale = np.abs(ref["g"]).sum() * max(float(np.abs(H.double().numpy()).max()), 1.0)
        assert np.abs(dW).max() <= 1e-5 * scale + 1e-30
