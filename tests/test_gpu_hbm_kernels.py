"""The HBM-bound kernels at sizes their single-pass designs must get right:

* H1 (k_validate + k_flags_compact, decoupled look-back over 4096-row tiles)
  bit-exact against the oracle's bookkeeping over the WHOLE Qwen-7B
  mini-batch (6.2M packed rows, ~1500 tiles: long look-back chains) and over
  a batch with more sequences than the kernel caches in shared memory
  (S > 4096: cu_seqlens read from global memory), plus the malformed cases.
* H2 (k_grpo_seg: one pass, segmented by group id) against the oracle with
  groups that are NOT contiguous in sequence order, with the many-groups
  fallback (G > 512), and the split-group statistics path.
* C4 (rl_loss_stats_reduce): rank-order combination of gathered stats.
"""
import numpy as np
import pytest

import oracle
from tests.gpu_util import dev_tensors
from workload import CONFIGS, custom_layout, make_layout

pytestmark = pytest.mark.gpu


def _prepare(rl, lay):
    import torch
    d = dev_tensors(lay)
    R = lay.num_rows
    row_seq = torch.full((max(R, 1),), -7, dtype=torch.int32, device="cuda")
    act = torch.full((max(R, 1),), -7, dtype=torch.int32, device="cuda")
    n = torch.zeros(1, dtype=torch.int64, device="cuda")
    acc = torch.full((1,), 11, dtype=torch.int64, device="cuda")
    rl.rl_batch_prepare(rl.Head(64, lay.vocab), rl.Batch(d["cu"], d["targets"], d["mask"],
                                                        d["err"]), row_seq, act, n, acc)
    torch.cuda.synchronize()
    return (row_seq.cpu().numpy()[:R], act.cpu().numpy(), int(n.item()), int(acc.item()),
            int(d["err"].item()))


def _check(rl, lay):
    row_seq, act, n, acc, err = _prepare(rl, lay)
    ref = oracle.bookkeeping(lay.cu_seqlens, lay.mask, lay.targets, lay.vocab)
    assert n == ref["n_active"] and acc == 11 + ref["n_active"] and err == ref["err"]
    np.testing.assert_array_equal(row_seq, ref["row_seq"])
    np.testing.assert_array_equal(act[:n], ref["active_idx"])


@pytest.mark.slow
def test_h1_whole_qwen7b_minibatch(rl):
    _check(rl, make_layout(CONFIGS["qwen7b"], seed=0))


def test_h1_many_sequences_global_cu(rl):
    rng = np.random.default_rng(31)
    S = 5000                                       # > the 4096 cached in shared memory
    lay = custom_layout(rng.integers(0, 6, S), rng.integers(0, 20, S), np.arange(S) // 10,
                        np.ones(S), vocab=777, num_groups=S // 10)
    lay.targets[::53] = 777                        # some out-of-range targets
    _check(rl, lay)


def test_h1_tile_boundaries(rl):
    """Rows exactly at / around multiples of the 4096-row tile."""
    for R in (4095, 4096, 4097, 8192, 3 * 4096 + 1):
        lens = [R // 3, R // 3, R - 2 * (R // 3)]
        lay = custom_layout([5, 0, 7], [x - p for x, p in zip(lens, [5, 0, 7])], [0, 0, 0],
                            np.ones(3), vocab=100, num_groups=1, seed=R)
        _check(rl, lay)


def test_grpo_segmented_noncontiguous(rl):
    import torch
    rng = np.random.default_rng(8)
    for S, G in ((4096, 256), (777, 300), (3000, 700)):   # 700 > 512: per-group fallback
        gos = rng.integers(0, G, S).astype(np.int32)       # interleaved, not contiguous
        r = rng.choice([-5.0, 5.0], S).astype(np.float32)
        r[gos == 1] = 5.0                                  # zero variance
        gos[5] = -3                                        # invalid id -> A = 0, error bit
        err = torch.zeros(1, dtype=torch.int32, device="cuda")
        adv = torch.full((S,), 9.0, device="cuda")
        rl.rl_grpo_advantage(torch.as_tensor(r, device="cuda"), torch.as_tensor(gos, device="cuda"),
                             G, adv, err_flags=err)
        s = torch.zeros(G, 3, dtype=torch.float64, device="cuda")
        m = torch.zeros(G, 2, dtype=torch.float64, device="cuda")
        rl.rl_grpo_group_stats(torch.as_tensor(r, device="cuda"),
                               torch.as_tensor(gos, device="cuda"), G, s, m)
        torch.cuda.synchronize()
        ref, rerr = oracle.grpo_advantage(r, gos, G)
        a = adv.cpu().double().numpy()
        np.testing.assert_allclose(a, ref, rtol=1e-5, atol=1e-5)
        assert (a[ref == 0] == 0).all() and int(err.item()) == rerr
        ref_s, ref_m, _ = oracle.grpo_group_stats(r, gos, G)
        np.testing.assert_allclose(s.cpu().numpy(), ref_s, rtol=1e-12, atol=1e-9)
        np.testing.assert_array_equal(m.cpu().numpy(), ref_m)


def test_grpo_deterministic(rl):
    import torch
    rng = np.random.default_rng(9)
    S, G = 4096, 256
    gos = torch.as_tensor(np.repeat(np.arange(G), 16).astype(np.int32), device="cuda")
    r = torch.as_tensor(rng.normal(size=S).astype(np.float32), device="cuda")
    outs = []
    for _ in range(3):
        adv = torch.empty(S, device="cuda")
        rl.rl_grpo_advantage(r, gos, G, adv)
        outs.append(adv.cpu())
    assert all(torch.equal(outs[0], o) for o in outs[1:])


def test_loss_stats_reduce_rank_order(rl):
    import torch
    from paper_2509_15965_b200 import rlhead as R
    rng = np.random.default_rng(4)
    parts = []
    for q in range(5):
        parts.append(R.rl_loss_stats(*rng.normal(size=5).tolist(), float(rng.uniform(0, 9)), 0,
                                     *[int(x) for x in rng.integers(0, 1000, 3)]))
    g = torch.frombuffer(bytearray(b"".join(bytes(p) for p in parts)),
                         dtype=torch.uint8).clone().cuda()
    out = rl.new_stats()
    rl.rl_loss_stats_reduce(g, out)
    s = rl.read_stats(out)
    exp = {k: 0.0 for k in ("loss_sum", "ratio_sum", "entropy_sum", "kl_sum", "objective")}
    for p in parts:                           # the same rank-order fp64 sums
        for k in exp:
            exp[k] += getattr(p, k)
    for k, v in exp.items():
        assert s[k] == v, k
    assert s["ratio_max"] == max(p.ratio_max for p in parts)
    for k in ("clip_lo_count", "clip_hi_count", "tokens"):
        assert s[k] == sum(getattr(p, k) for p in parts)
