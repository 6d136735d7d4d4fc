"""REINFORCE++-style batch-normalised advantage (NEXT-1, DESIGN.md §3 #33) on
the GPU vs the oracle: random batches with and without the group baseline,
the exact-zero degenerate cases, invalid group ids (A = 0 + device error
word read back with rl_read_device_error), and the two-phase multi-rank form
(local statistics, SUM/MAX combine, then A from the combined statistics)."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _run(rl, r, gos, G, **kw):
    import torch
    dev = "cuda"
    rd = torch.as_tensor(r, dtype=torch.float32, device=dev)
    gd = torch.as_tensor(gos, dtype=torch.int32, device=dev)
    adv = torch.full((len(r),), 9.0, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    rl.rl_batch_norm_advantage(rd, gd, G, adv, err_flags=err, **kw)
    code = rl.rl_read_device_error(err)
    return adv.cpu().double().numpy(), code


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("gb", [True, False])
def test_batch_adv_random(rl, seed, gb):
    rng = np.random.default_rng(seed)
    S = int(rng.integers(2, 3000))
    G = int(rng.integers(1, 200))
    gos = rng.integers(0, G, S).astype(np.int32)
    r = (rng.choice([-5.0, 5.0], S) if seed % 2 else rng.normal(0, 3, S)).astype(np.float32)
    for unbiased in (True, False):
        A, code = _run(rl, r, gos, G, group_baseline=gb, unbiased=unbiased)
        Ao, err = oracle.batch_norm_advantage(r, gos, G, group_baseline=gb, unbiased=unbiased)
        assert code == err == 0
        assert np.all(np.abs(A - Ao) <= 1e-5 * np.maximum(1.0, np.abs(Ao)))


def test_batch_adv_degenerate_invalid(rl):
    r = np.array([0.7] * 7 + [5, 5, 5], dtype=np.float32)
    gos = np.array([0] * 7 + [1] * 3, dtype=np.int32)
    A, code = _run(rl, r, gos, 2, group_baseline=True)
    assert code == 0 and (A == 0.0).all()
    A, _ = _run(rl, np.full(6, 2.5, np.float32), np.zeros(6, np.int32), 1, group_baseline=False)
    assert (A == 0.0).all()
    r = np.array([5, -5, 5, -5, 100.0], dtype=np.float32)
    gos = np.array([0, 0, 1, 1, 9], dtype=np.int32)
    A, code = _run(rl, r, gos, 2, group_baseline=False, unbiased=False, eps=0.0)
    Ao, err = oracle.batch_norm_advantage(r, gos, 2, group_baseline=False, unbiased=False, eps=0.0)
    assert code == err == rl.RL_DEVERR_GROUP
    assert A[4] == 0.0 and np.abs(A - Ao).max() <= 1e-6


def test_batch_adv_two_phase_matches_whole(rl):
    import torch
    dev = "cuda"
    rng = np.random.default_rng(11)
    S, G = 1024, 64
    gos = np.repeat(np.arange(G), S // G).astype(np.int32)
    r = rng.choice([-5.0, 5.0], S).astype(np.float32)
    whole, _ = _run(rl, r, gos, G, group_baseline=True)
    # two "ranks", whole groups each (group sums local), batch stats combined
    halves = [slice(0, S // 2), slice(S // 2, S)]
    stats = []
    for h in halves:
        st = torch.empty(5, dtype=torch.float64, device=dev)
        rl.rl_batch_norm_advantage(torch.as_tensor(r[h], device=dev),
                                   torch.as_tensor(gos[h], device=dev), G, None,
                                   group_baseline=True, batch_stats_out=st)
        stats.append(st)
    comb = torch.cat([stats[0][:3] + stats[1][:3], torch.maximum(stats[0][3:], stats[1][3:])])
    out = []
    for h in halves:
        a = torch.empty(S // 2, device=dev)
        rl.rl_batch_norm_advantage(torch.as_tensor(r[h], device=dev),
                                   torch.as_tensor(gos[h], device=dev), G, a,
                                   group_baseline=True, batch_stats_in=comb)
        out.append(a.cpu().double().numpy())
    A2 = np.concatenate(out)
    Ao, _ = oracle.batch_norm_advantage(r, gos, G, group_baseline=True)
    assert np.abs(A2 - Ao).max() <= 1e-5 * max(1.0, np.abs(Ao).max())
    assert np.abs(A2 - whole).max() <= 1e-6
