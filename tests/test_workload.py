"""The seeded generator reproduces the shapes of the paper's workloads
(DESIGN.md §4). Shape/statistics checks only; no method arithmetic here."""
import numpy as np
import pytest

from workload import CONFIGS, make_layout, sub_layout


def test_tiny_layout():
    lay = make_layout(CONFIGS["tiny"], seed=0)
    assert lay.num_seqs == 8 and lay.num_groups == 2
    assert (np.asarray(lay.resp_len) <= 32).all() and (np.asarray(lay.resp_len) >= 1).all()
    assert sorted(set(lay.rewards.tolist())) <= [-5.0, 5.0]
    assert (lay.rewards[4:] == 5.0).all() and (lay.rewards[:4] == 5.0).sum() == 1


@pytest.mark.parametrize("name,lo,hi", [("qwen1.5b", 5e5, 9e5), ("qwen7b", 4.5e6, 7e6)])
def test_reasoning_long_tail(name, lo, hi):
    cfg = CONFIGS[name]
    lay = make_layout(cfg, seed=0)
    r = np.asarray(lay.resp_len)
    assert lo < lay.num_tokens < hi
    assert r.max() <= cfg.lmax and r.min() >= 16
    assert np.median(r) < r.mean()                         # right-skewed
    assert 0.005 < (r > cfg.lmax / 2).mean() < 0.08        # a thin long tail
    g = lay.rewards.reshape(cfg.prompts, cfg.group)
    assert (g[0] == 5).all() and (g[1] == -5).all()


def test_openvla_layout():
    cfg = CONFIGS["openvla"]
    lay = make_layout(cfg, seed=0)
    assert lay.num_seqs == 256 and lay.num_tokens == 256 * 7 * 64 == lay.num_rows
    assert lay.targets.min() >= cfg.vocab - 256
    assert set(np.unique(lay.rewards).tolist()) <= {0.0, 1.0}


def test_sub_layout_rows():
    lay = make_layout(CONFIGS["tiny"], seed=1)
    sub, rows = sub_layout(lay, [3, 1])
    assert sub.num_rows == len(rows)
    np.testing.assert_array_equal(sub.targets, lay.targets[rows])
    assert sub.group_of_seq.tolist() == [lay.group_of_seq[3], lay.group_of_seq[1]]
