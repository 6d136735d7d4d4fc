"""Host-side data-parallel logic on CPU: LPT sharding bound, micro-batch
packing, and the world-size-2 gloo reduction path (N all-reduce, dW SUM,
stats SUM/MAX) reproducing the whole-batch oracle."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import oracle
from paper_2509_15965_b200.dp import lpt_shard, pack_micro_batches, shard_layout
from workload import CONFIGS, make_layout, make_tensors_host, sub_layout


@given(st.lists(st.integers(0, 10000), min_size=0, max_size=60), st.integers(1, 8))
@settings(max_examples=200, deadline=None)
def test_lpt_bound_and_cover(weights, world):
    bins, loads = lpt_shard(weights, world)
    items = sorted(i for b in bins for i in b)
    assert items == list(range(len(weights)))
    for r, b in enumerate(bins):
        assert loads[r] == sum(weights[i] for i in b)
    if weights:
        assert loads.max() - loads.min() <= max(weights)   # S:L479-style bound
    assert lpt_shard(weights, world)[0] == bins             # deterministic


@given(st.lists(st.integers(0, 500), min_size=0, max_size=80), st.integers(1, 1000))
@settings(max_examples=200, deadline=None)
def test_micro_batch_packing(rows, budget):
    mbs = pack_micro_batches(rows, budget)
    covered = [s for s0, s1 in mbs for s in range(s0, s1)]
    assert covered == list(range(len(rows)))
    for s0, s1 in mbs:
        tot = sum(rows[s0:s1])
        assert tot <= budget or s1 - s0 == 1


def test_shard_keeps_groups_whole():
    lay = make_layout(CONFIGS["qwen1.5b"], seed=0)
    seen = {}
    for r in range(4):
        seqs, loads = shard_layout(lay, r, 4)
        for s in seqs:
            g = int(lay.group_of_seq[s])
            assert seen.setdefault(g, r) == r
    assert len(seen) == lay.num_groups
    assert loads.max() / loads.mean() < 1.05


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _stats_bytes(d):
    from paper_2509_15965_b200 import rlhead as R
    s = R.rl_loss_stats(d["loss_sum"], d["ratio_sum"], d["entropy_sum"], d["kl_sum"],
                        d["objective"], d["ratio_max"], 0, d["clip_lo_count"],
                        d["clip_hi_count"], d["tokens"])
    return bytes(s)


def _host_combine(gathered, out):
    """Test-side stand-in for rl_loss_stats_reduce on CPU tensors: rank-order
    sums of the gathered structs, max of ratio_max."""
    from paper_2509_15965_b200 import rlhead as R
    n = R.STATS_BYTES
    raw = gathered.numpy().tobytes()
    parts = [R.rl_loss_stats.from_buffer_copy(raw[q * n:(q + 1) * n]) for q in range(len(raw) // n)]
    t = parts[0]
    for v in parts[1:]:
        for k in ("loss_sum", "ratio_sum", "entropy_sum", "kl_sum", "objective", "clip_lo_count",
                  "clip_hi_count", "tokens"):
            setattr(t, k, getattr(t, k) + getattr(v, k))
        t.ratio_max = max(t.ratio_max, v.ratio_max)
    out.copy_(torch_u8(bytes(t)))


def torch_u8(b):
    import torch
    return torch.frombuffer(bytearray(b), dtype=torch.uint8).clone()


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    from paper_2509_15965_b200 import rlhead as R
    from paper_2509_15965_b200.dp import all_reduce_, reduce_stats_
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = CONFIGS["tiny"]
    lay = make_layout(cfg, seed=3)
    H, W = make_tensors_host(cfg, lay.num_rows, seed=3)
    adv_all, _ = oracle.grpo_advantage(lay.rewards, lay.group_of_seq, lay.num_groups)
    seqs, _ = shard_layout(lay, rank, world)
    mine, rows = sub_layout(lay, seqs)
    old = np.zeros(lay.num_rows)
    # C1: N = all-reduce(SUM) of the local active counts
    n = torch.tensor([mine.num_tokens], dtype=torch.int64)
    all_reduce_(n, "sum")
    out = oracle.policy_loss_fwd_bwd(H[rows], W, mine.cu_seqlens, mine.mask, mine.targets,
                                     old[rows], adv_all[seqs], n_global=int(n.item()))
    # C3: dW all-reduce SUM; C4: stats SUM / MAX
    dW = torch.from_numpy(out["dW"].copy())
    all_reduce_(dW, "sum")
    st = torch.frombuffer(bytearray(_stats_bytes(out["stats"])), dtype=torch.uint8).clone()
    reduce_stats_(st, combine=_host_combine)   # one all-gather (C4)
    if rank == 0:
        np.save(os.path.join(out_dir, "dW.npy"), dW.numpy())
        with open(os.path.join(out_dir, "stats.bin"), "wb") as f:
            f.write(st.numpy().tobytes())
        with open(os.path.join(out_dir, "n.txt"), "w") as f:
            f.write(str(int(n.item())))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_world_matches_whole_batch(tmp_path, world):
    """world 4 on the tiny config (2 prompt groups) leaves two ranks with no
    sequences: they must still join every collective with zero contributions."""
    import torch.multiprocessing as mp

    from paper_2509_15965_b200 import rlhead as R
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    cfg = CONFIGS["tiny"]
    lay = make_layout(cfg, seed=3)
    H, W = make_tensors_host(cfg, lay.num_rows, seed=3)
    adv, _ = oracle.grpo_advantage(lay.rewards, lay.group_of_seq, lay.num_groups)
    ref = oracle.policy_loss_fwd_bwd(H, W, lay.cu_seqlens, lay.mask, lay.targets,
                                     np.zeros(lay.num_rows), adv)
    assert int(open(tmp_path / "n.txt").read()) == ref["n_active"]
    np.testing.assert_allclose(np.load(tmp_path / "dW.npy"), ref["dW"], atol=1e-14)
    st = R.rl_loss_stats.from_buffer_copy((tmp_path / "stats.bin").read_bytes())
    assert st.loss_sum == pytest.approx(ref["stats"]["loss_sum"], abs=1e-12)
    assert st.tokens == ref["stats"]["tokens"]
    assert st.ratio_max == pytest.approx(ref["stats"]["ratio_max"], rel=1e-6)


@given(st.integers(1, 300000), st.integers(1, 8))
@settings(max_examples=200, deadline=None)
def test_vocab_shards_cover_and_align(V, P):
    from paper_2509_15965_b200.tp import vocab_shards
    if -(-(-(-V // P)) // 256) * 256 * (P - 1) >= V:      # too many shards for this vocab
        return
    sh = vocab_shards(V, P)
    assert sh[0][0] == 0 and sum(s for _, s in sh) == V
    for (o1, s1), (o2, _) in zip(sh, sh[1:]):
        assert o2 == o1 + s1 and s1 % 256 == 0


def test_shard_layout_split_groups_partition():
    """Split-group sharding assigns single sequences by LPT: a partition of all
    sequences, loads within one sequence's weight of each other."""
    from paper_2509_15965_b200.dp import shard_layout
    from workload import CONFIGS, make_layout
    lay = make_layout(CONFIGS["qwen1.5b"], 0)
    cu = lay.cu_seqlens.astype(np.int64)
    tok = np.add.reduceat(lay.mask.astype(np.int64), cu[:-1])
    for world in (2, 3, 8):
        got = [shard_layout(lay, r, world, split_groups=True, work_weighted=False)
               for r in range(world)]
        seqs = sorted(s for g, _ in got for s in g)
        assert seqs == list(range(lay.num_seqs))
        loads = got[0][1]
        assert loads.max() - loads.min() <= tok.max()
        for r, (g, _) in enumerate(got):
            assert int(tok[g].sum()) == int(loads[r])


def test_shard_work_weighted():
    """Default LPT weights: response tokens x 3 for groups whose rewards differ
    (forward + backward), x 1 for all-equal groups (A = 0: the backward skips
    their rows). Loads are those weights; whole groups; LPT bound holds."""
    from paper_2509_15965_b200.dp import group_has_gradient, shard_layout
    from workload import CONFIGS, make_layout
    lay = make_layout(CONFIGS["qwen7b"], 0)
    cu = lay.cu_seqlens.astype(np.int64)
    tok = np.add.reduceat(lay.mask.astype(np.int64), cu[:-1])
    hg = group_has_gradient(lay)
    assert not hg[0] and not hg[1] and hg.sum() > lay.num_groups // 2   # forced A = 0 groups
    w_g = np.bincount(lay.group_of_seq, weights=tok * np.where(hg[lay.group_of_seq], 3, 1),
                      minlength=lay.num_groups)
    for world in (2, 4, 8):
        got = [shard_layout(lay, r, world) for r in range(world)]
        loads = got[0][1]
        for r, (seqs, _) in enumerate(got):
            assert int(w_g[np.unique(lay.group_of_seq[seqs])].sum()) == int(loads[r])
        assert loads.max() - loads.min() <= w_g.max()


def test_shard_rows_and_dw_output_args():
    """dw_output="shard" (FSDP / ZeRO-2 gradient: owned rows only): the owned
    rows follow the header's
    owner(j) = min(j / ceil(V / P), P - 1) rule and tile [0, V)."""
    from paper_2509_15965_b200.dp import PolicyLossStep, shard_rows
    for V, P in ((152064, 4), (32064, 3), (10, 4), (7, 8)):
        spans = [shard_rows(V, P, q) for q in range(P)]
        assert spans[0][0] == 0 and spans[-1][1] == V
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        rows = -(-V // P)
        for q, (r0, r1) in enumerate(spans):
            assert all(min(j // rows, P - 1) == q for j in range(r0, r1, max(1, (r1 - r0) // 7)))
    with pytest.raises(ValueError):
        PolicyLossStep(None, None, None, dw_output="bogus")
