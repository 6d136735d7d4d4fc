"""The C-ABI calls are CUDA-graph capturable (no allocation, no host sync,
stream-ordered): a whole mini-batch step captured once and replayed gives the
same result as eager execution (bit-identical: same kernels, same order)."""
import pytest

from workload import HeadConfig, make_layout, make_tensors_host

pytestmark = pytest.mark.gpu


def test_step_graph_replay_matches_eager(rl):
    import torch
    from paper_2509_15965_b200.dp import PolicyLossStep, device_batch
    cfg = HeadConfig("small-bf16", 192, 1000, 6, 4, 96, "bf16", "reasoning")
    lay = make_layout(cfg, seed=61)
    H, W = make_tensors_host(cfg, lay.num_rows, seed=61)
    dev = "cuda"
    Hd, Wd = H.to(dev), W.to(dev)
    db = device_batch(lay, 2048, device=dev)
    old = torch.zeros(lay.num_rows, device=dev)
    gh = torch.empty_like(Hd)
    step = PolicyLossStep(rl.Head(cfg.hidden, cfg.vocab), Wd, db)
    step.run(Hd, old, gh)                       # eager (also sizes the workspaces)
    torch.cuda.synchronize()
    gw_eager = step.grad_w.clone()
    st_eager = step.stats.clone()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            step.run(Hd, old, gh)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(step.grad_w, gw_eager)
    assert torch.equal(step.stats, st_eager)
