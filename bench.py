#!/usr/bin/env python
"""Benchmark of the GRPO policy-loss head: fwd+bwd tokens/s on 1..8 B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config qwen7b]
    torchrun --nproc-per-node N bench.py --gpus N ...     (one rank per GPU)
    python bench.py --impl reference ...                  (CPU float64 oracle arm)

A "step" is one GRPO mini-batch of the config (BASELINE.json configs[3],
Qwen-7B head: 128 prompts x G=16, long-tailed responses up to 16k tokens,
~5.6M masked tokens) through the whole hot path: N all-reduce, GRPO
advantages, every micro-batch through rl_policy_loss_fwd_bwd (projection,
online LSE, loss, dZ recompute, dH, dW), dW all-reduce. Strong scaling: the
mini-batch is fixed and its prompt groups are LPT-sharded over the ranks.
value = masked response tokens of the mini-batch / device time per step
(CUDA events, max over ranks). Inputs (44 GB of hidden rows) exceed L2.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "policy-loss fwd+bwd tokens/s at 1/2/4/8 B200; % bf16 tensor-core peak"



# micro-batch row budget per head, from same-box A/B runs (profiles/r2/SUMMARY.md §3)
MB_ROWS_DEFAULT = {"qwen1.5b": 32768, "openvla": 32768}
# sequence-level DP sharding per head (N > 1): OpenVLA's few large groups leave whole-group
# LPT shards 2.6% apart at 4 GPUs (profiles/r2/r2_vla: +3.1% with split groups)
SPLIT_GROUPS_DEFAULT = {"openvla": 1}

def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="qwen7b")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--mb-rows", type=int, default=None,
                   help="rows per micro-batch; default per head (MB_ROWS_DEFAULT): 16k for "
                        "the Qwen-7B/32B heads (same-box: 24k -1.4%%, 32k -2.6%%, 8k -2.6%%), "
                        "32k for Qwen-1.5B and OpenVLA (h <= 4096 and short steps: +2.0%% / "
                        "+1.4%% over 16k; profiles/r2/SUMMARY.md)")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--max-mb", type=int, default=0, help="debug: first micro-batches only")
    p.add_argument("--mb-offset", type=int, default=0,
                   help="debug, with --max-mb: start at this micro-batch (the first ones hold "
                        "the forced A = 0 groups)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-sample-tokens", type=int, default=512,
                   help="masked tokens per --impl reference step")
    p.add_argument("--cpu-baseline-tokens", type=int, default=1536,
                   help="masked tokens of the cpu_baseline leg (about 10-30 s of oracle work)")
    p.add_argument("--cpu-1t-tokens", type=int, default=64,
                   help="masked tokens of the cpu_baseline leg's 1-thread run (SURVEY M.7)")
    p.add_argument("--collective", default="nvls", choices=["nvls", "symm", "nccl"],
                   help="N>1 dW reduction: reduce-scatter fused into the last dW GEMM epilogue "
                        "+ NVLink all-gather (symm); NVLS in-switch sum after the last dW GEMM "
                        "(nvls); or NCCL all-reduce / reduce-scatter (nccl)")
    p.add_argument("--dw-output", default="full", choices=["full", "shard"],
                   help="N>1: every rank ends with the whole reduced dW (full), or only its "
                        "owned rows (shard: FSDP / ZeRO-2 gradient reduce-scatter, no "
                        "broadcast / all-gather)")
    p.add_argument("--split-groups", type=int, default=None,
                   help="N>1: LPT over single sequences (group statistics all-reduced) "
                        "instead of whole groups -- finer balance for few large groups; "
                        "default per head (SPLIT_GROUPS_DEFAULT: on for OpenVLA, whose 4-GPU "
                        "whole-group shards differ by 2.6%%)")
    p.add_argument("--pipeline", type=int, default=0,
                   help="1: two-stream micro-batch pipeline (bwd(i) beside fwd(i+1))")
    p.add_argument("--phases", action="store_true",
                   help="per-phase step times (always on for N > 1)")
    p.add_argument("--no-aux", action="store_true",
                   help="skip the auxiliary lines (forward-only path, HBM kernels)")
    a = p.parse_args()
    if a.mb_rows is None:
        a.mb_rows = MB_ROWS_DEFAULT.get(a.config, 16384)
    if a.split_groups is None:
        a.split_groups = SPLIT_GROUPS_DEFAULT.get(a.config, 0)
    return a


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return dict(hbm=float(d["hbm_gbs"]), bf16=float(d["bf16_tflops"]),
                    bf16_sus=float(d["bf16_tflops_sustained"]), src="measured")
    except Exception:
        return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="fallback")


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.index)], stdout=open(self.path, "w"),
                stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
                pw.append(float(f[3]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": []}
        loaded = [s for s, p in zip(sm, pw) if p > 300.0] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


_W64 = {}


def _oracle_weight(cfg, seed):
    """The config's W as float64 (exact bf16/fp32 values), built once outside
    any timed region (the conversion is a fixed cost that does not scale with
    the sampled token count)."""
    import torch

    from workload import make_tensors_torch
    key = (cfg.name, seed)
    if key not in _W64:
        _, W = make_tensors_torch(cfg, 0, seed=seed, hidden=False)
        _W64[key] = W.to(torch.float64).numpy()
    return _W64[key]


def _blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 0) for i in threadpool_info()] or [0])
    except Exception:
        return 0


def cpu_baseline(cfg, layout, seed, tokens, threads=None):
    """The oracle as it stands on this host, on a bounded sample: the first
    `tokens` response rows of sequence 0 (with its prompt rows), fwd+bwd.
    W is converted to float64 before the clock starts; threads=k limits the
    BLAS pool to k threads for the timed call."""
    import contextlib

    import oracle
    from workload import make_tensors_torch, sub_layout
    sub, _ = sub_layout(layout, [0])
    P = int(sub.prompt_len[0]) if sub.prompt_len is not None else 0
    R = min(sub.num_rows, P + tokens)
    cu = np.array([0, R], dtype=np.int32)
    mask, targets = sub.mask[:R], sub.targets[:R]
    H, _ = make_tensors_torch(cfg, R, seed=seed, weight=False)
    W64 = _oracle_weight(cfg, seed)
    old = np.zeros(R)
    adv = np.array([1.0])
    lim = contextlib.nullcontext()
    if threads is not None:
        from threadpoolctl import threadpool_limits
        lim = threadpool_limits(limits=threads)
    with lim:
        blas = _blas_threads()
        t0 = time.perf_counter()
        out = oracle.policy_loss_fwd_bwd(H, W64, cu, mask, targets, old, adv)
        dt = time.perf_counter() - t0
    n = int(out["n_active"])
    return {"value": n / dt, "unit": "tokens/s", "cores": blas or os.cpu_count(),
            "host_cpus": os.cpu_count(), "blas_threads": blas, "kind": "oracle", "seconds": dt,
            "sample": f"{n} masked tokens of sequence 0 ({cfg.name}, fwd+bwd incl. dW [V,h] fp64)"}


def cpu_tiny_end_to_end(seed=0):
    """the tiny config (BJ configs[0]) through the whole oracle path
    end to end: bookkeeping, GRPO advantages, fwd+bwd of the full batch."""
    import oracle
    from workload import CONFIGS, make_layout, make_tensors_host
    cfg = CONFIGS["tiny"]
    lay = make_layout(cfg, seed=seed)
    H, W = make_tensors_host(cfg, lay.num_rows, seed=seed)
    t0 = time.perf_counter()
    adv, _ = oracle.grpo_advantage(lay.rewards, lay.group_of_seq, lay.num_groups)
    out = oracle.policy_loss_fwd_bwd(H, W, lay.cu_seqlens, lay.mask, lay.targets,
                                     np.zeros(lay.num_rows), adv)
    dt = time.perf_counter() - t0
    return {"workload": "tiny (2 prompts x G=4, h=64, V=1000), whole batch",
            "tokens": int(out["n_active"]), "seconds": round(dt, 4),
            "value": round(int(out["n_active"]) / dt, 1), "unit": "tokens/s"}


def cpu_baseline_m7(cfg, layout, seed, tokens, tokens_1t, tokens_global):
    """all host threads on `tokens`, 1 thread on `tokens_1t`,
    the tiny config end to end, and the full config's time extrapolated from
    the all-thread per-token rate (labelled as such)."""
    cb = cpu_baseline(cfg, layout, seed, tokens)
    one = cpu_baseline(cfg, layout, seed, tokens_1t, threads=1)
    cb["one_thread"] = {"value": one["value"], "seconds": round(one["seconds"], 3),
                        "sample": one["sample"], "cores": 1}
    cb["tiny_end_to_end"] = cpu_tiny_end_to_end(seed)
    cb["full_config_extrapolated"] = {
        "tokens": int(tokens_global), "seconds": round(tokens_global / cb["value"], 1),
        "hours": round(tokens_global / cb["value"] / 3600.0, 2),
        "note": "extrapolated: full mini-batch tokens / the all-thread sample's tokens/s "
                "(not run)"}
    return cb


def workload_name(cfg):
    return (f"{cfg.name} head (h={cfg.hidden}, V={cfg.vocab}), {cfg.prompts} prompts x "
            f"G={cfg.group}, responses <= {cfg.lmax}")


def run_reference(args, cfg):
    """--impl reference: the CPU float64 oracle, timed on this host."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from workload import make_layout
    layout = make_layout(cfg, seed=args.seed)
    for _ in range(args.warmup):
        cpu_baseline(cfg, layout, args.seed, 8)
    vals = []
    for _ in range(args.steps):
        vals.append(cpu_baseline(cfg, layout, args.seed, args.cpu_sample_tokens))
    v = statistics.median([x["value"] for x in vals])
    cb = dict(vals[-1])
    cb["value"] = v
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * statistics.median([x["seconds"] for x in vals]),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(cfg), "sample": cb["sample"]},
            "gpus_used": 0, "host_only": "the CPU float64 oracle on the host cores",
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def relaunch_under_torchrun(args):
    """`python bench.py --gpus N` (N > 1) without a torchrun environment:
    re-exec as one rank per GPU (the driver's own launch form) and pass the
    ranks' output and exit code through."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    print(f"[bench] --gpus {args.gpus} without WORLD_SIZE: relaunching under torchrun",
          file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def main():
    args = parse()
    from workload import CONFIGS, make_layout, make_tensors_torch, ratio_noise, sub_layout
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args)
    if int(os.environ.get("WORLD_SIZE", "1")) != args.gpus:
        print(f"[bench] --gpus {args.gpus} but WORLD_SIZE={os.environ.get('WORLD_SIZE')}: "
              "launch one rank per GPU (torchrun --nproc-per-node N ... --gpus N)",
              file=sys.stderr, flush=True)
        return 2

    import torch
    import torch.distributed as dist

    import paper_2509_15965_b200 as rl
    from paper_2509_15965_b200.dp import PolicyLossStep, device_batch, shard_layout

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    layout = make_layout(cfg, seed=args.seed)
    split = bool(args.split_groups) and world > 1
    seqs, loads = shard_layout(layout, rank, world, split_groups=split)
    mine, _ = sub_layout(layout, seqs)
    db = device_batch(mine, args.mb_rows, device=dev, global_groups=split)
    if args.max_mb:  # debug: the sequences of max_mb micro-batches only
        i0 = min(args.mb_offset, len(db.mbs) - 1)
        s_beg = db.mbs[i0][0]
        s_end = db.mbs[min(i0 + args.max_mb, len(db.mbs)) - 1][1]
        mine, _ = sub_layout(mine, np.arange(s_beg, s_end))
        db = device_batch(mine, args.mb_rows, device=dev, global_groups=split)
    _, W = make_tensors_torch(cfg, 0, seed=args.seed, device=dev, hidden=False)
    H, _ = make_tensors_torch(cfg, mine.num_rows, seed=args.seed + 7919 * (rank + 1), device=dev,
                              weight=False)
    head = rl.Head(cfg.hidden, cfg.vocab, cfg.dtype)
    max_mb = max(r1 - r0 for _, _, r0, r1, _ in db.mbs)

    # old log-probs from the inference-worker call + delta ~ N(0, 0.05^2) (M.2)
    old = torch.empty(max(mine.num_rows, 1), dtype=torch.float32, device=dev)
    ws = rl.Workspace(dev)
    for (s0, s1, r0, r1, cu_mb) in db.mbs:
        rl.rl_logprob_fwd(head, H[r0:r1], W, rl.Batch(cu_mb, db.targets[r0:r1], db.mask[r0:r1],
                                                      num_rows=r1 - r0), old[r0:r1], ws=ws)
    old += torch.as_tensor(ratio_noise(old.shape[0], args.seed + rank), dtype=torch.float32,
                           device=dev)
    del ws
    collective = args.collective if world > 1 else "none"
    try:
        step = PolicyLossStep(head, W, db, group=group,
                              collective=collective if collective in ("symm", "nvls")
                              else "nccl",
                              pipeline=bool(args.pipeline), split_groups=split,
                              dw_output=args.dw_output if world > 1 else "full")
    except Exception as e:  # symmetric memory unavailable: NCCL all-reduce instead
        print(f"[bench] collective={collective} unavailable ({e}); using nccl", file=sys.stderr)
        collective = "nccl"
        step = PolicyLossStep(head, W, db, group=group, collective="nccl",
                              pipeline=bool(args.pipeline), split_groups=split,
                              dw_output=args.dw_output if world > 1 else "full")
    gh = torch.empty(max_mb, cfg.hidden, dtype=H.dtype, device=dev)
    tokens_local = int(sum(int(mine.mask[r0:r1].sum()) for _, _, r0, r1, _ in db.mbs))
    tok_t = torch.tensor([tokens_local], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(tok_t)
    tokens_global = int(tok_t.item())

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ------------------------------------------------------ device-timed run
    for i in range(args.warmup):
        if i == args.warmup - 1:
            nw = rl.rl_launch_count()
        step.run(H, old, gh)
    per_step_launches = rl.rl_launch_count() - nw
    barrier()
    clk = Clocks(local)
    clk.start()
    # every launch of the timed steps is traced (the roofline's time is the sum
    # over ALL dominant-kernel launches; checked against rl_launch_count below)
    tr = rl.Trace(per_step_launches * args.steps + 4096).start()
    n0 = rl.rl_launch_count()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    e0, e1 = evs[0], evs[-1]
    barrier()
    e0.record()
    for i in range(args.steps):
        step.run(H, old, gh)
        evs[i + 1].record()
    barrier()
    launches = rl.rl_launch_count() - n0
    tr.stop()
    clocks = clk.stop()
    if len(tr.kinds) != launches:
        raise RuntimeError(f"trace holds {len(tr.kinds)} of {launches} launches: roofline invalid")
    ms = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms_per_step = float(ms.item())
    value = tokens_global / (ms_per_step / 1e3)
    per_step = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]   # this rank

    # per-phase device time of one extra (untimed) step, max over ranks: the
    # fixed costs that decide strong scaling (zero dW, N all-reduce, advantage,
    # micro-batches, dW reduction, stats all-gather)
    phases = None
    if world > 1 or args.phases:
        step.timer.enabled = True
        step.run(H, old, gh)
        torch.cuda.synchronize()
        ph = step.timer.ms()
        step.timer.enabled = False
        keys = ["zero_dw", "count_allreduce", "advantage", "micro_batches", "dw_reduce",
                "stats_gather"]
        t = torch.tensor([ph.get(k, 0.0) for k in keys], dtype=torch.float64, device=dev)
        t_min = t.clone()
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dist.all_reduce(t_min, op=dist.ReduceOp.MIN)
        phases = {k: round(float(v), 3) for k, v in zip(keys, t.tolist())}
        if world > 1:   # max - min of a phase: the slowest rank's lead (imbalance / waiting)
            phases["min_over_ranks"] = {k: round(float(v), 3) for k, v in zip(keys, t_min.tolist())}
        phases["note"] = "one extra untimed step, ms per phase, max over ranks"

    # roofline of the dominant kernel (GEMM kinds: 2hV flops per token per launch)
    pk = peaks()
    kinds = tr.by_kind()
    per_kind = {k: {"launches": c, "ms_total": round(t, 3)} for k, (c, t) in kinds.items()}
    units = rl.rlhead.GEMM_FLOP_UNITS        # a fused dH+dW launch does 2 x 2hV per token
    gemm = {k: kinds[k] for k in units if k in kinds}
    dom = max(gemm, key=lambda k: gemm[k][1])
    # rows each GEMM kind runs over: every active row for the forward (and the
    # recompute); in skip mode the backward GEMMs (dH, dW) only see the rows with
    # dL/dlogp != 0 -- here all tokens but those of A = 0 groups and the clipped
    # ones (token-mean loss, no KL in the bench)
    st_loc = rl.read_stats(step.stats_local)
    adv_np = step.adv[:mine.num_seqs].cpu().numpy()
    cu_np = mine.cu_seqlens.astype(np.int64)
    seq_tok = np.add.reduceat(mine.mask.astype(np.int64), cu_np[:-1]) if mine.num_rows else \
        np.zeros(0, np.int64)
    seq_tok = np.where(cu_np[1:] > cu_np[:-1], seq_tok, 0)
    grad_rows = int(seq_tok[adv_np != 0].sum()) - st_loc["clip_lo_count"] - st_loc["clip_hi_count"]
    skip = "dz_from_q" in kinds and os.environ.get("RLHEAD_BWD_SKIP", "1") != "0"
    rows_of = {"gemm_lse": tokens_local, "gemm_dz": tokens_local,
               "gemm_dh": grad_rows if skip else tokens_local,
               "gemm_dw": grad_rows if skip else tokens_local,
               "gemm_dhdw": grad_rows if skip else tokens_local}
    dom_flops = units[dom] * 2.0 * cfg.hidden * cfg.vocab * rows_of[dom] * args.steps
    achieved = dom_flops / (gemm[dom][1] / 1e3) / 1e12
    # executed tensor work per token from the GEMM launches actually traced:
    # 8hV with the dZ recompute GEMM, 6hV in q mode, (2 + 4 f) hV in skip mode
    # (f = share of tokens with a non-zero gradient)
    exec_units = sum(units[k] * gemm[k][0] * rows_of[k] for k in gemm) / \
        max(gemm["gemm_lse"][0] * tokens_local, 1)
    step_tflops_exec = exec_units * 2.0 * cfg.hidden * cfg.vocab * value / 1e12
    step_tflops_alg = 6.0 * cfg.hidden * cfg.vocab * value / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            tpt = json.load(open(prof)).get(cfg.name, {}).get(dom)
            if tpt:
                traffic = tpt * rows_of[dom] / max(gemm[dom][0] / args.steps, 1)
        except Exception:
            traffic = None
    roof = {"bound": "tensor", "kernel": f"k_tc_gemm[{dom}]", "achieved": round(achieved, 1),
            "peak": pk["bf16_sus"], "unit": "TFLOP/s", "frac": round(achieved / pk["bf16_sus"], 4),
            "traffic": traffic, "peak_kind": f"bf16 sustained ({pk['src']})",
            "frac_of_burst": round(achieved / pk["bf16"], 4),
            "executed_flops_per_token": f"{exec_units:.4g} x 2hV",
            "backward_rows": {"tokens": tokens_local, "with_gradient": grad_rows,
                              "skip_zero_gradient_rows": skip},
            "step_executed_tflops": round(step_tflops_exec / world, 1),
            "step_executed_frac_burst": round(step_tflops_exec / world / pk["bf16"], 4),
            "step_algorithmic_frac_burst": round(step_tflops_alg / world / pk["bf16"], 4)}
    if skip:
        roof["algorithmic_note"] = ("6hV per token counts the dH/dW work of the rows whose "
                                    "dL/dlogp is exactly 0, which skip mode does not execute; "
                                    "step_executed_* is the hardware's share")

    # ------------------------------------ auxiliary measurements (M.1, M.4)
    aux = None
    if not args.no_aux:
        aux = run_aux(rl, head, H, W, db, mine, step, kinds, tokens_local, tokens_global, cfg,
                      pk, world, args.steps)

    # ------------------------------------------------ end-to-end (host data)
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, rl, step, db, mine, H, old, gh, dev, world, tokens_global)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_m7(cfg, layout, args.seed, args.cpu_baseline_tokens,
                              args.cpu_1t_tokens, tokens_global)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": world,
            "gpus_active": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": cfg.dtype,
            "step_ms_rank0": {"median": round(statistics.median(per_step), 3),
                              "min": round(min(per_step), 3), "max": round(max(per_step), 3)},
            "data": "synthetic",
            "config": {"workload": workload_name(cfg),
                       "global_batch_tokens": tokens_global, "micro_batch_rows": args.mb_rows,
                       "micro_batches_per_rank": len(db.mbs), "parallelism": f"dp{world}",
                       "dw_collective": collective, "pipeline": bool(args.pipeline),
                       "dw_output": args.dw_output if world > 1 else "local",
                       "sharding": "sequences (split groups)" if split else "whole groups",
                       "l2": "inputs > L2 (hidden rows of the mini-batch ~ "
                             f"{mine.num_rows * cfg.hidden * 2 / 1e9:.1f} GB per rank)",
                       "lpt_load_max_over_mean": round(float(loads.max() / loads.mean()), 4),
                       "partial": bool(args.max_mb)},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clocks, "kernels": per_kind, "phases_ms": phases, "aux": aux,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_aux(rl, head, H, W, db, mine, step, kinds, tokens_local, tokens_global, cfg, pk, world,
            steps):
    """SURVEY M.1/M.4 side numbers (not the headline):
    * fwd_only: the inference-worker path (rl_logprob_fwd over every micro-
      batch: H1 + H3 + H4), tokens/s, device time, max over ranks;
    * bookkeeping: H1 (rl_batch_prepare) once over the rank's whole mini-batch
      (all packed rows in one call), algorithmic bytes / time vs the HBM peak;
    * merge: the H4-merge + H5 kernel inside the timed steps (live per-launch
      events), algorithmic bytes 12 n_vt + 30 per active row."""
    import torch
    import torch.distributed as dist
    dev = H.device

    def max_ms(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    out = {}
    ws = step.ws
    lp = step.logp
    mb0 = db.mbs[0]
    rl.rl_logprob_fwd(head, H[mb0[2]:mb0[3]], W, rl.Batch(mb0[4], db.targets[mb0[2]:mb0[3]],
                      db.mask[mb0[2]:mb0[3]], num_rows=mb0[3] - mb0[2]), lp[mb0[2]:mb0[3]], ws=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for (s0, s1, r0, r1, cu_mb) in db.mbs:
        rl.rl_logprob_fwd(head, H[r0:r1], W, rl.Batch(cu_mb, db.targets[r0:r1], db.mask[r0:r1],
                                                      num_rows=r1 - r0), lp[r0:r1], ws=ws)
    e1.record()
    torch.cuda.synchronize()
    ms = max_ms(e0.elapsed_time(e1))
    fwd_tflops = 2.0 * cfg.hidden * cfg.vocab * tokens_global / (ms / 1e3) / 1e12 / world
    out["fwd_only"] = {"metric": "logprob fwd tokens/s (inference worker)",
                       "value": round(tokens_global / (ms / 1e3), 1), "unit": "tokens/s",
                       "ms": round(ms, 3), "tflops_per_gpu": round(fwd_tflops, 1),
                       "frac_of_burst": round(fwd_tflops / pk["bf16"], 4)}
    # H1 over the whole local mini-batch
    R = mine.num_rows
    S = int(db.cu.shape[0]) - 1
    row_seq = torch.empty(max(R, 1), dtype=torch.int32, device=dev)
    act = torch.empty(max(R, 1), dtype=torch.int32, device=dev)
    na = torch.zeros(1, dtype=torch.int64, device=dev)
    wsp = rl.Workspace(dev)
    b = rl.Batch(db.cu, db.targets, db.mask)
    rl.rl_batch_prepare(head, b, row_seq=row_seq, active_idx=act, n_active=na, ws=wsp)
    torch.cuda.synchronize()
    reps = 5
    e0.record()
    for _ in range(reps):
        rl.rl_batch_prepare(head, b, row_seq=row_seq, active_idx=act, n_active=na, ws=wsp)
    e1.record()
    torch.cuda.synchronize()
    ms = max_ms(e0.elapsed_time(e1) / reps)
    T = int(mine.num_tokens)
    nbytes = R * (4 + 1 + 4) + 4 * (S + 1) + 4 * T   # targets+mask in, row_seq out, cu, active out
    gbs = nbytes / (ms / 1e3) / 1e9
    out["bookkeeping"] = {"rows": R, "ms": round(ms, 4), "bytes": nbytes, "gbs": round(gbs, 1),
                          "frac_hbm": round(gbs / pk["hbm"], 4),
                          "note": "H1 once over the rank's whole mini-batch; bytes algorithmic"}
    del wsp
    if "merge" in kinds:
        n, t = kinds["merge"]
        n_vt = -(-cfg.vocab // 256)
        nb = (12 * n_vt + 30) * tokens_local * steps
        g = nb / (t / 1e3) / 1e9
        out["merge"] = {"launches": n, "ms_per_launch": round(t / max(n, 1), 4),
                        "gbs": round(g, 1), "frac_hbm": round(g / pk["hbm"], 4),
                        "bytes_per_token": 12 * n_vt + 30}
    if world == 1 and cfg.dtype == "bf16":
        out["torch_eager_reference"] = torch_reference(H, W, db, mine, step, cfg)
    return out


def torch_reference(H, W, db, mine, step, cfg, n_mb=2, chunk=4096):
    """A library baseline for context (not the headline, not the oracle): the
    same micro-batch step written the usual way in PyTorch on the GPU --
    cuBLAS bf16 logits materialised per row chunk, log-softmax, gather, the
    clipped surrogate, autograd for dL/dH and dL/dW (bf16 parameter grads) --
    over the first `n_mb` micro-batches, CUDA-event timed after a warm-up."""
    import torch
    dev = H.device
    Wp = W.detach().clone().requires_grad_(True)
    old = step.logp.detach().clone() + 0.01       # any fixed old log-probs

    def one(r0, r1, s0, s1):
        mask = db.mask[r0:r1].bool()
        rows = torch.nonzero(mask).squeeze(1)
        if rows.numel() == 0:
            return 0
        lens = torch.as_tensor(db.mbs_cu_np[s0 + 1:s1 + 1] - db.mbs_cu_np[s0:s1], device=dev)
        seq = torch.repeat_interleave(torch.arange(s1 - s0, device=dev), lens)[rows]
        A = step.adv[s0:s1][seq]
        N = float(db.num_tokens)
        for c0 in range(0, rows.numel(), chunk):
            rr = rows[c0:c0 + chunk]
            h = H[r0:r1][rr].detach().requires_grad_(True)
            z = (h @ Wp.t()).float()
            logp = torch.log_softmax(z, dim=-1).gather(1, db.targets[r0:r1][rr].long()[:, None])[:, 0]
            r = torch.exp(torch.clamp(logp - old[r0:r1][rr], -20, 20))
            a = A[c0:c0 + chunk]
            loss = torch.maximum(-a * r, -a * torch.clamp(r, 0.8, 1.2)).sum() / N
            loss.backward()
        return rows.numel()

    mbs = db.mbs[:n_mb]
    db.mbs_cu_np = db.cu.cpu().numpy().astype(np.int64)
    for (s0, s1, r0, r1, _) in mbs[:1]:
        one(r0, r1, s0, s1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tok = 0
    for (s0, s1, r0, r1, _) in mbs:
        tok += one(r0, r1, s0, s1)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    del Wp
    torch.cuda.empty_cache()
    return {"value": round(tok / (ms / 1e3), 1), "unit": "tokens/s", "tokens": tok,
            "ms": round(ms, 3), "micro_batches": len(mbs), "row_chunk": chunk,
            "what": "PyTorch eager bf16 on this GPU: cuBLAS logits materialised per chunk, "
                    "log_softmax, clipped surrogate, autograd dH/dW (bf16 grads); context only"}


def run_e2e(args, rl, step, db, mine, H, old, gh, dev, world, tokens_global):
    """Same metric through the public API with HOST buffers on both sides.
    Every step copies its inputs from pinned host memory (hidden streamed per
    micro-batch on a copy stream, double-buffered, the next step's first
    micro-batches prefetched under this step's last ones) and reads its
    results back on a second copy stream: each micro-batch's log-probs (the
    inference worker's output) as soon as its call is enqueued, this
    rank's slab of the reduced dW (the rows a sharded optimizer owns) and the
    loss statistics at the end of the step."""
    import torch
    import torch.distributed as dist
    R = mine.num_rows
    host_H = torch.empty(H.shape, dtype=H.dtype, pin_memory=True)
    host_H.copy_(H)
    small = dict(targets=db.targets, mask=db.mask, cu=db.cu, gos=db.gos, rewards=db.rewards,
                 old=old)
    small.update({f"cu_mb{i}": mb[4] for i, mb in enumerate(db.mbs)})
    host_small = {k: v.detach().to("cpu").pin_memory() for k, v in small.items()}
    dev_small = {k: torch.empty_like(v, device=dev) for k, v in host_small.items()}
    max_mb = gh.shape[0]
    bufs = [torch.empty(max_mb, H.shape[1], dtype=H.dtype, device=dev) for _ in range(2)]
    copy_s = torch.cuda.Stream(device=dev)
    d2h_s = torch.cuda.Stream(device=dev)
    ready = [torch.cuda.Event() for _ in range(2)]
    freed = [torch.cuda.Event() for _ in range(2)]
    comp = torch.cuda.current_stream()
    stats_host = torch.empty(rl.rlhead.STATS_BYTES, dtype=torch.uint8, pin_memory=True)
    logp_host = torch.empty(max(R, 1), dtype=torch.float32, pin_memory=True)
    rank = dist.get_rank() if world > 1 else 0
    V = step.grad_w.shape[0]
    slab = -(-V // world)
    v0, v1 = min(rank * slab, V), min((rank + 1) * slab, V)
    dw_host = torch.empty((v1 - v0, step.grad_w.shape[1]), dtype=torch.float32, pin_memory=True)
    h2d = sum(v.numel() * v.element_size() for v in host_small.values()) + \
        sum((r1 - r0) * H.shape[1] * H.element_size() for _, _, r0, r1, _ in db.mbs)
    d2h = 4 * sum(r1 - r0 for _, _, r0, r1, _ in db.mbs) + dw_host.numel() * 4 + \
        rl.rlhead.STATS_BYTES

    n_mb = len(db.mbs)
    # micro-batches are numbered c = step * n_mb + i across the steps of one run
    # so the copy of the next step's first micro-batches overlaps this step's
    # last ones (a training loop prefetching its next batch); buffer = c % 2.
    state = {"base": 0, "total": 0, "issued": 0}

    def issue_copy(c):
        _, _, r0, r1, _ = db.mbs[c % n_mb]
        with torch.cuda.stream(copy_s):
            copy_s.wait_event(freed[c % 2])
            bufs[c % 2][:r1 - r0].copy_(host_H[r0:r1], non_blocking=True)
            ready[c % 2].record(copy_s)
        state["issued"] = c + 1

    def hidden_for_mb(i):
        c = state["base"] + i
        comp.wait_event(ready[c % 2])
        _, _, r0, r1, _ = db.mbs[i]
        return bufs[c % 2][:r1 - r0]

    def after_mb(i):
        c = state["base"] + i
        freed[c % 2].record(comp)
        _, _, r0, r1, _ = db.mbs[i]
        with torch.cuda.stream(d2h_s):       # this micro-batch's log-probs -> host
            d2h_s.wait_event(freed[c % 2])
            logp_host[r0:r1].copy_(step.logp[r0:r1], non_blocking=True)
        if c + 2 < state["total"]:
            issue_copy(c + 2)

    orig = (step.db.targets, step.db.mask, step.db.cu, step.db.gos, step.db.rewards,
            list(step.db.mbs))

    def one():
        for k, v in host_small.items():
            dev_small[k].copy_(v, non_blocking=True)
        step.db.targets, step.db.mask, step.db.cu = (dev_small["targets"], dev_small["mask"],
                                                     dev_small["cu"])
        step.db.gos, step.db.rewards = dev_small["gos"], dev_small["rewards"]
        step.db.mbs = [(s0, s1, r0, r1, dev_small[f"cu_mb{i}"])
                       for i, (s0, s1, r0, r1, _) in enumerate(orig[5])]
        b = state["base"]
        for c in range(state["issued"], min(b + 2, state["total"])):
            issue_copy(c)            # not prefetched by the previous step
        step.run(None, dev_small["old"], gh, hidden_for_mb=hidden_for_mb, after_mb=after_mb)
        done = torch.cuda.Event()
        done.record(comp)
        with torch.cuda.stream(d2h_s):       # reduced dW slab + stats -> host
            d2h_s.wait_event(done)
            dw_host.copy_(step.grad_w[v0:v1], non_blocking=True)
            stats_host.copy_(step.stats, non_blocking=True)
        comp.wait_stream(d2h_s)              # the next step zeroes dW/stats after the read
        state["base"] = b + n_mb

    def run(k):
        state.update(base=0, total=k * n_mb, issued=0)
        for e in freed:
            e.record(comp)
        for _ in range(k):
            one()

    run(max(1, min(args.warmup, 2)))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run(args.steps)
    e1.record()
    torch.cuda.synchronize()
    (step.db.targets, step.db.mask, step.db.cu, step.db.gos, step.db.rewards) = orig[:5]
    step.db.mbs = orig[5]
    ms = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    v = tokens_global / (float(ms.item()) / 1e3)
    # the host copies are the step's results: same values as the device run
    ok = bool(torch.equal(logp_host[:R], step.logp[:R].cpu())) and \
        bool(torch.equal(dw_host, step.grad_w[v0:v1].cpu()))
    del host_H
    return {"value": round(v, 1), "unit": "tokens/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": round(float(ms.item()), 3),
            "d2h": "per micro-batch logp [rows] fp32 + this rank's dW slab "
                   f"[{v1 - v0}, {step.grad_w.shape[1]}] fp32 + 72 B stats (bytes per rank)",
            "host_results_match_device": ok}


if __name__ == "__main__":
    sys.exit(main())
