"""bench.py's reference arm (the CPU oracle, `--impl reference`) runs without a
GPU: check its one JSON line carries the contract's keys (metric/unit/value,
steps/warmup, e2e with zero copy bytes, cpu_baseline with cores and sample)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "tiny", "--steps", "2", "--warmup", "1",
                          "--cpu-sample-tokens", "16"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["steps"] == 2 and d["warmup"] == 1 and d["value"] > 0
    assert d["unit"] == d["e2e"]["unit"] == "tokens/s" and d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["sample"] and cb["value"] == d["value"]


def test_reference_arm_under_torchrun_rank0_only():
    """Under torchrun (N > 1) rank 0 alone runs and prints; the others exit 0."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node=2", "--master-addr", "127.0.0.1", "--master-port",
                          str(port), os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--config", "tiny", "--steps", "1", "--warmup", "1",
                          "--cpu-sample-tokens", "16"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1 and json.loads(lines[0])["n_gpus"] == 2


def test_cpu_baseline_leg_bounded_oracle_sample():
    """The N=1 cpu_baseline leg times the oracle on the first `tokens` masked rows
    of sequence 0: the reported sample size is the active-row count, bounded by
    the request, and value = tokens / seconds."""
    sys.path.insert(0, ROOT)
    import bench
    from workload import CONFIGS, make_layout
    cfg = CONFIGS["tiny"]
    cb = bench.cpu_baseline(cfg, make_layout(cfg, seed=0), 0, 8)
    assert cb["kind"] == "oracle" and cb["unit"] == "tokens/s" and cb["cores"] >= 1
    n = int(cb["sample"].split()[0])
    assert 1 <= n <= 8
    assert abs(cb["value"] - n / cb["seconds"]) <= 1e-9 * cb["value"]


def test_gpu_arm_refuses_world_mismatch():
    """--gpus N must equal the torchrun world: a mismatch exits 2 before any
    device work (without WORLD_SIZE, --gpus N > 1 relaunches under torchrun)."""
    env = dict(os.environ, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--config", "tiny"], capture_output=True, text=True, timeout=300,
                         cwd=ROOT, env=env)
    assert out.returncode == 2, (out.returncode, out.stderr[-2000:])
    assert "WORLD_SIZE=3" in out.stderr


def test_cpu_baseline_m7_pieces():
    """all-thread sample, 1-thread sample, tiny end to end, and the
    full config's extrapolated time, labelled as extrapolated."""
    sys.path.insert(0, ROOT)
    import bench
    from workload import CONFIGS, make_layout
    cfg = CONFIGS["tiny"]
    lay = make_layout(cfg, seed=0)
    cb = bench.cpu_baseline_m7(cfg, lay, 0, 8, 4, lay.num_tokens)
    assert cb["one_thread"]["cores"] == 1 and cb["one_thread"]["value"] > 0
    assert cb["tiny_end_to_end"]["tokens"] == lay.num_tokens
    ex = cb["full_config_extrapolated"]
    assert "extrapolated" in ex["note"]
    assert abs(ex["seconds"] - lay.num_tokens / cb["value"]) <= 0.06
