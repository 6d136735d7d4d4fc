"""The C-ABI library loads and exports every symbol include/rlhead.h declares;
host-side validation rejects bad arguments before touching the GPU (so these
run on a CPU-only box)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rlhead.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"RL_API\s+[\w\s\*]*?\b(rl_\w+)\s*\(", src)))


def test_header_declares_the_three_entry_points():
    names = _declared()
    for n in ("rl_logprob_fwd", "rl_grpo_advantage", "rl_policy_loss_fwd_bwd"):
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_2509_15965_b200 import rlhead
    for name in _declared():
        assert hasattr(rlhead.lib, name), name
    assert sorted(rlhead.EXPORTED) == _declared()


def test_workspace_size_and_validation_host_only():
    from paper_2509_15965_b200 import rlhead as R
    hd = R.rl_head(3584, 152064, R.RL_BF16, 3584, 1.0)
    n_f = R.lib.rl_workspace_size(C.byref(hd), 65536, 0)
    n_b = R.lib.rl_workspace_size(C.byref(hd), 65536, 1)
    # dZ chunk bf16 [Rp, Vp] dominates the backward workspace
    assert n_b - n_f >= 65536 * 152064 * 2
    # bookkeeping-only prefix (rl_batch_prepare): ~21 B/row, independent of V and h
    n_p = R.lib.rl_workspace_size(C.byref(hd), 65536, 2)
    assert 0 < n_p <= 65536 * 24 + 4096 and n_p < n_f
    assert R.lib.rl_workspace_size(C.byref(hd), 65536, 3) == 0
    assert R.lib.rl_workspace_size(C.byref(R.rl_head(100, 10, R.RL_BF16, 100, 1.0)), 10, 0) == 0
    assert R.lib.rl_workspace_size(C.byref(R.rl_head(64, 10, R.RL_BF16, 64, 0.0)), 10, 0) == 0
    assert R.lib.rl_workspace_size(C.byref(R.rl_head(100, 10, R.RL_F32, 100, 1.0)), 10, 0) > 0
    # NULL arguments are rejected on the host (nothing launched)
    st = R.lib.rl_logprob_fwd(None, None, None, None, None, None, None, None, 0, None)
    assert st == R.RL_ERR_INVALID_ARG
    b = R.rl_batch(4, 1, None, None, None, None)
    st = R.lib.rl_batch_prepare(C.byref(hd), C.byref(b), None, None, None, None, None, None, 0,
                                None)
    assert st == R.RL_ERR_INVALID_ARG
    assert R.lib.rl_status_string(3) == b"RL_ERR_WORKSPACE"
    assert R.lib.rl_grpo_advantage(None, None, -1, 1, None, None, 1e-6, 1, None, None, None) \
        == R.RL_ERR_INVALID_ARG
    # the DP dW sum (collective "nvls") validates before touching a device pointer
    peers = (C.c_void_p * 2)(16, 32)
    dw = R.lib.rl_dw_reduce_rows_f32
    assert dw(None, None, 0, 2, 10, 8, 5, 1, None) == R.RL_ERR_INVALID_ARG      # no peers
    assert dw(peers, None, 0, 0, 10, 8, 5, 1, None) == R.RL_ERR_INVALID_ARG     # world 0
    assert dw(peers, None, 2, 2, 10, 8, 5, 1, None) == R.RL_ERR_INVALID_ARG     # rank >= world
    assert dw(peers, None, 0, 2, 10, 6, 5, 1, None) == R.RL_ERR_INVALID_ARG     # cols % 4
    assert dw(peers, None, 0, 2, 11, 8, 5, 1, None) == R.RL_ERR_INVALID_ARG     # 2 x 5 < 11 rows
    bad = (C.c_void_p * 2)(16, 40)
    assert dw(bad, None, 0, 2, 10, 8, 5, 1, None) == R.RL_ERR_INVALID_ARG       # misaligned peer
    assert dw(peers, C.c_void_p(8), 0, 2, 10, 8, 5, 1, None) == R.RL_ERR_INVALID_ARG  # mc align
    one = (C.c_void_p * 1)(16)
    assert dw(one, None, 0, 1, 10, 8, 10, 1, None) == R.RL_OK                   # world 1: no-op


def test_struct_layouts_match_header(tmp_path):
    """ctypes mirrors of the header structs have the C compiler's sizes and
    field offsets."""
    import shutil
    import subprocess
    from paper_2509_15965_b200 import rlhead as R
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    structs = {"rl_batch": R.rl_batch, "rl_head": R.rl_head, "rl_loss_params": R.rl_loss_params,
               "rl_loss_stats": R.rl_loss_stats, "rl_peer_group": R.rl_peer_group,
               "rl_value_params": R.rl_value_params}
    lines = ["#include <stdio.h>", "#include <stddef.h>", f'#include "{HEADER}"', "int main(){"]
    for s, cls in structs.items():
        lines.append(f'printf("{s} %zu\\n", sizeof({s}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{s}.{f} %zu\\n", offsetof({s}, {f}));')
    lines.append("return 0;}")
    src = tmp_path / "s.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "s"
    subprocess.run(["gcc", str(src), "-o", str(exe)], check=True)
    out = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                 check=True).stdout.splitlines())
    for s, cls in structs.items():
        assert int(out[s]) == C.sizeof(cls), s
        for f, _ in cls._fields_:
            assert int(out[f"{s}.{f}"]) == getattr(cls, f).offset, (s, f)


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2509_15965_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
