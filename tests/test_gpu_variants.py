"""The tensor-core GEMM variants (1-CTA tiles, 2-CTA 256-wide tiles, 2-CTA
512-wide dH/dW tiles) all pass the bf16 parity tests. The variant is fixed per
process (read once from the environment), so each runs in a subprocess."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [{"RLHEAD_CTA_GROUP": "1"},
                                 {"RLHEAD_CTA_GROUP": "2", "RLHEAD_WIDE": "0"},
                                 {"RLHEAD_CTA_GROUP": "2", "RLHEAD_WIDE": "1",
                                  "RLHEAD_FUSED_BWD": "1"},
                                 {"RLHEAD_CTA_GROUP": "2", "RLHEAD_WIDE": "1",
                                  "RLHEAD_GROUP_M": "16", "RLHEAD_GROUP_M_BWD": "4"},
                                 {"RLHEAD_DW_RED": "0"},
                                 {"RLHEAD_DW_RED": "1", "RLHEAD_FUSED_BWD": "1"}],
                         ids=["cta1", "cta2-narrow", "cta2-wide-fused", "cta2-unfused-raster",
                              "dw-load-store", "dw-red-fused"])
def test_variant_parity(env):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        "tests/test_gpu_parity.py", "-k", "bf16 or qwen15b or determinism"],
                       cwd=ROOT, env={**os.environ, **env}, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
