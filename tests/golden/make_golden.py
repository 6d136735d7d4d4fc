"""Writes tests/golden/tiny_oracle.npz: the tiny GRPO config (BASELINE.json
configs[0]) run through the CPU oracle ONLY (plus the seeded generator).
Re-run after an intentional oracle change; the commit must cite why.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from workload import CONFIGS, make_layout, make_tensors_host  # noqa: E402


def main():
    cfg = CONFIGS["tiny"]
    lay = make_layout(cfg, seed=0)
    H, W = make_tensors_host(cfg, lay.num_rows, seed=0)
    adv, _ = oracle.grpo_advantage(lay.rewards, lay.group_of_seq, lay.num_groups)
    fwd = oracle.logprob_fwd(H, W, lay.cu_seqlens, lay.mask, lay.targets)
    # old_logp = logp - ln r*, r* = 1 + 0.1 * (-1)^t (inside the clip band)
    t = np.arange(lay.num_rows)
    old = fwd["logp"] - np.log(1.0 + 0.1 * np.where(t % 2 == 0, 1.0, -1.0))
    out = oracle.policy_loss_fwd_bwd(H, W, lay.cu_seqlens, lay.mask, lay.targets, old, adv)
    np.savez_compressed(os.path.join(os.path.dirname(__file__), "tiny_oracle.npz"),
                        adv=adv, logp=fwd["logp"], entropy=fwd["entropy"], lse=fwd["lse"],
                        old_logp=old, loss=out["loss"], dH=out["dH"], dW=out["dW"],
                        n_active=out["n_active"])


if __name__ == "__main__":
    main()
