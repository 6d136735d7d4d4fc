"""CPU float64 oracle for the GRPO policy-loss head -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import anything under
``oracle/``. The product path (``paper_2509_15965_b200``) never imports it
and shares no code, header, constant or helper with it.

Every function is the plain definition of what the hot path computes
(SURVEY.md §8(c) O.1), evaluated in float64 on the exact values
of the (bf16 or fp32) input tensors, and cites the PAPER.md passage it
follows. The paper prints no value for this path, so every function is pinned
by closed forms, brute force, invariants and an independent autograd /
finite-difference check in ``tests/test_oracle_pins.py``. The *readings* of
points the paper leaves open (std estimator, eps, clip range, clamp, zero-
variance rule) are "parity unpinned" against the paper itself:
no printed number distinguishes them.
"""
from .head import (  # noqa: F401
    ERR_CU_SEQLENS, ERR_TARGET, ERR_GROUP,
    bookkeeping, logprob_fwd, grpo_group_stats, grpo_advantage,
    grpo_advantage_from_stats, batch_norm_advantage, policy_loss_fwd_bwd, LossParams,
)
