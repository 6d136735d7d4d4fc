"""Seeded synthetic workloads for the GRPO policy-loss head.

This module holds NONE of the method's arithmetic. It only draws what a
micro-batch looks like -- packed ragged sequences, response masks, group ids,
rewards, target ids and the hidden / vocab-weight tensor values -- following
the input recipe in DESIGN.md §4. Both sides of the
parity tests (the CPU oracle in ``oracle/`` and the CUDA path in
``paper_2509_15965_b200/``) consume it; neither side is imported here.

Paper anchors for the shapes (PAPER.md = /root/reference/PAPER.md):
  * G responses per query, "e.g., 8"; group 16/32/32, sequence
    length 28672 (tab:math-eval-config).
  * rule-based reward "+5 if ... correct else -5".
  * long-tailed response lengths, "fluctuate across responses of the same
    query, and even more so across different queries".
  * embodied: 256 envs (ManiSkill) x 64 steps (LIBERO); OpenVLA
    emits 7 action tokens per step (BASELINE.json configs[2]).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = ["HeadConfig", "CONFIGS", "Layout", "make_layout", "custom_layout",
           "make_tensors_host", "make_tensors_torch", "sub_layout", "ratio_noise"]


@dataclass(frozen=True)
class HeadConfig:
    """One BASELINE.json config (BJ:L7-L11)."""
    name: str
    hidden: int          # h
    vocab: int           # V
    prompts: int         # prompts (reasoning) / env groups (embodied)
    group: int           # G responses per prompt / envs per group
    lmax: int            # max response length (reasoning) / rows per trajectory
    dtype: str           # "f32" | "bf16"
    kind: str            # "tiny" | "reasoning" | "embodied"
    steps: int = 0       # embodied: env steps per trajectory
    action_tokens: int = 0


CONFIGS = {
    # BJ:L7  tiny GRPO: 2 prompts x G=4, <=32 tokens, h=64, V=1000, fp32
    "tiny": HeadConfig("tiny", 64, 1000, 2, 4, 32, "f32", "tiny"),
    # BJ:L8  Qwen-1.5B head, 64 prompts x G=8, up to 8k tokens, bf16
    "qwen1.5b": HeadConfig("qwen1.5b", 1536, 151936, 64, 8, 8192, "bf16", "reasoning"),
    # BJ:L9  OpenVLA head, 256 envs x 7 action tokens x 64 steps, bf16
    "openvla": HeadConfig("openvla", 4096, 32064, 32, 8, 448, "bf16", "embodied",
                          steps=64, action_tokens=7),
    # BJ:L10 Qwen-7B head, 128 prompts x G=16, up to 16k tokens, bf16
    "qwen7b": HeadConfig("qwen7b", 3584, 152064, 128, 16, 16384, "bf16", "reasoning"),
    # BJ:L11 Qwen-32B head, 256 prompts x G=16, up to 28k tokens, bf16
    "qwen32b": HeadConfig("qwen32b", 5120, 152064, 256, 16, 28672, "bf16", "reasoning"),
}


@dataclass
class Layout:
    """Host-side description of one packed ragged (mini-)batch.

    Row t of the packed batch belongs to sequence s iff
    cu_seqlens[s] <= t < cu_seqlens[s+1]. Each sequence is its prompt rows
    (mask 0) followed by its response rows (mask 1). ``targets[t]`` is the
    (pre-shifted) token id row t predicts.
    """
    cu_seqlens: np.ndarray      # int32 [S+1]
    mask: np.ndarray            # uint8 [R]
    targets: np.ndarray         # int32 [R]
    group_of_seq: np.ndarray    # int32 [S]
    rewards: np.ndarray         # float32 [S]
    num_groups: int
    vocab: int
    prompt_len: np.ndarray = field(default=None)   # int32 [S]
    resp_len: np.ndarray = field(default=None)     # int32 [S]

    @property
    def num_rows(self) -> int:
        return int(self.cu_seqlens[-1])

    @property
    def num_seqs(self) -> int:
        return int(self.cu_seqlens.shape[0] - 1)

    @property
    def num_tokens(self) -> int:
        """Masked response rows (the loss tokens)."""
        return int(np.count_nonzero(self.mask))


def _pack(prompt_len, resp_len, group_of_seq, rewards, vocab, num_groups, rng,
          target_lo=0):
    prompt_len = np.asarray(prompt_len, dtype=np.int64)
    resp_len = np.asarray(resp_len, dtype=np.int64)
    seq_len = prompt_len + resp_len
    cu = np.zeros(seq_len.shape[0] + 1, dtype=np.int64)
    np.cumsum(seq_len, out=cu[1:])
    R = int(cu[-1])
    assert R < 2**31, "packed rows must fit int32"
    mask = np.zeros(R, dtype=np.uint8)
    for s in range(seq_len.shape[0]):
        mask[cu[s] + prompt_len[s]: cu[s + 1]] = 1
    targets = rng.integers(target_lo, vocab, size=R, dtype=np.int64).astype(np.int32)
    return Layout(cu_seqlens=cu.astype(np.int32), mask=mask, targets=targets,
                  group_of_seq=np.asarray(group_of_seq, dtype=np.int32),
                  rewards=np.asarray(rewards, dtype=np.float32),
                  num_groups=int(num_groups), vocab=int(vocab),
                  prompt_len=prompt_len.astype(np.int32),
                  resp_len=resp_len.astype(np.int32))


def make_layout(cfg: HeadConfig, seed: int = 0) -> Layout:
    """The packed mini-batch of a config."""
    rng = np.random.default_rng(seed)
    G, P = cfg.group, cfg.prompts
    if cfg.kind == "tiny":
        # 2 prompts x G=4; response lengths U{1..32}; prompt rows U{2..8}.
        plen = np.repeat(rng.integers(2, 9, size=P), G)
        rlen = rng.integers(1, cfg.lmax + 1, size=P * G)
        # Constructed rewards: prompt 0 has 1 of 4 correct, prompt 1 is
        # all-correct (the zero-variance group). +-5 per P:L833.
        rewards = np.full(P * G, -5.0)
        rewards[int(rng.integers(0, G))] = 5.0
        rewards[G:2 * G] = 5.0
        gos = np.repeat(np.arange(P), G)
        return _pack(plen, rlen, gos, rewards, cfg.vocab, P, rng)
    if cfg.kind == "reasoning":
        # Per-prompt difficulty u_p ~ N(0, 0.6^2), per-response noise
        # e ~ N(0, 0.45^2); L = clamp(round(exp(ln(Lmax/8) + u_p + e)), 16, Lmax).
        u = rng.normal(0.0, 0.6, size=P)
        e = rng.normal(0.0, 0.45, size=(P, G))
        L = np.exp(math.log(cfg.lmax / 8.0) + u[:, None] + e)
        rlen = np.clip(np.rint(L), 16, cfg.lmax).astype(np.int64).reshape(-1)
        # Prompt length U{64..512}, shared by the G responses of a prompt.
        plen = np.repeat(rng.integers(64, 513, size=P), G)
        # Rewards +-5, Bernoulli(p_p), p_p ~ U(0,1); prompt 0 forced
        # all-correct and prompt 1 all-wrong (zero-variance groups).
        pp = rng.uniform(0.0, 1.0, size=P)
        ok = rng.uniform(0.0, 1.0, size=(P, G)) < pp[:, None]
        ok[0, :] = True
        ok[1, :] = False
        rewards = np.where(ok, 5.0, -5.0).reshape(-1)
        gos = np.repeat(np.arange(P), G)
        return _pack(plen, rlen, gos, rewards, cfg.vocab, P, rng)
    if cfg.kind == "embodied":
        # One sequence per env trajectory: steps x action_tokens rows, all
        # response rows (no prompt rows). Groups of G envs. Reward = success
        # in {0,1}, Bernoulli(p_g), p_g ~ U(0,1); group 0 all-success, group 1
        # all-fail. Targets are action bins: the last 256 ids of the vocab.
        n_env = P * G
        rows = cfg.steps * cfg.action_tokens
        plen = np.zeros(n_env, dtype=np.int64)
        rlen = np.full(n_env, rows, dtype=np.int64)
        pg = rng.uniform(0.0, 1.0, size=P)
        ok = rng.uniform(0.0, 1.0, size=(P, G)) < pg[:, None]
        ok[0, :] = True
        ok[1, :] = False
        rewards = ok.astype(np.float64).reshape(-1)
        gos = np.repeat(np.arange(P), G)
        return _pack(plen, rlen, gos, rewards, cfg.vocab, P, rng,
                     target_lo=cfg.vocab - 256)
    raise ValueError(cfg.kind)


def custom_layout(prompt_len, resp_len, group_of_seq, rewards, vocab, num_groups,
                  seed: int = 0) -> Layout:
    """Hand-built layout (edge cases in tests): explicit per-sequence lengths."""
    rng = np.random.default_rng(seed)
    return _pack(prompt_len, resp_len, group_of_seq, rewards, vocab, num_groups, rng)


def sub_layout(layout: Layout, seqs):
    """(layout, rows): the packed batch made of the given whole sequences, in the
    given order, and the parent rows it was cut from."""
    seqs = np.asarray(seqs, dtype=np.int64)
    cu = layout.cu_seqlens.astype(np.int64)
    rows = [np.arange(cu[s], cu[s + 1]) for s in seqs]
    rows = np.concatenate(rows) if rows else np.zeros(0, dtype=np.int64)
    lens = cu[seqs + 1] - cu[seqs]
    ncu = np.zeros(len(seqs) + 1, dtype=np.int64)
    np.cumsum(lens, out=ncu[1:])
    return Layout(cu_seqlens=ncu.astype(np.int32), mask=layout.mask[rows].copy(),
                  targets=layout.targets[rows].copy(),
                  group_of_seq=layout.group_of_seq[seqs].copy(),
                  rewards=layout.rewards[seqs].copy(), num_groups=layout.num_groups,
                  vocab=layout.vocab,
                  prompt_len=None if layout.prompt_len is None else layout.prompt_len[seqs].copy(),
                  resp_len=None if layout.resp_len is None else layout.resp_len[seqs].copy()), rows


def _torch_dtype(dtype: str):
    import torch
    return {"f32": torch.float32, "bf16": torch.bfloat16}[dtype]


def make_tensors_torch(cfg: HeadConfig, num_rows: int, seed: int = 0, device="cpu",
                       chunk_rows: int = 1 << 16, weight=True, hidden=True):
    """hidden [num_rows, h] ~ N(0,1) and W [V, h] ~ N(0, (4/sqrt(h))^2), cast to
    the config dtype (logit std ~= 4, a peaked softmax). Generated in row chunks
    with a torch generator on ``device`` so the 40 GB Qwen-7B batch never
    exists in fp32."""
    import torch
    dt = _torch_dtype(cfg.dtype)
    g = torch.Generator(device=device)
    H = Wt = None
    if weight:
        g.manual_seed(seed * 1000003 + 1)
        Wt = torch.empty(cfg.vocab, cfg.hidden, dtype=dt, device=device)
        for r0 in range(0, cfg.vocab, chunk_rows):
            r1 = min(cfg.vocab, r0 + chunk_rows)
            Wt[r0:r1] = (torch.randn(r1 - r0, cfg.hidden, generator=g, device=device)
                         * (4.0 / math.sqrt(cfg.hidden))).to(dt)
    if hidden:
        g.manual_seed(seed * 1000003 + 2)
        H = torch.empty(num_rows, cfg.hidden, dtype=dt, device=device)
        for r0 in range(0, num_rows, chunk_rows):
            r1 = min(num_rows, r0 + chunk_rows)
            H[r0:r1] = torch.randn(r1 - r0, cfg.hidden, generator=g, device=device).to(dt)
    return H, Wt


def make_tensors_host(cfg: HeadConfig, num_rows: int, seed: int = 0):
    """Same recipe as make_tensors_torch on the CPU; returns torch CPU tensors
    of the config dtype (exact values the GPU will see after .to('cuda'))."""
    return make_tensors_torch(cfg, num_rows, seed, device="cpu")


def ratio_noise(n: int, seed: int = 0, sigma: float = 0.05) -> np.ndarray:
    """delta ~ N(0, sigma^2) for old_logp = logp + delta (perf runs, M.2)."""
    return np.random.default_rng(seed + 7919).normal(0.0, sigma, size=n)
