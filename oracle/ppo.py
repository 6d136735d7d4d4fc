"""CPU float64 oracle of the PPO pieces (NEXT-4) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py may import this module.
The paper trains OpenVLA with PPO as well as GRPO (tab:maniskill-eval
"RLinf-OpenVLA-PPO") and cites PPO for the RLHF workflow with a critic
(P:L184). PAPER.md gives no formula, so the textbook definitions are used
(DESIGN.md §3 #30-#32):

* value head: v_t = <w_v, h_t> + b_v on the rows that predict a value;
* GAE over each trajectory (Schulman et al.), steps in order t = 0..T_s-1:
    delta_t = r_t + gamma * (1 - done_t) * V_{t+1} - V_t,
    A_t     = delta_t + gamma * lambda * (1 - done_t) * A_{t+1},
  with V_{T_s} = the trajectory's bootstrap value and A_{T_s} = 0;
  returns R_t = A_t + V_t;
* clipped value loss: L_v = (1/N_v) sum_t 0.5 max((v_t - R_t)^2,
  (clip(v_t, v_old - eps_v, v_old + eps_v) - R_t)^2), gradient through the
  larger term (the unclipped one on ties); the clipped term carries no
  gradient outside [v_old - eps_v, v_old + eps_v] (inside, it equals the
  unclipped term).
"""
from __future__ import annotations

import math

import numpy as np

from .head import _as64, _take_rows, bookkeeping


def gae(rewards, values, dones, bootstrap, cu_steps, gamma, lam):
    """Plain reverse loop per trajectory. cu_steps [S+1] offsets into the
    step arrays; bootstrap [S] = V after the last step. Returns (adv, ret)."""
    r = _as64(rewards).reshape(-1)
    v = _as64(values).reshape(-1)
    d = np.asarray(dones).reshape(-1)
    vb = _as64(bootstrap).reshape(-1)
    cu = [int(x) for x in np.asarray(cu_steps).reshape(-1)]
    adv = np.zeros_like(r)
    for s in range(len(cu) - 1):
        next_v, next_a = float(vb[s]), 0.0
        for t in range(cu[s + 1] - 1, cu[s] - 1, -1):
            nonterm = 0.0 if d[t] else 1.0
            delta = float(r[t]) + gamma * nonterm * next_v - float(v[t])
            next_a = delta + gamma * lam * nonterm * next_a
            adv[t] = next_a
            next_v = float(v[t])
    return adv, adv + v


def value_fwd(hidden, w_v, b_v, cu_seqlens, mask, vocab_dummy=1):
    """v_t on the active rows (mask != 0), 0 elsewhere."""
    bk = bookkeeping(cu_seqlens, mask, np.zeros(np.asarray(mask).shape[0], np.int64), vocab_dummy)
    R = np.asarray(mask).shape[0]
    out = np.zeros(R)
    idx = bk["active_idx"].astype(np.int64)
    if len(idx):
        out[idx] = _as64(_take_rows(hidden, idx)) @ _as64(w_v).reshape(-1) + float(b_v)
    return out


def value_loss_fwd_bwd(hidden, w_v, b_v, cu_seqlens, mask, returns, old_values, clip_eps,
                       n_global=None):
    """Clipped value loss and its gradients. Returns dict(loss, values, g (dL/dv),
    dH [R,h], dw [h], db, clipfrac_count, tokens)."""
    H_rows_mask = np.asarray(mask).reshape(-1)
    R = H_rows_mask.shape[0]
    bk = bookkeeping(cu_seqlens, mask, np.zeros(R, np.int64), 1)
    idx = bk["active_idx"].astype(np.int64)
    N = len(idx) if n_global is None else int(n_global)
    scale = 1.0 / N if N > 0 else 0.0
    w = _as64(w_v).reshape(-1)
    ret = _as64(returns).reshape(-1)
    vold = _as64(old_values).reshape(-1)
    h = w.shape[0]
    values = np.zeros(R)
    g = np.zeros(R)
    dH = np.zeros((R, h))
    losses = []
    nclip = 0
    if len(idx):
        Hs = _as64(_take_rows(hidden, idx))
        vs = Hs @ w + float(b_v)
        for j, t in enumerate(idx):
            v = float(vs[j])
            lo, hi = vold[t] - clip_eps, vold[t] + clip_eps
            vc = min(max(v, lo), hi)
            a, b = (v - ret[t]) ** 2, (vc - ret[t]) ** 2
            losses.append(0.5 * max(a, b))
            if a >= b:
                dv = v - ret[t]
            else:
                dv = (vc - ret[t]) if lo <= v <= hi else 0.0
                nclip += 1
            values[t] = v
            g[t] = scale * dv
        dH[idx] = g[idx][:, None] * w[None, :]
        dw = (g[idx][:, None] * Hs).sum(axis=0)
        db = math.fsum(g[idx])
    else:
        dw, db = np.zeros(h), 0.0
    return dict(loss=math.fsum(losses) * scale, loss_sum=math.fsum(losses), values=values, g=g,
                dH=dH, dw=dw, db=db, clip_count=nclip, tokens=len(idx))
