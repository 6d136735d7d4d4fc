"""CPU float64 oracle of the GRPO policy-loss head -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this module. It shares no code with the
CUDA path. Plain NumPy float64 (OpenBLAS dgemm as the only library step),
obviously-correct loops over rows/groups, ``math.fsum`` for scalar sums.

Citations: P:Lnnn = /root/reference/PAPER.md line nnn; "reading #k" =
DESIGN.md §3 row k (the paper is silent there).

Pins (tests/test_oracle_pins.py): brute-force mpmath softmax, closed forms
(zero logits, GRPO +-5 groups, ratio = 1, clip quadrants), invariants,
torch float64 autograd of the definitional loss, central finite
differences. Parity against the paper's *readings* (#5-#8, #12-#16) is
"parity unpinned": PAPER.md prints no number that fixes them.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

# Device error-word bits ("Device validation"). Restated here
# from the spec, not shared with include/rlhead.h.
ERR_CU_SEQLENS = 1   # cu_seqlens[0] != 0, decreasing, or cu[S] != num_rows
ERR_TARGET = 2       # a target id outside [0, V)
ERR_GROUP = 4        # a group id outside [0, num_groups)

_CHUNK = 512         # rows per float64 logits chunk


# --------------------------------------------------------------------------
# H1: packing / index bookkeeping (packed ragged batch, response mask).
# P:L202-203 ("per response ... or at least a micro-batch of responses"),
# BASELINE.json north_star ("packed variable-length sequences with a
# response mask and group ids").
# --------------------------------------------------------------------------
def bookkeeping(cu_seqlens, mask, targets, vocab):
    """Validate a packed batch and list its active rows.

    Returns dict(row_seq int32[R], active bool[R], active_idx int32[T],
    n_active int, err int).

    * cu_seqlens must satisfy cu[0] = 0, cu[s] <= cu[s+1], cu[S] = R
      (R = len(mask)). If not, ERR_CU_SEQLENS is raised in ``err``, every row
      is inactive and row_seq = -1 everywhere (reading #23).
    * row_seq[t] = the s with cu[s] <= t < cu[s+1].
    * row t is active iff the batch is well formed, mask[t] != 0 and
      0 <= targets[t] < V. An out-of-range target of a masked-in row raises
      ERR_TARGET and the row becomes inactive.
    * active_idx lists the active rows in increasing (packed) order.
    """
    cu = [int(x) for x in np.asarray(cu_seqlens).reshape(-1)]
    mask = np.asarray(mask).reshape(-1)
    targets = np.asarray(targets).reshape(-1)
    R = mask.shape[0]
    S = len(cu) - 1
    err = 0
    ok = S >= 0 and len(cu) >= 1 and cu[0] == 0 and cu[-1] == R
    for s in range(S):
        if cu[s] > cu[s + 1]:
            ok = False
    row_seq = np.full(R, -1, dtype=np.int32)
    active = np.zeros(R, dtype=bool)
    if not ok:
        err |= ERR_CU_SEQLENS
        return dict(row_seq=row_seq, active=active,
                    active_idx=np.zeros(0, dtype=np.int32), n_active=0, err=err)
    for s in range(S):
        for t in range(cu[s], cu[s + 1]):
            row_seq[t] = s
    for t in range(R):
        if mask[t] != 0:
            y = int(targets[t])
            if 0 <= y < vocab:
                active[t] = True
            else:
                err |= ERR_TARGET
    active_idx = np.array([t for t in range(R) if active[t]], dtype=np.int32)
    return dict(row_seq=row_seq, active=active, active_idx=active_idx,
                n_active=int(active_idx.shape[0]), err=err)


# --------------------------------------------------------------------------
# H3 + H4: projection z = tau^-1 W h, log-softmax at the target, entropy.
# "computes logarithmic probabilities for these responses" (
# reading #1: natural-log softmax over the full V at the pre-shifted target).
# Entropy (reading #4): Shannon entropy in nats of softmax(z).
# --------------------------------------------------------------------------
def _as64(x):
    """float64 copy of a numpy array or torch tensor (exact for bf16/fp32)."""
    if hasattr(x, "detach"):
        x = x.detach().to("cpu")
        import torch
        x = x.to(torch.float64).numpy()
    return np.asarray(x, dtype=np.float64)


def _row_softmax_stats(Hrows, W, targets_rows, inv_temperature):
    """For a chunk of rows: z = tau^-1 H W^T; lse, logp, p, entropy."""
    Z = (Hrows @ W.T) * inv_temperature                 # [n, V] float64
    m = Z.max(axis=1, keepdims=True)
    lse = (m + np.log(np.exp(Z - m).sum(axis=1, keepdims=True)))[:, 0]
    P = np.exp(Z - lse[:, None])
    zy = Z[np.arange(Z.shape[0]), targets_rows]
    logp = zy - lse
    entropy = lse - (P * Z).sum(axis=1)
    return Z, P, lse, logp, entropy


def logprob_fwd(hidden, weight, cu_seqlens, mask, targets, inv_temperature=1.0,
                rows=None):
    """Per-row log-prob / entropy / lse of the target token (fp64).

    hidden [R, h], weight [V, h] (nn.Linear layout). Inactive rows (see
    ``bookkeeping``) get 0 in all three outputs. ``rows`` restricts the work to
    a subset of rows (sampled parity at full size); other rows are left 0.
    Returns dict(logp, entropy, lse, err, active).
    """
    W = _as64(weight)
    V = W.shape[0]
    bk = bookkeeping(cu_seqlens, mask, targets, V)
    R = np.asarray(mask).shape[0]
    logp = np.zeros(R)
    ent = np.zeros(R)
    lse = np.zeros(R)
    want = bk["active_idx"] if rows is None else np.array(
        [t for t in np.asarray(rows).reshape(-1) if bk["active"][t]], dtype=np.int64)
    targets = np.asarray(targets).reshape(-1)
    for c0 in range(0, len(want), _CHUNK):
        idx = want[c0:c0 + _CHUNK]
        Hc = _as64(_take_rows(hidden, idx))
        _, _, l, lp, e = _row_softmax_stats(Hc, W, targets[idx].astype(np.int64), inv_temperature)
        logp[idx], ent[idx], lse[idx] = lp, e, l
    return dict(logp=logp, entropy=ent, lse=lse, err=bk["err"], active=bk["active"])


def _take_rows(x, idx):
    """Rows ``idx`` of a numpy array or torch tensor (any device)."""
    idx = np.asarray(idx, dtype=np.int64)
    if hasattr(x, "detach"):
        import torch
        return x[torch.as_tensor(idx, device=x.device)]
    return np.asarray(x)[idx]


# --------------------------------------------------------------------------
# H2: GRPO group-relative advantage.
# GRPO generates G responses per query; "normalization must
# aggregate all responses for a query"; rewards +-5.
# Formula (reading #5): A_i = (r_i - mu_g) / (sigma_g + eps) within the group,
# sigma unbiased (n-1) by default (reading #6), eps = 1e-6 (reading #7),
# A = 0 exactly when n_g = 1 or max_g r = min_g r (reading #8).
# --------------------------------------------------------------------------
def grpo_group_stats(rewards, group_of_seq, num_groups):
    """Per-group sufficient statistics of the rewards.

    sum_stats[g] = (n_g, sum r, sum r^2) and max_stats[g] = (max r, -min r),
    over the sequences with a valid group id (others raise ERR_GROUP). Groups
    with no member: (0, 0, 0) and (-inf, -inf).
    """
    r = _as64(rewards).reshape(-1)
    gos = np.asarray(group_of_seq).reshape(-1)
    sum_stats = np.zeros((num_groups, 3))
    max_stats = np.full((num_groups, 2), -np.inf)
    err = 0
    members = [[] for _ in range(num_groups)]
    for i in range(r.shape[0]):
        g = int(gos[i])
        if 0 <= g < num_groups:
            members[g].append(float(r[i]))
        else:
            err |= ERR_GROUP
    for g in range(num_groups):
        xs = members[g]
        if xs:
            sum_stats[g] = (len(xs), math.fsum(xs), math.fsum(x * x for x in xs))
            max_stats[g] = (max(xs), -min(xs))
    return sum_stats, max_stats, err


def grpo_advantage(rewards, group_of_seq, num_groups, eps=1e-6, unbiased=True):
    """A_i per sequence, the plain two-pass definition (mean, then squared
    deviations). Sequences with an invalid group id get A = 0 and ERR_GROUP."""
    r = _as64(rewards).reshape(-1)
    gos = np.asarray(group_of_seq).reshape(-1)
    adv = np.zeros(r.shape[0])
    err = 0
    for i in range(r.shape[0]):
        if not (0 <= int(gos[i]) < num_groups):
            err |= ERR_GROUP
    for g in range(num_groups):
        idx = [i for i in range(r.shape[0]) if int(gos[i]) == g]
        n = len(idx)
        if n == 0:
            continue
        xs = [float(r[i]) for i in idx]
        if n == 1 or max(xs) == min(xs):
            continue                       # A = 0 exactly (reading #8)
        mu = math.fsum(xs) / n
        var = math.fsum((x - mu) ** 2 for x in xs) / ((n - 1) if unbiased else n)
        sigma = math.sqrt(var)
        for i, x in zip(idx, xs):
            adv[i] = (x - mu) / (sigma + eps)
    return adv, err


def grpo_advantage_from_stats(rewards, group_of_seq, sum_stats, max_stats, eps=1e-6,
                              unbiased=True):
    """A_i from (possibly all-reduced) group statistics: the split-group form
    (a group's responses on several DP ranks).
    mu = S1/n, var = (S2 - n mu^2) / (n - 1 | n); A = 0 if n <= 1 or max = min."""
    r = _as64(rewards).reshape(-1)
    gos = np.asarray(group_of_seq).reshape(-1)
    G = np.asarray(sum_stats).shape[0]
    adv = np.zeros(r.shape[0])
    for i in range(r.shape[0]):
        g = int(gos[i])
        if not (0 <= g < G):
            continue
        n, s1, s2 = (float(v) for v in sum_stats[g])
        mx, negmn = float(max_stats[g][0]), float(max_stats[g][1])
        if n <= 1 or mx == -negmn:
            continue
        mu = s1 / n
        var = max(s2 - n * mu * mu, 0.0) / ((n - 1) if unbiased else n)
        adv[i] = (float(r[i]) - mu) / (math.sqrt(var) + eps)
    return adv


def batch_norm_advantage(rewards, group_of_seq, num_groups, group_baseline=True, eps=1e-6,
                         unbiased=True):
    """REINFORCE++-style advantage, NEXT-1 (P:L654 names REINFORCE++ among the
    supported algorithms; no formula is printed -- DESIGN.md §3 reading #33):
    normalisation over the whole batch instead of per query.

      x_s = r_s - mu_g(s)   (group_baseline; mu_g the plain mean of s's group)
          = r_s             (otherwise)
      A_s = (x_s - mean_B x) / (std_B x + eps)   over the sequences of the batch
            with a valid group id (std over n-1 if unbiased else n);
      A_s = 0 exactly when fewer than 2 valid sequences or max_B x == min_B x,
      and for sequences with an invalid group id (ERR_GROUP).
    Plain two-pass definition (means with math.fsum, then deviations)."""
    r = _as64(rewards).reshape(-1)
    gos = np.asarray(group_of_seq).reshape(-1)
    S = r.shape[0]
    adv = np.zeros(S)
    err = 0
    valid = [i for i in range(S) if 0 <= int(gos[i]) < num_groups]
    if len(valid) < S:
        err |= ERR_GROUP
    x = {}
    for i in valid:
        x[i] = float(r[i])
    if group_baseline:
        for g in range(num_groups):
            idx = [i for i in valid if int(gos[i]) == g]
            if not idx:
                continue
            mu_g = math.fsum(float(r[i]) for i in idx) / len(idx)
            for i in idx:
                x[i] = float(r[i]) - mu_g
    n = len(valid)
    if n < 2:
        return adv, err
    xs = [x[i] for i in valid]
    if max(xs) == min(xs):
        return adv, err
    mu = math.fsum(xs) / n
    var = math.fsum((v - mu) ** 2 for v in xs) / ((n - 1) if unbiased else n)
    sigma = math.sqrt(var)
    for i in valid:
        adv[i] = (x[i] - mu) / (sigma + eps)
    return adv, err


# --------------------------------------------------------------------------
# H5: ratio, clipped surrogate, token-level mean; H6-H8: backward.
# "Token-Level Loss: ... compute the average over tokens, as in DAPO";
# "discard minibatches with too large importance ratio" (P:L830 -> ratio
# statistics are emitted). Surrogate (readings #12-#15):
#   d = logp - old, r = exp(clamp(d, -c, c)),
#   l = max(-A r, -A clip(r, 1-eps_lo, 1+eps_hi)),  L = sum_t m_t l_t / N,
#   dL/dlogp = -(m/N) A r * act * [|d| <= c],
#   act = not((A > 0 and r > 1+eps_hi) or (A < 0 and r < 1-eps_lo)).
# Backward through softmax: dz = tau^-1 g (onehot(y) - p); dH = dz W;
# dW = sum_t dz_t^T h_t (BASELINE.json north_star: "dL/dhidden and dL/dW").
#
# NEXT-1 variants (DESIGN.md §3 #25-#28; the algorithms the paper cites,
# PPO/DAPO/GRPO P:L184; all off by default):
#   dual clip (A < 0): l = min(max(-A r, -A clip(r)), -A c_dual), grad 0 if r > c_dual;
#   KL to a reference policy, k3 estimator: k = e^{q} - q - 1, q = clamp(ref - logp),
#     dk/dlogp = 1 - e^{q} (0 if clamped);
#   entropy bonus: - c_ent H_t, dH_t/dz_j = -p_j (z_j - E_p[z]);
#   aggregation: token mean (w_t = 1/N) or seq-mean-token-mean
#     (w_t = 1 / (S n_s), n_s = active tokens of t's sequence, S = sequences
#     with n_s >= 1 over the mini-batch).
#   L = sum_t m_t w_t (l_t + beta k_t - c_ent H_t).
# --------------------------------------------------------------------------
@dataclass
class LossParams:
    clip_lo: float = 0.2
    clip_hi: float = 0.2
    logratio_clamp: float = 20.0
    loss_scale: float | None = None     # None -> 1 / n_global (token mean)
    dual_clip: float = 0.0              # c_dual > 1 enables dual clip for A < 0
    kl_coef: float = 0.0                # beta
    entropy_coef: float = 0.0           # c_ent
    seq_mean: bool = False              # seq-mean-token-mean aggregation


def _surrogate(logp, old, A, p: LossParams):
    d = logp - old
    c = p.logratio_clamp
    r = math.exp(min(max(d, -c), c))
    lo, hi = 1.0 - p.clip_lo, 1.0 + p.clip_hi
    rc = min(max(r, lo), hi)
    loss = max(-A * r, -A * rc)
    clipped_hi = A > 0 and r > hi
    clipped_lo = A < 0 and r < lo
    act = not (clipped_hi or clipped_lo)
    if p.dual_clip > 0 and A < 0:
        loss = min(loss, -A * p.dual_clip)
        if r > p.dual_clip:
            act = False
    inrange = abs(d) <= c
    dl_dlogp = (-A * r) if (act and inrange) else 0.0
    return r, loss, dl_dlogp, clipped_lo, clipped_hi


def _kl_k3(logp, ref, c):
    """k3 estimator of KL(pi || ref) at one token and its d/dlogp."""
    q0 = ref - logp
    q = min(max(q0, -c), c)
    k = math.exp(q) - q - 1.0
    dk = (1.0 - math.exp(q)) if abs(q0) <= c else 0.0
    return k, dk


def policy_loss_fwd_bwd(hidden, weight, cu_seqlens, mask, targets, old_logp, adv_seq,
                        params: LossParams | None = None, n_global=None,
                        inv_temperature=1.0, want_grads=True, ref_logp=None, n_seqs_global=None,
                        adv_per_token=False):
    """Forward + backward of the masked clipped-ratio loss (token mean by default).

    hidden [R, h]; weight [V, h]; old_logp [R]; adv_seq [S] (one advantage per
    sequence, broadcast to its rows). n_global = the loss normaliser N (masked
    tokens of the whole mini-batch over all ranks, reading #13); defaults to
    this batch's active count. loss_scale, when given, replaces 1/N (and
    1/S under seq_mean). ref_logp [R] is needed when kl_coef > 0;
    n_seqs_global = S for seq_mean (default: this batch's non-empty sequences).

    Returns dict(loss, loss_sum, logp, entropy, lse, g, ge, dH [R,h], dW [V,h],
    stats{loss_sum, ratio_sum, entropy_sum, kl_sum, objective, ratio_max,
    clip_lo_count, clip_hi_count, tokens}, err). Inactive rows: logp = entropy
    = lse = g = 0 and dH row = 0.
    """
    p = params or LossParams()
    W = _as64(weight)
    V, h = W.shape
    bk = bookkeeping(cu_seqlens, mask, targets, V)
    R = np.asarray(mask).shape[0]
    targets = np.asarray(targets).reshape(-1).astype(np.int64)
    old = _as64(old_logp).reshape(-1)
    adv = _as64(adv_seq).reshape(-1)
    ref = None if ref_logp is None else _as64(ref_logp).reshape(-1)
    if p.kl_coef > 0 and ref is None:
        raise ValueError("kl_coef > 0 needs ref_logp")
    N = bk["n_active"] if n_global is None else int(n_global)
    # per-token weights w_t
    S_count = np.bincount(bk["row_seq"][bk["active"]], minlength=max(len(adv), 1))
    if p.seq_mean:
        S = int((S_count > 0).sum()) if n_seqs_global is None else int(n_seqs_global)
        base = (1.0 / S if S > 0 else 0.0) if p.loss_scale is None else float(p.loss_scale)
    else:
        base = (1.0 / N if N > 0 else 0.0) if p.loss_scale is None else float(p.loss_scale)

    def weight_of(t):
        if p.seq_mean:
            return base / S_count[bk["row_seq"][t]]
        return base

    logp = np.zeros(R)
    ent = np.zeros(R)
    lse = np.zeros(R)
    g = np.zeros(R)
    ge = np.zeros(R)
    dH = np.zeros((R, h)) if want_grads else None
    dW = np.zeros((V, h)) if want_grads else None
    losses, ratios, ents, kls, objs = [], [], [], [], []
    ratio_max = 0.0
    n_lo = n_hi = 0
    act_rows = bk["active_idx"].astype(np.int64)
    for c0 in range(0, len(act_rows), _CHUNK):
        idx = act_rows[c0:c0 + _CHUNK]
        Hc = _as64(_take_rows(hidden, idx))
        Z, P, l, lp, e = _row_softmax_stats(Hc, W, targets[idx], inv_temperature)
        logp[idx], ent[idx], lse[idx] = lp, e, l
        gc = np.zeros(len(idx))
        gec = np.zeros(len(idx))
        for j, t in enumerate(idx):
            # GRPO: one advantage per sequence; PPO/GAE (NEXT-4): one per token
            A = float(adv[t] if adv_per_token else adv[bk["row_seq"][t]])
            r, loss, dldlp, clo, chi = _surrogate(float(lp[j]), float(old[t]), A, p)
            k, dk = (0.0, 0.0) if ref is None else _kl_k3(float(lp[j]), float(ref[t]),
                                                            p.logratio_clamp)
            w = weight_of(t)
            losses.append(loss)
            ratios.append(r)
            ents.append(float(e[j]))
            kls.append(k)
            objs.append(w * (loss + p.kl_coef * k - p.entropy_coef * float(e[j])))
            ratio_max = max(ratio_max, r)
            n_lo += int(clo)
            n_hi += int(chi)
            gc[j] = w * (dldlp + p.kl_coef * dk)
            gec[j] = w * p.entropy_coef
        g[idx] = gc
        ge[idx] = gec
        if want_grads:
            onehot = np.zeros_like(P)
            onehot[np.arange(len(idx)), targets[idx]] = 1.0
            Ez = (P * Z).sum(axis=1, keepdims=True)
            # d(-c H)/dz = +c p (z - E_p z)
            dZ = inv_temperature * (gc[:, None] * (onehot - P) + gec[:, None] * P * (Z - Ez))
            dH[idx] = dZ @ W
            dW += dZ.T @ Hc
    loss_sum = math.fsum(losses)
    objective = math.fsum(objs)
    stats = dict(loss_sum=loss_sum, ratio_sum=math.fsum(ratios), entropy_sum=math.fsum(ents),
                 kl_sum=math.fsum(kls), objective=objective, ratio_max=ratio_max,
                 clip_lo_count=n_lo, clip_hi_count=n_hi, tokens=len(act_rows))
    return dict(loss=objective, loss_sum=loss_sum, logp=logp, entropy=ent, lse=lse, g=g, ge=ge,
                dH=dH, dW=dW, stats=stats, err=bk["err"], active=bk["active"],
                row_seq=bk["row_seq"], n_active=bk["n_active"],
                n_seqs=int((S_count > 0).sum()))


# --------------------------------------------------------------------------
# NEXT-3: vocab-parallel head (tensor parallelism over the vocabulary, as
# the paper's actor TP 2/4/8). A rank holding vocab rows
# [off, off + V_p) reports per active row (compact order) the partial
#   m_p = max_{j in shard} z_j, s_p = sum e^{z_j - m_p},
#   u_p = sum e^{z_j - m_p} (z_j - m_p), zy_p = z_y if y in shard else 0;
# the log-softmax over the union of shards is then
#   lse = log sum_p e^{m_p} s_p,  E_p[z] = sum_p e^{m_p}(u_p + m_p s_p) / sum_p e^{m_p} s_p,
#   entropy = lse - E_p[z],  logp = sum_p zy_p - lse.
# --------------------------------------------------------------------------
def logprob_shard_partials(hidden, weight_shard, vocab_offset, vocab_total, cu_seqlens, mask,
                           targets, inv_temperature=1.0):
    """float64 [4, T] partials of one vocab shard for the active rows."""
    Ws = _as64(weight_shard)
    bk = bookkeeping(cu_seqlens, mask, targets, vocab_total)
    idx = bk["active_idx"].astype(np.int64)
    targets = np.asarray(targets).reshape(-1).astype(np.int64)
    out = np.zeros((4, len(idx)))
    for c0 in range(0, len(idx), _CHUNK):
        rows = idx[c0:c0 + _CHUNK]
        Z = (_as64(_take_rows(hidden, rows)) @ Ws.T) * inv_temperature
        m = Z.max(axis=1)
        E = np.exp(Z - m[:, None])
        out[0, c0:c0 + len(rows)] = m
        out[1, c0:c0 + len(rows)] = E.sum(axis=1)
        out[2, c0:c0 + len(rows)] = (E * (Z - m[:, None])).sum(axis=1)
        yl = targets[rows] - vocab_offset
        own = (yl >= 0) & (yl < Ws.shape[0])
        out[3, c0:c0 + len(rows)] = np.where(own, Z[np.arange(len(rows)), np.clip(yl, 0, Ws.shape[0] - 1)], 0.0)
    return out


def merge_shard_partials(parts):
    """parts [P, 4, T] -> dict(lse, entropy, logp) per compact row (float64)."""
    parts = np.asarray(parts, dtype=np.float64)
    m, s, u, zy = parts[:, 0], parts[:, 1], parts[:, 2], parts[:, 3]
    M = m.max(axis=0)                          # shift for range only
    w = np.exp(m - M) * s                      # e^{m_p - M} s_p
    S = w.sum(axis=0)
    lse = M + np.log(S)
    Ez = (np.exp(m - M) * (u + m * s)).sum(axis=0) / S
    return dict(lse=lse, entropy=lse - Ez, logp=zy.sum(axis=0) - lse)


# --------------------------------------------------------------------------
# NEXT-2: minibatch early stop and deferred normalisation.
# "Minibatch Early-Stop: We discard minibatches with too large importance
# ratio to stabilize training" (reading #29): the update of a
# mini-batch is discarded (gradient zeroed) when its largest token ratio
# exceeds max_ratio, or its token-mean ratio exceeds max_mean_ratio (a
# threshold <= 0 disables that test). Elastic pipelining lets
# micro-batches run before N is known: they use loss_scale = 1 and the
# accumulated gradient is multiplied by 1/N at the end (the loss is linear).
# --------------------------------------------------------------------------
def minibatch_early_stop(stats, max_ratio=0.0, max_mean_ratio=0.0):
    """True if the mini-batch's update is discarded.

    PARITY UNPINNED: the statistic and threshold are a reading (#29); PAPER.md
    prints nothing that fixes them, so no pin exists outside this rule."""
    if max_ratio > 0 and float(stats["ratio_max"]) > max_ratio:
        return True
    if max_mean_ratio > 0 and stats["tokens"] > 0 and \
            float(stats["ratio_sum"]) / float(stats["tokens"]) > max_mean_ratio:
        return True
    return False


def scale_by_inverse_count(x, count):
    """x / count (0 when count == 0): the deferred 1/N of streaming mode."""
    x = np.asarray(x, dtype=np.float64)
    return x * (1.0 / count) if count > 0 else np.zeros_like(x)
