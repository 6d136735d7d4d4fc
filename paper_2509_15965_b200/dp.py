"""Host-side data-parallel driver of the policy-loss head.

* ``lpt_shard``: whole prompt groups -> DP ranks, greedy least-loaded by token
  count (longest first). This is the paper's weighted load-balancing channel
  ("each data item can be assigned a weight value") used as a
  sharder; it keeps every GRPO group on one rank so advantages are
  rank-local. Bound: max - min load <= max item weight.
* ``pack_micro_batches``: whole sequences packed greedily, in order, into
  micro-batches of at most ``budget`` rows ("the micro-batch defines
  forward/backward units, while the global-batch determines when model
  updates occur").
* ``PolicyLossStep``: one mini-batch step on this rank: N all-reduce, GRPO
  advantages, every micro-batch through ``rl_policy_loss_fwd_bwd``, dW SUM
  all-reduce (the loss is normalised by the global N, so gradients add;
  a DDP-style mean would be off by world_size), stats all-reduce.

Collectives go through torch.distributed (NCCL over NVLink on the B200 box,
gloo on CPU in the tests); nothing else crosses ranks. ``collective="symm"``
replaces the dW all-reduce (the one exchange that follows a GEMM) by the
reduce-scatter fused into the last micro-batch's dW GEMM epilogue plus an
NVLink all-gather over torch symmetric memory.
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass, field

import numpy as np


def lpt_shard(weights, world: int):
    """Assign items (e.g. prompt groups, weight = token count) to ``world``
    bins: heaviest first onto the currently lightest bin (ties: lower bin id,
    then lower item id). Returns (list of item-id lists per bin, loads)."""
    weights = np.asarray(weights, dtype=np.int64)
    order = sorted(range(len(weights)), key=lambda i: (-int(weights[i]), i))
    heap = [(0, r) for r in range(world)]
    bins = [[] for _ in range(world)]
    loads = np.zeros(world, dtype=np.int64)
    for i in order:
        load, r = heapq.heappop(heap)
        bins[r].append(i)
        loads[r] = load + int(weights[i])
        heapq.heappush(heap, (int(loads[r]), r))
    for b in bins:
        b.sort()
    return bins, loads


def pack_micro_batches(seq_rows, budget: int):
    """Contiguous [s0, s1) sequence ranges, each <= budget rows (a single
    longer sequence gets a micro-batch of its own)."""
    out, s0, rows = [], 0, 0
    for s, n in enumerate(np.asarray(seq_rows, dtype=np.int64)):
        if s > s0 and rows + int(n) > budget:
            out.append((s0, s))
            s0, rows = s, 0
        rows += int(n)
    if len(seq_rows) > s0 or not out:
        out.append((s0, len(seq_rows)))
    return out


def group_has_gradient(layout):
    """Per group: True unless all its rewards are equal -- a GRPO group whose
    rewards are all equal has A = 0 for every member, so its tokens need the
    forward only (the backward GEMMs skip rows with dL/dlogp = 0). A host-side
    scheduling estimate, not numerics."""
    G = layout.num_groups
    r = np.asarray(layout.rewards, dtype=np.float64)
    g = np.asarray(layout.group_of_seq, dtype=np.int64)
    mx = np.full(G, -np.inf)
    mn = np.full(G, np.inf)
    np.maximum.at(mx, g, r)
    np.minimum.at(mn, g, r)
    return mx > mn


def shard_layout(layout, rank: int, world: int, split_groups: bool = False,
                 work_weighted: bool = True):
    """This rank's sequences, LPT by work: whole groups (advantages rank-local),
    or with ``split_groups`` single sequences (finer balance; the group
    statistics are then all-reduced). The weight of a group is
    its response tokens x 3 (forward 2hV + backward 4hV per token) when its
    rewards differ, x 1 when they are all equal (A = 0: forward only, the
    backward skips those rows); ``work_weighted=False`` weighs tokens only.
    The returned loads are the weights, in those units."""
    G = layout.num_groups
    cu = layout.cu_seqlens.astype(np.int64)
    seq_tokens = np.add.reduceat(layout.mask.astype(np.int64), cu[:-1]) \
        if layout.num_rows else np.zeros(layout.num_seqs, np.int64)
    seq_tokens = np.where(cu[1:] > cu[:-1], seq_tokens, 0)
    if work_weighted and G > 0:
        seq_tokens = seq_tokens * np.where(group_has_gradient(layout)[layout.group_of_seq], 3, 1)
    if split_groups:
        bins, loads = lpt_shard(seq_tokens, world)
        return list(bins[rank]), loads
    g_tokens = np.bincount(layout.group_of_seq, weights=seq_tokens, minlength=G).astype(np.int64)
    bins, loads = lpt_shard(g_tokens, world)
    mine = set(bins[rank])
    seqs = [s for s in range(layout.num_seqs) if int(layout.group_of_seq[s]) in mine]
    return seqs, loads


# ------------------------------------------------------------ collectives ----
def _world(group=None) -> int:
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group)
    return 1


def _symm_dw_buffers(R, weight, group):
    """C3 over NVLink peer memory: dW [V, h] and the staging
    buffer [P, ceil(V/P), h] (fp32) in torch symmetric memory. The last
    micro-batch's dW epilogue stores (partial + tile) into the owners' staging
    slots; _symm_dw_finish sums them in rank order and broadcasts."""
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm_mem
    V, h = weight.shape
    dev = weight.device
    grp = group if group is not None else dist.group.WORLD
    P = _world(group)
    rows = -(-V // P)
    t = symm_mem.empty(V * h, dtype=torch.float32, device=dev)
    hdl = symm_mem.rendezvous(t, grp)
    stg = symm_mem.empty(P * rows * h, dtype=torch.float32, device=dev)
    hdl_s = symm_mem.rendezvous(stg, grp)
    pg = R.PeerGroup(hdl.rank, P, rows, list(hdl_s.buffer_ptrs))
    return t.view(V, h), stg, pg, list(hdl.buffer_ptrs), hdl


def _symm_dw_finish(R, hdl, staging, grad_w, pg, out_peers, shard=False):
    """shard=False: every rank ends with the whole reduced dW (multicast or
    P2P broadcast of each owner's slab). shard=True: each rank keeps only its
    own summed slab (FSDP / ZeRO-2 gradient semantics: the optimizer updates
    the owned rows; the other rows of grad_w hold this rank's local partial)."""
    hdl.barrier(channel=0)         # every rank's slots in every staging buffer written
    if shard:
        own = [p if q == pg.rank else 0 for q, p in enumerate(out_peers)]
        R.rl_reduce_bcast_rows_f32(staging, grad_w, pg.rank, pg.world, pg.rows_per_rank, own)
    else:
        R.rl_reduce_bcast_rows_f32(staging, grad_w, pg.rank, pg.world, pg.rows_per_rank,
                                   out_peers, mc_ptr=hdl.multicast_ptr)
    hdl.barrier(channel=0)         # every slab stored (staging free for the next step)


def shard_rows(V: int, world: int, rank: int):
    """Rows [r0, r1) of dW [V, h] that rank owns in the fused reduce-scatter
    (rows_per_rank = ceil(V / world); the header's owner(j) rule)."""
    rows = -(-V // world)
    r0 = min(rank * rows, V)
    return r0, min(r0 + rows, V)


def all_reduce_(t, op="sum", group=None):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX,
                        group=group)
    return t


def reduce_stats_(stats_u8, group=None, combine=None):
    """C4: ONE all-gather of every rank's 72-B rl_loss_stats, combined on the
    device in rank order by rl_loss_stats_reduce (fp64/int64 fields summed,
    ratio_max maxed; deterministic) -- instead of three all-reduces (SUM
    fp64, MAX fp32, SUM int64). ``combine(gathered, out)`` replaces the
    combiner (the CPU gloo tests pass a host one; there is no librlhead
    kernel on a CPU tensor)."""
    import torch
    import torch.distributed as dist
    P = _world(group)
    if P <= 1:
        return stats_u8
    gathered = torch.empty(P * stats_u8.numel(), dtype=torch.uint8, device=stats_u8.device)
    dist.all_gather_into_tensor(gathered, stats_u8, group=group)
    if combine is None:
        from . import rlhead as R
        combine = R.rl_loss_stats_reduce
    combine(gathered, stats_u8)
    return stats_u8


class PhaseTimer:
    """Per-phase device time of a step (CUDA events on the current stream):
    record(name) closes the phase that started at the previous record. Used
    to break the multi-GPU step into its fixed costs (bench --phases)."""

    def __init__(self, enabled: bool):
        self.enabled = enabled
        self.marks = []

    def reset(self):
        self.marks = []

    def record(self, name):
        if not self.enabled:
            return
        import torch
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.marks.append((name, e))

    def ms(self) -> dict:
        out = {}
        for (_, a), (name, b) in zip(self.marks[:-1], self.marks[1:]):
            out[name] = out.get(name, 0.0) + a.elapsed_time(b)
        return out


@dataclass
class DeviceBatch:
    """One rank's packed batch resident on the device, plus its micro-batches."""
    cu: object            # int32 [S+1] (whole local batch)
    targets: object       # int32 [R]
    mask: object          # uint8 [R]
    gos: object           # int32 [S] local group ids
    rewards: object       # float32 [S]
    num_groups: int
    mbs: list             # [(s0, s1, r0, r1, cu_mb tensor)]
    num_rows: int
    num_tokens: int
    seq_rows: np.ndarray = field(default=None)


def device_batch(layout, mb_rows: int, device="cuda", global_groups: bool = False) -> DeviceBatch:
    """global_groups: keep the mini-batch-wide group ids (split-group mode, whose
    group statistics are all-reduced by id); else local ids 0..G'-1."""
    import torch
    cu_np = layout.cu_seqlens.astype(np.int64)
    seq_rows = cu_np[1:] - cu_np[:-1]
    if global_groups:
        uniq = np.arange(layout.num_groups)
        gos_local = np.asarray(layout.group_of_seq)
    else:  # local group ids 0..G'-1 (keeps the GRPO launch small)
        uniq, gos_local = np.unique(layout.group_of_seq, return_inverse=True)
    mbs = []
    for s0, s1 in pack_micro_batches(seq_rows, mb_rows):
        r0, r1 = int(cu_np[s0]), int(cu_np[s1])
        cu_mb = torch.as_tensor((cu_np[s0:s1 + 1] - r0).astype(np.int32), device=device)
        mbs.append((s0, s1, r0, r1, cu_mb))
    return DeviceBatch(
        cu=torch.as_tensor(layout.cu_seqlens, device=device),
        targets=torch.as_tensor(layout.targets, device=device),
        mask=torch.as_tensor(layout.mask, device=device),
        gos=torch.as_tensor(gos_local.astype(np.int32), device=device),
        rewards=torch.as_tensor(layout.rewards, device=device),
        num_groups=len(uniq), mbs=mbs, num_rows=layout.num_rows,
        num_tokens=layout.num_tokens, seq_rows=seq_rows)


class PolicyLossStep:
    """One GRPO mini-batch step of the head on this rank."""

    def __init__(self, head, weight, db: DeviceBatch, params=None, group=None,
                 advantage: str = "grpo", collective: str = "nccl", split_groups: bool = False,
                 want_entropy: bool = False, phases: bool = False, pipeline: bool = False,
                 dw_output: str = "full"):
        import torch
        from . import rlhead as R
        self.R = R
        if dw_output not in ("full", "shard"):
            raise ValueError(f"unknown dw_output {dw_output!r}")
        # "shard": after run(), grad_w_shard (rows shard_rows(V, world, rank))
        # holds this rank's slab of the reduced dW and no broadcast runs
        # (symm: the fused reduce-scatter's owner sum only; nccl: one
        # reduce_scatter over the dW rows padded to world x ceil(V / world))
        self.dw_output = dw_output
        if advantage not in ("grpo", "reinforce_pp"):
            raise ValueError(f"unknown advantage {advantage!r}")
        if collective not in ("nccl", "symm", "nvls"):
            raise ValueError(f"unknown collective {collective!r}")
        self.advantage = advantage
        self.split_groups = split_groups
        self.head, self.W, self.db = head, weight, db
        self.params = params or R.LossParams()
        self.group = group
        dev = weight.device
        # C1: (N, S) in one int64[2] tensor -> one all-reduce per step
        self.counts = torch.zeros(2, dtype=torch.int64, device=dev)
        self.n_global = self.counts[0:1]
        self.n_seqs = self.counts[1:2]
        self.params.n_tokens_global = self.n_global
        self.params.n_seqs_global = self.n_seqs
        self.adv = torch.empty(max(db.cu.shape[0] - 1, 1), dtype=torch.float32, device=dev)
        self.symm = None
        P = _world(group)
        rank = 0
        if P > 1:
            import torch.distributed as dist
            rank = dist.get_rank(group)
        V, h = weight.shape
        self._gw_pad = None
        self.nvls = None
        if collective == "symm" and P > 1:
            self.grad_w, self.staging, self.peer_group, self.out_peers, self.symm = \
                _symm_dw_buffers(R, weight, group)
        elif collective == "nvls" and P > 1:
            # dW in symmetric memory, summed after the last dW GEMM by
            # rl_dw_reduce_rows_f32 (NVLS in-switch reduce; P2P without NVLS)
            import torch.distributed._symmetric_memory as symm_mem
            import torch.distributed as dist
            t = symm_mem.empty(V * h, dtype=torch.float32, device=dev)
            self.nvls = symm_mem.rendezvous(t, group if group is not None else dist.group.WORLD)
            self.grad_w = t.view(V, h)
        elif dw_output == "shard" and P > 1:
            # rows padded to P x ceil(V / P) so reduce_scatter's chunks are equal
            self._gw_pad = torch.zeros(P * -(-V // P), h, dtype=torch.float32, device=dev)
            self.grad_w = self._gw_pad[:V]
        else:
            self.grad_w = torch.zeros(V, h, dtype=torch.float32, device=dev)
        r0, r1 = shard_rows(V, P, rank)
        self.grad_w_shard = self.grad_w[r0:r1]
        if self._gw_pad is not None:
            self._shard_out = torch.empty(-(-V // P), h, dtype=torch.float32, device=dev)
        self.stats = R.new_stats(dev)
        self.stats_local = R.new_stats(dev)
        self.logp = torch.empty(max(db.num_rows, 1), dtype=torch.float32, device=dev)
        self.entropy = (torch.empty(max(db.num_rows, 1), dtype=torch.float32, device=dev)
                        if want_entropy else None)
        self.ws = R.Workspace(dev)
        self.ws_prep = R.Workspace(dev)
        self.timer = PhaseTimer(phases)
        # two-stream micro-batch pipeline (split fwd/bwd API, two workspaces)
        self.pipeline = bool(pipeline) and head.dtype == "bf16"
        if self.pipeline:
            self.ws_pipe = [R.Workspace(dev), R.Workspace(dev)]
            self.aux_stream = torch.cuda.Stream(device=dev)

    def _rs_group(self, last: int):
        """The fused reduce-scatter's peer group for the last micro-batch; with a
        single micro-batch grad_w holds no partial yet, so the epilogue need not
        read it (no_partial)."""
        if last == 0:
            import dataclasses
            return dataclasses.replace(self.peer_group, no_partial=True)
        return self.peer_group

    def count_tokens(self):
        """N = masked tokens (and S = non-empty sequences, for seq-mean
        aggregation) of the whole mini-batch over all ranks."""
        R = self.R
        self.counts.zero_()
        R.rl_batch_prepare(self.head, R.Batch(self.db.cu, self.db.targets, self.db.mask),
                           n_accum=self.n_global, nseq_accum=self.n_seqs, ws=self.ws_prep)
        all_reduce_(self.counts, "sum", self.group)

    def advantages(self):
        """GRPO (groups are rank-local under LPT sharding) or the REINFORCE++
        batch normalisation, whose 5 batch statistics span all ranks (C2')."""
        R, db = self.R, self.db
        if self.advantage == "grpo" and not self.split_groups:
            R.rl_grpo_advantage(db.rewards, db.gos, db.num_groups, self.adv)
            return
        import torch
        dev = self.adv.device
        G = max(db.num_groups, 1)
        gsum = torch.empty(G, 3, dtype=torch.float64, device=dev)
        gmax = torch.empty(G, 2, dtype=torch.float64, device=dev)
        R.rl_grpo_group_stats(db.rewards, db.gos, db.num_groups, gsum, gmax)
        if self.split_groups:          # C2: a group's members may sit on several ranks
            all_reduce_(gsum, "sum", self.group)
            all_reduce_(gmax, "max", self.group)
        if self.advantage == "grpo":
            R.rl_grpo_advantage(db.rewards, db.gos, db.num_groups, self.adv, sum_stats=gsum,
                                max_stats=gmax)
            return
        bst = torch.empty(5, dtype=torch.float64, device=dev)
        R.rl_batch_norm_advantage(db.rewards, db.gos, db.num_groups, None, group_baseline=True,
                                  group_sum_stats=gsum, batch_stats_out=bst)
        all_reduce_(bst[:3], "sum", self.group)
        all_reduce_(bst[3:], "max", self.group)
        R.rl_batch_norm_advantage(db.rewards, db.gos, db.num_groups, self.adv,
                                  group_baseline=True, group_sum_stats=gsum, batch_stats_in=bst)

    def run(self, hidden, old_logp, grad_hidden, hidden_for_mb=None, after_mb=None):
        """hidden [R, h] (or ``hidden_for_mb(i)`` -> the micro-batch's rows, for
        streaming). grad_hidden is [R, h], or a reused buffer of at least the
        largest micro-batch (its rows then hold the last micro-batch's dH,
        which the trunk backward would consume before the next one)."""
        R, tm = self.R, self.timer
        tm.reset()
        tm.record("start")
        self.grad_w.zero_()
        self.stats.zero_()
        tm.record("zero_dw")
        self.count_tokens()
        tm.record("count_allreduce")
        self.advantages()
        tm.record("advantage")
        full_gh = grad_hidden.shape[0] >= self.db.num_rows
        last = len(self.db.mbs) - 1
        if self.pipeline:
            self._run_pipelined(hidden, old_logp, grad_hidden, full_gh, hidden_for_mb, after_mb)
        for i, (s0, s1, r0, r1, cu_mb) in enumerate([] if self.pipeline else self.db.mbs):
            hs = hidden_for_mb(i) if hidden_for_mb else hidden[r0:r1]
            gh = grad_hidden[r0:r1] if full_gh else grad_hidden[:r1 - r0]
            b = R.Batch(cu_mb, self.db.targets[r0:r1], self.db.mask[r0:r1], num_rows=r1 - r0)
            self.params.dw_reduce_scatter = (self._rs_group(last) if self.symm is not None and
                                             i == last else None)
            R.rl_policy_loss_fwd_bwd(self.head, hs, self.W, b, old_logp[r0:r1], self.adv[s0:s1],
                                     self.params, self.logp[r0:r1], gh, self.grad_w,
                                     entropy=None if self.entropy is None else self.entropy[r0:r1],
                                     stats=self.stats, ws=self.ws)
            if after_mb:
                after_mb(i)
        self.params.dw_reduce_scatter = None
        tm.record("micro_batches")
        if self.symm is not None:
            _symm_dw_finish(R, self.symm, self.staging, self.grad_w, self.peer_group,
                            self.out_peers, shard=self.dw_output == "shard")
        elif self.nvls is not None:
            hdl = self.nvls
            hdl.barrier(channel=0)      # every rank's dW GEMMs done
            R.rl_dw_reduce_rows_f32(self.grad_w, hdl.rank, hdl.world_size,
                                    -(-self.grad_w.shape[0] // hdl.world_size),
                                    list(hdl.buffer_ptrs), mc_ptr=hdl.multicast_ptr or 0,
                                    broadcast=self.dw_output == "full")
            hdl.barrier(channel=0)      # every owned slab summed (and broadcast)
        elif self._gw_pad is not None:
            import torch.distributed as dist
            dist.reduce_scatter_tensor(self._shard_out, self._gw_pad, group=self.group)
            self.grad_w_shard.copy_(self._shard_out[:self.grad_w_shard.shape[0]])
        else:
            all_reduce_(self.grad_w, "sum", self.group)
        tm.record("dw_reduce")
        self.stats_local.copy_(self.stats)    # this rank's own sums (for reporting)
        reduce_stats_(self.stats, self.group)
        tm.record("stats_gather")
        return self.stats


    def _run_pipelined(self, hidden, old_logp, grad_hidden, full_gh, hidden_for_mb, after_mb):
        """Micro-batches through the split API on two streams and two workspaces:
        fwd(i) (H1-H5) on the current stream, bwd(i) (H6-H8) on an auxiliary
        stream once fwd(i) is done, so bwd(i)'s memory-bound dZ pass runs beside
        fwd(i+1)'s GEMM; fwd(i+2) waits for bwd(i) (its workspace). dW and the
        stats accumulate in stream order as in the serial loop (same values)."""
        import torch
        R = self.R
        main = torch.cuda.current_stream()
        aux = self.aux_stream
        aux.wait_stream(main)                 # dW/stats zeroed, N and A ready
        last = len(self.db.mbs) - 1
        ev_b = {}
        for i, (s0, s1, r0, r1, cu_mb) in enumerate(self.db.mbs):
            ws = self.ws_pipe[i % 2]
            if i >= 2:
                main.wait_event(ev_b.pop(i - 2))
            hs = hidden_for_mb(i) if hidden_for_mb else hidden[r0:r1]
            gh = grad_hidden[r0:r1] if full_gh else grad_hidden[:r1 - r0]
            b = R.Batch(cu_mb, self.db.targets[r0:r1], self.db.mask[r0:r1], num_rows=r1 - r0)
            args = (self.head, hs, self.W, b, old_logp[r0:r1], self.adv[s0:s1], self.params,
                    self.logp[r0:r1], gh, self.grad_w)
            kw = dict(entropy=None if self.entropy is None else self.entropy[r0:r1],
                      stats=self.stats, ws=ws)
            self.params.dw_reduce_scatter = None
            R.rl_policy_loss_fwd(*args, **kw)
            ev_f = torch.cuda.Event()
            ev_f.record(main)
            if after_mb:
                after_mb(i)                   # hidden rows are in the workspace now
            with torch.cuda.stream(aux):
                aux.wait_event(ev_f)
                self.params.dw_reduce_scatter = (self._rs_group(last)
                                                 if self.symm is not None and i == last else None)
                R.rl_policy_loss_bwd(*args, **kw, stream=aux)
                ev_b[i] = torch.cuda.Event()
                ev_b[i].record(aux)
        main.wait_stream(aux)


class StreamingPolicyLoss:
    """Micro-batch streaming interface (NEXT-2; P:L433-436 elastic pipelining:
    "output data can be forwarded once a configured size of data batch is
    ready ... the micro-batch defines forward/backward units, while the
    global-batch determines when model updates occur").

    Micro-batches are fed as they arrive (e.g. from a data channel), before the
    global batch -- and so N -- is known: each runs at once with loss_scale = 1
    while its token count accumulates on the device. ``finish()`` all-reduces
    N, applies the deferred 1/N to dW (the caller applies the same factor to
    the trunk gradients it accumulated from each micro-batch's dL/dH),
    all-reduces dW and the stats, and evaluates the minibatch early stop
    ("discard minibatches with too large importance ratio") on the
    device: ``stop_flag`` = 1 and dW = 0 when the update is discarded.
    """

    def __init__(self, head, weight, params=None, group=None, max_ratio: float = 0.0,
                 max_mean_ratio: float = 0.0, collective: str = "nccl"):
        import torch
        from . import rlhead as R
        self.R = R
        self.head, self.W, self.group = head, weight, group
        self.params = params or R.LossParams()
        self.params.loss_scale = 1.0
        self.params.n_tokens_global = None
        if self.params.seq_mean:
            raise ValueError("streaming mode defers 1/N: token-mean aggregation only")
        dev = weight.device
        self.max_ratio, self.max_mean_ratio = max_ratio, max_mean_ratio
        self.n_tokens = torch.zeros(1, dtype=torch.int64, device=dev)
        self.stop_flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self.symm = None
        if collective == "symm" and _world(group) > 1:
            self.grad_w, self.staging, self.peer_group, self.out_peers, self.symm = \
                _symm_dw_buffers(R, weight, group)
        else:
            self.grad_w = torch.zeros(weight.shape[0], weight.shape[1], dtype=torch.float32,
                                      device=dev)
        self.sent = False
        self.stats = R.new_stats(dev)
        self.ws = R.Workspace(dev)
        self.ws_prep = R.Workspace(dev)

    def begin(self):
        self.n_tokens.zero_()
        self.stop_flag.zero_()
        self.grad_w.zero_()
        self.stats.zero_()
        self.sent = False

    def feed(self, hidden, batch, old_logp, adv, logp, grad_hidden, entropy=None,
             last: bool = False):
        """last=True on this rank's final micro-batch of the global batch lets its
        dW epilogue run the fused reduce-scatter (collective="symm")."""
        R = self.R
        if self.sent:
            # the fused reduce-scatter already shipped this rank's partial: a
            # later micro-batch's dW would never reach the reduction
            raise RuntimeError("feed() after the micro-batch marked last=True; call begin() "
                               "to start the next global batch")
        R.rl_batch_prepare(self.head, batch, n_accum=self.n_tokens, ws=self.ws_prep)
        fuse = self.symm is not None and last and not self.sent
        self.params.dw_reduce_scatter = self.peer_group if fuse else None
        R.rl_policy_loss_fwd_bwd(self.head, hidden, self.W, batch, old_logp, adv, self.params,
                                 logp, grad_hidden, self.grad_w, entropy=entropy,
                                 stats=self.stats, ws=self.ws)
        self.params.dw_reduce_scatter = None
        self.sent = self.sent or fuse

    def _send_partial(self):
        """No last=True feed on this rank: send the accumulated partial through a
        one-row, fully masked micro-batch (its dW GEMM has K = 0 and only ships
        the partial to the owners)."""
        import torch
        R, dev, h = self.R, self.grad_w.device, self.W.shape[1]
        dt = self.W.dtype
        b = R.Batch(torch.tensor([0, 1], dtype=torch.int32, device=dev),
                    torch.zeros(1, dtype=torch.int32, device=dev),
                    torch.zeros(1, dtype=torch.uint8, device=dev))
        hid = torch.zeros(1, h, dtype=dt, device=dev)
        one = torch.zeros(1, device=dev)
        self.params.dw_reduce_scatter = self.peer_group
        R.rl_policy_loss_fwd_bwd(self.head, hid, self.W, b, one, one, self.params,
                                 torch.empty(1, device=dev), torch.empty_like(hid), self.grad_w,
                                 ws=self.ws)
        self.params.dw_reduce_scatter = None
        self.sent = True

    def finish(self):
        R = self.R
        all_reduce_(self.n_tokens, "sum", self.group)
        if self.symm is not None:
            if not self.sent:
                self._send_partial()
            _symm_dw_finish(R, self.symm, self.staging, self.grad_w, self.peer_group,
                            self.out_peers)
        else:
            all_reduce_(self.grad_w, "sum", self.group)
        R.rl_scale_by_inverse_count(self.grad_w, self.n_tokens)
        reduce_stats_(self.stats, self.group)
        R.rl_minibatch_early_stop(self.stats, self.stop_flag, self.grad_w, self.max_ratio,
                                  self.max_mean_ratio)
        return self.stats
