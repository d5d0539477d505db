"""One synchronous training step of the paper's large-vocabulary LM output path (§4.2, §6.4),
composed from the libtfs C-ABI calls.  One process per GPU; GPU r is both replica r (a worker)
and shard r of the vocabulary-sharded tables (a "PS task", R-26).

Per step on rank r:
  sample      s = first S distinct log-uniform draws            tfs_log_uniform_sample
  Part        x and y||s by owner = id mod R                    tfs_partition
  route ids   all-to-all-v over NCCL (Send/Recv worker->PS)     Router
  Gather      rows of the local shard for every requester       tfs_gather
  route rows  all-to-all-v back                                             Router
  Stitch      h, W_true, W_s, b rows in token order             tfs_stitch
  softmax     loss + dh, dW_true, dW_s, db                      tfs_sampled_softmax_fwd_bwd
  reduce      sum gradient rows per id, grouped by owner        tfs_sort_reduce
  route grads all-to-all-v to the owners                                    Router
  SGD         T[id] -= lr * sum over sources, fixed order       tfs_scatter_add_sgd

With R = 1 the routes are the identity and the whole step is free of host synchronisation,
so it is captured once into a CUDA graph and replayed (the sampler reads its step counter from
device memory, advanced inside the graph).  Part and Stitch are identity maps then (Gather
writes rows in place), and the SGD is split into a plan (id sort, tfs_scatter_plan) built on a
side stream while the softmax runs, and its apply (tfs_scatter_add_sgd_planned).  With R > 1 each route needs its counts on the host
(an all-to-all of R counts, then one device->host read).
"""
from __future__ import annotations

import contextlib
from dataclasses import dataclass

import torch

from . import ops
from ._lib import TFS_BF16, TFS_F32, TFS_REMOVE_ACCIDENTAL_HITS, TFS_SUBTRACT_LOG_Q


@dataclass
class StepConfig:
    vocab: int
    dim: int
    tokens: int                 # B per replica
    num_sampled: int            # S per replica (ignored when full_softmax)
    lr: float = 0.1
    seed: int = 7
    unique: bool = True
    flags: int = TFS_SUBTRACT_LOG_Q | TFS_REMOVE_ACCIDENTAL_HITS
    operand_dtype: int = TFS_BF16
    # candidates = all V classes (config F).  R > 1: the vocabulary-sharded full softmax of
    # P:706-714 (W / b never move; every shard scores all R*B tokens against its classes).
    full_softmax: bool = False
    # R > 1 fixed-capacity routes: distinct ids per (requester, owner) pair are expected near
    # n / R (ids mod R); slots per owner = min(n, ceil(route_slack * n / R) + route_pad).
    # An overflow is reported as TFS_ERR_CAPACITY (never silent).
    route_slack: float = 1.25
    route_pad: int = 64
    # R > 1 transport: "p2p" = one-sided NVLink (peer loads of the owners' rows, id / gradient
    # stores into the owners' inboxes, device barriers; tables and inboxes in symmetric memory)
    # or "nccl" = equal-split all-to-alls of slot regions.
    route: str = "p2p"
    # sparse optimizer of the ScatterAdd step: "sgd" (the paper's
    # experiments), "momentum" (mu) or "adagrad" (accumulators start at adagrad_init); R = 1
    optimizer: str = "sgd"
    momentum: float = 0.9
    adagrad_init: float = 0.1


class Router:
    """All-to-all-v over a torch.distributed process group (NCCL on GPUs, gloo on CPU).

    Payload rows destined to rank o are contiguous and ordered by o (what Part and
    sort-reduce produce); the receive buffer is ordered by source rank (R-2, O4)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.R = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.group_name = (group if group is not None else dist.group.WORLD).group_name

    def exchange_counts(self, send_counts: torch.Tensor):
        """send_counts int64 [R, k]: row o = counts of k payload kinds destined to rank o.
        Returns (send, recv) as k lists of R Python ints (one device->host read)."""
        recv = torch.empty_like(send_counts)
        self.dist.all_to_all_single(recv, send_counts.contiguous(), group=self.group)
        both = torch.stack([send_counts, recv]).cpu().tolist()
        k = send_counts.shape[1]
        send = [[both[0][o][j] for o in range(self.R)] for j in range(k)]
        rcv = [[both[1][o][j] for o in range(self.R)] for j in range(k)]
        return send, rcv

    def a2a(self, out: torch.Tensor, inp: torch.Tensor):
        """Equal-split all-to-all of [R, ...] buffers (fixed size: no host counts, capturable)."""
        self.dist.all_to_all_single(out, inp, group=self.group)
        return out

    def route(self, payload: torch.Tensor, send_counts, recv_counts) -> torch.Tensor:
        n_send = sum(send_counts)
        out = torch.empty((sum(recv_counts),) + tuple(payload.shape[1:]), dtype=payload.dtype,
                          device=payload.device)
        self.dist.all_to_all_single(out, payload[:n_send].contiguous(),
                                    output_split_sizes=list(recv_counts),
                                    input_split_sizes=list(send_counts), group=self.group)
        return out


class _PhaseTimer:
    SPIN_CYCLES = 200_000  # ~0.1 ms at 1.9 GHz: lets the host queue the phase ahead

    def __init__(self, st, name):
        self.st, self.name = st, name

    def __enter__(self):
        torch.cuda._sleep(self.SPIN_CYCLES)
        self.start = torch.cuda.Event(enable_timing=True)
        self.end = torch.cuda.Event(enable_timing=True)
        self.start.record()

    def __exit__(self, *exc):
        self.end.record()
        self.st.phase_events.append((self.name, self.start, self.end))
        return False


class ShardedStep:
    """Owns rank r's shard of E, W, b and the per-step buffers; ``run`` does one step."""

    def __init__(self, cfg: StepConfig, E: torch.Tensor, W: torch.Tensor, b: torch.Tensor,
                 router: Router | None = None):
        self.cfg = cfg
        self.E, self.W, self.b = E, W, b
        self.router = router
        self.R = router.R if router is not None else 1
        self.rank = router.rank if router is not None else 0
        dev = E.device
        self.device = dev
        V, d, B = cfg.vocab, cfg.dim, cfg.tokens
        self.full_sharded = cfg.full_softmax and self.R > 1
        if self.full_sharded:
            if cfg.route != "p2p" or cfg.operand_dtype != TFS_BF16 or cfg.optimizer != "sgd":
                raise ValueError("the sharded full softmax runs over p2p with bf16 operands and "
                                 "SGD")
            S = 0  # no candidate rows travel: the softmax runs where W lives
        else:
            S = V if cfg.full_softmax else cfg.num_sampled
        self.B, self.S, self.d = B, S, d
        self.c = 1.0 / (self.R * B)  # R-13: mean over the global batch
        f32 = dict(dtype=torch.float32, device=dev)
        i64 = dict(dtype=torch.int64, device=dev)
        self.x = torch.zeros(B, **i64)
        self.y = torch.zeros(B, **i64)
        self.qw = torch.zeros(B + S, **i64)          # y || s
        self.err = ops.ErrorSlot(dev)
        self.step_dev = torch.zeros(1, **i64)
        if cfg.full_softmax:
            self.qw[B:] = torch.arange(S, **i64)
            self.les = torch.zeros(S, **f32)
            self.ley = torch.zeros(B, **f32)
            self.num_tries = torch.full((1,), V, **i64)
            self.flags = TFS_REMOVE_ACCIDENTAL_HITS
            self.sampler = None
        else:
            self.sampler = ops.Sampler(V, S, cfg.unique, dev)
            self.les = torch.empty(S, **f32)
            self.ley = torch.empty(B, **f32)
            self.num_tries = torch.empty(1, **i64)
            self.flags = cfg.flags
        R = self.R
        L = ops._lib.lib()
        self.side_stream = torch.cuda.Stream(device=dev)
        # bf16 operand mode: the Gathers round h / W rows to bf16 on the way (the only values
        # the bf16 softmax consumes), halving their writes and skipping its conversion pass.
        bf16_rows = cfg.operand_dtype == TFS_BF16 and (self.R == 1 or cfg.route == "p2p")
        rdt = dict(dtype=torch.bfloat16 if bf16_rows else torch.float32, device=dev)
        self.h = torch.empty((B, d), **rdt)
        self.w_rows = torch.empty((B + S, d), **rdt)
        self.b_rows = torch.empty(B + S, **f32)
        self.ssm_out = {"loss": torch.empty(B, **f32), "lse": torch.empty(B, **f32),
                        "loss_sum": torch.zeros(1, **f32), "dh": torch.empty((B, d), **f32)}
        self.dw = torch.empty((B + S, d), **f32)    # dW_true || dW_s (aligned with y || s)
        self.db = torch.empty(B + S, **f32)
        self.ssm_out.update({"dw_true": self.dw[:B], "db_true": self.db[:B], "dw_s": self.dw[B:],
                             "db_s": self.db[B:]})
        self.ws_ssm = ops.ssm_workspace(B, S, d, cfg.operand_dtype, dev, V)
        if cfg.optimizer not in ("sgd", "momentum", "adagrad"):
            raise ValueError(f"unknown optimizer {cfg.optimizer!r}")
        if cfg.optimizer != "sgd" and R != 1:
            raise ValueError("sparse Momentum / Adagrad are wired into the R = 1 step")
        self.slots = None
        if cfg.optimizer != "sgd":  # fp32 slot tables shaped like E, W, b
            init = 0.0 if cfg.optimizer == "momentum" else cfg.adagrad_init
            self.slots = tuple(torch.full_like(t, init) for t in (E, W, b))
        if R == 1:
            self.plan_e = ops.ScatterPlan(B, E.shape[0], d, dev)
            self.plan_w = ops.ScatterPlan(B + S, W.shape[0], d, dev)
            self.ev = {k: torch.cuda.Event() for k in ("h", "q", "plan_w", "ssm")}
        else:
            # Slot layout of the three exchanges (ids forward, rows forward, gradients back):
            # region o of each buffer goes to / comes from rank o.
            #   ids   int64 [R, cap_e + cap_w]          E ids | W ids
            #   rows  f32   [R, rstride]                 E rows | W rows | b   (rows of d)
            #   grads f32   [R, rstride]                 dE rows | dW rows | db
            if cfg.route not in ("p2p", "nccl"):
                raise ValueError(f"unknown route transport {cfg.route!r}")
            if cfg.route == "p2p":
                self._symm_tables()
            if self.full_sharded:
                self._init_full_sharded()

            def cap_for(n):
                return int(min(n, -(-cfg.route_slack * n // R) + cfg.route_pad))
            self.set_route_caps(cap_for(B), cap_for(B + S))
            self.ev = {k: torch.cuda.Event()
                       for k in ("route_e", "ids", "own", "h", "q", "ssm", "red_e", "b2")}
        self.graph = None
        self.phase_events = None  # list of (phase, start, end) when instrumented
        self.ssm_events = None    # 8 timing events recorded inside the softmax call (bench)

    def _symm(self, shape, dtype):
        """A symmetric-memory tensor of this shape on every rank and the int64 tensor of the R
        peer base pointers (device); the handle also provides the device barriers."""
        import torch.distributed._symmetric_memory as symm_mem
        t = symm_mem.empty(shape, dtype=dtype, device=self.device)
        h = symm_mem.rendezvous(t, self.router.group_name)
        ptrs = torch.tensor(list(h.buffer_ptrs), dtype=torch.int64, device=self.device)
        return t, h, ptrs

    def _symm_tables(self):
        """Move this rank's shards of E, W, b into symmetric memory (equal shapes on every rank:
        ceil(V / R) rows) so that peers can read them over NVLink."""
        V, R, d = self.cfg.vocab, self.R, self.d
        rows = -(-V // R)
        self.shard_rows = rows
        for name in ("E", "W", "b"):
            src = getattr(self, name)
            shape = (rows, d) if src.dim() == 2 else (rows,)
            t, h, ptrs = self._symm(shape, src.dtype)
            t[:src.shape[0]].copy_(src)
            setattr(self, name, t[:src.shape[0]])
            setattr(self, "tab_" + name, ptrs)
            setattr(self, "hdl_" + name, h)

    def _init_full_sharded(self):
        """Buffers of the vocabulary-sharded full softmax (R > 1).  h and y live in symmetric
        memory (every shard all-gathers them), and so do the per-token (max, sum) pairs, the dh
        partials and the loss partial that the other shards pull."""
        R, B, d, V, dev = self.R, self.B, self.d, self.cfg.vocab, self.device
        M = R * B
        f32 = dict(dtype=torch.float32, device=dev)
        i64 = dict(dtype=torch.int64, device=dev)
        self.M, self.nloc = M, self.W.shape[0]
        self.h, _, self.tab_h = self._symm((B, d), torch.bfloat16)
        self.y, _, self.tab_y = self._symm((B,), torch.int64)
        self.h_all = torch.empty((M, d), dtype=torch.bfloat16, device=dev)
        self.y_all = torch.empty(M, **i64)
        g = torch.arange(M, **i64)
        self.ag_ids = (g % B) * R + g // B      # global token g = rank g // B, row g % B
        self.cand = torch.arange(self.nloc, **i64) * R + self.rank   # this shard's classes
        self.W_bf = self.W.to(torch.bfloat16)   # operand shadow, refreshed by the W update
        self.rowstats, _, self.tab_rowstats = self._symm((M, 2), torch.float32)
        self.lse_all = torch.empty(M, **f32)
        dh_part, _, self.tab_dh = self._symm((M, d), torch.float32)
        self.full_out = {"dh": dh_part, "dw_s": torch.empty((self.nloc, d), **f32),
                         "db_s": torch.empty(self.nloc, **f32), "z_label": torch.empty(M, **f32)}
        self.loss_part, _, self.tab_loss = self._symm((4,), torch.float32)
        self.ws_full = ops.ssm_workspace(M, self.nloc, d, TFS_BF16, dev, V)

    def _refresh_shadow(self):
        if self.full_sharded:
            self.W_bf.copy_(self.W)

    def set_route_caps(self, cap_e: int, cap_w: int):
        """(Re)allocate the R > 1 slot buffers for cap_e / cap_w distinct ids per owner."""
        R, B, S, d, V, dev = self.R, self.B, self.S, self.d, self.cfg.vocab, self.device
        f32 = dict(dtype=torch.float32, device=dev)
        i64 = dict(dtype=torch.int64, device=dev)
        ce, cw = int(min(cap_e, B)), int(min(cap_w, B + S))
        self.cap_e, self.cap_w = ce, cw
        self.istride = ce + cw
        self.off_w, self.off_b = ce * d, (ce + cw) * d
        self.rstride = -(-((ce + cw) * d + cw) // 4) * 4  # 16-byte aligned regions
        if self.cfg.route == "p2p":
            # inboxes: region r of owner o's inbox is written by requester r over NVLink
            self.recv_ids, self.hdl_ids, self.tab_ids = self._symm((R, self.istride), torch.int64)
            self.recv_grads, _, self.tab_grads = self._symm((R, self.rstride), torch.float32)
        else:
            self.send_ids = torch.empty((R, self.istride), **i64)
            self.recv_ids = torch.empty((R, self.istride), **i64)
            self.send_rows = torch.empty((R, self.rstride), **f32)
            self.recv_rows = torch.empty((R, self.rstride), **f32)
            self.send_grads = torch.empty((R, self.rstride), **f32)
            self.recv_grads = torch.empty((R, self.rstride), **f32)
        self.route_e = ops.RoutePlan(B, V, R, ce, d, dev)
        self.route_w = ops.RoutePlan(B + S, V, R, cw, d, dev)
        self.own_e = ops.SlotScatterPlan(R, ce, self.E.shape[0], d, dev)
        self.own_w = ops.SlotScatterPlan(R, cw, self.W.shape[0], d, dev)
        self.counts = torch.zeros((2, R), **i64)  # distinct ids per owner of the last step
        self.graph = None

    def calibrate_routes(self, margin: float = 1.25, pad: int = 64):
        """Shrink the slot capacities to margin x the largest per-owner distinct-id count of
        the last eager step (max over ranks) + pad: the fixed-size exchanges then move little
        padding.  Overflow in a later step is still reported (TFS_ERR_CAPACITY)."""
        c = self.counts.max(dim=1).values.clone()
        self.router.dist.all_reduce(c, op=self.router.dist.ReduceOp.MAX, group=self.router.group)
        ce, cw = (int(v * margin) + pad for v in c.tolist())
        self.set_route_caps(ce, cw)
        return ce, cw

    # ------------------------------------------------------------------------------------------
    def _sample(self, step: int | None):
        B = self.B
        if self.sampler is None:
            return
        self.sampler.sample(self.cfg.seed, 0 if step is None else step, self.rank, self.y,
                            step_dev=self.step_dev if step is None else None, err=self.err,
                            out=(self.qw[B:], self.les, self.ley, self.num_tries))

    def _softmax(self):
        B = self.B
        ops.sampled_softmax(self.h, self.y, self.w_rows[:B], self.b_rows[:B], self.ley,
                            self.qw[B:], self.w_rows[B:], self.b_rows[B:], self.les,
                            flags=self.flags, grad_scale=self.c,
                            operand_dtype=self.cfg.operand_dtype, vocab=self.cfg.vocab,
                            out=self.ssm_out, ws=self.ws_ssm, events=self.ssm_events)

    def _apply_e(self):
        cfg = self.cfg
        if self.slots is None:
            self.plan_e.apply(self.E, self.ssm_out["dh"], cfg.lr)
        else:
            self.plan_e.apply_opt(cfg.optimizer, self.E, self.ssm_out["dh"], cfg.lr, self.slots[0],
                                  cfg.momentum)

    def _apply_w(self):
        cfg = self.cfg
        if self.slots is None:
            self.plan_w.apply(self.W, self.dw, cfg.lr, table2=self.b, grad2=self.db)
        else:
            self.plan_w.apply_opt(cfg.optimizer, self.W, self.dw, cfg.lr, self.slots[1],
                                  cfg.momentum, table2=self.b, grad2=self.db,
                                  slot2=self.slots[2])

    def _ph(self, name: str):
        """Phase marker: with ``self.phase_events`` set (bench instrumentation, eager only) the
        phase is bracketed by CUDA events on the current stream, preceded by a short device
        spin so the host has queued the whole phase before its start event fires."""
        if self.phase_events is None:
            return contextlib.nullcontext()
        return _PhaseTimer(self, name)

    def _local_step(self, step: int | None):
        """R = 1: every route is the identity (send buffer == receive buffer).

        The embedding lookup (E) and the softmax-row lookup (W, b) are independent until the
        sampled softmax, and so are their sparse updates afterwards: outside instrumentation
        the E path runs on a side stream concurrently with the W path (fork / join through
        stream waits, which CUDA-graph capture records as graph edges)."""
        if self.phase_events is not None:
            return self._local_step_serial(step)
        V, B = self.cfg.vocab, self.B
        main = torch.cuda.current_stream()
        side = self.side_stream
        side.wait_stream(main)
        # With one shard Part is the identity (every id local, positions 0..n-1) and so is
        # Stitch: each Gather writes its rows straight to their final place.  The ScatterAdd
        # plans (id sorts) depend only on the ids, so they are built on the side stream while
        # the main stream samples, gathers and runs the sampled softmax.
        ev = self.ev
        with torch.cuda.stream(side):                      # E path: h first (the softmax
            ops.gather(self.E, self.x, out=self.h, err=self.err)   # waits for it), then the
            ev["h"].record(side)                           # plan of the E update
            self.plan_e.build(self.x, err=self.err)
        self.qw[:B].copy_(self.y)                          # W path
        self._sample(step)
        ev["q"].record(main)
        with torch.cuda.stream(side):
            side.wait_event(ev["q"])
            self.plan_w.build(self.qw, err=self.err)
            ev["plan_w"].record(side)
        ops.gather2(self.W, self.b, self.qw, self.w_rows, self.b_rows, err=self.err)
        main.wait_event(ev["h"])
        self._softmax()
        ev["ssm"].record(main)
        with torch.cuda.stream(side):
            side.wait_event(ev["ssm"])
            self._apply_e()
        main.wait_event(ev["plan_w"])
        self._apply_w()
        main.wait_stream(side)

    def _local_step_serial(self, step: int | None):
        """The same step on one stream, bracketed into phases (bench instrumentation)."""
        V, B = self.cfg.vocab, self.B
        with self._ph("sample"):
            self.qw[:B].copy_(self.y)
            self._sample(step)
        with self._ph("gather"):  # one shard: Part / Stitch are the identity (see _local_step)
            ops.gather(self.E, self.x, out=self.h, err=self.err)
            ops.gather2(self.W, self.b, self.qw, self.w_rows, self.b_rows, err=self.err)
        with self._ph("sampled_softmax"):
            self._softmax()
        with self._ph("scatter_plan"):
            self.plan_e.build(self.x, err=self.err)
            self.plan_w.build(self.qw, err=self.err)
        with self._ph("scatter_sgd"):
            self._apply_e()
            self._apply_w()

    def _dist_step_p2p(self, step: int | None):
        """R > 1 over NVLink, one-sided: three device barriers, no collectives, no host sync.

        B0 (start): every owner finished the previous update, so its table is stable and its
        inbox free.  The requester pulls its h / W / b rows straight from the owners' tables
        (tfs_gather_peers) and stores its distinct ids into the owners' inboxes (route plan,
        push).  B1: all ids have arrived; each owner builds the plan of its inbox (merge of R
        ascending runs) on the side stream while the softmax runs.  The requester stores its
        per-id gradient sums into the same inbox slots (reduce, push).  B2: all gradients have
        arrived; each owner applies its planned ScatterAdd-SGD."""
        V, B, R, d = self.cfg.vocab, self.B, self.R, self.d
        ev, rank = self.ev, self.rank
        main, side = torch.cuda.current_stream(), self.side_stream
        self.hdl_ids.barrier(channel=0)                             # B0
        side.wait_stream(main)
        io = rank * self.istride
        with torch.cuda.stream(side):                               # E path: h first
            ops.gather_peers(self.tab_E, self.shard_rows, d, self.x, V, R, self.h, err=self.err)
            ev["h"].record(side)
            self.route_e.build_push(self.x, self.tab_ids, io, counts=self.counts[0],
                                    err=self.err)
        self.qw[:B].copy_(self.y)                                   # W path
        self._sample(step)
        ev["q"].record(main)
        with torch.cuda.stream(side):     # W route plan + id push, then the owner plans
            side.wait_event(ev["q"])
            self.route_w.build_push(self.qw, self.tab_ids, io + self.cap_e,
                                    counts=self.counts[1], err=self.err)
            self.hdl_ids.barrier(channel=1)                         # B1
            self.own_e.build(self.recv_ids, self.istride, err=self.err)
            self.own_w.build(self.recv_ids[:, self.cap_e:], self.istride, err=self.err)
            ev["own"].record(side)
        ops.gather_peers2(self.tab_W, self.tab_b, self.shard_rows, d, self.qw, V, R, self.w_rows,
                          self.b_rows, err=self.err)
        main.wait_event(ev["h"])
        self._softmax()
        ev["ssm"].record(main)
        ro = rank * self.rstride
        with torch.cuda.stream(side):                               # E gradients, in parallel
            side.wait_event(ev["ssm"])
            self.route_e.reduce_push(self.ssm_out["dh"], d, self.tab_grads, ro)
            ev["red_e"].record(side)
        self.route_w.reduce_push(self.dw, d, self.tab_grads, ro + self.off_w, rows2=self.db,
                                 out2_tab=self.tab_grads, out2_off=ro + self.off_b)
        main.wait_event(ev["red_e"])
        self.hdl_ids.barrier(channel=2)                             # B2
        ev["b2"].record(main)
        gr, rs = self.recv_grads, self.rstride
        with torch.cuda.stream(side):                               # E update, in parallel
            side.wait_event(ev["b2"])
            self.own_e.apply(self.E, gr, rs, self.cfg.lr)
        main.wait_event(ev["own"])
        self.own_w.apply(self.W, gr[:, self.off_w:], rs, self.cfg.lr, table2=self.b,
                         grad2=gr[:, self.off_b:], grad2_stride=rs)
        main.wait_stream(side)

    def _dist_step_full(self, step: int | None):
        """Vocabulary-sharded full softmax over NVLink ("the multiplication and
        gradient calculation are colocated with the shards"): W and b never move.

        B0: the previous step is applied everywhere.  Each rank pulls its h rows from the E
        owners and pushes its distinct x ids into their inboxes.  B1: h, y and the ids are
        in place; every rank all-gathers h and y (peer loads), scores all R*B tokens against
        its own classes and publishes per-token (max, sum) pairs.  B2: every rank combines all
        pairs into the global lse, forms G = c (p - onehot) on its classes, its dh partial,
        dW / db of its classes (applied locally, dense) and the loss of the labels it holds.
        B3: each rank pulls and sums its tokens' dh partials and the loss partials, then pushes
        per-id dh sums to the E owners.  B4: the E owners apply their planned ScatterAdd-SGD."""
        V, B, R, d, M = self.cfg.vocab, self.B, self.R, self.d, self.M
        ev, rank, lr = self.ev, self.rank, self.cfg.lr
        main, side = torch.cuda.current_stream(), self.side_stream
        L = ops._lib.lib()
        bar = self.hdl_ids.barrier
        bar(channel=0)                                              # B0
        side.wait_stream(main)
        with torch.cuda.stream(side):
            self.route_e.build_push(self.x, self.tab_ids, rank * self.istride,
                                    counts=self.counts[0], err=self.err)
            ev["q"].record(side)
        ops.gather_peers(self.tab_E, self.shard_rows, d, self.x, V, R, self.h, err=self.err)
        main.wait_event(ev["q"])
        bar(channel=1)                                              # B1
        ev["ids"].record(main)
        with torch.cuda.stream(side):                               # E owner plan, in parallel
            side.wait_event(ev["ids"])
            self.own_e.build(self.recv_ids, self.istride, err=self.err)
            ev["own"].record(side)
        # all-gathers of h (bf16) and y (int64) as bit copies of float words
        ops.gather_peers(self.tab_h, B, d // 2, self.ag_ids, M, R,
                         self.h_all.view(torch.float32), err=self.err)
        ops.gather_peers(self.tab_y, B, 2, self.ag_ids, M, R, self.y_all.view(torch.float32),
                         err=self.err)
        tev = self.ssm_events  # optional timing: 4 events around the two softmax halves
        if tev is not None:
            tev[0].record()
        ops.ssm_partial_stats(self.h_all, self.y_all, self.cand, self.W_bf, self.b, vocab=V,
                              ws=self.ws_full, out=self.rowstats)
        if tev is not None:
            tev[1].record()
        bar(channel=2)                                              # B2
        ops.lse_combine_peers(self.tab_rowstats, R, M, self.lse_all)
        fo = self.full_out
        if tev is not None:
            tev[2].record()
        ops.ssm_backward_from_lse(self.h_all, self.y_all, self.cand, self.W_bf, self.b,
                                  self.lse_all, grad_scale=self.c, ws=self.ws_full, vocab=V,
                                  out=fo)
        if tev is not None:
            tev[3].record()
        ops.label_loss_sum(self.lse_all, fo["z_label"], self.y_all, R, rank, self.c,
                           self.loss_part)
        ev["ssm"].record(main)
        with torch.cuda.stream(side):                  # W / b: local dense SGD, in parallel
            side.wait_event(ev["ssm"])
            ops.dense_sgd(self.W, fo["dw_s"], lr, shadow=self.W_bf)
            ops.dense_sgd(self.b, fo["db_s"], lr)
        bar(channel=3)                                              # B3
        ops.reduce_peers(self.tab_dh, R, rank * B * d, B * d, self.ssm_out["dh"])
        ops.reduce_peers(self.tab_loss, R, 0, 1, self.ssm_out["loss_sum"])
        self.route_e.reduce_push(self.ssm_out["dh"], d, self.tab_grads, rank * self.rstride)
        bar(channel=4)                                              # B4
        main.wait_event(ev["own"])
        self.own_e.apply(self.E, self.recv_grads, self.rstride, lr)
        main.wait_stream(side)

    def _dist_step(self, step: int | None):
        if self.full_sharded:
            self._dist_step_full(step)
        elif self.cfg.route == "p2p":
            self._dist_step_p2p(step)
        else:
            self._dist_step_nccl(step)

    def _dist_step_nccl(self, step: int | None):
        """R > 1, host-synchronisation free (capturable): plans -> ids a2a -> owner Gather ->
        rows a2a -> Stitch -> softmax -> per-id gradient sums -> gradients a2a -> owner SGD.

        Only distinct ids travel; every exchange is an equal-split all-to-all of slot regions
        (tfs_route_*), so no count ever reaches the host.  The E route plan is built on the
        side stream while the main stream samples; the owner-side ScatterAdd plans (a function
        of the received ids only) are built on the side stream while the softmax runs."""
        V, B, R, d = self.cfg.vocab, self.B, self.R, self.d
        rt, ev = self.router, self.ev
        main, side = torch.cuda.current_stream(), self.side_stream
        side.wait_stream(main)
        with torch.cuda.stream(side):
            self.route_e.build(self.x, self.send_ids, self.istride, counts=self.counts[0],
                               err=self.err)
            ev["route_e"].record(side)
        self.qw[:B].copy_(self.y)
        self._sample(step)
        self.route_w.build(self.qw, self.send_ids[:, self.cap_e:], self.istride,
                           counts=self.counts[1], err=self.err)
        main.wait_event(ev["route_e"])
        rt.a2a(self.recv_ids, self.send_ids)                        # ids -> owners
        ev["ids"].record(main)
        with torch.cuda.stream(side):                               # owner plans (backward)
            side.wait_event(ev["ids"])
            self.own_e.build(self.recv_ids, self.istride, err=self.err)
            self.own_w.build(self.recv_ids[:, self.cap_e:], self.istride, err=self.err)
            ev["own"].record(side)
        ce, cw, rs = self.cap_e, self.cap_w, self.rstride
        rows = self.send_rows
        ops.gather_slots(self.E, self.recv_ids, self.istride, R, ce, rows, rs, err=self.err)
        ops.gather_slots(self.W, self.recv_ids[:, ce:], self.istride, R, cw, rows[:, self.off_w:],
                         rs, err=self.err)
        ops.gather_slots(self.b, self.recv_ids[:, ce:], self.istride, R, cw, rows[:, self.off_b:],
                         rs, err=self.err)
        rt.a2a(self.recv_rows, self.send_rows)                      # rows -> requesters
        got = self.recv_rows
        self.route_e.unpack(got, rs, d, self.h)
        self.route_w.unpack(got[:, self.off_w:], rs, d, self.w_rows)
        self.route_w.unpack(got[:, self.off_b:], rs, 1, self.b_rows)
        self._softmax()
        g = self.send_grads
        self.route_e.reduce(self.ssm_out["dh"], d, g, rs)
        self.route_w.reduce(self.dw, d, g[:, self.off_w:], rs, rows2=self.db,
                            out2=g[:, self.off_b:], out2_stride=rs)
        rt.a2a(self.recv_grads, self.send_grads)                    # gradients -> owners
        main.wait_event(ev["own"])
        gr = self.recv_grads
        self.own_e.apply(self.E, gr, rs, self.cfg.lr)
        self.own_w.apply(self.W, gr[:, self.off_w:], rs, self.cfg.lr, table2=self.b,
                         grad2=gr[:, self.off_b:], grad2_stride=rs)
        main.wait_stream(side)

    # ------------------------------------------------------------------------------------------
    def run(self, x: torch.Tensor, y: torch.Tensor, step: int):
        """One step on device-resident x, y (int64 [B]).  Returns the device loss_sum [1]."""
        self.x.copy_(x)
        self.y.copy_(y)
        if self.R == 1:
            self._local_step(step)
        else:
            self._dist_step(step)
        return self.ssm_out["loss_sum"]

    def capture(self, first_step: int = 0):
        """Capture the whole step (inputs read from self.x / self.y, step counter from
        self.step_dev, advanced by one inside the graph) into a CUDA graph.  Any R: the R > 1
        step has no host synchronisation (fixed-capacity all-to-alls over NCCL)."""
        saved = (self.E.clone(), self.W.clone(), self.b.clone())
        saved_slots = None if self.slots is None else tuple(t.clone() for t in self.slots)
        self.step_dev.fill_(first_step)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        step_fn = self._local_step if self.R == 1 else self._dist_step
        with torch.cuda.stream(s):
            step_fn(None)                # warm-up (lazy init of kernels / attributes)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        for dst, src in zip((self.E, self.W, self.b), saved):  # undo the warm-up update
            dst.copy_(src)
        self._refresh_shadow()
        if saved_slots is not None:
            for dst, src in zip(self.slots, saved_slots):
                dst.copy_(src)
        del saved, saved_slots
        self.step_dev.fill_(first_step)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph(keep_graph=True)  # raw graph kept for inspection
        with torch.cuda.graph(self.graph):
            step_fn(None)
            self.step_dev.add_(1)
        self.graph.instantiate()
        torch.cuda.synchronize()
        return self.graph

    def replay(self):
        self.graph.replay()
        return self.ssm_out["loss_sum"]
