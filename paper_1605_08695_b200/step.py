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
    full_softmax: bool = False  # candidates = all V classes (config F; R must be 1)


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
        S = V if cfg.full_softmax else cfg.num_sampled
        if cfg.full_softmax and self.R != 1:
            raise ValueError("full softmax (config F) is a single-GPU configuration")
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
            self.qw[B:] = torch.arange(V, **i64)
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
        self.part_x = (torch.empty(B, **i64), torch.empty(B, **i64), torch.empty(R, **i64))
        self.part_w = (torch.empty(B + S, **i64), torch.empty(B + S, **i64), torch.empty(R, **i64))
        self.ws_part = ops._ws(L.tfs_partition_workspace_bytes(B + S, R), dev)
        self.ws_part_x = ops._ws(L.tfs_partition_workspace_bytes(B, R), dev)
        self.side_stream = torch.cuda.Stream(device=dev)
        self.h = torch.empty((B, d), **f32)
        self.w_rows = torch.empty((B + S, d), **f32)
        self.b_rows = torch.empty(B + S, **f32)
        self.ssm_out = {"loss": torch.empty(B, **f32), "lse": torch.empty(B, **f32),
                        "loss_sum": torch.zeros(1, **f32), "dh": torch.empty((B, d), **f32)}
        self.dw = torch.empty((B + S, d), **f32)    # dW_true || dW_s (aligned with y || s)
        self.db = torch.empty(B + S, **f32)
        self.ssm_out.update({"dw_true": self.dw[:B], "db_true": self.db[:B], "dw_s": self.dw[B:],
                             "db_s": self.db[B:]})
        self.ws_ssm = ops.ssm_workspace(B, S, d, cfg.operand_dtype, dev, V)
        if R == 1:
            self.plan_e = ops.ScatterPlan(B, E.shape[0], d, dev)
            self.plan_w = ops.ScatterPlan(B + S, W.shape[0], d, dev)
            self.ev = {k: torch.cuda.Event() for k in ("h", "q", "plan_w", "ssm")}
        else:
            self.ws_sr_e = ops._ws(L.tfs_sort_reduce_workspace_bytes(B, d), dev)
            self.ws_sr_w = ops._ws(L.tfs_sort_reduce_workspace_bytes(B + S, d), dev)
            self.sr_e = (torch.empty(B, **i64), torch.empty((B, d), **f32), None,
                         torch.empty(R, **i64), torch.empty(1, **i64))
            self.sr_w = (torch.empty(B + S, **i64), torch.empty((B + S, d), **f32),
                         torch.empty(B + S, **f32), torch.empty(R, **i64), torch.empty(1, **i64))
        self.graph = None
        self.phase_events = None  # list of (phase, start, end) when instrumented

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
                            out=self.ssm_out, ws=self.ws_ssm)

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
        with torch.cuda.stream(side):                      # E path
            self.plan_e.build(self.x, err=self.err)
            ops.gather(self.E, self.x, out=self.h, err=self.err)
            ev["h"].record(side)
        self.qw[:B].copy_(self.y)                          # W path
        self._sample(step)
        ev["q"].record(main)
        with torch.cuda.stream(side):
            side.wait_event(ev["q"])
            self.plan_w.build(self.qw, err=self.err)
            ev["plan_w"].record(side)
        ops.gather(self.W, self.qw, out=self.w_rows, err=self.err)
        ops.gather(self.b, self.qw, out=self.b_rows.view(-1, 1), err=self.err)
        main.wait_event(ev["h"])
        self._softmax()
        ev["ssm"].record(main)
        with torch.cuda.stream(side):
            side.wait_event(ev["ssm"])
            self.plan_e.apply(self.E, self.ssm_out["dh"], self.cfg.lr)
        main.wait_event(ev["plan_w"])
        self.plan_w.apply(self.W, self.dw, self.cfg.lr, table2=self.b, grad2=self.db)
        main.wait_stream(side)

    def _local_step_serial(self, step: int | None):
        """The same step on one stream, bracketed into phases (bench instrumentation)."""
        V, B = self.cfg.vocab, self.B
        with self._ph("sample"):
            self.qw[:B].copy_(self.y)
            self._sample(step)
        with self._ph("gather"):  # one shard: Part / Stitch are the identity (see _local_step)
            ops.gather(self.E, self.x, out=self.h, err=self.err)
            ops.gather(self.W, self.qw, out=self.w_rows, err=self.err)
            ops.gather(self.b, self.qw, out=self.b_rows.view(-1, 1), err=self.err)
        with self._ph("sampled_softmax"):
            self._softmax()
        with self._ph("scatter_plan"):
            self.plan_e.build(self.x, err=self.err)
            self.plan_w.build(self.qw, err=self.err)
        with self._ph("scatter_sgd"):
            self.plan_e.apply(self.E, self.ssm_out["dh"], self.cfg.lr)
            self.plan_w.apply(self.W, self.dw, self.cfg.lr, table2=self.b, grad2=self.db)

    def _dist_step(self, step: int | None):
        """R > 1: Part -> route -> Gather -> route back -> Stitch -> softmax -> sort-reduce ->
        route -> ScatterAdd-SGD on the owner."""
        V, B, R, d = self.cfg.vocab, self.B, self.R, self.d
        rt = self.router
        self.qw[:B].copy_(self.y)
        self._sample(step)
        xl, xpos, xcnt = ops.partition(self.x, V, R, err=self.err, out=self.part_x,
                                       ws=self.ws_part_x)
        wl, wpos, wcnt = ops.partition(self.qw, V, R, err=self.err, out=self.part_w, ws=self.ws_part)
        (sx, sw), (rx, rw) = rt.exchange_counts(torch.stack([xcnt, wcnt], dim=1))
        ids_x = rt.route(xl, sx, rx)
        ids_w = rt.route(wl, sw, rw)
        # Gather on the owner (colocated with the shard), send the rows back.
        rows_e = ops.gather(self.E, ids_x, err=self.err)
        rows_w = ops.gather(self.W, ids_w, err=self.err)
        rows_b = ops.gather(self.b, ids_w, err=self.err)
        back_e = rt.route(rows_e, rx, sx)
        back_w = rt.route(rows_w, rw, sw)
        back_b = rt.route(rows_b, rw, sw)
        ops.stitch(xpos, back_e, out=self.h)
        ops.stitch(wpos, back_w, out=self.w_rows)
        ops.stitch(wpos, back_b.view(-1), out=self.b_rows)
        self._softmax()
        # Sparse gradients: sum per id locally, route to the owners, apply there.
        le, ge, _, ce, _ = ops.sort_reduce(self.x, V, R, self.ssm_out["dh"], err=self.err,
                                           out=self.sr_e, ws=self.ws_sr_e)
        lw, gw, gb, cw, _ = ops.sort_reduce(self.qw, V, R, self.dw, rows2=self.db, err=self.err,
                                            out=self.sr_w, ws=self.ws_sr_w)
        (se, sw2), (re, rw2) = rt.exchange_counts(torch.stack([ce, cw], dim=1))
        r_ids_e = rt.route(le, se, re)
        r_g_e = rt.route(ge, se, re)
        r_ids_w = rt.route(lw, sw2, rw2)
        r_g_w = rt.route(gw, sw2, rw2)
        r_g_b = rt.route(gb, sw2, rw2)
        ops.scatter_add_sgd(self.E, r_ids_e, r_g_e, self.cfg.lr, err=self.err)
        ops.scatter_add_sgd(self.W, r_ids_w, r_g_w, self.cfg.lr, table2=self.b, grad2=r_g_b,
                            err=self.err)

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
        """R = 1 only: capture the whole step (inputs read from self.x / self.y, step counter
        from self.step_dev, advanced by one inside the graph) into a CUDA graph."""
        assert self.R == 1
        saved = (self.E.clone(), self.W.clone(), self.b.clone())
        self.step_dev.fill_(first_step)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self._local_step(None)       # warm-up (lazy init of kernels / attributes)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        for dst, src in zip((self.E, self.W, self.b), saved):  # undo the warm-up update
            dst.copy_(src)
        del saved
        self.step_dev.fill_(first_step)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._local_step(None)
            self.step_dev.add_(1)
        torch.cuda.synchronize()
        return self.graph

    def replay(self):
        self.graph.replay()
        return self.ssm_out["loss_sum"]
