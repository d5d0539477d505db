"""Torch-tensor front end of the libtfs C ABI: one function per entry point of include/tfs.h,
same names, argument marshalling only (every step runs in the CUDA kernels of libtfs.so).

Tensors must live on the current CUDA device; calls are enqueued on the current torch stream.
Data errors (bad ids / positions) land in a device error slot; ``ErrorSlot.check()`` reads it
(that read synchronises, so hot loops check once at the end).
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import (TFS_BF16, TFS_BF16_OPERANDS, TFS_F32, TFS_LABEL_IN_CANDIDATES,
                   TFS_REMOVE_ACCIDENTAL_HITS, TFS_SUBTRACT_LOG_Q, SsmArgs, TfsError, check)

INT64_MAX = (1 << 63) - 1


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ws(nbytes: int, device) -> torch.Tensor:
    """Zero-filled: the segmented-sum workspaces hold arrival counters that must start at zero
    (every call leaves them zero again; include/tfs.h)."""
    return torch.zeros(max(int(nbytes), 256), dtype=torch.uint8, device=device)


class ErrorSlot:
    """Device-resident tfs_device_error {int32 code; int32 pad; int64 index}."""

    def __init__(self, device=None):
        self.buf = torch.zeros(2, dtype=torch.int64, device=device or "cuda")
        self.reset()

    def reset(self):
        self.buf[0] = 0
        self.buf[1] = INT64_MAX

    @property
    def ptr(self):
        return ctypes.c_void_p(self.buf.data_ptr())

    def read(self):
        v = self.buf.tolist()
        return int(v[0]) & 0xFFFFFFFF, int(v[1])

    def check(self, what: str):
        code, idx = self.read()
        if code != 0:
            raise TfsError(code, what, idx)


def _err(err):
    return None if err is None else err.ptr


# ---------------------------------------------------------------------------------------------
def partition(ids, vocab: int, num_shards: int, assignments=None, err: ErrorSlot = None,
              out=None, ws=None):
    """Part: returns (local_ids, positions, counts), shard-major, stable."""
    n = ids.numel()
    dev = ids.device
    if out is None:
        out = (torch.empty(n, dtype=torch.int64, device=dev),
               torch.empty(n, dtype=torch.int64, device=dev),
               torch.empty(num_shards, dtype=torch.int64, device=dev))
    local, pos, counts = out
    L = _lib.lib()
    if ws is None:
        ws = _ws(L.tfs_partition_workspace_bytes(n, num_shards), dev)
    check(L.tfs_partition(_p(ids), n, vocab, num_shards, _p(assignments), _p(local), _p(pos),
                          _p(counts), _p(ws), ws.numel(), _err(err), _stream()), "tfs_partition")
    return local, pos, counts


def gather(table, ids, out_dtype=torch.float32, err: ErrorSlot = None, out=None):
    """Gather: out[j] = table[ids[j]] (fp32 copy or bf16 RNE)."""
    rows = table.shape[0]
    dim = 1 if table.dim() == 1 else table.shape[1]
    n = ids.numel()
    if out is None:
        out = torch.empty((n, dim), dtype=out_dtype, device=table.device)
    od = TFS_BF16 if out.dtype == torch.bfloat16 else TFS_F32
    check(_lib.lib().tfs_gather(_p(table), rows, dim, TFS_F32, _p(ids), n, _p(out), od, _err(err),
                                _stream()), "tfs_gather")
    return out


def gather2(table, table2, ids, out, out2, err: ErrorSlot = None):
    """Gather of a row table and its width-1 companion in one pass: out[j] = table[ids[j]]
    (fp32 or bf16 per out.dtype), out2[j] = table2[ids[j]]."""
    od = TFS_BF16 if out.dtype == torch.bfloat16 else TFS_F32
    check(_lib.lib().tfs_gather2(_p(table), table.shape[0], table.shape[1], _p(table2), _p(ids),
                                 ids.numel(), _p(out), od, _p(out2), _err(err), _stream()),
          "tfs_gather2")
    return out, out2


def stitch(positions, rows, err: ErrorSlot = None, out=None):
    """Stitch: out[positions[j]] = rows[j]."""
    n = positions.numel()
    if out is None:
        out = torch.empty_like(rows)
    row_bytes = rows[0].numel() * rows.element_size() if n else 4
    L = _lib.lib()
    ws = _ws(L.tfs_stitch_workspace_bytes(n), rows.device) if err is not None else None
    check(L.tfs_stitch(_p(positions), _p(rows), n, row_bytes, _p(out), _p(ws),
                       0 if ws is None else ws.numel(), _err(err), _stream()), "tfs_stitch")
    return out


class Sampler:
    """Log-uniform candidate sampler with its device state."""

    def __init__(self, vocab: int, num_sampled: int, unique: bool = True, device=None):
        self.vocab, self.num_sampled, self.unique = vocab, num_sampled, bool(unique)
        self.device = torch.device(device or "cuda")
        L = _lib.lib()
        self.state = _ws(L.tfs_sampler_state_bytes(vocab), self.device)
        md = ctypes.c_int64(0)
        check(L.tfs_sampler_init(vocab, num_sampled, int(unique), _p(self.state), ctypes.byref(md),
                                 _stream()), "tfs_sampler_init")
        self.max_draws = int(md.value)
        self.ws = _ws(L.tfs_sampler_workspace_bytes(self.max_draws), self.device)

    def sample(self, seed: int, step: int, replica: int, labels, step_dev=None,
               err: ErrorSlot = None, out=None):
        """Returns (sampled int64[S], log_ec_sampled f32[S], log_ec_labels f32[B], T int64[1])."""
        S = self.num_sampled
        dev = self.device
        if out is None:
            out = (torch.empty(S, dtype=torch.int64, device=dev),
                   torch.empty(S, dtype=torch.float32, device=dev),
                   torch.empty(labels.numel(), dtype=torch.float32, device=dev),
                   torch.empty(1, dtype=torch.int64, device=dev))
        s, les, ley, T = out
        check(_lib.lib().tfs_log_uniform_sample(
            _p(self.state), self.vocab, S, int(self.unique), self.max_draws, seed, step,
            _p(step_dev), replica, _p(labels), labels.numel(), _p(s), _p(les), _p(ley), _p(T),
            _p(self.ws), self.ws.numel(), _err(err), _stream()), "tfs_log_uniform_sample")
        return s, les, ley, T


def ssm_workspace(B: int, S: int, dim: int, operand_dtype: int, device, vocab: int = 0):
    """Zero-filled: with vocab > 0 its head holds the candidate map, which must start (and
    stays) zero."""
    n = _lib.lib().tfs_ssm_workspace_bytes(B, S, dim, operand_dtype, vocab)
    return torch.zeros(max(int(n), 256), dtype=torch.uint8, device=device)


def sampled_softmax(h, labels, w_true, b_true, log_ec_true, sampled, w_s, b_s, log_ec_s, *,
                    flags=TFS_SUBTRACT_LOG_Q | TFS_REMOVE_ACCIDENTAL_HITS, grad_scale=1.0,
                    operand_dtype=TFS_BF16, vocab: int = 0, out=None, ws=None, events=None,
                    rows_ready=None):
    """Sampled softmax forward + backward.  Returns a dict of fp32 tensors:
    loss, lse, loss_sum, dh, dw_true, db_true, dw_s, db_s.  vocab > 0: labels and sampled lie
    in [0, vocab) (enables the candidate map; ws must come from ssm_workspace(..., vocab))."""
    B, d = h.shape
    S = sampled.numel()
    dev = h.device
    if h.dtype == torch.bfloat16:  # operands already rounded (e.g. by a bf16 Gather)
        assert w_true.dtype == torch.bfloat16 and w_s.dtype == torch.bfloat16
        assert operand_dtype == TFS_BF16
        flags |= TFS_BF16_OPERANDS
    if out is None:
        f = lambda *s: torch.empty(*s, dtype=torch.float32, device=dev)
        out = {"loss": f(B), "lse": f(B), "loss_sum": f(1), "dh": f(B, d), "dw_true": f(B, d),
               "db_true": f(B), "dw_s": f(S, d), "db_s": f(S)}
    if ws is None:
        ws = ssm_workspace(B, S, d, operand_dtype, dev, vocab)
    a = SsmArgs(B, S, d, operand_dtype, flags, float(grad_scale),
                _p(h), _p(labels), _p(w_true), _p(b_true), _p(log_ec_true), _p(sampled), _p(w_s),
                _p(b_s), _p(log_ec_s), _p(out["loss"]), _p(out["lse"]), _p(out["loss_sum"]),
                _p(out["dh"]), _p(out["dw_true"]), _p(out["db_true"]), _p(out["dw_s"]),
                _p(out["db_s"]), int(vocab), None, 0)
    if rows_ready is not None:  # torch.cuda.Event: recorded once dw_true/db_true/dw_s/db_s are final
        a.rows_ready_event = ctypes.c_void_p(rows_ready.cuda_event)
    if events is not None:  # 8 torch.cuda.Event (timing), recorded inside the call
        arr = (ctypes.c_void_p * 8)(*[ctypes.c_void_p(e.cuda_event) for e in events])
        a.timing_events = ctypes.cast(arr, ctypes.c_void_p)
    check(_lib.lib().tfs_sampled_softmax_fwd_bwd(ctypes.byref(a), _p(ws), ws.numel(), _stream()),
          "tfs_sampled_softmax_fwd_bwd")
    return out


def _slice_args(h, labels, sampled, w_s, b_s, flags, grad_scale, vocab, lse=None, dh=None,
                dw_s=None, db_s=None):
    B, d = h.shape
    if h.dtype == torch.bfloat16:
        assert w_s.dtype == torch.bfloat16
        flags |= TFS_BF16_OPERANDS
    return SsmArgs(B, sampled.numel(), d, TFS_BF16, flags, float(grad_scale), _p(h), _p(labels),
                   None, None, None, _p(sampled), _p(w_s), _p(b_s), None, None, _p(lse), None,
                   _p(dh), None, None, _p(dw_s), _p(db_s), int(vocab), None, 0)


def ssm_partial_stats(h, labels, sampled, w_s, b_s, *, flags=TFS_LABEL_IN_CANDIDATES,
                      vocab: int = 0, ws=None, out=None):
    """First half of a vocabulary-sharded full softmax on one shard: per token the
    (max, sum 2^x) pair, log2 domain, over this shard's candidate logits.  Returns fp32
    [B, 2].  ws (from ssm_workspace(B, S, d, TFS_BF16, vocab)) must be passed on to
    ssm_backward_from_lse."""
    B = h.shape[0]
    out = torch.empty(B, 2, dtype=torch.float32, device=h.device) if out is None else out
    a = _slice_args(h, labels, sampled, w_s, b_s, flags, 1.0, vocab)
    check(_lib.lib().tfs_ssm_partial_stats(ctypes.byref(a), _p(out), _p(ws), ws.numel(),
                                           _stream()), "tfs_ssm_partial_stats")
    return out


def ssm_backward_from_lse(h, labels, sampled, w_s, b_s, lse, *, grad_scale, ws,
                          flags=TFS_LABEL_IN_CANDIDATES, vocab: int = 0, out=None):
    """Second half: with the global lse, this shard's G = c (p - onehot), its dh partial
    (G W_s), dw_s = G^T h, db_s, and the label logits z_label of the labels it holds."""
    B, d = h.shape
    S = sampled.numel()
    if out is None:
        f = lambda *s: torch.empty(*s, dtype=torch.float32, device=h.device)
        out = {"dh": f(B, d), "dw_s": f(S, d), "db_s": f(S), "z_label": f(B)}
    a = _slice_args(h, labels, sampled, w_s, b_s, flags, grad_scale, vocab, lse, out["dh"],
                    out["dw_s"], out["db_s"])
    check(_lib.lib().tfs_ssm_backward_from_lse(ctypes.byref(a), _p(out["z_label"]), _p(ws),
                                               ws.numel(), _stream()),
          "tfs_ssm_backward_from_lse")
    return out


def lse_combine_peers(stats_tab, R: int, n: int, lse):
    """lse[t] from every shard's (m, s) pair (peer pointers, rank order)."""
    check(_lib.lib().tfs_lse_combine_peers(_p(stats_tab), int(R), int(n), _p(lse), _stream()),
          "tfs_lse_combine_peers")
    return lse


def reduce_peers(src_tab, R: int, offset: int, n: int, out):
    """out[i] = sum_r src_tab[r][offset + i] (peer pointers, rank order)."""
    check(_lib.lib().tfs_reduce_peers(_p(src_tab), int(R), int(offset), int(n), _p(out),
                                      _stream()), "tfs_reduce_peers")
    return out


def label_loss_sum(lse, z_label, labels, R: int, shard: int, c: float, out):
    check(_lib.lib().tfs_label_loss_sum(_p(lse), _p(z_label), _p(labels), labels.numel(), int(R),
                                        int(shard), float(c), _p(out), _stream()),
          "tfs_label_loss_sum")
    return out


def dense_sgd(table, grad, lr: float, shadow=None):
    """table -= lr * grad; shadow (bf16, same shape) = bf16(table) when given."""
    check(_lib.lib().tfs_dense_sgd(_p(table), _p(grad), table.numel(), float(lr), _p(shadow),
                                   _stream()), "tfs_dense_sgd")
    return table


def sort_reduce(ids, vocab: int, num_shards: int, rows, rows2=None, err: ErrorSlot = None,
                out=None, ws=None):
    """Sum gradient rows of equal ids; unique ids in (owner, local) order.
    Returns (local int64[n], sums [n, dim], sums2 [n] | None, counts int64[R], U int64[1]);
    only the first U entries are meaningful."""
    n = ids.numel()
    dim = rows.shape[1] if rows.dim() == 2 else 1
    dev = ids.device
    if out is None:
        out = (torch.empty(n, dtype=torch.int64, device=dev),
               torch.empty((n, dim), dtype=torch.float32, device=dev),
               None if rows2 is None else torch.empty(n, dtype=torch.float32, device=dev),
               torch.empty(num_shards, dtype=torch.int64, device=dev),
               torch.empty(1, dtype=torch.int64, device=dev))
    local, sums, sums2, counts, U = out
    L = _lib.lib()
    if ws is None:
        ws = _ws(L.tfs_sort_reduce_workspace_bytes(n, dim), dev)
    check(L.tfs_sort_reduce(_p(ids), n, vocab, num_shards, _p(rows), dim, _p(rows2), _p(local),
                            _p(sums), _p(sums2), _p(counts), _p(U), _p(ws), ws.numel(), _err(err),
                            _stream()), "tfs_sort_reduce")
    return local, sums, sums2, counts, U


def scatter_add_sgd(table, ids, grad, lr: float, table2=None, grad2=None, err: ErrorSlot = None,
                    ws=None):
    """ScatterAdd-SGD: table[ids[i]] -= lr * grad[i], duplicates summed in a fixed
    order; optional width-1 companion (table2, grad2).  In place."""
    rows = table.shape[0]
    dim = 1 if table.dim() == 1 else table.shape[1]
    n = ids.numel()
    L = _lib.lib()
    if ws is None:
        ws = _ws(L.tfs_scatter_add_sgd_workspace_bytes(n, dim), table.device)
    check(L.tfs_scatter_add_sgd(_p(table), rows, dim, _p(ids), _p(grad), n, float(lr),
                                _p(table2), _p(grad2), _p(ws), ws.numel(), _err(err), _stream()),
          "tfs_scatter_add_sgd")
    return table


class ScatterPlan:
    """Planned ScatterAdd-SGD: the id sort / segmentation (``build``, ids only) split from the
    row reduction + table update (``apply``); identical results to scatter_add_sgd."""

    def __init__(self, n: int, rows: int, dim: int, device):
        L = _lib.lib()
        self.n, self.rows, self.dim = int(n), int(rows), int(dim)
        self.plan = _ws(L.tfs_scatter_plan_bytes(n), device)
        self.ws = _ws(L.tfs_scatter_apply_workspace_bytes(n, dim), device)

    def build(self, ids, err: ErrorSlot = None):
        assert ids.numel() == self.n
        check(_lib.lib().tfs_scatter_plan(_p(ids), self.n, self.rows, _p(self.plan),
                                          self.plan.numel(), _err(err), _stream()),
              "tfs_scatter_plan")
        return self

    def apply_opt(self, kind: str, table, grad, lr: float, slot, mu: float = 0.0, table2=None,
                  grad2=None, slot2=None, mirror=None):
        """Sparse Momentum ("momentum") / Adagrad ("adagrad") / "sgd" with the fp32 slot
        tables (tfs_scatter_opt_planned); mirror: optional bf16 copy of the table kept in step."""
        from ._lib import SparseOpt
        k = {"sgd": 0, "momentum": 1, "adagrad": 2}[kind]
        o = SparseOpt(k, float(lr), float(mu), _p(slot), _p(slot2), _p(mirror))
        check(_lib.lib().tfs_scatter_opt_planned(
            _p(table), self.rows, self.dim, _p(self.plan), self.plan.numel(), self.n, _p(grad),
            _p(table2), _p(grad2), ctypes.byref(o), _p(self.ws), self.ws.numel(), _stream()),
            "tfs_scatter_opt_planned")
        return table

    def apply(self, table, grad, lr: float, table2=None, grad2=None):
        assert table.shape[0] == self.rows
        check(_lib.lib().tfs_scatter_add_sgd_planned(
            _p(table), self.rows, self.dim, _p(self.plan), self.plan.numel(), self.n, _p(grad),
            float(lr), _p(table2), _p(grad2), _p(self.ws), self.ws.numel(), _stream()),
            "tfs_scatter_add_sgd_planned")
        return table


class RoutePlan:
    """Requester side of a fixed-capacity route between R shards (tfs_route_*): the plan of
    ``n`` ids (built from ids only), its send ids in slot layout, the Stitch of received rows
    and the reduction of gradient rows into slots.  Slot regions are ``stride`` elements
    apart; each holds ``cap`` slots."""

    def __init__(self, n: int, vocab: int, R: int, cap: int, dim: int, device):
        L = _lib.lib()
        self.n, self.vocab, self.R, self.cap = int(n), int(vocab), int(R), int(cap)
        self.plan = _ws(L.tfs_route_plan_bytes(n, R), device)
        self.ws = _ws(L.tfs_route_reduce_workspace_bytes(n, dim), device)

    def build(self, ids, send, send_stride: int, counts=None, err: ErrorSlot = None):
        assert ids.numel() == self.n
        check(_lib.lib().tfs_route_plan(_p(ids), self.n, self.vocab, self.R, self.cap,
                                        _p(self.plan), self.plan.numel(), _p(send),
                                        int(send_stride), _p(counts), _err(err), _stream()),
              "tfs_route_plan")
        return self

    def build_push(self, ids, dst_tab, dst_off: int, counts=None, err: ErrorSlot = None):
        """Plan + send ids stored straight into the owners' inboxes (dst_tab: int64 tensor of R
        peer pointers) at element offset dst_off."""
        assert ids.numel() == self.n
        check(_lib.lib().tfs_route_plan_push(_p(ids), self.n, self.vocab, self.R, self.cap,
                                             _p(self.plan), self.plan.numel(), _p(dst_tab),
                                             int(dst_off), _p(counts), _err(err), _stream()),
              "tfs_route_plan_push")
        return self

    def reduce_push(self, rows, dim: int, out_tab, out_off: int, rows2=None, out2_tab=None,
                    out2_off: int = 0):
        check(_lib.lib().tfs_route_reduce_push(_p(self.plan), self.plan.numel(), self.n,
                                               self.vocab, self.R, self.cap, _p(rows), int(dim),
                                               _p(rows2), _p(out_tab), int(out_off),
                                               _p(out2_tab), int(out2_off), _p(self.ws),
                                               self.ws.numel(), _stream()),
              "tfs_route_reduce_push")

    def unpack(self, slots, slots_stride: int, dim: int, out):
        check(_lib.lib().tfs_route_unpack(_p(self.plan), self.plan.numel(), self.n, self.vocab,
                                          self.R, self.cap, _p(slots), int(slots_stride),
                                          int(dim), _p(out), _stream()), "tfs_route_unpack")
        return out

    def reduce(self, rows, dim: int, out, out_stride: int, rows2=None, out2=None,
               out2_stride: int = 0):
        check(_lib.lib().tfs_route_reduce(_p(self.plan), self.plan.numel(), self.n, self.vocab,
                                          self.R, self.cap, _p(rows), int(dim), _p(rows2),
                                          _p(out), int(out_stride), _p(out2), int(out2_stride),
                                          _p(self.ws), self.ws.numel(), _stream()),
              "tfs_route_reduce")
        return out


def gather_peers(shard_tab, shard_rows: int, dim: int, ids, vocab: int, R: int, out,
                 err: ErrorSlot = None):
    """One-sided routed Gather: out[t] = row id//R of shard id%R through peer pointers."""
    od = TFS_BF16 if out.dtype == torch.bfloat16 else TFS_F32
    check(_lib.lib().tfs_gather_peers(_p(shard_tab), int(shard_rows), int(dim), _p(ids),
                                      ids.numel(), int(vocab), int(R), _p(out), od, _err(err),
                                      _stream()), "tfs_gather_peers")
    return out


def gather_peers2(shard_tab, shard_tab2, shard_rows: int, dim: int, ids, vocab: int, R: int,
                  out, out2, err: ErrorSlot = None):
    """tfs_gather_peers plus the width-1 companion shards (e.g. b with W) in one pass."""
    od = TFS_BF16 if out.dtype == torch.bfloat16 else TFS_F32
    check(_lib.lib().tfs_gather_peers2(_p(shard_tab), int(shard_rows), int(dim), _p(shard_tab2),
                                       _p(ids), ids.numel(), int(vocab), int(R), _p(out), od,
                                       _p(out2), _err(err), _stream()), "tfs_gather_peers2")
    return out, out2


def gather_peers2_bf16(mirror_tab, shard_tab2, shard_rows: int, dim: int, ids, vocab: int,
                       R: int, out, out2, err: ErrorSlot = None):
    """tfs_gather_peers2 from the owners' bf16 mirrors (bf16 rows out)."""
    assert out.dtype == torch.bfloat16
    check(_lib.lib().tfs_gather_peers2_bf16(_p(mirror_tab), int(shard_rows), int(dim),
                                            _p(shard_tab2), _p(ids), ids.numel(), int(vocab),
                                            int(R), _p(out), _p(out2), _err(err), _stream()),
          "tfs_gather_peers2_bf16")
    return out, out2


def gather_slots(table, ids, ids_stride: int, num_slots: int, cap: int, out, out_stride: int,
                 err: ErrorSlot = None):
    """Owner side: rows of the received slot ids (-1 = padding) into slot layout."""
    rows = table.shape[0]
    dim = 1 if table.dim() == 1 else table.shape[1]
    check(_lib.lib().tfs_gather_slots(_p(table), rows, dim, _p(ids), int(ids_stride),
                                      int(num_slots), int(cap), _p(out), int(out_stride),
                                      _err(err), _stream()), "tfs_gather_slots")
    return out


class SlotScatterPlan:
    """Owner side: planned ScatterAdd-SGD over R x cap received slots (tfs_scatter_*_slots)."""

    def __init__(self, R: int, cap: int, rows: int, dim: int, device):
        L = _lib.lib()
        self.R, self.cap, self.rows, self.dim = int(R), int(cap), int(rows), int(dim)
        n = self.R * self.cap
        self.plan = _ws(L.tfs_scatter_plan_bytes(n), device)
        self.ws = _ws(L.tfs_scatter_apply_workspace_bytes(n, dim), device)

    def build(self, ids, ids_stride: int, sorted_runs: bool = True, err: ErrorSlot = None):
        """sorted_runs: every region is ascending ids + trailing -1 (as tfs_route_plan sends)."""
        check(_lib.lib().tfs_scatter_plan_slots(_p(ids), int(ids_stride), self.R, self.cap,
                                                self.rows, int(sorted_runs), _p(self.plan),
                                                self.plan.numel(), _err(err), _stream()),
              "tfs_scatter_plan_slots")
        return self

    def apply(self, table, grad, grad_stride: int, lr: float, table2=None, grad2=None,
              grad2_stride: int = 0):
        check(_lib.lib().tfs_scatter_add_sgd_planned_slots(
            _p(table), self.rows, self.dim, _p(self.plan), self.plan.numel(), self.R, self.cap,
            _p(grad), int(grad_stride), float(lr), _p(table2), _p(grad2), int(grad2_stride),
            _p(self.ws), self.ws.numel(), _stream()), "tfs_scatter_add_sgd_planned_slots")
        return table


def debug_gemm_bf16(A, B, ksplit: int = 1, a_mn: bool = False, b_mn: bool = False):
    """C[ks] = sum_k A(m, k) B(n, k) on the tcgen05 path (diagnostics).  A is [M, K] (K-major)
    or, with a_mn, [K, M] (MN-major); likewise B is [N, K] or [K, N]."""
    M, K = (A.shape[1], A.shape[0]) if a_mn else A.shape
    N = B.shape[1] if b_mn else B.shape[0]
    C = torch.empty((M, N), dtype=torch.float32, device=A.device)
    L = _lib.lib()
    ws = _ws(L.tfs_debug_gemm_workspace_bytes(M, N, K, ksplit), A.device)
    check(L.tfs_debug_gemm_bf16(_p(A), A.stride(0), int(a_mn), _p(B), B.stride(0), int(b_mn),
                                M, N, K, ksplit, _p(C), _p(ws), ws.numel(), _stream()),
          "tfs_debug_gemm_bf16")
    return C
