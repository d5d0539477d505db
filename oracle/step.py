"""Oracle training step: O1-O13 of DESIGN.md §3, one synchronous step over R replicas.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Composes the C oracle functions in the
paper's order: Part -> route to the owner (Send/Recv) -> Gather
colocated with the shard -> route back -> Stitch -> sampled softmax
 -> sparse gradients -> one synchronous SGD apply of the
sum over replicas (Fig. 4b at P:820-827, R-15).

Shards are simulated: shard o of a logical table T[V, d] is T[o::R] (rows i with i mod R == o,
local row i div R; R-1).  Every replica reads the pre-step tables.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import (LABEL_IN_CANDIDATES, REMOVE_ACCIDENTAL_HITS, SUBTRACT_LOG_Q, gather, partition,
               sample, sampled_softmax, scatter_add_sgd, stitch)


@dataclass
class StepConfig:
    vocab: int
    dim: int
    num_sampled: int
    num_shards: int          # R = replicas = shards
    lr: float = 0.1
    seed: int = 7
    step: int = 0
    unique: bool = True
    flags: int = SUBTRACT_LOG_Q | REMOVE_ACCIDENTAL_HITS
    bf16: bool = False
    full_softmax: bool = False   # candidates = all V classes, no sampler (config F)
    # full softmax with the label among the candidates (R-30: the vocabulary-sharded full
    # softmax of P:706-714 -- G = c (p - onehot) rounded as a whole in bf16 mode); the plain
    # full softmax (R = 1) keeps the separate true-class term with the hit excluded (R-9)
    label_in: bool = False
    inplace: bool = False        # update E, W, b in place (same arithmetic; saves table copies)
    # also return, per table, lr x the sum over contributions of the abs_* term sums: the
    # element-wise scale of the update's rounding error (tests' parity bound)
    abs_bounds: bool = False


@dataclass
class ReplicaTrace:
    send_local_x: np.ndarray = None
    send_pos_x: np.ndarray = None
    counts_x: np.ndarray = None
    send_local_w: np.ndarray = None
    send_pos_w: np.ndarray = None
    counts_w: np.ndarray = None
    sampled: np.ndarray = None
    num_tries: int = 0
    log_ec_s: np.ndarray = None
    log_ec_y: np.ndarray = None
    h: np.ndarray = None
    w_rows: np.ndarray = None     # [B+S, d]: W_true then W_s
    b_rows: np.ndarray = None     # [B+S]
    ssm: dict = field(default_factory=dict)
    abs_delta: tuple = None       # (E, W, b) update scales, traces[0] only, cfg.abs_bounds
    amb_delta: tuple = None       # (E, W, b) bf16 rounding-tie allowances (R-34), likewise


def _route(send_local, counts, R):
    """O4: owner o receives, from every source r in rank order, r's slice destined to o."""
    recv = []
    for o in range(R):
        parts = []
        for r in range(R):
            off = np.concatenate([[0], np.cumsum(counts[r])])
            parts.append(send_local[r][off[o]:off[o + 1]])
        recv.append(np.concatenate(parts) if parts else np.empty(0, np.int64))
    return recv


def _route_back(rows_at_owner, counts, R):
    """Reverse of _route: replica r gets back, in owner order, the rows it asked for."""
    back = []
    for r in range(R):
        parts = []
        for o in range(R):
            start = sum(int(counts[rr][o]) for rr in range(r))
            parts.append(rows_at_owner[o][start:start + int(counts[r][o])])
        back.append(np.concatenate(parts))
    return back


def step(E, W, b, xs, ys, cfg: StepConfig):
    """One oracle step.  E, W: float32 [V, d]; b: float32 [V]; xs, ys: R arrays of int64 [B].

    Returns (E', W', b', traces) where traces[r] holds replica r's intermediates.
    """
    R = cfg.num_shards
    V, d = E.shape
    B = len(xs[0])
    c = 1.0 / (R * B)                                  # R-13: mean over the global batch
    traces = [ReplicaTrace() for _ in range(R)]

    # O7 sampler (per replica, R-7) -- needed before Part of q_W = y || s.
    for r in range(R):
        t = traces[r]
        if cfg.full_softmax:
            t.sampled = np.arange(V, dtype=np.int64)
            t.num_tries = V
            t.log_ec_s = np.zeros(V)
            t.log_ec_y = np.zeros(B)
        else:
            t.sampled, t.num_tries, t.log_ec_s, t.log_ec_y = sample(
                V, cfg.num_sampled, cfg.unique, cfg.seed, cfg.step, r, ys[r])

    # O3 Part of both lookups.
    for r in range(R):
        t = traces[r]
        t.send_local_x, t.send_pos_x, t.counts_x = partition(xs[r], V, R)
        qw = np.concatenate([ys[r], t.sampled])
        t.send_local_w, t.send_pos_w, t.counts_w = partition(qw, V, R)

    # O4 route ids; O5 gather on the owner's shard; route rows back; O6 stitch.
    cx = [t.counts_x for t in traces]
    cw = [t.counts_w for t in traces]
    recv_x = _route([t.send_local_x for t in traces], cx, R)
    recv_w = _route([t.send_local_w for t in traces], cw, R)
    rows_e = [gather(E[o::R], recv_x[o]) for o in range(R)]
    rows_w = [gather(W[o::R], recv_w[o]) for o in range(R)]
    rows_b = [gather(b[o::R].reshape(-1, 1), recv_w[o])[:, 0] for o in range(R)]
    back_e = _route_back(rows_e, cx, R)
    back_w = _route_back(rows_w, cw, R)
    back_b = _route_back(rows_b, cw, R)
    for r in range(R):
        t = traces[r]
        t.h = stitch(t.send_pos_x, back_e[r])
        t.w_rows = stitch(t.send_pos_w, back_w[r])
        t.b_rows = stitch(t.send_pos_w, back_b[r])

    # O8-O11 sampled softmax per replica; O12 sparse accumulation over all replicas.
    ids_e, g_e, ids_w, g_w, g_b = [], [], [], [], []
    for r in range(R):
        t = traces[r]
        S = t.sampled.size
        # Config F (full softmax): every class is a candidate, no log-Q correction, and the
        # true class is excluded from the candidates (R-9) -- exactly the full softmax; or,
        # label_in, the label's own column carries its gradient (R-30).
        if cfg.full_softmax:
            flags = LABEL_IN_CANDIDATES if cfg.label_in else REMOVE_ACCIDENTAL_HITS
        else:
            flags = cfg.flags
        t.ssm = sampled_softmax(
            t.h, ys[r], t.w_rows[:B], t.b_rows[:B], t.log_ec_y, t.sampled, t.w_rows[B:B + S],
            t.b_rows[B:B + S], t.log_ec_s, flags=flags, grad_scale=c, bf16=cfg.bf16)
        ids_e.append(xs[r])
        g_e.append(t.ssm["dh"])
        ids_w.append(np.concatenate([ys[r], t.sampled]))
        g_w.append(np.concatenate([t.ssm["dw_true"], t.ssm["dw_s"]]))
        g_b.append(np.concatenate([t.ssm["db_true"], t.ssm["db_s"]]))

    # O13 one synchronous SGD apply of the summed sparse gradient.
    E2 = scatter_add_sgd(E, np.concatenate(ids_e), np.concatenate(g_e), cfg.lr, cfg.inplace)
    W2 = scatter_add_sgd(W, np.concatenate(ids_w), np.concatenate(g_w), cfg.lr, cfg.inplace)
    b2 = scatter_add_sgd(b, np.concatenate(ids_w), np.concatenate(g_b), cfg.lr, cfg.inplace)
    if cfg.abs_bounds:
        # per touched entry: lr x sum over its contributions of their absolute term sums
        aE, aW, ab = np.zeros(E.shape), np.zeros(W.shape), np.zeros(b.shape)
        for r in range(R):
            t = traces[r]
            np.add.at(aE, xs[r], cfg.lr * t.ssm["abs_dh"])
            q = np.concatenate([ys[r], t.sampled])
            # g_t = c (p_t - 1) is a difference: its scale is c (p_t + 1), p_t = e^{-loss_t}
            dbt = t.ssm["db_true"]
            sg = np.where(dbt == 0, 0.0, c * (np.exp(-t.ssm["loss"]) + 1.0))
            hs = np.abs(t.ssm["dw_true"]) / np.maximum(np.abs(dbt), 1e-300)[:, None]
            np.add.at(aW, q, cfg.lr * np.concatenate([sg[:, None] * hs, t.ssm["abs_dw_s"]]))
            np.add.at(ab, q, cfg.lr * np.concatenate([sg, t.ssm["abs_db_s"]]))
        traces[0].abs_delta = (aE, aW, ab)
        # bf16 rounding ties (R-34): lr x the amb_* allowances of the contributions
        mE, mW, mb = np.zeros(E.shape), np.zeros(W.shape), np.zeros(b.shape)
        for r in range(R):
            t = traces[r]
            np.add.at(mE, xs[r], cfg.lr * t.ssm["amb_dh"])
            q = np.concatenate([ys[r], t.sampled])
            np.add.at(mW, q, cfg.lr * np.concatenate([np.zeros_like(t.ssm["dw_true"]),
                                                     t.ssm["amb_dw_s"]]))
            np.add.at(mb, q, cfg.lr * np.concatenate([np.zeros_like(t.ssm["db_true"]),
                                                     t.ssm["amb_db_s"]]))
        traces[0].amb_delta = (mE, mW, mb)
    return E2, W2, b2, traces
