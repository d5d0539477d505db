"""CPU ORACLE for the sharded-embedding + sampled-softmax step (arXiv 1605.08695, §4.2 / §6.4).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product package
``paper_1605_08695_b200`` never imports it, and it never imports the product package.

The arithmetic lives in ``oracle.cpp`` (single-threaded C++17, fp64 accumulation), loaded with
ctypes; ``step.py`` composes those functions into one synchronous training step exactly in the
order of DESIGN.md §3 (O1-O13).  This module is argument marshalling only.

Parity status: every function is pinned by ``tests/test_oracle_*.py`` except the
two rows the survey marks "parity unpinned": throughput (the paper prints no words/sec) and the
sampler's bit-compatibility with TensorFlow's own sampler (no TF here; R-17 defines ours).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.cpp")

OK, INVALID, OUT_OF_RANGE, BAD_POSITIONS, EXHAUSTED = 0, 1, 2, 3, 8
SUBTRACT_LOG_Q, REMOVE_ACCIDENTAL_HITS, LABEL_IN_CANDIDATES = 1, 2, 4


class OracleError(RuntimeError):
    def __init__(self, status: int, bad: int = -1):
        super().__init__(f"oracle status {status} (bad index {bad})")
        self.status = status
        self.bad = bad


def build(force: bool = False) -> str:
    """Compile liboracle.so with g++ (single-threaded, -O2)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", _SRC, "-o", _SO])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_SO)
        _declare(_lib)
    return _lib


P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int32
U32 = ctypes.c_uint32
U64 = ctypes.c_uint64


class _SsmIO(ctypes.Structure):
    _fields_ = [
        ("B", I64), ("S", I64), ("dim", I32), ("bf16", I32), ("flags", U32),
        ("grad_scale", ctypes.c_double),
        ("h", P), ("labels", P), ("w_true", P), ("b_true", P), ("log_ec_true", P),
        ("sampled", P), ("w_s", P), ("b_s", P), ("log_ec_s", P),
        ("n_tok", I64), ("tok_idx", P), ("n_col", I64), ("col_idx", P),
        ("loss", P), ("lse", P), ("z_true", P), ("dh", P), ("dw_true", P), ("db_true", P),
        ("dw_s", P), ("db_s", P),
        ("abs_loss", P), ("abs_dh", P), ("abs_dw_s", P), ("abs_db_s", P),
        ("amb_dh", P), ("amb_dw_s", P), ("amb_db_s", P),
    ]


def _declare(L):
    L.orc_partition.argtypes = [P, I64, I64, I32, P, P, P, P, P]
    L.orc_gather.argtypes = [P, I64, I32, P, I64, I32, P, P]
    L.orc_stitch.argtypes = [P, P, I64, I64, P, P]
    L.orc_bf16_round.argtypes = [ctypes.c_float]
    L.orc_bf16_round.restype = ctypes.c_float
    L.orc_bf16_round_array.argtypes = [P, I64, P]
    L.orc_philox4x32_10.argtypes = [P, P, P]
    L.orc_log_uniform_thresholds.argtypes = [I64, P]
    L.orc_log_uniform_prob.argtypes = [I64, I64]
    L.orc_log_uniform_prob.restype = ctypes.c_double
    L.orc_log_uniform_sample.argtypes = [I64, I32, I32, U64, U64, U32, P, I64, I64, P, P, P, P]
    L.orc_sampled_softmax.argtypes = [ctypes.POINTER(_SsmIO)]
    L.orc_scatter_add_sgd.argtypes = [P, I64, I32, P, P, I64, ctypes.c_double, P]
    L.orc_scatter_opt.argtypes = [ctypes.c_int, P, P, I64, I32, P, P, I64, ctypes.c_double,
                                  ctypes.c_double, P]
    L.orc_sort_reduce.argtypes = [P, I64, I32, P, I32, P, P, P, P]
    for f in (L.orc_partition, L.orc_gather, L.orc_stitch, L.orc_log_uniform_sample,
              L.orc_sampled_softmax, L.orc_scatter_add_sgd, L.orc_sort_reduce,
              L.orc_scatter_opt):
        f.restype = ctypes.c_int


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _check(status, bad=None):
    if status != OK:
        raise OracleError(status, int(bad.value) if bad is not None else -1)


# ---------------------------------------------------------------------------------------------
def partition(ids, vocab: int, num_shards: int, assignments=None):
    """Part.  Returns (local_ids, positions, counts)."""
    ids = _c(ids, np.int64)
    n = ids.size
    asg = None if assignments is None else _c(assignments, np.int32)
    local = np.empty(n, np.int64)
    pos = np.empty(n, np.int64)
    counts = np.empty(num_shards, np.int64)
    bad = I64(-1)
    st = lib().orc_partition(_ptr(ids), n, vocab, num_shards, _ptr(asg), _ptr(local), _ptr(pos),
                             _ptr(counts), ctypes.byref(bad))
    _check(st, bad)
    return local, pos, counts


def gather(table, ids, bf16: bool = False):
    """Gather.  fp32 rows, or bf16 bit patterns (uint16) when bf16=True."""
    table = _c(table, np.float32)
    rows, dim = table.shape
    ids = _c(ids, np.int64)
    out = np.empty((ids.size, dim), np.uint16 if bf16 else np.float32)
    bad = I64(-1)
    st = lib().orc_gather(_ptr(table), rows, dim, _ptr(ids), ids.size, int(bf16), _ptr(out),
                          ctypes.byref(bad))
    _check(st, bad)
    return out


def stitch(positions, rows):
    """Stitch: out[positions[j]] = rows[j]."""
    positions = _c(positions, np.int64)
    rows = np.ascontiguousarray(rows)
    n = positions.size
    row_bytes = rows.nbytes // max(n, 1) if n else max(rows.itemsize, 1)
    out = np.empty_like(rows)
    bad = I64(-1)
    st = lib().orc_stitch(_ptr(positions), _ptr(rows), n, row_bytes, _ptr(out), ctypes.byref(bad))
    _check(st, bad)
    return out


def bf16_round(x):
    x = _c(x, np.float32)
    out = np.empty_like(x)
    lib().orc_bf16_round_array(_ptr(x), x.size, _ptr(out))
    return out


def philox4x32_10(ctr, key):
    c = _c(ctr, np.uint32)
    k = _c(key, np.uint32)
    out = np.empty(4, np.uint32)
    lib().orc_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def log_uniform_thresholds(vocab: int):
    thr = np.empty(vocab, np.uint64)
    lib().orc_log_uniform_thresholds(vocab, _ptr(thr))
    return thr


def log_uniform_prob(vocab: int, k: int) -> float:
    return lib().orc_log_uniform_prob(vocab, k)


def sample(vocab, num_sampled, unique, seed, step, replica, labels, max_draws=None):
    """Log-uniform candidate sampler.  Returns (s int64[S], T, log_ec_s f64[S], log_ec_y f64)."""
    labels = _c(labels, np.int64)
    if max_draws is None:
        max_draws = 1 << 40
    s = np.empty(num_sampled, np.int64)
    les = np.empty(num_sampled, np.float64)
    ley = np.empty(labels.size, np.float64)
    T = I64(0)
    st = lib().orc_log_uniform_sample(vocab, num_sampled, int(unique), seed, step, replica,
                                      _ptr(labels), labels.size, max_draws, _ptr(s), _ptr(les),
                                      _ptr(ley), ctypes.byref(T))
    _check(st)
    return s, int(T.value), les, ley


def sampled_softmax(h, labels, w_true, b_true, log_ec_true, sampled, w_s, b_s, log_ec_s, *,
                    flags=SUBTRACT_LOG_Q | REMOVE_ACCIDENTAL_HITS, grad_scale=1.0, bf16=False,
                    tok_idx=None, col_idx=None):
    """Sampled softmax forward + backward (O9-O11).  Returns a dict of fp64 arrays:
    loss, lse, z_true, dh, dw_true, db_true, dw_s, db_s, and abs_loss / abs_dh / abs_dw_s /
    abs_db_s -- the sums of absolute values of the terms forming those outputs (the scale of
    the rounding error of any evaluation order; abs of dw_true / db_true is the value itself)
    -- and, in bf16 mode, amb_dh / amb_dw_s / amb_db_s: one bf16 unit (2^-8) of the terms whose
    G rounding is a tie within 2^-14 (R-34: either neighbour is a correct rounding).
    flags may include LABEL_IN_CANDIDATES (R-30: sharded full softmax; w_true, b_true,
    log_ec_true are then unused and may be None)."""
    h = _c(h, np.float32)
    B, d = h.shape
    w_s = _c(w_s, np.float32).reshape(-1, d)
    S = w_s.shape[0]
    labels = _c(labels, np.int64)
    if w_true is None:  # label-in mode: no true-class operand
        w_true, b_true, log_ec_true = np.zeros((B, d)), np.zeros(B), np.zeros(B)
    w_true = _c(w_true, np.float32).reshape(B, d)
    b_true = _c(b_true, np.float32)
    le_t = _c(log_ec_true, np.float64)
    sampled = _c(sampled, np.int64)
    b_s = _c(b_s, np.float32)
    le_s = _c(log_ec_s, np.float64)
    ti = None if tok_idx is None else _c(tok_idx, np.int64)
    ci = None if col_idx is None else _c(col_idx, np.int64)
    nt = B if ti is None else ti.size
    nc = S if ci is None else ci.size
    out = {
        "loss": np.empty(nt), "lse": np.empty(nt), "z_true": np.empty(nt),
        "dh": np.empty((nt, d)), "dw_true": np.empty((nt, d)), "db_true": np.empty(nt),
        "dw_s": np.empty((nc, d)), "db_s": np.empty(nc),
        "abs_loss": np.empty(nt), "abs_dh": np.empty((nt, d)), "abs_dw_s": np.empty((nc, d)),
        "abs_db_s": np.empty(nc),
        "amb_dh": np.zeros((nt, d)), "amb_dw_s": np.zeros((nc, d)), "amb_db_s": np.zeros(nc),
    }
    io = _SsmIO(B, S, d, int(bf16), flags, grad_scale, _ptr(h), _ptr(labels), _ptr(w_true),
                _ptr(b_true), _ptr(le_t), _ptr(sampled), _ptr(w_s), _ptr(b_s), _ptr(le_s),
                nt, _ptr(ti), nc, _ptr(ci),
                _ptr(out["loss"]), _ptr(out["lse"]), _ptr(out["z_true"]), _ptr(out["dh"]),
                _ptr(out["dw_true"]), _ptr(out["db_true"]), _ptr(out["dw_s"]), _ptr(out["db_s"]),
                _ptr(out["abs_loss"]), _ptr(out["abs_dh"]), _ptr(out["abs_dw_s"]),
                _ptr(out["abs_db_s"]), _ptr(out["amb_dh"]), _ptr(out["amb_dw_s"]),
                _ptr(out["amb_db_s"]))
    _check(lib().orc_sampled_softmax(ctypes.byref(io)))
    return out


def scatter_opt(kind, table, slot, ids, grad, lr, mu=0.0, inplace=False):
    """Sparse Momentum ("momentum") / Adagrad ("adagrad") on distinct-id sums (R-29).
    Returns (table, slot) (copies unless inplace)."""
    k = {"momentum": 1, "adagrad": 2}[kind]
    if not inplace:
        table = np.array(table, dtype=np.float32, copy=True)
        slot = np.array(slot, dtype=np.float32, copy=True)
    rows = table.shape[0]
    dim = 1 if table.ndim == 1 else table.shape[1]
    ids = _c(ids, np.int64)
    grad = _c(grad, np.float64).reshape(ids.size, dim)
    bad = I64(-1)
    st = lib().orc_scatter_opt(k, _ptr(table), _ptr(slot), rows, dim, _ptr(ids), _ptr(grad),
                               ids.size, float(lr), float(mu), ctypes.byref(bad))
    _check(st, bad)
    return table, slot


def scatter_add_sgd(table, ids, grad, lr, inplace=False):
    """Sparse SGD.  Returns the updated COPY of table (or updates a
    C-contiguous float32 `table` in place when inplace=True -- same arithmetic)."""
    if inplace:
        assert table.dtype == np.float32 and table.flags["C_CONTIGUOUS"]
    else:
        table = np.array(table, dtype=np.float32, copy=True, order="C")
    rows = table.shape[0]
    dim = 1 if table.ndim == 1 else table.shape[1]
    ids = _c(ids, np.int64)
    grad = _c(grad, np.float64)
    bad = I64(-1)
    st = lib().orc_scatter_add_sgd(_ptr(table), rows, dim, _ptr(ids), _ptr(grad), ids.size,
                                   float(lr), ctypes.byref(bad))
    _check(st, bad)
    return table


def sort_reduce(ids, num_shards, rows):
    """Unique (owner, local) ids with fp64 row sums.  Returns (local, sums, counts)."""
    ids = _c(ids, np.int64)
    rows = _c(rows, np.float64)
    dim = 1 if rows.ndim == 1 else rows.shape[1]
    n = ids.size
    local = np.empty(n, np.int64)
    sums = np.empty((n, dim))
    counts = np.empty(num_shards, np.int64)
    u = I64(0)
    _check(lib().orc_sort_reduce(_ptr(ids), n, num_shards, _ptr(rows), dim, _ptr(local),
                                 _ptr(sums), _ptr(counts), ctypes.byref(u)))
    k = int(u.value)
    return local[:k], (sums[:k, 0] if rows.ndim == 1 else sums[:k]), counts
