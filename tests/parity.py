"""Element-wise, cancellation-aware parity metric (reading R-19, round 2).

Every floating-point output o_i of the method is a sum of terms (a dot product, a gradient
sum over tokens or classes, a sum of duplicate-id rows).  Any evaluation order -- the GPU's
fp32 tensor-core accumulation, its fixed-order segment sums, the oracle's fp64 loops -- commits
a rounding error bounded by a multiple of the sum of the ABSOLUTE values of those terms, a_i
(the oracle returns a_i next to o_i: ``abs_*`` outputs of ``oracle.sampled_softmax``).  So the
check is, element by element,

    |g_i - o_i| <= tol * a_i

with tol = 1e-5 (fp32 operands), 2e-2 (bf16 operands vs the fp64 unrounded oracle) and 2e-3
(bf16 operands vs the oracle's bf16-emulating mode).  Unlike a single normwise ratio
max|g - o| / max|o|, a wrong small entry (a low-probability class's dW_s row, a token's dh
entry formed by cancellation) cannot hide behind the tensor's largest entry.

Table updates T' = fl32(T - lr g) are compared as deltas with one more allowance: each side
rounds its new value to fp32 once, so the two may differ by one ulp of T' beyond tol * a_i.

Against the bf16-EMULATING oracle one more term is admitted (reading R-34): where the exact
pre-rounding G_tj lies within 2^-14 of a bf16 rounding midpoint, either neighbour is a correct
rounding (the GPU forms G from fp32 logits; the oracle from fp64 ones), so such terms may
differ by one bf16 unit; the oracle returns that allowance per element (amb_*), and the check
is |g_i - o_i| - amb_i <= tol * a_i.
"""
from __future__ import annotations

import numpy as np

TOL_F32, TOL_BF16_ACC, TOL_BF16_EMU = 1e-5, 2e-2, 2e-3


def elem_err(got, ref, scale, allow=None) -> float:
    """max_i (|got_i - ref_i| - allow_i)_+ / scale_i (0 / 0 counts as 0; a nonzero error on a
    zero scale is infinite)."""
    g = np.asarray(got, np.float64).ravel()
    o = np.asarray(ref, np.float64).ravel()
    a = np.asarray(scale, np.float64).ravel()
    if g.shape != o.shape or a.shape != o.shape:
        raise ValueError(f"shape mismatch {g.shape} {o.shape} {a.shape}")
    if o.size == 0:
        return 0.0
    diff = np.abs(g - o)
    if allow is not None:
        diff = np.maximum(diff - np.asarray(allow, np.float64).ravel(), 0.0)
    if not np.all(np.isfinite(g)):
        return float("inf")
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.where(diff == 0, 0.0, diff / a)
    return float(np.max(r))


def update_err(new_gpu, new_ref, scale, ulps: int = 1, allow=None) -> float:
    """Table rows after an update: max_i (|new_gpu - new_ref| - ulps x ulp(new_ref))_+ / scale_i,
    where scale_i = lr x the absolute term sum of that entry's gradient (ulps: the fp32
    roundings each side committed on the way, one per update step)."""
    g = np.asarray(new_gpu, np.float32).ravel()
    o = np.asarray(new_ref, np.float32).ravel()
    a = np.asarray(scale, np.float64).ravel()
    if o.size == 0:
        return 0.0
    if not np.all(np.isfinite(g)):
        return float("inf")
    diff = np.abs(g.astype(np.float64) - o.astype(np.float64))
    ex = diff - ulps * np.spacing(np.abs(o)).astype(np.float64)
    if allow is not None:
        ex = ex - np.asarray(allow, np.float64).ravel()
    ex = np.maximum(ex, 0.0)
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.where(ex == 0, 0.0, ex / a)
    return float(np.max(r))


def ssm_scales(o: dict, c: float) -> dict:
    """Per-output scale arrays of an oracle.sampled_softmax result with grad_scale c.
    g_t = c (p_t - 1) is itself a difference: its scale is c (p_t + 1), p_t = e^{-loss_t}."""
    sg = c * (np.exp(-o["loss"]) + 1.0)
    if np.all(o["db_true"] == 0):  # label-in mode: no true-class term
        sg = np.zeros_like(sg)
    hscale = np.abs(o["dw_true"]) / np.maximum(np.abs(o["db_true"]), 1e-300)[:, None]
    return {"loss": o["abs_loss"], "lse": o["abs_loss"], "dh": o["abs_dh"],
            "dw_true": sg[:, None] * hscale, "db_true": sg,
            "dw_s": o["abs_dw_s"], "db_s": o["abs_db_s"]}


def ssm_allow(o: dict) -> dict:
    """Per-output rounding-tie allowances (R-34) of an oracle.sampled_softmax result (zero in
    fp32 mode and for outputs without a bf16 G)."""
    z = lambda k: np.zeros_like(o[k])
    return {"loss": z("loss"), "lse": z("lse"), "dh": o["amb_dh"], "dw_true": z("dw_true"),
            "db_true": z("db_true"), "dw_s": o["amb_dw_s"], "db_s": o["amb_db_s"]}
