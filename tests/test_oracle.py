"""Pins for the CPU oracle (runs without a GPU: -m "not gpu").

Each test pins an oracle function to something other than itself: a worked example printed in
SPEC.md / the paper (tests/golden/), a textbook or library routine (numpy, torch bf16 casts,
Random123 known-answer vectors), a closed form, an invariant, brute force on tiny inputs, or
central finite differences.  A plausible slip in the oracle (dropped term, wrong sign, wrong
index, transposed operand) fails at least one of them.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
from oracle import step as ostep
import workloads

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


# ------------------------------------------------------------------------------------------ Part
def test_partition_spec_examples():
    for ex in _golden("spec_examples.json")["partition"]:
        local, pos, counts = oracle.partition(ex["indices"], 0, ex["num_shards"],
                                              assignments=ex["assignments"])
        off = np.concatenate([[0], np.cumsum(counts)])
        shards = [local[off[s]:off[s + 1]].tolist() for s in range(ex["num_shards"])]
        assert shards == ex["shards"], ex["cite"]
        # positions point back at the original slot of each element
        ids = np.asarray(ex["indices"], np.int64)
        assert np.array_equal(ids[pos], local)


@pytest.mark.parametrize("R", [1, 2, 3, 5, 8])
def test_partition_equals_stable_sort(R):
    rng = np.random.default_rng(R)
    V = 997
    ids = rng.integers(0, V, 501)
    local, pos, counts = oracle.partition(ids, V, R)
    order = sorted(range(ids.size), key=lambda i: ids[i] % R)  # Python's sort is stable
    assert pos.tolist() == order
    assert np.array_equal(local, ids[order] // R)
    assert counts.tolist() == [int(np.sum(ids % R == o)) for o in range(R)]
    assert counts.sum() == ids.size
    # every local id is a valid row of its shard: n_r = ceil((V - r) / R)   (R-28)
    off = np.concatenate([[0], np.cumsum(counts)])
    for o in range(R):
        n_o = -(-(V - o) // R)
        assert np.all(local[off[o]:off[o + 1]] < n_o)


@pytest.mark.parametrize("R", [1, 2, 3, 8])
def test_stitch_of_part_is_identity(R):
    """BJ check: Stitch(Part(x)) == x."""
    rng = np.random.default_rng(10 + R)
    x = rng.integers(0, 5000, 777)
    local, pos, counts = oracle.partition(x, 5000, R)
    owner = np.repeat(np.arange(R), counts)
    rebuilt = oracle.stitch(pos, (local * R + owner).reshape(-1, 1))[:, 0]
    assert np.array_equal(rebuilt, x)


def test_partition_errors():
    with pytest.raises(oracle.OracleError) as e:
        oracle.partition([3, 10, 2, 11], 10, 2)
    assert e.value.status == oracle.OUT_OF_RANGE and e.value.bad == 1
    with pytest.raises(oracle.OracleError) as e:
        oracle.partition([0, 1, 2], 0, 2, assignments=[0, 1, 2])
    assert e.value.bad == 2
    local, pos, counts = oracle.partition(np.zeros(0, np.int64), 10, 4)
    assert local.size == 0 and counts.tolist() == [0, 0, 0, 0]


# ---------------------------------------------------------------------------------------- Gather
def test_gather_spec_examples():
    for ex in _golden("spec_examples.json")["gather"]:
        out = oracle.gather(np.asarray(ex["params"], np.float32), ex["indices"])
        assert out.tolist() == ex["out"], ex["cite"]


def test_gather_equals_onehot_matmul():
    """gather == onehot(idx) . params, exactly (one nonzero term per output)."""
    rng = np.random.default_rng(1)
    params = rng.standard_normal((50, 17)).astype(np.float32)
    idx = rng.integers(0, 50, 40)
    onehot = np.zeros((40, 50))
    onehot[np.arange(40), idx] = 1.0
    ref = onehot @ params.astype(np.float64)
    assert np.array_equal(oracle.gather(params, idx).astype(np.float64), ref)


def test_gather_bf16_matches_torch_cast():
    rng = np.random.default_rng(2)
    params = (rng.standard_normal((20, 8)) * 3).astype(np.float32)
    idx = rng.integers(0, 20, 30)
    got = oracle.gather(params, idx, bf16=True)
    ref = torch.from_numpy(params[idx]).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(got, ref)


def test_gather_out_of_range():
    with pytest.raises(oracle.OracleError) as e:
        oracle.gather(np.zeros((4, 2), np.float32), [0, 3, 4, -1, 9])
    assert e.value.status == oracle.OUT_OF_RANGE and e.value.bad == 2


# ---------------------------------------------------------------------------------------- Stitch
def test_stitch_spec_and_scatter():
    for ex in _golden("spec_examples.json")["stitch"]:
        out = oracle.stitch(ex["positions"], np.asarray(ex["data"], np.float32))
        assert out.tolist() == ex["out"], ex["cite"]
    rng = np.random.default_rng(3)
    perm = rng.permutation(64)
    rows = rng.standard_normal((64, 5)).astype(np.float32)
    ref = np.empty_like(rows)
    ref[perm] = rows                                    # direct scatter
    assert np.array_equal(oracle.stitch(perm, rows), ref)


def test_stitch_bad_positions():
    rows = np.zeros((4, 1), np.float32)
    for pos, bad in (([0, 1, 1, 2], 2), ([0, 4, 1, 2], 1), ([3, 2, -1, 0], 2)):
        with pytest.raises(oracle.OracleError) as e:
            oracle.stitch(pos, rows)
        assert e.value.status == oracle.BAD_POSITIONS and e.value.bad == bad


# ------------------------------------------------------------------------------------------ bf16
def test_bf16_round_matches_torch():
    rng = np.random.default_rng(4)
    x = np.concatenate([rng.standard_normal(10000).astype(np.float32) * 10,
                        np.array([0.0, -0.0, 1.0, 1.00390625, 1.01171875, 65504.0, 3.4e38,
                                  1e-40, -1e-40, np.inf, -np.inf], np.float32)])
    # exact ties: 1 + 2^-8 rounds to 1 (even), 1 + 3*2^-8 rounds up to 1 + 2^-6
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float32).numpy()
    assert np.array_equal(oracle.bf16_round(x), ref)


# --------------------------------------------------------------------------------------- Sampler
def test_philox_known_answers():
    with open(os.path.join(GOLDEN, "philox4x32_10_kat.txt")) as f:
        lines = [l.split() for l in f if l.strip() and not l.startswith("#")]
    for w in lines:
        vals = [int(v, 16) for v in w]
        assert oracle.philox4x32_10(vals[0:4], vals[4:6]).tolist() == vals[6:10]


@pytest.mark.parametrize("V", [1000, 40000])
def test_log_uniform_probabilities(V):
    p = np.array([oracle.log_uniform_prob(V, k) for k in range(V)])
    assert abs(p.sum() - 1.0) < 1e-12                      # telescoping sum
    assert np.all(np.diff(p) < 0)                          # strictly decreasing in rank
    thr = oracle.log_uniform_thresholds(V)
    assert np.all(np.diff(thr.astype(np.float64)) > 0)     # strictly increasing thresholds
    assert thr[-1] == 1 << 53
    widths = np.diff(np.concatenate([[0], thr.astype(np.float64)])) / 2.0 ** 53
    assert np.max(np.abs(widths - p)) < 4.0 / 2.0 ** 53    # P(k) = Thr[k] - Thr[k-1]


def test_sampler_matches_float_inverse_cdf():
    """The integer threshold search is the log-uniform inverse CDF k = floor(e^{u ln(V+1)}) - 1
    (TF's formulation) up to rare boundary ties: an independent construction of R-6."""
    V, n, seed, step, rep = 40000, 4000, 99, 3, 1
    s, T, _, _ = oracle.sample(V, n, False, seed, step, rep, np.zeros(0, np.int64))
    assert T == n
    agree = 0
    for i in range(n):
        w = oracle.philox4x32_10([i, step >> 32, step & 0xffffffff, rep],
                                 [seed & 0xffffffff, seed >> 32])
        m = ((int(w[0]) << 32) | int(w[1])) >> 11
        k = math.floor(math.exp(m / 2.0 ** 53 * math.log(V + 1))) - 1
        agree += int(k == s[i])
    assert agree >= n - 2


def test_sampler_chi_square():
    V, n = 50, 200000
    s, _, _, _ = oracle.sample(V, n, False, 5, 0, 0, np.zeros(0, np.int64))
    p = np.array([oracle.log_uniform_prob(V, k) for k in range(V)])
    obs = np.bincount(s, minlength=V)
    chi2 = np.sum((obs - n * p) ** 2 / (n * p))
    assert chi2 < 100.0           # 49 dof: mean 49, sd ~10; 100 is > 5 sd


@pytest.mark.parametrize("V,S", [(1000, 64), (40000, 512), (1000, 999)])
def test_unique_sampler_is_first_distinct_in_draw_order(V, S):
    seed, step, rep = 7, 11, 2
    s, T, les, _ = oracle.sample(V, S, True, seed, step, rep, np.zeros(0, np.int64))
    draws, _, _, _ = oracle.sample(V, T, False, seed, step, rep, np.zeros(0, np.int64))
    first, seen = [], set()
    for k in draws.tolist():                           # brute force, sequential
        if k not in seen:
            seen.add(k)
            first.append(k)
    assert first == s.tolist() and len(first) == S
    assert draws[-1] not in set(draws[:-1].tolist())  # T-th draw completed the set
    assert np.all(np.isfinite(les))


def test_expected_counts_statistics():
    """ec(k) is the probability that k is among the T draws (unique mode) and S*p_k is the
    expected multiplicity (non-unique mode): Monte Carlo over seeds."""
    V, S, n_seeds = 1000, 64, 1500
    labels = np.arange(6, dtype=np.int64)
    inc = np.zeros(6)
    ec_mean = np.zeros(6)
    for seed in range(n_seeds):
        s, T, _, ley = oracle.sample(V, S, True, seed, 0, 0, labels)
        inc += np.isin(labels, s)
        ec_mean += np.exp(ley)
    inc /= n_seeds
    ec_mean /= n_seeds
    assert np.all(np.abs(inc - ec_mean) < 0.05 + 0.1 * ec_mean)
    cnt = np.zeros(6)
    for seed in range(300):
        s, T, _, ley = oracle.sample(V, S, False, seed, 0, 0, labels)
        cnt += np.bincount(s, minlength=V)[:6]
    mean = cnt / 300
    expect = np.exp(ley)                               # S * p_k, seed independent
    assert np.all(np.abs(mean - expect) < 4 * np.sqrt(expect / 300) + 0.05)


def test_sampler_exhaustion_and_counters():
    with pytest.raises(oracle.OracleError) as e:
        oracle.sample(1000, 999, True, 1, 0, 0, np.zeros(0, np.int64), max_draws=500)
    assert e.value.status == oracle.EXHAUSTED
    # paper §6.4 "a factor of 78": |V| / S rows of the 40,000-class softmax are transferred
    nums = _golden("paper_numbers.json")
    V, S = nums["vocab_lm1b_restricted"]["value"], nums["num_sampled"]["value"]
    assert round(V / S) == nums["reduction_factor"]["value"]
    assert round(V / (S + 1)) == nums["reduction_factor"]["value"]


# ------------------------------------------------------------------------------ Sampled softmax
def _ssm_inputs(rng, B, S, V, d, hit_frac=0.3):
    h = rng.standard_normal((B, d)).astype(np.float32) * 0.5
    labels = rng.integers(0, V, B)
    sampled = rng.choice(V, S, replace=False)
    # force some accidental hits
    nh = int(B * hit_frac)
    labels[:nh] = rng.choice(sampled, nh)
    W = rng.standard_normal((V, d)).astype(np.float32) * 0.5
    b = rng.standard_normal(V).astype(np.float32) * 0.1
    le = rng.standard_normal(V) * 0.3 - 2.0
    return h, labels, W, b, le, sampled


def _numpy_full_softmax(h, labels, W, b, c):
    """Textbook dense softmax cross-entropy and its gradients (fp64 numpy)."""
    logits = h.astype(np.float64) @ W.astype(np.float64).T + b
    m = logits.max(axis=1, keepdims=True)
    lse = (m + np.log(np.exp(logits - m).sum(axis=1, keepdims=True)))[:, 0]
    B = h.shape[0]
    loss = lse - logits[np.arange(B), labels]
    P = np.exp(logits - lse[:, None])
    onehot = np.zeros_like(P)
    onehot[np.arange(B), labels] = 1.0
    dlog = c * (P - onehot)
    return loss, lse, dlog @ W.astype(np.float64), dlog.T @ h.astype(np.float64), dlog.sum(0)


def test_full_vocab_candidates_equal_full_softmax():
    """BJ check / S:583: all classes as candidates, no log-Q, hits excluded == full softmax."""
    rng = np.random.default_rng(5)
    B, V, d = 13, 37, 6
    h, labels, W, b, _, _ = _ssm_inputs(rng, B, V, V, d)
    sampled = np.arange(V)
    c = 1.0 / B
    o = oracle.sampled_softmax(h, labels, W[labels], b[labels], np.zeros(B), sampled, W, b,
                               np.zeros(V), flags=oracle.REMOVE_ACCIDENTAL_HITS, grad_scale=c)
    loss, lse, dh, dW, db = _numpy_full_softmax(h, labels, W, b, c)
    np.testing.assert_allclose(o["loss"], loss, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(o["lse"], lse, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(o["dh"], dh, rtol=1e-10, atol=1e-13)
    dW_o = o["dw_s"].copy()
    db_o = o["db_s"].copy()
    np.add.at(dW_o, labels, o["dw_true"])
    np.add.at(db_o, labels, o["db_true"])
    np.testing.assert_allclose(dW_o, dW, rtol=1e-10, atol=1e-13)
    np.testing.assert_allclose(db_o, db, rtol=1e-10, atol=1e-13)


def test_closed_form_zero_hidden():
    """h = 0, no log-Q, equal biases: loss_t = ln(1 + S - hits_t), G_tj = c / (1 + S - hits_t)."""
    rng = np.random.default_rng(6)
    B, S, V, d = 9, 11, 50, 4
    _, labels, W, _, _, sampled = _ssm_inputs(rng, B, S, V, d, hit_frac=0.5)
    h = np.zeros((B, d), np.float32)
    bb = np.full(V, 0.25, np.float32)
    c = 0.5
    o = oracle.sampled_softmax(h, labels, W[labels], bb[labels], np.zeros(B), sampled, W[sampled],
                               bb[sampled], np.zeros(S), flags=oracle.REMOVE_ACCIDENTAL_HITS,
                               grad_scale=c)
    hits = np.array([np.sum(sampled == y) for y in labels])
    np.testing.assert_allclose(o["loss"], np.log(1 + S - hits), rtol=1e-14)
    # db_s_j = sum over non-hit tokens of c / (1 + S - hits_t)
    ref = np.array([sum(c / (1 + S - hits[t]) for t in range(B) if labels[t] != sampled[j])
                    for j in range(S)])
    np.testing.assert_allclose(o["db_s"], ref, rtol=1e-13)
    np.testing.assert_allclose(o["db_true"], c * (1.0 / (1 + S - hits) - 1.0), rtol=1e-13)


def test_gradient_sum_and_bias_shift_invariants():
    rng = np.random.default_rng(7)
    B, S, V, d = 17, 23, 300, 8
    h, labels, W, b, le, sampled = _ssm_inputs(rng, B, S, V, d)
    args = (h, labels, W[labels], b[labels], le[labels], sampled, W[sampled], b[sampled],
            le[sampled])
    o = oracle.sampled_softmax(*args, grad_scale=0.1)
    # per token g_t + sum_j G_tj = 0  =>  total of all bias gradients is 0
    assert abs(o["db_true"].sum() + o["db_s"].sum()) < 1e-14
    shifted = list(args)
    shifted[3] = args[3] + np.float32(0.5)
    shifted[7] = args[7] + np.float32(0.5)
    o2 = oracle.sampled_softmax(*shifted, grad_scale=0.1)
    np.testing.assert_allclose(o2["loss"], o["loss"], rtol=1e-6)  # fp32 bias shift rounding


def test_log_q_correction_is_subtracted():
    """With flag 1 the logits are corrected by -ln ec: a shift of log_ec_s by +delta on every
    class equals lowering every sampled logit by delta (the loss rises)."""
    rng = np.random.default_rng(8)
    B, S, V, d = 5, 7, 40, 4
    h, labels, W, b, le, sampled = _ssm_inputs(rng, B, S, V, d, hit_frac=0.0)
    f = oracle.SUBTRACT_LOG_Q | oracle.REMOVE_ACCIDENTAL_HITS
    base = oracle.sampled_softmax(h, labels, W[labels], b[labels], le[labels], sampled,
                                  W[sampled], b[sampled], le[sampled], flags=f)
    moved = oracle.sampled_softmax(h, labels, W[labels], b[labels], le[labels], sampled,
                                   W[sampled], b[sampled] - np.float32(1.0), le[sampled], flags=f)
    shifted = oracle.sampled_softmax(h, labels, W[labels], b[labels], le[labels], sampled,
                                     W[sampled], b[sampled], le[sampled] + 1.0, flags=f)
    np.testing.assert_allclose(shifted["loss"], moved["loss"], rtol=1e-6)
    assert np.all(moved["loss"] < base["loss"])


def test_finite_differences():
    """central differences in f64, h = 1e-6 (on fp32-exact perturbations of the
    inputs the oracle reads as fp32 we use a dyadic step), relative error < 1e-5."""
    rng = np.random.default_rng(9)
    B, S, V, d = 4, 6, 30, 3
    h, labels, W, b, le, sampled = _ssm_inputs(rng, B, S, V, d, hit_frac=0.25)
    c = 0.25
    base = dict(h=h, w_true=W[labels], b_true=b[labels], w_s=W[sampled], b_s=b[sampled])

    def L(**kw):
        a = dict(base, **kw)
        o = oracle.sampled_softmax(a["h"], labels, a["w_true"], a["b_true"], le[labels], sampled,
                                   a["w_s"], a["b_s"], le[sampled], grad_scale=c)
        return c * o["loss"].sum()

    o = oracle.sampled_softmax(h, labels, base["w_true"], base["b_true"], le[labels], sampled,
                               base["w_s"], base["b_s"], le[sampled], grad_scale=c)
    eps = 2.0 ** -12  # exactly representable; fp32 inputs keep every bit of the perturbation
    checks = []
    for name, grad in (("h", o["dh"]), ("w_true", o["dw_true"]), ("w_s", o["dw_s"]),
                       ("b_true", o["db_true"]), ("b_s", o["db_s"])):
        arr = base[name]
        for idx in np.ndindex(arr.shape):
            p = arr.copy(); p[idx] += eps
            m = arr.copy(); m[idx] -= eps
            fd = (L(**{name: p}) - L(**{name: m})) / (2 * eps)
            checks.append((fd, grad[idx]))
    fd = np.array([a for a, _ in checks])
    an = np.array([g for _, g in checks])
    rel = np.abs(fd - an) / np.maximum(np.abs(an), 1e-3 * np.abs(an).max())
    assert rel.max() < 1e-5


def test_bf16_mode_rounding_points():
    """bf16 mode = fp32-operand definition evaluated on RNE-rounded h / W_true / W_s with G
    rounded to bf16 before the dh / dW_s / db_s reductions (R-18), recomputed with numpy+torch."""
    rng = np.random.default_rng(10)
    B, S, V, d = 8, 12, 60, 16
    h, labels, W, b, le, sampled = _ssm_inputs(rng, B, S, V, d)
    c = 0.125
    o = oracle.sampled_softmax(h, labels, W[labels], b[labels], le[labels], sampled, W[sampled],
                               b[sampled], le[sampled], grad_scale=c, bf16=True)
    r = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).double().numpy()
    hb, wt, ws = r(h), r(W[labels]), r(W[sampled])
    z = (hb * wt).sum(1) + b[labels] - le[labels]
    Z = hb @ ws.T + b[sampled] - le[sampled]
    mask = labels[:, None] == sampled[None, :]
    Zm = np.where(mask, -np.inf, Z)
    mu = np.maximum(z, Zm.max(1))
    lse = mu + np.log(np.exp(z - mu) + np.exp(Zm - mu[:, None]).sum(1))
    np.testing.assert_allclose(o["lse"], lse, rtol=1e-13)
    G = np.where(mask, 0.0, c * np.exp(Z - lse[:, None]))
    Gr = torch.from_numpy(G.astype(np.float32)).to(torch.bfloat16).double().numpy()
    g = c * (np.exp(z - lse) - 1.0)
    np.testing.assert_allclose(o["dh"], g[:, None] * wt + Gr @ ws, rtol=1e-11, atol=1e-14)
    np.testing.assert_allclose(o["dw_s"], Gr.T @ hb, rtol=1e-11, atol=1e-14)
    np.testing.assert_allclose(o["db_s"], Gr.sum(0), rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(o["dw_true"], g[:, None] * hb, rtol=1e-13)


def test_subset_outputs_match_full():
    rng = np.random.default_rng(11)
    B, S, V, d = 10, 9, 80, 5
    h, labels, W, b, le, sampled = _ssm_inputs(rng, B, S, V, d)
    args = (h, labels, W[labels], b[labels], le[labels], sampled, W[sampled], b[sampled],
            le[sampled])
    full = oracle.sampled_softmax(*args, grad_scale=0.3)
    ti, ci = np.array([7, 2, 2]), np.array([0, 8])
    sub = oracle.sampled_softmax(*args, grad_scale=0.3, tok_idx=ti, col_idx=ci)
    for k in ("loss", "lse", "dh", "dw_true", "db_true"):
        assert np.array_equal(sub[k], full[k][ti])
    for k in ("dw_s", "db_s"):
        assert np.array_equal(sub[k], full[k][ci])


# ----------------------------------------------------------------------------- ScatterAdd / SGD
def test_scatter_sgd_spec_examples():
    g = _golden("spec_examples.json")
    ex = g["apply_sgd"][0]
    out = oracle.scatter_add_sgd(np.array([[ex["W"]]], np.float32), [0], [[ex["g"]]], ex["alpha"])
    assert out[0, 0] == np.float32(ex["out"]), ex["cite"]
    for ex in g["apply_sparse"]:
        t = np.zeros((ex["rows"], ex["dim"]), np.float32)
        grads = np.asarray(ex["grads"], np.float64).reshape(-1, ex["dim"])
        out = oracle.scatter_add_sgd(t, ex["ids"], grads, ex["alpha"])
        assert out.tolist() == ex["out"], ex["cite"]


def test_scatter_sgd_equals_dense_onehot_gradient():
    """sparse gradient via scatter-add == dense one-hot^T . rows gradient."""
    rng = np.random.default_rng(12)
    V, d, n = 40, 6, 100
    T = rng.standard_normal((V, d)).astype(np.float32)
    ids = rng.integers(0, 10, n)                 # heavy duplicates
    G = rng.standard_normal((n, d))
    onehot = np.zeros((n, V))
    onehot[np.arange(n), ids] = 1.0
    dense = onehot.T @ G
    ref = T.copy()
    touched = np.unique(ids)
    ref[touched] = (T[touched].astype(np.float64) - 0.3 * dense[touched]).astype(np.float32)
    out = oracle.scatter_add_sgd(T, ids, G, 0.3)
    np.testing.assert_array_max_ulp(out, ref, maxulp=1)
    untouched = np.setdiff1d(np.arange(V), touched)
    assert np.array_equal(out[untouched], T[untouched])
    assert np.array_equal(oracle.scatter_add_sgd(T, ids, G, 0.0), T)    # alpha = 0


def test_scatter_sgd_out_of_range():
    with pytest.raises(oracle.OracleError) as e:
        oracle.scatter_add_sgd(np.zeros((3, 2), np.float32), [0, 2, 3, 5], np.zeros((4, 2)), 1.0)
    assert e.value.bad == 2


def test_sort_reduce_brute_force():
    rng = np.random.default_rng(13)
    ids = rng.integers(0, 30, 200)
    rows = rng.standard_normal((200, 3))
    for R in (1, 2, 3, 8):
        local, sums, counts = oracle.sort_reduce(ids, R, rows)
        ref = {}
        for i, k in enumerate(ids.tolist()):
            ref.setdefault((k % R, k // R), np.zeros(3))
            ref[(k % R, k // R)] += rows[i]
        keys = sorted(ref)
        assert local.tolist() == [k[1] for k in keys]
        assert counts.tolist() == [sum(1 for k in keys if k[0] == o) for o in range(R)]
        np.testing.assert_allclose(sums, np.array([ref[k] for k in keys]), rtol=1e-14)


# ------------------------------------------------------------------------------------------ Step
def _tiny_step(R, bf16=False, full=False):
    w = workloads.WORKLOADS["T"]
    E, W, b = workloads.tables(w.vocab, w.dim)
    xs, ys = zip(*[workloads.batch(w, R, r) for r in range(R)])
    cfg = ostep.StepConfig(vocab=w.vocab, dim=w.dim, num_sampled=w.num_sampled, num_shards=R,
                           lr=1.0, bf16=bf16, full_softmax=full)
    return E, W, b, xs, ys, cfg, ostep.step(E, W, b, list(xs), list(ys), cfg)


@pytest.mark.parametrize("R", [1, 2, 3, 5])
def test_step_lookup_is_plain_definition(R):
    """O6 invariant: h_r == E[x_r], W rows == W[y_r || s_r], bit for bit, for any R."""
    E, W, b, xs, ys, cfg, (E2, W2, b2, tr) = _tiny_step(R)
    for r in range(R):
        assert np.array_equal(tr[r].h, E[xs[r]])
        q = np.concatenate([ys[r], tr[r].sampled])
        assert np.array_equal(tr[r].w_rows, W[q])
        assert np.array_equal(tr[r].b_rows, b[q])
        assert tr[r].counts_x.sum() == len(xs[r])


def test_step_touches_only_read_rows():
    """training modifies only the rows read by the sparse multiplication."""
    E, W, b, xs, ys, cfg, (E2, W2, b2, tr) = _tiny_step(2)
    V = E.shape[0]
    te = np.unique(np.concatenate(xs))
    tw = np.unique(np.concatenate([np.concatenate([ys[r], tr[r].sampled]) for r in range(2)]))
    ue = np.setdiff1d(np.arange(V), te)
    uw = np.setdiff1d(np.arange(V), tw)
    assert np.array_equal(E2[ue], E[ue]) and np.array_equal(W2[uw], W[uw])
    assert np.array_equal(b2[uw], b[uw])
    assert np.any(E2[te] != E[te]) and np.any(W2[tw] != W[tw])


def test_step_r1_is_sequential_sgd():
    """with one replica the synchronous step is plain SGD on that replica's batch,
    recomputed here with the textbook dense formulas for the full-softmax variant (config F)."""
    E, W, b, xs, ys, cfg, (E2, W2, b2, tr) = _tiny_step(1, full=True)
    x, y = xs[0], ys[0]
    B = x.size
    loss, lse, dh, dW, db = _numpy_full_softmax(E[x], y, W, b, 1.0 / B)
    np.testing.assert_allclose(tr[0].ssm["loss"], loss, rtol=1e-12)
    dE = np.zeros(E.shape)
    np.add.at(dE, x, dh)
    touched = np.unique(x)
    refE = E.copy()
    refE[touched] = (E[touched] - 1.0 * dE[touched]).astype(np.float32)
    np.testing.assert_array_max_ulp(E2, refE, maxulp=1)
    refW = (W - 1.0 * dW).astype(np.float32)
    np.testing.assert_array_max_ulp(W2, refW, maxulp=1)
    np.testing.assert_array_max_ulp(b2, (b - db).astype(np.float32), maxulp=1)


# ------------------------------------------------- sparse Momentum / Adagrad (R-29)
def test_momentum_closed_form_constant_gradient():
    """k updates of one row with a constant gradient g: m_k = g (1 - mu^k) / (1 - mu) and
    w_k = w_0 - lr g sum_{i<=k} (1 - mu^i) / (1 - mu) (geometric series)."""
    mu, lr, g, k = 0.9, 0.05, np.array([0.3, -1.25, 2.0]), 12
    w = np.array([[1.0, -2.0, 0.5]], np.float32)
    m = np.zeros((1, 3), np.float32)
    for _ in range(k):
        w, m = oracle.scatter_opt("momentum", w, m, [0], g.reshape(1, 3), lr, mu)
    m_k = g * (1 - mu ** k) / (1 - mu)
    series = (k - mu * (1 - mu ** k) / (1 - mu)) / (1 - mu)
    assert np.allclose(m[0], m_k, rtol=1e-5)
    assert np.allclose(w[0], np.array([1.0, -2.0, 0.5]) - lr * g * series, rtol=1e-5, atol=1e-6)


def test_momentum_zero_is_sgd_and_duplicates_summed_once():
    rng = np.random.default_rng(3)
    T0 = rng.standard_normal((20, 4)).astype(np.float32)
    ids = np.array([3, 7, 3, 3, 19, 7])
    g = rng.standard_normal((6, 4))
    w_m, m = oracle.scatter_opt("momentum", T0, np.zeros_like(T0), ids, g, 0.1, 0.0)
    w_s = oracle.scatter_add_sgd(T0, ids, g, 0.1)
    assert np.array_equal(w_m, w_s)                       # mu = 0 is plain SGD
    # one call with duplicates == one occurrence per id carrying the sum
    uniq = np.array([3, 7, 19])
    gs = np.stack([g[ids == u].sum(axis=0) for u in uniq])
    w_u, m_u = oracle.scatter_opt("momentum", T0, np.zeros_like(T0), uniq, gs, 0.1, 0.0)
    assert np.allclose(w_m, w_u, rtol=0, atol=1e-7) and np.allclose(m, m_u, rtol=0, atol=1e-7)
    untouched = np.setdiff1d(np.arange(20), ids)
    assert np.array_equal(w_m[untouched], T0[untouched]) and not m[untouched].any()


def test_adagrad_closed_form_constant_gradient():
    """k updates with a constant gradient g and accumulator start a0:
    w_k = w_0 - lr g sum_{i<=k} 1 / sqrt(a0 + i g^2)."""
    lr, a0, k = 0.1, 0.1, 9
    g = np.array([0.5, -3.0, 0.01])
    w = np.array([[0.25, 1.0, -1.0]], np.float32)
    a = np.full((1, 3), a0, np.float32)
    for _ in range(k):
        w, a = oracle.scatter_opt("adagrad", w, a, [0], g.reshape(1, 3), lr)
    i = np.arange(1, k + 1)[:, None]
    want = np.array([0.25, 1.0, -1.0]) - lr * g * (1.0 / np.sqrt(a0 + i * g ** 2)).sum(axis=0)
    assert np.allclose(a[0], a0 + k * g ** 2, rtol=1e-5)
    assert np.allclose(w[0], want, rtol=1e-5, atol=1e-6)


def test_adagrad_step_bounded_by_lr():
    """|delta w| = lr |g| / sqrt(a + g^2) <= lr for a >= 0 (the update is scale-free)."""
    rng = np.random.default_rng(4)
    T0 = rng.standard_normal((50, 8)).astype(np.float32)
    ids = rng.integers(0, 50, 200)
    g = rng.standard_normal((200, 8)) * 100.0
    w, a = oracle.scatter_opt("adagrad", T0, np.zeros_like(T0), ids, g, 0.01)
    assert np.all(np.abs(w.astype(np.float64) - T0) <= 0.01 * (1 + 1e-6))


# ------------------------------------------------------- round 2 pins (VERDICT r1 "What's weak" 1)
def test_log_uniform_closed_form_values():
    """SURVEY c.4 prints p(k) for V = 1000, 40000, 800000 (k = 0, 1, V-1); the oracle's p_k
    must agree to half a unit in the last printed digit."""
    from decimal import Decimal
    g = _golden("log_uniform_closed_form.json")
    for v in g["values"]:
        printed = Decimal(v["p"])
        half_unit = Decimal(1).scaleb(printed.as_tuple().exponent) / 2
        got = oracle.log_uniform_prob(v["V"], v["k"])
        assert abs(Decimal(got) - printed) <= half_unit, (v, got)
    # k = 0 special case: p(0) = ln 2 / ln(V + 1) (the telescoping sum's first term)
    for V in (1000, 40000, 800000):
        assert abs(oracle.log_uniform_prob(V, 0) - math.log(2) / math.log(V + 1)) < 1e-16


def test_log_q_shift_invariance_pins_true_logit_correction():
    """R-10: ln ec is subtracted from the TRUE logit and from every sampled logit.  With the
    same value k for every label and every class, the correction shifts all logits of a token
    by -k, which the softmax cannot see: loss and every gradient equal the uncorrected ones.
    (Dropping the correction on either side breaks the equality.)"""
    rng = np.random.default_rng(21)
    B, S, V, d = 9, 13, 200, 5
    h, labels, W, b, _, sampled = _ssm_inputs(rng, B, S, V, d, hit_frac=0.3)
    plain = oracle.sampled_softmax(h, labels, W[labels], b[labels], np.zeros(B), sampled,
                                   W[sampled], b[sampled], np.zeros(S),
                                   flags=oracle.REMOVE_ACCIDENTAL_HITS, grad_scale=0.2)
    for k in (-3.0, 0.75, 11.0):
        cor = oracle.sampled_softmax(h, labels, W[labels], b[labels], np.full(B, k), sampled,
                                     W[sampled], b[sampled], np.full(S, k), grad_scale=0.2)
        np.testing.assert_allclose(cor["loss"], plain["loss"], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(cor["lse"], plain["lse"] - k, rtol=1e-12, atol=1e-11)
        for key in ("dh", "dw_true", "db_true", "dw_s", "db_s"):
            np.testing.assert_allclose(cor[key], plain[key], rtol=1e-10, atol=1e-15)
    # the true-logit correction alone: raising ln ec(y_t) lowers z_t, so every loss rises
    up = oracle.sampled_softmax(h, labels, W[labels], b[labels], np.full(B, 1.0), sampled,
                                W[sampled], b[sampled], np.zeros(S), grad_scale=0.2)
    assert np.all(up["loss"] > plain["loss"])


def test_label_in_candidates_equals_textbook_full_softmax():
    """R-30 (the sharded full softmax): all V classes as candidates with the label
    among them (flag 4, no true-class term) == the textbook dense softmax cross-entropy, loss
    and every gradient; and == the excluded-hit form with a separate true logit (R-9)."""
    rng = np.random.default_rng(22)
    B, V, d = 11, 29, 7
    h, labels, W, b, _, _ = _ssm_inputs(rng, B, V, V, d)
    c = 1.0 / B
    o = oracle.sampled_softmax(h, labels, None, None, None, np.arange(V), W, b, np.zeros(V),
                               flags=oracle.LABEL_IN_CANDIDATES, grad_scale=c)
    loss, lse, dh, dW, db = _numpy_full_softmax(h, labels, W, b, c)
    np.testing.assert_allclose(o["loss"], loss, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(o["lse"], lse, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(o["dh"], dh, rtol=1e-10, atol=1e-13)
    np.testing.assert_allclose(o["dw_s"], dW, rtol=1e-10, atol=1e-13)
    np.testing.assert_allclose(o["db_s"], db, rtol=1e-10, atol=1e-13)
    assert np.all(o["dw_true"] == 0) and np.all(o["db_true"] == 0)
    # a token whose label is missing from the candidates is an error in label-in mode
    keep = np.setdiff1d(np.arange(V), [labels[0]])
    with pytest.raises(oracle.OracleError):
        oracle.sampled_softmax(h, labels, None, None, None, keep, W[keep], b[keep],
                               np.zeros(keep.size), flags=oracle.LABEL_IN_CANDIDATES,
                               grad_scale=c)


def test_label_in_bf16_rounding_point():
    """bf16 emulation of the sharded full softmax (R-18 + R-30): operands rounded RNE, and
    G = c (p - onehot) rounded to bf16 AS A WHOLE at the label column (the GPU's epilogue
    forms c p - c in fp32, then rounds), recomputed with numpy + torch casts."""
    rng = np.random.default_rng(23)
    B, V, d = 10, 40, 16
    h, labels, W, b, _, _ = _ssm_inputs(rng, B, V, V, d)
    c = 0.05
    o = oracle.sampled_softmax(h, labels, None, None, None, np.arange(V), W, b, np.zeros(V),
                               flags=oracle.LABEL_IN_CANDIDATES, grad_scale=c, bf16=True)
    r = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).double().numpy()
    hb, wb = r(h), r(W)
    Z = hb @ wb.T + b
    m = Z.max(1)
    lse = m + np.log(np.exp(Z - m[:, None]).sum(1))
    onehot = np.zeros_like(Z)
    onehot[np.arange(B), labels] = 1.0
    Gr = r((c * (np.exp(Z - lse[:, None]) - onehot)).astype(np.float32))
    np.testing.assert_allclose(o["lse"], lse, rtol=1e-13)
    np.testing.assert_allclose(o["loss"], lse - Z[np.arange(B), labels], rtol=1e-12)
    np.testing.assert_allclose(o["dh"], Gr @ wb, rtol=1e-11, atol=1e-14)
    np.testing.assert_allclose(o["dw_s"], Gr.T @ hb, rtol=1e-11, atol=1e-14)
    np.testing.assert_allclose(o["db_s"], Gr.sum(0), rtol=1e-12, atol=1e-15)


def test_abs_term_sums_bound_the_outputs():
    """abs_* (the element-wise parity scale) are >= |output|, and equal it where every term is
    non-negative: G >= 0 in sampled mode, so with h >= 0, abs_dw_s == dw_s and
    abs_db_s == db_s; abs_loss = |lse| + |z|."""
    rng = np.random.default_rng(24)
    B, S, V, d = 12, 17, 300, 6
    h, labels, W, b, le, sampled = _ssm_inputs(rng, B, S, V, d)
    h = np.abs(h)
    o = oracle.sampled_softmax(h, labels, W[labels], b[labels], le[labels], sampled, W[sampled],
                               b[sampled], le[sampled], grad_scale=0.1)
    for k in ("dh", "dw_s", "db_s"):
        assert np.all(o["abs_" + k] >= np.abs(o[k]) * (1 - 1e-15))
    np.testing.assert_allclose(o["abs_dw_s"], o["dw_s"], rtol=1e-14)
    np.testing.assert_allclose(o["abs_db_s"], o["db_s"], rtol=1e-14)
    np.testing.assert_allclose(o["abs_loss"], np.abs(o["lse"]) + np.abs(o["z_true"]), rtol=1e-15)
    assert np.any(o["abs_dh"] > np.abs(o["dh"]) * 1.01)   # dh does cancel (g_t < 0 <= G)


def test_bf16_rounding_ties_are_flagged():
    """R-34: a G whose exact value is a bf16 rounding tie (within 2^-14) is flagged, and its
    term enters amb_* at one bf16 unit.  h = 0, equal biases, no log-Q: G_tj = c / (1 + S) for
    tokens without hits; with c = (1 + S)(1 + 2^-8), G = 1 + 2^-8 is exactly the midpoint of the
    bf16 neighbours 1 and 1 + 2^-7 (ties to even -> 1).  fp32 mode flags nothing."""
    rng = np.random.default_rng(25)
    B, S, V, d = 6, 9, 400, 4
    _, labels, W, _, _, sampled = _ssm_inputs(rng, B, S, V, d, hit_frac=0.0)
    labels = np.setdiff1d(np.arange(V), sampled)[:B]           # no accidental hits
    h = np.zeros((B, d), np.float32)
    bb = np.full(V, 0.5, np.float32)
    c = (1 + S) * (1 + 2.0 ** -8)
    args = (h, labels, W[labels], bb[labels], np.zeros(B), sampled, W[sampled], bb[sampled],
            np.zeros(S))
    o = oracle.sampled_softmax(*args, flags=oracle.REMOVE_ACCIDENTAL_HITS, grad_scale=c, bf16=True)
    np.testing.assert_array_equal(o["db_s"], np.full(S, B * 1.0))          # ties to even: 1.0
    np.testing.assert_allclose(o["amb_db_s"], np.full(S, B * 2.0 ** -8), rtol=1e-15)
    assert np.all(o["amb_dh"] <= o["abs_dh"] * 2.0 ** -8 * (1 + 1e-12))
    f = oracle.sampled_softmax(*args, flags=oracle.REMOVE_ACCIDENTAL_HITS, grad_scale=c)
    assert not f["amb_db_s"].any() and not f["amb_dh"].any() and not f["amb_dw_s"].any()
    # away from a tie nothing is flagged
    g = oracle.sampled_softmax(*args, flags=oracle.REMOVE_ACCIDENTAL_HITS, grad_scale=c * 1.001,
                               bf16=True)
    assert not g["amb_db_s"].any()
