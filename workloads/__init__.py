"""Seeded synthetic inputs shared by the CUDA path's tests/bench and by the oracle.

This module holds NO arithmetic of the method: only the workload shapes (BASELINE.json
``configs``) and seeded random inputs -- Zipf-distributed token ids laid out as
LM1B-style sequences, and uniformly initialised fp32 tables.  Both sides receive the same bytes.
Random numbers the method itself draws (the candidate sampler) are NOT generated here: each
side implements the counter-based Philox generator independently (R-17).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    vocab: int          # V
    dim: int            # d
    tokens: int         # B = tokens per replica per step (weak scaling) ...
    num_sampled: int    # S per replica per step (0 => full softmax over all V classes)
    shards: int         # default R
    zipf_s: float = 1.0
    strong: bool = False  # ... or global tokens split over R replicas (strong scaling)
    seq_len: int = 20     # LM1B unroll: 20 input words -> 20 next words (21-id sequences)

    def tokens_per_replica(self, R: int) -> int:
        return self.tokens // R if self.strong else self.tokens


# BASELINE.json configs[0..4] (names T, L, F, X, Z as in SURVEY.md §8(d)).
WORKLOADS = {
    "T": Workload("T", 1000, 64, 32, 64, 2),
    "L": Workload("L", 40_000, 512, 128 * 20, 512, 1),
    "F": Workload("F", 40_000, 512, 128 * 20, 0, 1),
    "X": Workload("X", 800_000, 512, 128 * 20, 8192, 1),
    "Z": Workload("Z", 800_000, 512, 65_536, 8192, 1, zipf_s=1.1, strong=True),
}

DATA_SEED = 1234
TABLE_SEED = 42
SAMPLER_SEED = 7


def zipf_ids(rng: np.random.Generator, vocab: int, s: float, n: int) -> np.ndarray:
    """n ids with P(id = k) proportional to (k+1)^-s on [0, vocab): frequency rank = id."""
    w = 1.0 / np.arange(1, vocab + 1, dtype=np.float64) ** s
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    u = rng.random(n)
    ids = np.searchsorted(cdf, u, side="right")
    return np.minimum(ids, vocab - 1).astype(np.int64)


def batch(w: Workload, R: int, replica: int, step: int = 0, seed: int = DATA_SEED):
    """(x, y) int64[B] for one replica: ceil(B/20) sequences of 21 Zipf ids; x = words 0..19,
    y = words 1..20 of each sequence (next-word prediction), flattened row-major."""
    B = w.tokens_per_replica(R)
    L = w.seq_len
    n_seq = -(-B // L)
    rng = np.random.Generator(np.random.PCG64([seed, step, replica]))
    seqs = zipf_ids(rng, w.vocab, w.zipf_s, n_seq * (L + 1)).reshape(n_seq, L + 1)
    x = np.ascontiguousarray(seqs[:, :L]).reshape(-1)[:B]
    y = np.ascontiguousarray(seqs[:, 1:]).reshape(-1)[:B]
    return x, y


def tables(vocab: int, dim: int, seed: int = TABLE_SEED):
    """Logical unsharded tables: E, W ~ U(-0.5, 0.5) [V, d]; b ~ U(-0.1, 0.1) [V]; fp32."""
    rng = np.random.Generator(np.random.PCG64(seed))
    E = (rng.random((vocab, dim), dtype=np.float32) - np.float32(0.5))
    W = (rng.random((vocab, dim), dtype=np.float32) - np.float32(0.5))
    b = (rng.random(vocab, dtype=np.float32) - np.float32(0.5)) * np.float32(0.2)
    return E, W, b



def shard_rows_count(vocab: int, num_shards: int, shard: int) -> int:
    """Rows of shard r under the id-mod-R layout: n_r = ceil((V - r) / R)."""
    return -(-(vocab - shard) // num_shards)


def tables_device(vocab: int, dim: int, num_shards: int, shard: int, device, seed: int = TABLE_SEED):
    """Bench-scale variant of ``tables``: shard r's rows generated directly on the GPU with a
    seeded torch generator (same distributions; a different stream of random numbers than the
    numpy generator, so parity tests use ``tables``).  Returns (E_r, W_r, b_r)."""
    import torch
    n = shard_rows_count(vocab, num_shards, shard)
    g = torch.Generator(device=device)
    g.manual_seed(seed * 1000003 + shard)
    E = torch.rand((n, dim), generator=g, device=device, dtype=torch.float32).sub_(0.5)
    W = torch.rand((n, dim), generator=g, device=device, dtype=torch.float32).sub_(0.5)
    b = torch.rand(n, generator=g, device=device, dtype=torch.float32).sub_(0.5).mul_(0.2)
    return E, W, b
