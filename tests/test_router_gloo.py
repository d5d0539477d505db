"""Host-side routing logic of the R > 1 step on CPU: two gloo ranks exchange counts and
payloads through paper_1605_08695_b200.step.Router exactly as the NCCL path does, and the
result is checked against the oracle's routing (oracle/step.py O4: owner o receives, from every
source rank in order, that source's slice destined to o; rows come back in request order).

The CUDA kernels are not involved (no GPU here): the per-rank Part and Gather are computed with
the oracle, which is test infrastructure; only the Router (the product's routing code) moves data.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from oracle import step as ostep
import workloads


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1605_08695_b200.step import Router
        rt = Router()
        w = workloads.WORKLOADS["T"]
        V, R = w.vocab, world
        E, W, b = workloads.tables(V, w.dim)
        xs = [workloads.batch(w, R, r)[0] for r in range(R)]
        x = xs[rank]
        local, pos, counts = oracle.partition(x, V, R)
        (send,), (recv,) = rt.exchange_counts(torch.from_numpy(counts).view(R, 1))
        ids = rt.route(torch.from_numpy(local), send, recv).numpy()
        # oracle routing of every rank's request, then this rank's view
        parts = [oracle.partition(xx, V, R) for xx in xs]
        want = ostep._route([p[0] for p in parts], [p[2] for p in parts], R)[rank]
        ok_ids = np.array_equal(ids, want)
        # owner gathers from its shard and routes the rows back; requester stitches
        rows = oracle.gather(E[rank::R], ids)
        back = rt.route(torch.from_numpy(rows), recv, send).numpy()
        h = oracle.stitch(pos, back)
        ok_h = np.array_equal(h, E[x])
        # gradient route: sort-reduce by (owner, local), route, owner applies
        g = np.random.default_rng(rank).standard_normal((x.size, w.dim))
        l2, s2, c2 = oracle.sort_reduce(x, R, g)
        (sg,), (rg,) = rt.exchange_counts(torch.from_numpy(c2).view(R, 1))
        rids = rt.route(torch.from_numpy(l2), sg, rg).numpy()
        rrows = rt.route(torch.from_numpy(s2), sg, rg).numpy()
        shard = oracle.scatter_add_sgd(E[rank::R], rids, rrows, 1.0)
        # reference: the same update from all ranks' gradients on the unsharded table
        allg = [np.random.default_rng(r).standard_normal((xs[r].size, w.dim)) for r in range(R)]
        ref = oracle.scatter_add_sgd(E, np.concatenate(xs), np.concatenate(allg), 1.0)[rank::R]
        ok_g = np.allclose(shard, ref, rtol=0, atol=1e-5)
        q.put((rank, ok_ids, ok_h, ok_g, sum(recv)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_router_gloo_matches_oracle_routing(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_ids, ok_h, ok_g, nrecv in res:
        assert ok_ids, f"rank {rank}: routed ids differ from the oracle's route"
        assert ok_h, f"rank {rank}: stitched rows differ from E[x]"
        assert ok_g, f"rank {rank}: routed sparse update differs from the unsharded update"
    w = workloads.WORKLOADS["T"]
    assert sum(r[4] for r in res) == world * w.tokens_per_replica(world)


def _slot_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1605_08695_b200.step import Router
        rt = Router()
        R, cap = world, 6
        # requester r sends to owner o the distinct local ids it needs, padded with -1
        need = [[np.unique(np.arange(o + r, 40, R) // R)[:cap] for o in range(R)]
                for r in range(R)]
        send = np.full((R, cap + 3), -7, np.int64)   # 3 trailing elements outside the slots
        for o in range(R):
            send[o, :cap] = -1
            send[o, :need[rank][o].size] = need[rank][o]
        recv = torch.empty((R, cap + 3), dtype=torch.int64)
        rt.a2a(recv, torch.from_numpy(send))
        ok = all(np.array_equal(recv.numpy()[src, :need[src][rank].size], need[src][rank])
                 and np.all(recv.numpy()[src, need[src][rank].size:cap] == -1)
                 for src in range(R))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_fixed_capacity_slot_exchange_gloo():
    """Router.a2a: region o of the send buffer lands in region `rank` of owner o's receive
    buffer, in source-rank order (the R > 1 step's slot exchanges)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slot_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == {0: True, 1: True}
