"""Host-side logic of the R > 1 path on CPU, with two gloo ranks (no GPU here):

* the communicator bootstrap -- every rank's 64-byte CUDA IPC handle all-gathered in rank order
  (paper_1605_08695_b200.step.exchange_handles, the torch.distributed plumbing the one-process-
  per-GPU tfs_comm relies on);
* the symmetric heap: every rank must size (and carve) the same heap, whatever its shard's row
  count -- tfs_step_heap_bytes is host arithmetic of libtfs, evaluated on each rank for ragged
  vocabularies and compared across ranks;
* the oracle's view of the exchanges those heaps carry (O4: owner o receives, from every source
  rank in order, that source's distinct ids destined to o), checked against the slot layout the
  step uses (distinct ids ascending per owner region).
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


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
        import oracle
        import workloads
        from paper_1605_08695_b200 import step as gstep
        # 1. IPC handle exchange, rank order
        mine = bytes([rank + 1]) * 32 + bytes(range(32))
        allh = gstep.exchange_handles(mine)
        ok_h = all(allh[64 * r:64 * r + 64] == bytes([r + 1]) * 32 + bytes(range(32))
                   for r in range(world))
        # 2. symmetric heap sizes agree (ragged V, sampled and sharded-full configs)
        sizes = []
        for V, S in ((1000, 64), (4003, 0), (800_000, 8192)):
            cfg = gstep.StepConfig(vocab=V, dim=64, tokens=32, num_sampled=S, num_shards=world)
            sizes.append(gstep.heap_bytes(cfg))
        got = [None] * world
        dist.all_gather_object(got, sizes)
        ok_heap = all(g == sizes for g in got) and all(s > 64 * 1024 for s in sizes)
        # 3. slot layout of the id push: region `rank` of owner o = the distinct local ids this
        #    rank needs from o, ascending; the owner's receive order is the source-rank order
        w = workloads.WORKLOADS["T"]
        V, R = w.vocab, world
        xs = [workloads.batch(w, R, r)[0] for r in range(R)]
        x = xs[rank]
        local, pos, counts = oracle.partition(x, V, R)
        off = np.concatenate([[0], np.cumsum(counts)])
        regions = [np.unique(local[off[o]:off[o + 1]]) for o in range(R)]
        recv = [None] * world
        dist.all_gather_object(recv, regions)
        mine_in = [recv[src][rank] for src in range(world)]       # what owner `rank` receives
        want = [np.unique(xs[src][xs[src] % R == rank] // R) for src in range(R)]
        ok_ids = all(np.array_equal(a, b) for a, b in zip(mine_in, want))
        q.put((rank, ok_h, ok_heap, ok_ids))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_comm_bootstrap_and_symmetric_layout_gloo(world):
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
    for rank, ok_h, ok_heap, ok_ids in res:
        assert ok_h, f"rank {rank}: IPC handles not all-gathered in rank order"
        assert ok_heap, f"rank {rank}: symmetric heap sizes differ across ranks"
        assert ok_ids, f"rank {rank}: routed id regions differ from the oracle's route"
