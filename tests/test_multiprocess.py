"""N > 1 on CPU: two gloo ranks shard the SBS stream by the rule the GPU
path uses (batch t of a call -> rank t % N), each running its own cursor
(here the oracle's, so it runs without a GPU); rank 0 gathers the shards
and checks they reassemble the single-process stream exactly -- no data
exchange is needed on the path, only for this check.  Also checks the
max-over-ranks timing reduction the bench uses."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch

    import oracle as O
    from paper_2105_00619_b200.shard import shard_batch_count, shard_batches
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    labels = (np.arange(5000) % 10).astype(np.int32)
    off, mem = O.class_index(labels, 10)
    B, calls, per_call = 64, 3, 10
    cur = O.Cursor(O.sbs_plan([0.1] * 10, B), off, mem, B, 1234)
    mine = []
    for _ in range(calls):
        ex, _ = cur.next(per_call)  # every rank advances the whole stream
        ex = ex.reshape(per_call, B)
        idx = shard_batches(per_call, rank, world)
        assert len(idx) == shard_batch_count(per_call, rank, world)
        mine.append(ex[idx])
    mine = torch.from_numpy(np.concatenate(mine))
    gathered = [torch.zeros_like(mine) for _ in range(world)] if rank == 0 else None
    if rank == 0:
        dist.gather(mine, gathered, dst=0)
    else:
        dist.gather(mine, dst=0)
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        full = O.Cursor(O.sbs_plan([0.1] * 10, B), off, mem, B, 1234)
        ok = True
        for c in range(calls):
            want = full.next(per_call)[0].reshape(per_call, B)
            for r in range(world):
                part = gathered[r].numpy()[c * (per_call // world):(c + 1) * (per_call // world)]
                ok &= bool(np.array_equal(part, want[r::world]))
        q.put((ok, float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_sharded_stream(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    ok, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    assert ok
    assert tmax == float(world)


def test_interleave_roundtrip():
    from paper_2105_00619_b200.shard import interleave, shard_batches
    B, n = 4, 11
    stream = list(range(n * B))
    for world in (1, 2, 3, 4):
        parts = [[x for t in shard_batches(n, r, world) for x in stream[t * B:(t + 1) * B]] for r in range(world)]
        assert interleave(parts, B) == stream
