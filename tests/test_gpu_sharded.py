"""Dataset-sharded global gather (sharded.py): two ranks each holding half
the dataset exchange the drawn rows and decode exactly the rows the
replicated-dataset stream would -- checked for every step on both ranks.
Both ranks share the box's one GPU; the exchange runs over gloo here (NCCL
all_to_all_single on a multi-GPU box)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import oracle as O
    import paper_2105_00619_b200 as pkg
    from paper_2105_00619_b200.sharded import ShardedGather
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    S = pkg.sampler
    N, P, B, nb, K = 6000, 768, 64, 3, 10
    full = O.synth_pixels(7, 0, N, P)
    per = (N + world - 1) // world
    local = torch.from_numpy(full[rank * per:(rank + 1) * per]).cuda()
    labels = (np.arange(N) % K).astype(np.int32)
    plan = S.plan([1.0 / K] * K, B, 42)
    offs, mem = S.class_index_dev(labels, K)
    cur = S.BatchCursor.from_device_index(plan, offs, mem)
    sg = ShardedGather(cur, local, N, rank, world, B, nb, exchange="gloo")
    ro, rm = O.class_index(labels, K)
    ref = O.Cursor(O.sbs_plan([1.0 / K] * K, B), ro, rm, B, 42)
    ok = True
    moved = 0
    for _ in range(3):
        out = torch.empty((B * nb, P), dtype=torch.uint8, device="cuda")
        send, recv = sg.step(out)
        pkg.codec.sync()
        moved += sum(recv) - recv[rank]
        ex, _ = ref.next(nb * world)
        mine = ex.reshape(nb * world, B)[rank::world].reshape(-1)
        ok &= bool(np.array_equal(out.cpu().numpy(), full[mine]))
    q.put((rank, ok, moved))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_gather_two_ranks(torch_cuda):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    assert all(moved > 0 for _, _, moved in res)  # rows really crossed ranks
