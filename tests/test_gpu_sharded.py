"""Dataset-sharded global gather (sharded.py): two ranks each holding half
the dataset decode exactly the rows the replicated-dataset stream would --
checked for every step on both ranks.  Both ranks share the box's one GPU.
ShardedGather exchanges the drawn rows (gloo here, NCCL all_to_all_single
on a multi-GPU box); PeerShardedGather maps the other rank's shard over CUDA
IPC and gathers straight from it inside the fused roundtrip kernel (peer
memory over NVLink on a multi-GPU box).  Also: the row-address kernels on
several shards in one process, vector and generic paths."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q, kind="a2a"):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import oracle as O
    import paper_2105_00619_b200 as pkg
    from paper_2105_00619_b200.sharded import PeerShardedGather, ShardedGather
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
    if kind == "peer":
        sg = PeerShardedGather(cur, local, N, rank, world, B, nb)
    else:
        sg = ShardedGather(cur, local, N, rank, world, B, nb, exchange="gloo")
    ro, rm = O.class_index(labels, K)
    ref = O.Cursor(O.sbs_plan([1.0 / K] * K, B), ro, rm, B, 42)
    ok = True
    moved = 0
    for _ in range(3):
        out = torch.empty((B * nb, P), dtype=torch.uint8, device="cuda")
        ex, _ = ref.next(nb * world)
        mine = ex.reshape(nb * world, B)[rank::world].reshape(-1)
        if kind == "peer":
            sg.step(out)
            moved += int(((mine // per) != rank).sum())
        else:
            send, recv = sg.step(out)
            moved += sum(recv) - recv[rank]
        pkg.codec.sync()
        ok &= bool(np.array_equal(out.cpu().numpy(), full[mine]))
    if kind == "peer":
        sg.close()
    q.put((rank, ok, moved))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["a2a", "peer"])
def test_sharded_gather_two_ranks(torch_cuda, kind):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, kind)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    assert all(moved > 0 for _, _, moved in res)  # rows really crossed ranks


@pytest.mark.parametrize("mode,P,dtype", [(1, 3072, "uint8"), (0, 768, "float32"), (2, 3072, "bfloat16"),
                                          (3, 3072, "uint8"), (1, 108, "uint8")])
def test_row_pointer_gather_three_shards(pkg, oracle_mod, torch_cuda, mode, P, dtype):
    """Three shards in separate allocations of one process: shard_row_ptrs +
    roundtrip_rows_dev / encode_rows_dev == the oracle on the replicated
    dataset (fused vector, two-launch lossless and generic paths)."""
    torch, C, O = torch_cuda, pkg.codec, oracle_mod
    rng = np.random.default_rng(5 + mode + P)
    N, B, nb, G = 900, 48, 3, 3
    full = rng.integers(0, 256, size=(N, P), dtype=np.uint8)
    per = (N + G - 1) // G
    shards = [torch.from_numpy(full[q * per:(q + 1) * per]).cuda() for q in range(G)]
    bases = torch.tensor([t.data_ptr() for t in shards], dtype=torch.int64, device="cuda")
    ex = rng.integers(0, N, size=B * nb).astype(np.int64)
    ptrs = C.shard_row_ptrs_dev(torch.from_numpy(ex).cuda(), bases, per, P)
    want_ptrs = np.array([shards[e // per].data_ptr() + (e - (e // per) * per) * P for e in ex], np.int64)
    assert np.array_equal(ptrs.cpu().numpy(), want_ptrs)
    pc = C.capacity(mode)
    L = C.layout(mode, pc, P, B, nb)
    cont, offs = C.alloc_stream(L)
    dt = getattr(torch, dtype)
    out = torch.empty((B * nb, P), dtype=dt, device="cuda")
    scale = 1.0 if dtype == "uint8" else float(np.float32(1) / np.float32(255))
    C.roundtrip_rows_dev(L, ptrs, cont, out, offsets=offs, aligned16=(P % 16 == 0), scale=scale)
    C.sync()
    rc, ro = O.encode_stream(full, ex, mode, pc, B, nb)
    assert np.array_equal(cont.cpu().numpy()[: rc.size], rc)
    kind = {"uint8": O.U8, "float32": O.F32, "bfloat16": O.BF16}[dtype]
    want = O.decode_stream(rc, ro, mode, pc, P, B, nb, out_dtype=kind, scale=scale)
    got = out.cpu()
    got = got.view(torch.int16).numpy() if dtype == "bfloat16" else got.numpy()
    assert np.array_equal(got.view(want.dtype), want)
    # encode_rows_dev alone, generic path forced (aligned16 = False)
    cont2, offs2 = C.alloc_stream(L)
    C.encode_rows_dev(L, ptrs, cont2, offs2, aligned16=False)
    C.sync()
    assert np.array_equal(cont2.cpu().numpy()[: rc.size], rc)
    if ro is not None:
        assert np.array_equal(offs2.cpu().numpy()[: ro.size], ro)
