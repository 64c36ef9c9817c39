"""Dataset-sharded global gather (optional): every rank holds
only its slice of the dataset and the rows a step draws are exchanged with
one all-to-all before the gather-encode.

Rank r owns dataset rows [r*per, min((r+1)*per, N)).  Per step:
  1. every rank draws the whole step's batches from its (identical) cursor
     and takes its own batches t % G == rank (no messages);
  2. owner(example) = example // per; a stable partition of each rank's
     draws by owner (the class-index kernel, K7) gives, for every (source,
     destination) pair, the rows to move and their order -- the same on both
     sides, so no index is exchanged;
  3. rows owned here are packed per destination (optb_gather_rows_dev) and
     exchanged (all_to_all_single over NCCL / NVLink, or point-to-point over
     gloo for CPU test runs);
  4. the gather-encode reads the received rows through the inverse of this
     rank's partition order (optb_inverse_perm_dev) -- bit-identical to the
     replicated-dataset path -- and decode runs as usual.
The exchange moves (G-1)/G of the step's rows across NVLink (~7x slower
than HBM), so this variant is exchange-bound and reported separately.

PeerShardedGather is the B200-native form of the same step: the shards are
mapped into every rank's address space (CUDA IPC over NVLink / NVSwitch peer
access), a tiny kernel turns the step's draws into absolute row addresses,
and ONE launch (optb_roundtrip_rows_dev) gathers each drawn row from the GPU
that owns it -- the NVLink transfer overlapped tile by tile with the packing
-- encodes it and decodes it: no staging buffer, no all-to-all, no host
synchronisation, no index exchange.
"""
from __future__ import annotations

import ctypes as ct

from . import _lib, codec
from ._lib import check, lib
from .sampler import class_index_dev


def _p(t):
    return ct.c_void_p(t.data_ptr())


class ShardedGather:
    def __init__(self, cursor, local_rows, n_examples: int, rank: int, world: int, batch: int,
                 batches_per_step: int, mode=codec.CodecMode.ExactInt128, group=None, device: int = 0,
                 exchange: str = "nccl"):
        self.cursor, self.local, self.N = cursor, local_rows, n_examples
        self.rank, self.world, self.B, self.nb = rank, world, batch, batches_per_step
        self.per = (n_examples + world - 1) // world
        self.P = local_rows.shape[1]
        self.group, self.device, self.exchange = group, device, exchange
        self.rows = batch * batches_per_step
        self.layout = codec.layout(mode, codec.capacity(mode), self.P, batch, batches_per_step)
        self.cont, self.offs = codec.alloc_stream(self.layout, device)
        self.ctx = _lib.context(device)

    def step(self, out):
        """One step on the current stream: exchange this step's rows,
        gather-encode, decode into `out`.  Returns (send_counts, recv_counts)."""
        import torch
        import torch.distributed as dist
        dev = torch.device("cuda", self.device)
        s = torch.cuda.current_stream(dev)
        sp = ct.c_void_p(s.cuda_stream)
        G, B, nb, P, rows = self.world, self.B, self.nb, self.P, self.rows
        ex_all, _ = self.cursor.next_dev(G * nb, stream=s)
        ex_by_rank = ex_all.view(nb, G, B).transpose(0, 1).reshape(G, rows).contiguous()
        owner = torch.empty((G, rows), dtype=torch.int32, device=dev)
        check(lib.optb_owner_labels_dev(self.ctx, _p(ex_by_rank), G * rows, self.per, G, _p(owner), sp))
        plans = []
        for q in range(G):  # stable partition of rank q's draws by owner
            offs_q, mem_q = class_index_dev(owner[q], G, device=self.device)
            plans.append((offs_q, mem_q))
        offs_host = torch.stack([p[0] for p in plans]).cpu()  # [G, G+1]
        send_counts = [int(offs_host[q, self.rank + 1] - offs_host[q, self.rank]) for q in range(G)]
        recv_counts = [int(offs_host[self.rank, r + 1] - offs_host[self.rank, r]) for r in range(G)]
        send = torch.empty((max(sum(send_counts), 1), P), dtype=torch.uint8, device=dev)
        at = 0
        for q in range(G):
            offs_q, mem_q = plans[q]
            lo, n = int(offs_host[q, self.rank]), send_counts[q]
            if n:
                ids = ex_by_rank[q][mem_q[lo:lo + n]].contiguous()
                check(lib.optb_gather_rows_dev(self.ctx, _p(self.local), self.local.stride(0), _p(ids), n,
                                               self.rank * self.per, P, _p(send[at:]), P, sp))
            at += n
        recv = torch.empty((max(rows, 1), P), dtype=torch.uint8, device=dev)
        if self.exchange == "nccl":
            s.synchronize()
            dist.all_to_all_single(recv[:rows], send[:sum(send_counts)],
                                   [c for c in recv_counts], [c for c in send_counts], group=self.group)
        else:  # gloo: point-to-point on host copies (CPU test runs)
            s.synchronize()
            send_h = send[:sum(send_counts)].cpu()
            recv_h = torch.empty((rows, P), dtype=torch.uint8)
            so = [sum(send_counts[:q]) for q in range(G)]
            ro = [sum(recv_counts[:r]) for r in range(G)]
            reqs = []
            for q in range(G):
                if q == self.rank:
                    recv_h[ro[q]:ro[q] + recv_counts[q]] = send_h[so[q]:so[q] + send_counts[q]]
                    continue
                if send_counts[q]:
                    reqs.append(dist.isend(send_h[so[q]:so[q] + send_counts[q]].contiguous(), q, group=self.group))
                if recv_counts[q]:
                    buf = torch.empty((recv_counts[q], P), dtype=torch.uint8)
                    reqs.append((dist.irecv(buf, q, group=self.group), buf, ro[q]))
            for r in reqs:
                if isinstance(r, tuple):
                    r[0].wait()
                    recv_h[r[2]:r[2] + r[1].shape[0]] = r[1]
                else:
                    r.wait()
            recv[:rows].copy_(recv_h)
        # received rows arrive source-major in partition order: invert it
        inv = torch.empty(rows, dtype=torch.int64, device=dev)
        check(lib.optb_inverse_perm_dev(self.ctx, _p(plans[self.rank][1]), rows, _p(inv), sp))
        codec.encode_dev(self.layout, recv, self.cont, self.offs, row_index=inv, stream=s)
        codec.decode_dev(self.layout, self.cont, out, offsets=self.offs, stream=s)
        return send_counts, recv_counts


class PeerShardedGather:
    """Dataset-sharded step over peer memory (see the module docstring).

    Every rank holds rows [rank*per, (rank+1)*per) in ``local_rows`` (a CUDA
    tensor, same row stride on every rank); construction is collective
    (exchanges the IPC handles, then a barrier).  ``step(out)`` enqueues the
    step on the current stream and returns immediately."""

    def __init__(self, cursor, local_rows, n_examples: int, rank: int, world: int, batch: int,
                 batches_per_step: int, mode=codec.CodecMode.ExactInt128, group=None, device: int = 0,
                 out_dtype=None, scale: float = 1.0):
        import torch
        import torch.distributed as dist
        self.cursor, self.local, self.N = cursor, local_rows, n_examples
        self.rank, self.world, self.B, self.nb = rank, world, batch, batches_per_step
        self.per = (n_examples + world - 1) // world
        self.P = local_rows.shape[1]
        self.stride = local_rows.stride(0)
        self.device, self.scale, self.group = device, scale, group
        self.rows = batch * batches_per_step
        self.layout = codec.layout(mode, codec.capacity(mode), self.P, batch, batches_per_step)
        self.cont, self.offs = codec.alloc_stream(self.layout, device)
        dev = torch.device("cuda", device)
        handle = (ct.c_uint8 * 64)()
        off = ct.c_uint64()
        check(lib.optb_ipc_export(ct.c_void_p(local_rows.data_ptr()), handle, ct.byref(off)))
        mine = (bytes(handle), off.value, self.stride)
        everyone = [None] * world
        dist.all_gather_object(everyone, mine, group=group)
        if any(e[2] != self.stride for e in everyone):
            raise ValueError("PeerShardedGather: shards must share one row stride")
        bases, self._opened = [], []
        err = ""
        try:
            for q, (h, o, _) in enumerate(everyone):
                if q == rank:
                    bases.append(local_rows.data_ptr())
                    continue
                p = ct.c_void_p()
                check(lib.optb_ipc_open(device, (ct.c_uint8 * 64).from_buffer_copy(h), o, ct.byref(p)))
                self._opened.append((p.value, o))
                bases.append(p.value)
        except Exception as e:  # noqa: BLE001 -- decided collectively below
            err = str(e)
        # every rank must agree before anyone relies on the mappings (a rank
        # that cannot map a peer, e.g. one GPU visible per process, must not
        # leave the others waiting in a later collective)
        nccl = dist.get_backend(group) == "nccl"
        flag = torch.tensor([0 if err else 1], dtype=torch.int32, device=dev if nccl else "cpu")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        if int(flag.item()) == 0:
            for p_, o_ in self._opened:
                lib.optb_ipc_close(ct.c_void_p(p_), o_)
            self._opened = None
            raise RuntimeError("PeerShardedGather: peer shards could not be mapped on every rank"
                               + (f" ({err})" if err else ""))
        self.aligned16 = all(b % 16 == 0 for b in bases) and self.stride % 16 == 0
        self.bases = torch.tensor(bases, dtype=torch.int64, device=dev)
        self.ptrs = torch.empty(max(self.rows, 1), dtype=torch.int64, device=dev)
        self.ex = torch.empty(max(self.rows, 1), dtype=torch.int64, device=dev)
        self.cls = torch.empty(max(self.rows, 1), dtype=torch.int32, device=dev)
        torch.cuda.synchronize(dev)
        dist.barrier(group=group)  # every shard written and mapped before anyone reads

    def step(self, out, stream=None):
        """Draw this rank's batches of the step, resolve their rows to peer
        addresses, then gather (over NVLink) + encode + decode in one launch."""
        import torch
        dev = torch.device("cuda", self.device)
        s = stream or torch.cuda.current_stream(dev)
        ex, _ = self.cursor.next_dev(self.nb * self.world, shard=self.rank, n_shards=self.world,
                                     examples=self.ex, classes=self.cls, stream=s)
        codec.shard_row_ptrs_dev(ex, self.bases, self.per, self.stride, out=self.ptrs, stream=s)
        codec.roundtrip_rows_dev(self.layout, self.ptrs, self.cont, out, offsets=self.offs,
                                 aligned16=self.aligned16, scale=self.scale, stream=s)

    def close(self):
        """Collective: unmap the peers' shards once every rank is done."""
        import torch
        import torch.distributed as dist
        if getattr(self, "_opened", None) is None:
            return
        torch.cuda.synchronize(torch.device("cuda", self.device))
        dist.barrier(group=self.group)
        for p, o in self._opened:
            check(lib.optb_ipc_close(ct.c_void_p(p), o))
        self._opened = None
