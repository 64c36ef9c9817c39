"""Host mirror of ``optb::sampler`` (include/optb/sampler.hpp:14-68) over the
C ABI.  The class index, the per-class Fisher-Yates permutations and the
SplitMix64 chain all live on the GPU (sbs.cu); this module only validates,
moves results across the boundary and runs the host preprocessing hook.

Reference API                         here
------------------------------------  --------------------------------------
SamplerPlan / plan(weights, B, seed)  SamplerPlan / plan (optb_sbs_plan)
ClassIndex::from_labels               ClassIndex.from_labels (optb_class_index_dev)
BatchCursor(plan, index)              BatchCursor (optb_sbs_create)
.set_preprocess_hook(hook)            same; called per draw, class-major order
.next() -> vector<Draw>               .next() (optb_sbs_next_host)
                                      .next_dev(n, shard, n_shards) -> device tensors
"""
from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import check, lib
from .errors import Error


@dataclass
class SamplerPlan:
    """sampler.hpp:14-21"""
    class_weights: List[float] = field(default_factory=list)
    batch_size: int = 0
    counts: List[int] = field(default_factory=list)
    seed: int = 0

    def num_classes(self) -> int:
        return len(self.counts)


def plan(class_weights: Sequence[float], batch_size: int, seed: int) -> SamplerPlan:
    """sampler.cpp:11-51 (largest remainder, ties to the lower class)."""
    w = np.ascontiguousarray(np.asarray(class_weights, np.float64))
    counts = np.zeros(max(len(w), 1), np.uint64)
    check(lib.optb_sbs_plan(w.ctypes.data_as(_lib.f64p), len(w), batch_size,
                            counts.ctypes.data_as(_lib.u64p)))
    return SamplerPlan(list(map(float, w)), int(batch_size), [int(c) for c in counts[: len(w)]],
                       int(seed) & 0xFFFFFFFFFFFFFFFF)


@dataclass
class ClassIndex:
    """sampler.hpp:27-32"""
    by_class: List[List[int]] = field(default_factory=list)

    def num_classes(self) -> int:
        return len(self.by_class)

    @staticmethod
    def from_labels(labels: Sequence[int], num_classes: int) -> "ClassIndex":
        """sampler.cpp:53-65, as a GPU stable partition (optb_class_index_dev)."""
        offs, members = class_index_dev(labels, num_classes)
        o = offs.cpu().numpy()
        m = members.cpu().numpy()
        return ClassIndex([m[o[c]:o[c + 1]].tolist() for c in range(num_classes)])


def class_index_dev(labels, num_classes: int, device: int = 0):
    """Device ClassIndex: (class_offsets[C+1] u64, members[n] i64) tensors."""
    import torch
    dev = torch.device("cuda", device)
    lab = torch.as_tensor(np.asarray(labels, np.int32) if not torch.is_tensor(labels) else labels,
                          dtype=torch.int32).to(dev).contiguous()
    n = lab.numel()
    offs = torch.zeros(num_classes + 1, dtype=torch.int64, device=dev)  # u64 values < 2^63
    members = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    ctx = _lib.context(device)
    stream = ct.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    check(lib.optb_class_index_dev(ctx, ct.c_void_p(lab.data_ptr()), n, num_classes,
                                   ct.c_void_p(offs.data_ptr()), ct.c_void_p(members.data_ptr()), stream))
    check(lib.optb_ctx_sync(ctx, stream))
    return offs, members[:n]


@dataclass
class Draw:
    """sampler.hpp:34-37"""
    example: int = 0
    cls: int = 0


PreprocessHook = Callable[[int, int], None]


class BatchCursor:
    """sampler.hpp:45-68: single-consumer batch stream, draws without
    replacement inside each class, reshuffling a class when exhausted."""

    def __init__(self, plan_: SamplerPlan, index: ClassIndex, device: int = 0):
        if index.num_classes() != plan_.num_classes():  # sampler.cpp:69-72
            raise Error(f"sampler: index has {index.num_classes()} classes, "
                        f"plan has {plan_.num_classes()}")
        self._plan = plan_
        self._device = device
        self._hook: Optional[PreprocessHook] = None
        counts = np.asarray(plan_.counts, np.uint64)
        sizes = [len(v) for v in index.by_class]
        offs = np.zeros(len(sizes) + 1, np.uint64)
        offs[1:] = np.cumsum(sizes, dtype=np.uint64)
        members = np.asarray([e for v in index.by_class for e in v] or [0], np.int64)
        self._h = ct.c_void_p()
        check(lib.optb_sbs_create(_lib.context(device), counts.ctypes.data_as(_lib.u64p), len(sizes),
                                  plan_.batch_size, plan_.seed, offs.ctypes.data_as(_lib.u64p),
                                  ct.c_void_p(members.ctypes.data), 0, ct.byref(self._h)))

    @classmethod
    def from_device_index(cls, plan_: SamplerPlan, class_offsets, members, device: int = 0):
        """Cursor over a device ClassIndex (class_index_dev) without a host round trip."""
        self = cls.__new__(cls)
        self._plan, self._device, self._hook = plan_, device, None
        counts = np.asarray(plan_.counts, np.uint64)
        offs = np.ascontiguousarray(class_offsets.cpu().numpy().astype(np.uint64))
        if len(offs) != plan_.num_classes() + 1:
            raise Error(f"sampler: index has {len(offs) - 1} classes, plan has {plan_.num_classes()}")
        self._h = ct.c_void_p()
        check(lib.optb_sbs_create(_lib.context(device), counts.ctypes.data_as(_lib.u64p), len(counts),
                                  plan_.batch_size, plan_.seed, offs.ctypes.data_as(_lib.u64p),
                                  ct.c_void_p(members.data_ptr()), 1, ct.byref(self._h)))
        return self

    def __copy__(self) -> "BatchCursor":
        """A copy continues the identical stream independently (the reference
        class is copyable, sampler.hpp:45-68): optb_sbs_clone."""
        other = BatchCursor.__new__(BatchCursor)
        other._plan, other._device, other._hook = self._plan, self._device, self._hook
        other._h = ct.c_void_p()
        check(lib.optb_sbs_clone(self._h, ct.byref(other._h)))
        return other

    copy = __copy__

    def set_preprocess_hook(self, hook: Optional[PreprocessHook]) -> None:
        self._hook = hook

    def plan(self) -> SamplerPlan:
        return self._plan

    def set_force_serial(self, on: bool) -> None:
        """Testing aid: exact serial rejection path for every reshuffle."""
        check(lib.optb_sbs_set_force_serial(self._h, 1 if on else 0))

    def next_arrays(self, n_batches: int = 1):
        """n_batches consecutive batches as host arrays (examples i64, classes i32)."""
        rows = n_batches * self._plan.batch_size
        ex = np.zeros(max(rows, 1), np.int64)
        cl = np.zeros(max(rows, 1), np.int32)
        check(lib.optb_sbs_next_host(self._h, n_batches, ct.c_void_p(ex.ctypes.data),
                                     ct.c_void_p(cl.ctypes.data)))
        ex, cl = ex[:rows], cl[:rows]
        if self._hook is not None:  # sampler.cpp:99, emission order
            for c, e in zip(cl.tolist(), ex.tolist()):
                self._hook(c, e)
        return ex, cl

    def next(self) -> List[Draw]:
        """sampler.cpp:91-104"""
        ex, cl = self.next_arrays(1)
        return [Draw(int(e), int(c)) for e, c in zip(ex, cl)]

    def next_dev(self, n_batches: int, shard: int = 0, n_shards: int = 1, examples=None, classes=None,
                 stream=None):
        """Device draws of batches t < n_batches with t % n_shards == shard
        (optb_sbs_next_dev); the cursor advances by n_batches."""
        import torch
        dev = torch.device("cuda", self._device)
        out_b = (n_batches - shard + n_shards - 1) // n_shards if n_batches > shard else 0
        rows = out_b * self._plan.batch_size
        if examples is None:
            examples = torch.empty(max(rows, 1), dtype=torch.int64, device=dev)
        if classes is None:
            classes = torch.empty(max(rows, 1), dtype=torch.int32, device=dev)
        if stream is None:
            stream = torch.cuda.current_stream(dev)
        check(lib.optb_sbs_next_dev(self._h, n_batches, shard, n_shards, ct.c_void_p(examples.data_ptr()),
                                    ct.c_void_p(classes.data_ptr()), ct.c_void_p(stream.cuda_stream)))
        return examples[:rows], classes[:rows]

    def batches_drawn(self) -> int:
        return lib.optb_sbs_batches_drawn(self._h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None and getattr(lib, "optb_sbs_destroy", None) is not None:  # not at interpreter exit
            lib.optb_sbs_destroy(h)
        self._h = None
