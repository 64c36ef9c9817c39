"""The encode-while-train data path (optb_pipeline_*; reference pipeline.cpp).

    pipe = Pipeline(cursor, dataset, mode=CodecMode.ExactInt128, batch=512,
                    batches_per_step=97, out_dtype=torch.float32, scale=1/255)
    for step in range(n):
        pipe.step(layer_input)          # SBS -> gather-encode -> decode, async

Per step the native pipeline gathers the SBS-drawn rows of ``dataset`` (a
CUDA tensor, or a pinned CPU tensor read zero-copy over PCIe), packs them into
containers and decodes them into ``layer_input`` on the current stream, while
the next step's draws run on a side stream.  One ctypes call per step; the
gather-encode and decode are one fused launch where the mode allows it
(optb_roundtrip_dev), or two launches with ``split_kernels=True``.
"""
from __future__ import annotations

import ctypes as ct

from . import _lib
from ._lib import Epilogue, Layout, PipelineDesc, check, lib
from .codec import BF16, F16, F32, U8


class Pipeline:
    def __init__(self, cursor, dataset, mode, batch: int, batches_per_step: int, per_chunk=None,
                 shard: int = 0, n_shards: int = 1, out_dtype=None, scale: float = 1.0,
                 class_scale=None, class_bias=None, device: int = 0, record_timings: bool = False,
                 steps_per_draw: int = 1, split_kernels: bool = False, timing_stride: int = 1):
        import torch
        from . import codec
        out_dtype = out_dtype or torch.uint8
        dt = {torch.uint8: U8, torch.float32: F32, torch.float16: F16, torch.bfloat16: BF16}[out_dtype]
        P = dataset.shape[1]
        pc = per_chunk or codec.capacity(mode)
        self.layout = Layout(int(mode), pc, P, batch, batches_per_step)
        self.rows = batch * batches_per_step
        self.P = P
        self.device = device
        # objects the native pipeline points into: the cursor and class tables
        # for its lifetime, the dataset until set_dataset replaces it, and the
        # host buffers of the last two step_host calls (one per double-buffer
        # slot) until host_wait
        self._keep = (cursor, class_scale, class_bias)
        self._dataset = dataset
        self._host_bufs = []
        E = Epilogue(dt, float(scale), None if class_scale is None else ct.c_void_p(class_scale.data_ptr()),
                     None if class_bias is None else ct.c_void_p(class_bias.data_ptr()), None, 0)
        desc = PipelineDesc(self.layout, ct.c_void_p(dataset.data_ptr()), dataset.stride(0), cursor._h, shard,
                            n_shards, E, 1 if record_timings else 0, steps_per_draw, 1 if split_kernels else 0,
                            timing_stride)
        self._h = ct.c_void_p()
        check(lib.optb_pipeline_create(_lib.context(device), ct.byref(desc), ct.byref(self._h)))
        # one fused launch per step (optb_roundtrip_dev) on the vector path
        # (lossless: P % 512 == 0); the library falls back to two launches
        self.fused = (not split_kernels and P % 16 == 0 and dataset.stride(0) % 16 == 0
                      and dataset.data_ptr() % 16 == 0 and (int(mode) in (0, 1, 2) or P % 512 == 0))
        self.steps = 0

    @classmethod
    def warm(cls, mode, batch: int, batches_per_step: int, shape, directory: str, epoch: int = 0, per_chunk=None,
             out_dtype=None, scale: float = 1.0, device: int = 0, record_timings: bool = False):
        """Warm start (optb_pipeline_create_warm; PipelineConfig::warm_start,
        pipeline.cpp:154-177): the dumped epoch <directory>/batch_<epoch>_<k>.optb
        is loaded once and every step decodes it into the caller's buffer."""
        import torch
        from . import codec
        out_dtype = out_dtype or torch.uint8
        dt = {torch.uint8: U8, torch.float32: F32, torch.float16: F16, torch.bfloat16: BF16}[out_dtype]
        self = cls.__new__(cls)
        P = shape.pixel_count()
        self.layout = Layout(int(mode), per_chunk or codec.capacity(mode), P, batch, batches_per_step)
        self.rows, self.P, self.device = batch * batches_per_step, P, device
        self._keep, self._dataset, self._host_bufs = (), None, []
        self.fused, self.steps = False, 0
        E = Epilogue(dt, float(scale), None, None, None, 0)
        self._h = ct.c_void_p()
        check(lib.optb_pipeline_create_warm(_lib.context(device), ct.byref(self.layout), shape.height, shape.width,
                                            shape.channels, str(directory).encode(), epoch, ct.byref(E),
                                            1 if record_timings else 0, ct.byref(self._h)))
        return self

    def step(self, out, stream=None):
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        check(lib.optb_pipeline_step(self._h, ct.c_void_p(out.data_ptr()), ct.c_void_p(stream.cuda_stream)))
        self.steps += 1

    def step_host(self, dataset_host, out_host, stream=None):
        """The step on host buffers (optb_pipeline_step_host): ``dataset_host``
        ([N, >=P] u8 CPU tensor, pinned for overlap) is uploaded, the step
        runs, and the decoded rows land in ``out_host`` (CPU tensor shaped
        like ``step``'s ``out``) -- asynchronously; see host_wait()."""
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self._host_bufs = (self._host_bufs + [(dataset_host, out_host)])[-2:]
        check(lib.optb_pipeline_step_host(self._h, ct.c_void_p(dataset_host.data_ptr()), dataset_host.shape[0],
                                          dataset_host.stride(0), ct.c_void_p(out_host.data_ptr()),
                                          ct.c_void_p(stream.cuda_stream)))
        self.steps += 1

    def host_wait(self, stream=None):
        """Every step_host download has landed (stream None: block the host),
        or `stream` waits for them (device-side)."""
        check(lib.optb_pipeline_host_wait(self._h, None if stream is None else ct.c_void_p(stream.cuda_stream)))
        if stream is None:  # every transfer has landed
            self._host_bufs = []

    def set_dataset(self, dataset):
        """Rows for subsequent steps come from `dataset` (same shape)."""
        check(lib.optb_pipeline_set_dataset(self._h, ct.c_void_p(dataset.data_ptr()), dataset.stride(0)))
        self._dataset = dataset

    def timings(self, step: int):
        s, e, d = ct.c_float(), ct.c_float(), ct.c_float()
        check(lib.optb_pipeline_timings(self._h, step, ct.byref(s), ct.byref(e), ct.byref(d)))
        return s.value, e.value, d.value

    def draws(self, step: int):
        """(examples_ptr, classes_ptr) device pointers of a buffered step."""
        ex, cl = ct.c_void_p(), ct.c_void_p()
        check(lib.optb_pipeline_draws(self._h, step, ct.byref(ex), ct.byref(cl)))
        return ex.value, cl.value

    def containers_ptr(self) -> int:
        return lib.optb_pipeline_containers(self._h)

    def close(self):
        if getattr(self, "_h", None):
            lib.optb_pipeline_destroy(self._h)
            self._h = None

    def __del__(self):
        if lib is not None:  # module globals may already be gone at interpreter exit
            self.close()
