"""The decode layer (nn.hpp:38-42, nn.cpp:153-192) as a device op.

``decode_input`` validates the chunk list exactly like nn.cpp:158-175 and
writes the (rows, P) layer input directly on the GPU with the fused epilogue
(float(q)*scale, optionally stored as binary16 like the MixedPrecision tape,
nn.cpp:141-146/235, or as bf16).  ``DecodeLayer`` is a torch.nn.Module front
for a device stream of containers.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import codec
from .codec import CodecMode, EncodedBatch
from .errors import ShapeError


@dataclass
class DecodeLayer:
    """nn.hpp:38-42"""
    mode: CodecMode = CodecMode.ExactInt64
    n_images: int = 0
    scale: float = 1.0


def decode_input(layer: DecodeLayer, chunks: Sequence[EncodedBatch], dtype=None, device: int = 0):
    """nn::decode_input (nn.cpp:153-192) on the GPU; returns a torch tensor."""
    import torch
    dtype = dtype or torch.float32
    if len(chunks) == 0:
        raise ShapeError("layer 0: no encoded batches supplied")
    rows = 0
    for enc in chunks:
        if int(enc.mode) != int(layer.mode):
            raise ShapeError(f"layer 0: decode expects mode {codec.mode_name(layer.mode)} but batch uses "
                             f"{codec.mode_name(enc.mode)}")
        if enc.shape != chunks[0].shape:
            raise ShapeError("layer 0: encoded chunks disagree on image shape")
        rows += int(enc.n_images)
    if layer.n_images != 0 and rows != layer.n_images:
        raise ShapeError(f"layer 0: decode expects {layer.n_images} images, got {rows}")
    P = chunks[0].pixel_count()
    dev = torch.device("cuda", device)
    out = torch.empty((rows, P), dtype=dtype, device=dev)
    mode = CodecMode(int(layer.mode))
    # consecutive chunks with equal n form one stream (one launch each)
    row = 0
    k = 0
    while k < len(chunks):
        n = int(chunks[k].n_images)
        j = k
        while j < len(chunks) and int(chunks[j].n_images) == n:
            j += 1
        group = chunks[k:j]
        plane = torch.from_numpy(np.concatenate([np.ascontiguousarray(c.plane) for c in group])).to(dev)
        offs = None
        if codec.mode_has_offsets(mode):
            ost = codec.offsets_stride(mode, P, n)
            o = np.zeros(len(group) * ost, np.uint8)
            for g, c in enumerate(group):
                o[g * ost: g * ost + c.offsets.size] = c.offsets
            offs = torch.from_numpy(o).to(dev)
        L = codec.layout(mode, n, P, n, len(group))
        codec.decode_dev(L, plane, out[row: row + n * len(group)], offsets=offs, scale=layer.scale)
        row += n * len(group)
        k = j
    codec.sync(device)
    return out
