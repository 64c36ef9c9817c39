"""Host mirror of ``optb::codec`` (include/optb/codec.hpp) over the C ABI, plus
the device-resident stream API used by the network input path and the bench.

Reference API (codec.hpp:22-102)          here
----------------------------------------  -------------------------------------
CodecMode, capacity, capacity_is_hard,     same names (metadata from the C ABI)
mode_name, mode_has_offsets,
container_value_bytes, kFloat64AcceptLimit
ImageShape, Image, EncodedBatch            dataclasses; EncodedBatch.packed is a
                                           numpy view of the [P][Wc] LE words
encode(images, mode)                       -> optb_encode_host (GPU)
decode(enc)                                -> optb_decode_host (GPU)
roundtrip_error(images, mode)              encode + decode on the GPU
(runner.cpp:77-90 + dataset.cpp:16-22)     encode_dev(layout, dataset, row_index)
(codec::decode + nn.cpp:183-189)           decode_dev(layout, ..., out, scale)

Every function raises the errors.hpp-equivalent class with the reference's
message.  There is no CPU fallback: all pixel work runs in liboptb_cuda.so.
"""
from __future__ import annotations

import ctypes as ct
import enum
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import Epilogue, Layout, check, lib
from .errors import Error, FormatError, ShapeError


class CodecMode(enum.IntEnum):
    """codec.hpp:22-28"""
    ExactInt64 = 0
    ExactInt128 = 1
    Float64Faithful = 2
    LosslessOffset64 = 3
    LosslessOffset128 = 4


kFloat64AcceptLimit = 16  # codec.hpp:36

U8, F32, F16, BF16 = 0, 1, 2, 3  # OPTB_OUT_*


def capacity(mode) -> int:
    return lib.optb_capacity(int(mode))


def accept_limit(mode) -> int:
    return lib.optb_accept_limit(int(mode))


def capacity_is_hard(mode) -> bool:
    return bool(lib.optb_capacity_is_hard(int(mode)))


def mode_name(mode) -> str:
    return lib.optb_mode_name(int(mode)).decode()


def mode_has_offsets(mode) -> bool:
    return bool(lib.optb_mode_has_offsets(int(mode)))


def container_value_bytes(mode) -> int:
    return lib.optb_container_value_bytes(int(mode))


def offsets_stride(mode, pixels: int, per_chunk: int) -> int:
    return lib.optb_offsets_stride(int(mode), pixels, per_chunk)


@dataclass(frozen=True)
class ImageShape:
    """codec.hpp:45-54"""
    height: int = 0
    width: int = 0
    channels: int = 0

    def pixel_count(self) -> int:
        return self.height * self.width * self.channels


@dataclass
class Image:
    """codec.hpp:56-62: one 8-bit image, pixels row-major (h, w, c)."""
    shape: ImageShape
    pixels: np.ndarray

    def __eq__(self, other) -> bool:
        return (isinstance(other, Image) and self.shape == other.shape
                and np.array_equal(np.asarray(self.pixels, np.uint8), np.asarray(other.pixels, np.uint8)))


@dataclass
class EncodedBatch:
    """codec.hpp:64-86.  ``plane`` holds the container plane in the on-disk /
    device layout: P little-endian words of container_value_bytes(mode)
    bytes.  ``packed`` (integer modes, u64 or [P,2] lo/hi u64) and
    ``packed_f64`` are numpy views of it."""
    mode: CodecMode = CodecMode.ExactInt64
    shape: ImageShape = field(default_factory=ImageShape)
    n_images: int = 0
    plane: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    offsets: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))

    def pixel_count(self) -> int:
        return self.shape.pixel_count()

    @property
    def packed(self) -> np.ndarray:
        if self.mode == CodecMode.Float64Faithful:
            return np.zeros(0, np.uint64)
        w = self.plane.view(np.uint64)
        return w if container_value_bytes(self.mode) == 8 else w.reshape(-1, 2)

    @property
    def packed_f64(self) -> np.ndarray:
        if self.mode != CodecMode.Float64Faithful:
            return np.zeros(0, np.float64)
        return self.plane.view(np.float64)

    def container_byte_size(self) -> int:
        return self.pixel_count() * container_value_bytes(self.mode)

    def offsets_byte_size(self) -> int:
        return int(self.offsets.size)

    def byte_size(self) -> int:
        return self.container_byte_size() + self.offsets_byte_size()

    def lossy(self) -> bool:
        return self.mode == CodecMode.Float64Faithful and self.n_images > capacity(self.mode)

    def offset_bit(self, image: int, pixel: int) -> bool:
        bit = image * self.pixel_count() + pixel
        return bool((int(self.offsets[bit // 8]) >> (bit % 8)) & 1)

    def word(self, p: int) -> int:
        """container value of pixel p as a Python int (u128 semantics)."""
        wc = container_value_bytes(self.mode)
        return int.from_bytes(self.plane[p * wc:(p + 1) * wc].tobytes(), "little")


def _ptr(a: np.ndarray):
    return ct.c_void_p(a.ctypes.data) if a is not None else None


def _validate(images: Sequence[Image], mode) -> ImageShape:
    """codec.cpp:79-97 (shape checks host-side; capacity via the C ABI)."""
    if len(images) == 0:
        raise Error("encode: batch must contain at least one image")
    shape = images[0].shape
    if shape.pixel_count() == 0:
        raise ShapeError("encode: image extents must be positive")
    for i, img in enumerate(images):
        if img.shape != shape:
            raise ShapeError(f"encode: image {i} shape differs from image 0")
        if np.asarray(img.pixels).size != shape.pixel_count():
            raise ShapeError(f"encode: image {i} pixel buffer does not match shape")
    return shape


def encode(images: Sequence[Image], mode) -> EncodedBatch:
    """codec::encode (codec.cpp:106-146) on the GPU via optb_encode_host."""
    mode = CodecMode(int(mode))
    shape = _validate(images, mode)
    n, P = len(images), shape.pixel_count()
    L = Layout(int(mode), n, P, n, 1)
    check(lib.optb_layout_check(ct.byref(L)))
    src = np.ascontiguousarray(np.stack([np.asarray(im.pixels, np.uint8).reshape(-1) for im in images]))
    plane = np.zeros(P * container_value_bytes(mode), np.uint8)
    ost = offsets_stride(mode, P, n)
    offs = np.zeros(max(ost, 16), np.uint8)
    check(lib.optb_encode_host(_lib.context(), ct.byref(L), _ptr(src), _ptr(plane), _ptr(offs)))
    offsets = offs[: (n * P + 7) // 8].copy() if mode_has_offsets(mode) else np.zeros(0, np.uint8)
    return EncodedBatch(mode, shape, n, plane, offsets)


def decode(enc: EncodedBatch) -> list:
    """codec::decode (codec.cpp:148-208) on the GPU via optb_decode_host."""
    P, n = enc.pixel_count(), int(enc.n_images)
    if n == 0 or P == 0:
        raise FormatError("decode: empty encoded batch")
    mode = CodecMode(int(enc.mode))
    if enc.plane.size != P * container_value_bytes(mode):
        raise FormatError("decode: container plane size mismatch")
    ost = offsets_stride(mode, P, n)
    offs = np.zeros(max(ost, 16), np.uint8)
    if mode_has_offsets(mode):
        if enc.offsets.size != (n * P + 7) // 8:
            raise FormatError("decode: offset plane size mismatch")
        offs[: enc.offsets.size] = enc.offsets
    L = Layout(int(mode), n, P, n, 1)
    out = np.zeros((n, P), np.uint8)
    E = Epilogue(U8, 1.0, None, None, None, 0)
    plane = np.ascontiguousarray(enc.plane, np.uint8)
    check(lib.optb_decode_host(_lib.context(), ct.byref(L), _ptr(plane), _ptr(offs), ct.byref(E), _ptr(out)))
    return [Image(enc.shape, out[i].copy()) for i in range(n)]


def roundtrip_error(images: Sequence[Image], mode) -> list:
    """codec.cpp:210-224"""
    back = decode(encode(images, mode))
    return [int(np.max(np.abs(np.asarray(a.pixels, np.int32).reshape(-1) - b.pixels.astype(np.int32))))
            if a.shape.pixel_count() else 0 for a, b in zip(images, back)]


# ---------------------------------------------------------------- device streams
def layout(mode, per_chunk: int, pixels: int, batch: int, n_batches: int) -> Layout:
    L = Layout(int(mode), per_chunk, pixels, batch, n_batches)
    return L


def layout_chunks(L: Layout) -> int:
    return lib.optb_layout_chunks(ct.byref(L))


def container_bytes(L: Layout) -> int:
    return lib.optb_layout_container_bytes(ct.byref(L))


def offsets_bytes(L: Layout) -> int:
    return lib.optb_layout_offsets_bytes(ct.byref(L))


def _dptr(t):
    return None if t is None else ct.c_void_p(t.data_ptr())


def _stream(stream, device):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return ct.c_void_p(stream.cuda_stream)


def alloc_stream(L: Layout, device=0):
    """Device buffers for a stream's container planes and parity planes."""
    import torch
    dev = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
    cont = torch.empty(max(container_bytes(L), 16), dtype=torch.uint8, device=dev)
    ob = offsets_bytes(L)
    offs = torch.empty(max(ob, 16), dtype=torch.uint8, device=dev) if ob else None
    return cont, offs


def encode_dev(L: Layout, images, containers, offsets=None, row_index=None, stream=None):
    """Gather-encode on the device (optb_encode_dev): stream row r packs
    dataset row row_index[r] (identity if None) of ``images`` ([rows, P] u8,
    any row stride)."""
    dev = images.device.index or 0
    check(lib.optb_encode_dev(_lib.context(dev), ct.byref(L), _dptr(images), images.stride(0),
                              _dptr(row_index), _dptr(containers), _dptr(offsets), _stream(stream, dev)))


def decode_dev(L: Layout, containers, out, offsets=None, scale: float = 1.0, class_scale=None,
               class_bias=None, row_class=None, stream=None):
    """Decode on the device (optb_decode_dev) into ``out`` ([rows, >=P] tensor
    of u8 / f32 / f16 / bf16) -- the network's layer-0 input written directly."""
    import torch
    dt = {torch.uint8: U8, torch.float32: F32, torch.float16: F16, torch.bfloat16: BF16}[out.dtype]
    dev = out.device.index or 0
    E = Epilogue(dt, float(scale), _dptr(class_scale), _dptr(class_bias), _dptr(row_class), out.stride(0))
    check(lib.optb_decode_dev(_lib.context(dev), ct.byref(L), _dptr(containers), _dptr(offsets),
                              ct.byref(E), _dptr(out), _stream(stream, dev)))


def roundtrip_dev(L: Layout, images, containers, out, offsets=None, row_index=None, scale: float = 1.0,
                  class_scale=None, class_bias=None, row_class=None, stream=None):
    """encode_dev then decode_dev of the same stream (optb_roundtrip_dev): one
    fused launch on the vector path (lossless: P % 512 == 0), the two launches otherwise; the
    containers (and offsets) are materialised exactly as by the two calls."""
    import torch
    dt = {torch.uint8: U8, torch.float32: F32, torch.float16: F16, torch.bfloat16: BF16}[out.dtype]
    dev = out.device.index or 0
    E = Epilogue(dt, float(scale), _dptr(class_scale), _dptr(class_bias), _dptr(row_class), out.stride(0))
    check(lib.optb_roundtrip_dev(_lib.context(dev), ct.byref(L), _dptr(images), images.stride(0),
                                 _dptr(row_index), _dptr(containers), _dptr(offsets), ct.byref(E), _dptr(out),
                                 _stream(stream, dev)))


RT_KINDS = {0: "none", 1: "split", 2: "phase_ordered", 3: "interleaved", 4: "interleaved_deep",
            5: "interleaved_lane_st"}


def last_roundtrip_kind() -> str:
    """Kernel of this thread's most recent roundtrip_dev / pipeline step
    (optb_last_roundtrip_kind): "split" (two launches), "phase_ordered",
    "interleaved", "interleaved_deep" or "interleaved_lane_st".  The interleaved kernels read the
    containers back from L2, so their HBM bytes exclude the container re-read."""
    return RT_KINDS[lib.optb_last_roundtrip_kind()]


def roundtrip_hbm_bytes(L: Layout, out_elem_size: int, gathered: bool) -> int:
    """HBM bytes of one round trip of layout L by the kernel that last ran:
    rows in (+ 8 B row ids when gathered), containers (+ parity planes) out,
    decoded rows out, and the container (+ plane) re-read unless the
    interleaved kernel served it from L2 (SURVEY 8(d) per-image figures)."""
    rows = L.batch * L.n_batches
    cb, ob = container_bytes(L), offsets_bytes(L)
    b = rows * L.pixels + cb + ob + (rows * 8 if gathered else 0) + rows * L.pixels * out_elem_size
    if not last_roundtrip_kind().startswith("interleaved"):
        b += cb + ob
    return b


def encode_rows_dev(L: Layout, row_ptrs, containers, offsets=None, aligned16: bool = True, stream=None):
    """Gather-encode from absolute row addresses (optb_encode_rows_dev):
    stream row r packs the P bytes at row_ptrs[r] (int64 device tensor of
    addresses -- this GPU's HBM, a peer GPU's HBM opened over IPC, mapped
    host memory).  ``aligned16`` asserts 16-byte aligned rows (vector path)."""
    dev = containers.device.index or 0
    check(lib.optb_encode_rows_dev(_lib.context(dev), ct.byref(L), _dptr(row_ptrs), 1 if aligned16 else 0,
                                   _dptr(containers), _dptr(offsets), _stream(stream, dev)))


def roundtrip_rows_dev(L: Layout, row_ptrs, containers, out, offsets=None, aligned16: bool = True,
                       scale: float = 1.0, class_scale=None, class_bias=None, row_class=None, stream=None):
    """roundtrip_dev reading stream row r from row_ptrs[r] (optb_roundtrip_rows_dev)."""
    import torch
    dt = {torch.uint8: U8, torch.float32: F32, torch.float16: F16, torch.bfloat16: BF16}[out.dtype]
    dev = out.device.index or 0
    E = Epilogue(dt, float(scale), _dptr(class_scale), _dptr(class_bias), _dptr(row_class), out.stride(0))
    check(lib.optb_roundtrip_rows_dev(_lib.context(dev), ct.byref(L), _dptr(row_ptrs), 1 if aligned16 else 0,
                                      _dptr(containers), _dptr(offsets), ct.byref(E), _dptr(out),
                                      _stream(stream, dev)))


def shard_row_ptrs_dev(examples, bases, rows_per_shard: int, row_stride: int, out=None, stream=None):
    """Drawn example ids -> absolute row addresses in the shard that owns
    them (optb_shard_row_ptrs_dev); ``bases`` is an int64 device tensor of
    the shards' base addresses in this process."""
    import torch
    dev = examples.device.index or 0
    n = examples.numel()
    if out is None:
        out = torch.empty(max(n, 1), dtype=torch.int64, device=examples.device)
    check(lib.optb_shard_row_ptrs_dev(_lib.context(dev), _dptr(examples), n, _dptr(bases), bases.numel(),
                                      rows_per_shard, row_stride, _dptr(out), _stream(stream, dev)))
    return out[:n]


def sync(device: int = 0, stream=None) -> None:
    """Synchronise and raise any latched device-side FormatError (optb_ctx_sync)."""
    check(lib.optb_ctx_sync(_lib.context(device), _stream(stream, device)))


def dump_dev(L: Layout, containers, offsets, shape: ImageShape, directory: str, epoch: int) -> None:
    """pipeline::dump for a device stream (optb_dump_dev): chunk k ->
    <directory>/batch_<epoch>_<k>.optb in write_optb's format."""
    dev = containers.device.index or 0
    check(lib.optb_dump_dev(_lib.context(dev), ct.byref(L), _dptr(containers), _dptr(offsets), shape.height,
                            shape.width, shape.channels, str(directory).encode(), epoch))


def load_dev(L: Layout, shape: ImageShape, directory: str, epoch: int, device=0):
    """pipeline::load into device planes (optb_load_dev); validates headers."""
    cont, offs = alloc_stream(L, device)
    check(lib.optb_load_dev(_lib.context(device), ct.byref(L), shape.height, shape.width, shape.channels,
                            str(directory).encode(), epoch, _dptr(cont), _dptr(offs)))
    return cont, offs


def load_records_dev(path: str, shape: ImageShape, num_classes: int, max_records: int, device=0):
    """data::load_records (dataset.cpp:65-99) onto the device: returns
    (pixels [N, P] u8 HWC rows, labels [N] int32) tensors."""
    import torch
    dev = torch.device("cuda", device)
    P = shape.pixel_count()
    pixels = torch.empty((max(max_records, 1), max(P, 1)), dtype=torch.uint8, device=dev)
    labels = torch.empty(max(max_records, 1), dtype=torch.int32, device=dev)
    n = ct.c_uint64(0)
    check(lib.optb_load_records_dev(_lib.context(device), str(path).encode(), shape.height, shape.width,
                                    shape.channels, num_classes, _dptr(pixels), _dptr(labels), max_records,
                                    ct.byref(n)))
    return pixels[: n.value], labels[: n.value]


def write_optb(stream, enc: EncodedBatch) -> None:
    """codec::write_optb (codec.cpp:283-317): header + LE plane + parity plane."""
    if enc.n_images == 0:
        raise Error("optb: refusing to write an empty batch")
    hdr = b"OPTB" + (1).to_bytes(2, "little") + bytes([int(enc.mode), int(enc.n_images)])
    hdr += b"".join(int(v).to_bytes(4, "little") for v in (enc.shape.height, enc.shape.width, enc.shape.channels))
    stream.write(hdr + np.ascontiguousarray(enc.plane, np.uint8).tobytes()
                 + (np.ascontiguousarray(enc.offsets, np.uint8).tobytes() if mode_has_offsets(enc.mode) else b""))


def read_optb(stream) -> EncodedBatch:
    """codec::read_optb (codec.cpp:319-367) with the same checks and messages."""
    def take(n):
        b = stream.read(n)
        if len(b) != n:
            raise FormatError("optb: truncated stream")
        return b
    if take(4) != b"OPTB":
        raise FormatError("optb: bad magic")
    version = int.from_bytes(take(2), "little")
    if version != 1:
        raise FormatError(f"optb: unsupported version {version}")
    tag, n = take(1)[0], take(1)[0]
    if tag > 4:
        raise FormatError(f"optb: unknown mode tag {tag}")
    mode = CodecMode(tag)
    h, w, c = (int.from_bytes(take(4), "little") for _ in range(3))
    shape = ImageShape(h, w, c)
    P = shape.pixel_count()
    if n == 0 or P == 0:
        raise FormatError("optb: empty batch header")
    limit = capacity(mode) if capacity_is_hard(mode) else kFloat64AcceptLimit
    if n > limit:
        raise FormatError(f"optb: image count {n} exceeds {mode_name(mode)} capacity")
    plane = np.frombuffer(take(P * container_value_bytes(mode)), np.uint8).copy()
    offsets = np.frombuffer(take((n * P + 7) // 8), np.uint8).copy() if mode_has_offsets(mode) else np.zeros(0, np.uint8)
    return EncodedBatch(mode, shape, n, plane, offsets)


def encode_host(L: Layout, images: np.ndarray):
    """optb_encode_host over a whole host stream ([rows, P] u8)."""
    cont = np.zeros(container_bytes(L), np.uint8)
    ob = offsets_bytes(L)
    offs = np.zeros(max(ob, 16), np.uint8)
    images = np.ascontiguousarray(images, np.uint8)
    check(lib.optb_encode_host(_lib.context(), ct.byref(L), _ptr(images), _ptr(cont), _ptr(offs)))
    return cont, (offs[:ob] if ob else None)


def decode_host(L: Layout, cont: np.ndarray, offs: Optional[np.ndarray] = None, dtype=U8,
                scale: float = 1.0) -> np.ndarray:
    rows = L.batch * L.n_batches
    npdt = {U8: np.uint8, F32: np.float32, F16: np.uint16, BF16: np.uint16}[dtype]
    out = np.zeros((rows, L.pixels), npdt)
    E = Epilogue(dtype, float(scale), None, None, None, 0)
    ob = offsets_bytes(L)
    o = np.zeros(max(ob, 16), np.uint8)
    if offs is not None and ob:
        o[:ob] = offs[:ob]
    cont = np.ascontiguousarray(cont, np.uint8)
    check(lib.optb_decode_host(_lib.context(), ct.byref(L), _ptr(cont), _ptr(o), ct.byref(E), _ptr(out)))
    return out
