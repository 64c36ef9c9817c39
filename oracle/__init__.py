"""ctypes/numpy front for the oracle libraries.

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs -- never by the product
package ``paper_2105_00619_b200`` (which fails loudly without its CUDA
library instead of falling back to anything here).

* ``C``   -- liboptb_oracle.so, the C restatement (oracle/optb_oracle.c).
* ``REF`` -- oracle/_ref/liboptb_ref.so, the reference library compiled from
  its own sources (oracle/Makefile); ``None`` when it was never built.
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboptb_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "liboptb_ref.so")

EXACT64, EXACT128, F64, LOSSLESS64, LOSSLESS128 = range(5)
U8, F32, F16, BF16 = range(4)
MODES = (EXACT64, EXACT128, F64, LOSSLESS64, LOSSLESS128)
CAPACITY = {EXACT64: 8, EXACT128: 16, F64: 6, LOSSLESS64: 9, LOSSLESS128: 18}
ACCEPT = {EXACT64: 8, EXACT128: 16, F64: 16, LOSSLESS64: 9, LOSSLESS128: 18}
WC = {EXACT64: 8, EXACT128: 16, F64: 8, LOSSLESS64: 8, LOSSLESS128: 16}
HAS_OFFSETS = {EXACT64: False, EXACT128: False, F64: False, LOSSLESS64: True, LOSSLESS128: True}
NAMES = {EXACT64: "exact64", EXACT128: "exact128", F64: "f64", LOSSLESS64: "lossless64",
         LOSSLESS128: "lossless128"}

u8p = ct.POINTER(ct.c_uint8)
i64p = ct.POINTER(ct.c_int64)
u64p = ct.POINTER(ct.c_uint64)
i32p = ct.POINTER(ct.c_int32)
u32p = ct.POINTER(ct.c_uint32)
f32p = ct.POINTER(ct.c_float)
f64p = ct.POINTER(ct.c_double)


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def ptr(a, t=ct.c_void_p):
    if a is None:
        return None
    return ct.cast(a.ctypes.data, t)


def build(quiet: bool = True) -> None:
    """Compile the oracle (and, where /root/reference exists, oracle/_ref)."""
    out = subprocess.run(["make", "-s", "-f", os.path.join(HERE, "Makefile"), "all"],
                         capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)


def _load_c():
    if not os.path.exists(ORACLE_SO):
        build()
    lib = ct.CDLL(ORACLE_SO)
    sig = {
        "orc_encode": (ct.c_int, [ct.c_int, u8p, ct.c_uint32, ct.c_uint64, u8p, u8p, ct.c_char_p, ct.c_size_t]),
        "orc_decode": (ct.c_int, [ct.c_int, u8p, u8p, ct.c_uint32, ct.c_uint64, u8p, ct.c_char_p, ct.c_size_t]),
        "orc_roundtrip_error": (ct.c_int, [ct.c_int, u8p, ct.c_uint32, ct.c_uint64, i32p, ct.c_char_p, ct.c_size_t]),
        "orc_encode_stream": (ct.c_int, [ct.c_int, ct.c_uint32, ct.c_uint64, ct.c_uint64, ct.c_uint64, u8p, ct.c_uint64,
                                         i64p, u8p, u8p, ct.c_uint64, ct.c_char_p, ct.c_size_t]),
        "orc_decode_stream": (ct.c_int, [ct.c_int, ct.c_uint32, ct.c_uint64, ct.c_uint64, ct.c_uint64, u8p, u8p,
                                         ct.c_uint64, ct.c_int, ct.c_float, f32p, f32p, i32p, ct.c_void_p,
                                         ct.c_uint64, ct.c_char_p, ct.c_size_t]),
        "orc_float_to_half": (ct.c_uint16, [ct.c_float]),
        "orc_float_to_bf16": (ct.c_uint16, [ct.c_float]),
        "orc_mix": (ct.c_uint64, [ct.c_uint64]),
        "orc_next_u64": (ct.c_uint64, [u64p]),
        "orc_next_below": (ct.c_uint64, [u64p, ct.c_uint64]),
        "orc_sbs_plan": (ct.c_int, [f64p, ct.c_uint64, ct.c_uint64, u64p, ct.c_char_p, ct.c_size_t]),
        "orc_class_index": (ct.c_int, [i32p, ct.c_uint64, ct.c_uint64, u64p, i64p, ct.c_char_p, ct.c_size_t]),
        "orc_cursor_create": (ct.c_void_p, [u64p, ct.c_uint64, ct.c_uint64, ct.c_uint64, u64p, i64p,
                                            ct.POINTER(ct.c_int), ct.c_char_p, ct.c_size_t]),
        "orc_cursor_next": (None, [ct.c_void_p, ct.c_uint64, i64p, i32p]),
        "orc_cursor_rng_state": (ct.c_uint64, [ct.c_void_p]),
        "orc_cursor_destroy": (None, [ct.c_void_p]),
        "orc_synth_pixels": (None, [ct.c_uint64, ct.c_uint64, ct.c_uint64, ct.c_uint64, u8p]),
        "orc_fnv1a64": (ct.c_uint64, [ct.c_void_p, ct.c_size_t]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    return lib


def _load_ref():
    if not os.path.exists(REF_SO):
        return None
    lib = ct.CDLL(REF_SO)
    sig = {
        "ref_encode": (ct.c_int, [ct.c_int, u8p, ct.c_uint32, ct.c_uint32, ct.c_uint32, ct.c_uint32, u8p, u8p,
                                  ct.c_char_p, ct.c_size_t]),
        "ref_decode": (ct.c_int, [ct.c_int, u8p, u8p, ct.c_uint32, ct.c_uint32, ct.c_uint32, ct.c_uint32, u8p,
                                  ct.c_char_p, ct.c_size_t]),
        "ref_roundtrip_error": (ct.c_int, [ct.c_int, u8p, ct.c_uint32, ct.c_uint32, ct.c_uint32, ct.c_uint32, i32p,
                                           ct.c_char_p, ct.c_size_t]),
        "ref_write_optb": (ct.c_int, [ct.c_int, u8p, ct.c_uint32, ct.c_uint32, ct.c_uint32, ct.c_uint32, u8p,
                                      ct.c_size_t, ct.POINTER(ct.c_size_t), ct.c_char_p, ct.c_size_t]),
        "ref_decode_input": (ct.c_int, [ct.c_int, u8p, u8p, ct.c_uint64, u32p, ct.c_uint32, ct.c_uint32,
                                        ct.c_uint32, ct.c_uint32, ct.c_float, ct.c_int, ct.c_void_p,
                                        ct.c_char_p, ct.c_size_t]),
        "ref_float_to_half": (ct.c_uint16, [ct.c_float]),
        "ref_sbs_plan": (ct.c_int, [f64p, ct.c_uint64, ct.c_uint64, ct.c_uint64, u64p, ct.c_char_p, ct.c_size_t]),
        "ref_class_index": (ct.c_int, [i32p, ct.c_uint64, ct.c_uint64, u64p, i64p, ct.c_char_p, ct.c_size_t]),
        "ref_cursor_create": (ct.c_void_p, [f64p, ct.c_uint64, ct.c_uint64, ct.c_uint64, u64p, i64p,
                                            ct.POINTER(ct.c_int), ct.c_char_p, ct.c_size_t]),
        "ref_cursor_next": (None, [ct.c_void_p, ct.c_uint64, i64p, i32p]),
        "ref_cursor_destroy": (None, [ct.c_void_p]),
        "ref_dataset_create": (ct.c_void_p, [u8p, ct.c_uint64, ct.c_uint32, ct.c_uint32, ct.c_uint32]),
        "ref_dataset_destroy": (None, [ct.c_void_p]),
        "ref_bench_roundtrip": (ct.c_double, [ct.c_void_p, ct.c_int, i64p, ct.c_uint64, ct.c_uint64, ct.c_int,
                                              ct.c_int, u64p]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    return lib


C = _load_c()
REF = _load_ref()


def _check(code, buf):
    if code:
        raise OracleError(code, buf.value.decode())


# ------------------------------------------------------------------ codec
def encode(images: np.ndarray, mode: int):
    """images [n][P] u8 -> (plane [P*Wc] u8, offsets u8 or None)."""
    images = np.ascontiguousarray(images, dtype=np.uint8)
    n, P = images.shape
    plane = np.zeros(P * WC[mode], np.uint8)
    offs = np.zeros(max(1, (n * P + 7) // 8), np.uint8) if HAS_OFFSETS[mode] else None
    buf = ct.create_string_buffer(512)
    _check(C.orc_encode(mode, ptr(images, u8p), n, P, ptr(plane, u8p), ptr(offs, u8p), buf, 512), buf)
    if offs is not None:
        offs = offs[: (n * P + 7) // 8]
    return plane, offs


def decode(plane: np.ndarray, offsets, n: int, P: int, mode: int) -> np.ndarray:
    plane = np.ascontiguousarray(plane, dtype=np.uint8)
    out = np.zeros((n, P), np.uint8)
    offs = None if offsets is None else np.ascontiguousarray(offsets, np.uint8)
    buf = ct.create_string_buffer(512)
    _check(C.orc_decode(mode, ptr(plane, u8p), ptr(offs, u8p), n, P, ptr(out, u8p), buf, 512), buf)
    return out


def roundtrip_error(images: np.ndarray, mode: int) -> np.ndarray:
    images = np.ascontiguousarray(images, dtype=np.uint8)
    n, P = images.shape
    errs = np.zeros(n, np.int32)
    buf = ct.create_string_buffer(512)
    _check(C.orc_roundtrip_error(mode, ptr(images, u8p), n, P, ptr(errs, i32p), buf, 512), buf)
    return errs


def stream_chunks(batch: int, n_batches: int, per_chunk: int) -> int:
    return n_batches * ((batch + per_chunk - 1) // per_chunk)


def offsets_stride(mode: int, P: int, per_chunk: int) -> int:
    """Per-chunk offsets stride of the device layout (16-byte padded)."""
    if not HAS_OFFSETS[mode]:
        return 0
    return ((per_chunk * P + 7) // 8 + 15) // 16 * 16


def encode_stream(dataset: np.ndarray, row_index, mode: int, per_chunk: int, batch: int,
                  n_batches: int):
    dataset = np.ascontiguousarray(dataset, dtype=np.uint8)
    P = dataset.shape[1]
    chunks = stream_chunks(batch, n_batches, per_chunk)
    cont = np.zeros(chunks * P * WC[mode], np.uint8)
    ost = offsets_stride(mode, P, per_chunk)
    offs = np.zeros(max(1, chunks * ost), np.uint8) if ost else None
    idx = None if row_index is None else np.ascontiguousarray(row_index, np.int64)
    buf = ct.create_string_buffer(512)
    _check(C.orc_encode_stream(mode, per_chunk, P, batch, n_batches, ptr(dataset, u8p), P, ptr(idx, i64p),
                               ptr(cont, u8p), ptr(offs, u8p), ost, buf, 512), buf)
    return cont, offs


def decode_stream(cont, offs, mode: int, per_chunk: int, P: int, batch: int, n_batches: int,
                  out_dtype: int = U8, scale: float = 1.0, class_scale=None, class_bias=None,
                  row_class=None):
    rows = batch * n_batches
    dt = {U8: np.uint8, F32: np.float32, F16: np.uint16, BF16: np.uint16}[out_dtype]
    out = np.zeros((rows, P), dt)
    ost = offsets_stride(mode, P, per_chunk)
    buf = ct.create_string_buffer(512)
    cs = None if class_scale is None else np.ascontiguousarray(class_scale, np.float32)
    cb = None if class_bias is None else np.ascontiguousarray(class_bias, np.float32)
    rc = None if row_class is None else np.ascontiguousarray(row_class, np.int32)
    _check(C.orc_decode_stream(mode, per_chunk, P, batch, n_batches, ptr(np.ascontiguousarray(cont), u8p),
                               ptr(offs, u8p), ost, out_dtype, ct.c_float(scale), ptr(cs, f32p), ptr(cb, f32p),
                               ptr(rc, i32p), ptr(out), P, buf, 512), buf)
    return out


# ------------------------------------------------------------------ sampler
def sbs_plan(weights, batch: int) -> np.ndarray:
    w = np.ascontiguousarray(weights, np.float64)
    counts = np.zeros(len(w), np.uint64)
    buf = ct.create_string_buffer(512)
    _check(C.orc_sbs_plan(ptr(w, f64p), len(w), batch, ptr(counts, u64p), buf, 512), buf)
    return counts


def class_index(labels, n_classes: int):
    lab = np.ascontiguousarray(labels, np.int32)
    off = np.zeros(n_classes + 1, np.uint64)
    mem = np.zeros(max(1, len(lab)), np.int64)
    buf = ct.create_string_buffer(512)
    _check(C.orc_class_index(ptr(lab, i32p), len(lab), n_classes, ptr(off, u64p), ptr(mem, i64p), buf, 512), buf)
    return off, mem[: len(lab)]


class Cursor:
    """Oracle BatchCursor over (counts, class lists, seed) -- sampler.cpp:67-104."""

    def __init__(self, counts, class_offsets, members, batch: int, seed: int):
        self.counts = np.ascontiguousarray(counts, np.uint64)
        off = np.ascontiguousarray(class_offsets, np.uint64)
        mem = np.ascontiguousarray(members, np.int64)
        if mem.size == 0:
            mem = np.zeros(1, np.int64)
        st = ct.c_int(0)
        buf = ct.create_string_buffer(512)
        self.h = C.orc_cursor_create(ptr(self.counts, u64p), len(self.counts), batch, seed, ptr(off, u64p),
                                     ptr(mem, i64p), ct.byref(st), buf, 512)
        _check(st.value, buf)
        self.batch = batch

    def next(self, n_batches: int = 1):
        ex = np.zeros(n_batches * self.batch, np.int64)
        cl = np.zeros(n_batches * self.batch, np.int32)
        C.orc_cursor_next(self.h, n_batches, ptr(ex, i64p), ptr(cl, i32p))
        return ex, cl

    def rng_state(self) -> int:
        return C.orc_cursor_rng_state(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            C.orc_cursor_destroy(self.h)
            self.h = None


def mix(z: int) -> int:
    return C.orc_mix(z & 0xFFFFFFFFFFFFFFFF)


def synth_pixels(seed: int, first_row: int, n_rows: int, P: int) -> np.ndarray:
    out = np.zeros((n_rows, P), np.uint8)
    C.orc_synth_pixels(seed, first_row, n_rows, P, ptr(out, u8p))
    return out


def fnv1a64(a: np.ndarray) -> int:
    a = np.ascontiguousarray(a)
    return C.orc_fnv1a64(ptr(a), a.nbytes)


def float_to_half(v: float) -> int:
    return C.orc_float_to_half(ct.c_float(v))


def float_to_bf16(v: float) -> int:
    return C.orc_float_to_bf16(ct.c_float(v))


def records_to_hwc(raw: bytes, h: int, w: int, c: int):
    """data::load_records' record parse (dataset.cpp:65-99): each record is a
    label byte then C planes of H*W bytes; pixels[hw*C + c] = plane c [hw]
    (dataset.cpp:84-91).  Returns (pixels [N, P] u8, labels [N] int32)."""
    P = h * w * c
    arr = np.frombuffer(raw, np.uint8).reshape(-1, P + 1)
    labels = arr[:, 0].astype(np.int32)
    pixels = arr[:, 1:].reshape(-1, c, h * w).transpose(0, 2, 1).reshape(-1, P)
    return np.ascontiguousarray(pixels), labels


# ------------------------------------------------------------------ reference (compiled)
def ref_available() -> bool:
    return REF is not None


def ref_encode(images: np.ndarray, mode: int, shape=None):
    images = np.ascontiguousarray(images, dtype=np.uint8)
    n, P = images.shape
    h, w, c = shape or (1, P, 1)
    plane = np.zeros(P * WC[mode], np.uint8)
    offs = np.zeros(max(1, (n * P + 7) // 8), np.uint8)
    buf = ct.create_string_buffer(512)
    _check(REF.ref_encode(mode, ptr(images, u8p), n, h, w, c, ptr(plane, u8p), ptr(offs, u8p), buf, 512), buf)
    return plane, (offs[: (n * P + 7) // 8] if HAS_OFFSETS[mode] else None)


def ref_decode(plane, offsets, n: int, P: int, mode: int, shape=None) -> np.ndarray:
    h, w, c = shape or (1, P, 1)
    out = np.zeros((n, P), np.uint8)
    plane = np.ascontiguousarray(plane, np.uint8)
    offs = None if offsets is None else np.ascontiguousarray(offsets, np.uint8)
    buf = ct.create_string_buffer(512)
    _check(REF.ref_decode(mode, ptr(plane, u8p), ptr(offs, u8p), n, h, w, c, ptr(out, u8p), buf, 512), buf)
    return out
