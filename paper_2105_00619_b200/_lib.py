"""ctypes binding of liboptb_cuda.so (the C ABI in include/optb_cuda.h).

This is the reference-side binding a Python user of the path adds: every
function declared in optb_cuda.h is bound here with its exact C signature.
There is deliberately no fallback: if the CUDA library is missing the import
fails with an instruction to build it.
"""
from __future__ import annotations

import ctypes as ct
import os
import threading

from .errors import raise_for

PKG = os.path.dirname(os.path.abspath(__file__))
# OPTB_CUDA_LIB selects an alternative build of the same library (tuning
# experiments, tools/tune_vec.sh); the default is the in-tree build.
LIB_PATH = os.environ.get("OPTB_CUDA_LIB", os.path.join(PKG, "liboptb_cuda.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the sm_100a library first "
        "(python -m paper_2105_00619_b200.build, or __graft_entry__.build())")

lib = ct.CDLL(LIB_PATH)

vp = ct.c_void_p
u8p = ct.POINTER(ct.c_uint8)
u64p = ct.POINTER(ct.c_uint64)
i64p = ct.POINTER(ct.c_int64)
i32p = ct.POINTER(ct.c_int32)
f64p = ct.POINTER(ct.c_double)


class Layout(ct.Structure):
    """optb_layout"""
    _fields_ = [("mode", ct.c_int32), ("per_chunk", ct.c_uint32), ("pixels", ct.c_uint64),
                ("batch", ct.c_uint64), ("n_batches", ct.c_uint64)]


class Epilogue(ct.Structure):
    """optb_epilogue"""
    _fields_ = [("out_dtype", ct.c_int32), ("scale", ct.c_float), ("class_scale", vp),
                ("class_bias", vp), ("row_class", vp), ("out_row_stride", ct.c_uint64)]


class PipelineDesc(ct.Structure):
    """optb_pipeline_desc"""
    _fields_ = [("layout", Layout), ("dataset", vp), ("row_stride", ct.c_uint64), ("sbs", vp),
                ("shard", ct.c_uint32), ("n_shards", ct.c_uint32), ("epilogue", Epilogue),
                ("record_timings", ct.c_int32), ("steps_per_draw", ct.c_uint32), ("split_kernels", ct.c_uint32),
                ("timing_stride", ct.c_uint32)]


LP = ct.POINTER(Layout)
EP = ct.POINTER(Epilogue)
fp = ct.POINTER(ct.c_float)

# name -> (restype, argtypes); exactly the declarations of include/optb_cuda.h
SIGNATURES = {
    "optb_abi_version": (ct.c_uint32, []),
    "optb_capacity": (ct.c_uint32, [ct.c_int32]),
    "optb_accept_limit": (ct.c_uint32, [ct.c_int32]),
    "optb_capacity_is_hard": (ct.c_int32, [ct.c_int32]),
    "optb_mode_name": (ct.c_char_p, [ct.c_int32]),
    "optb_mode_has_offsets": (ct.c_int32, [ct.c_int32]),
    "optb_container_value_bytes": (ct.c_uint32, [ct.c_int32]),
    "optb_offsets_plane_bytes": (ct.c_uint64, [ct.c_uint32, ct.c_uint64]),
    "optb_offsets_stride": (ct.c_uint64, [ct.c_int32, ct.c_uint64, ct.c_uint32]),
    "optb_layout_chunks": (ct.c_uint64, [LP]),
    "optb_layout_rows": (ct.c_uint64, [LP]),
    "optb_layout_container_bytes": (ct.c_uint64, [LP]),
    "optb_layout_offsets_bytes": (ct.c_uint64, [LP]),
    "optb_layout_check": (ct.c_int, [LP]),
    "optb_last_error": (ct.c_char_p, []),
    "optb_ctx_create": (ct.c_int, [ct.c_int, ct.POINTER(vp)]),
    "optb_ctx_destroy": (None, [vp]),
    "optb_ctx_sync": (ct.c_int, [vp, vp]),
    "optb_ctx_launches": (ct.c_uint64, [vp]),
    "optb_encode_dev": (ct.c_int, [vp, LP, vp, ct.c_uint64, vp, vp, vp, vp]),
    "optb_decode_dev": (ct.c_int, [vp, LP, vp, vp, EP, vp, vp]),
    "optb_roundtrip_dev": (ct.c_int, [vp, LP, vp, ct.c_uint64, vp, vp, vp, EP, vp, vp]),
    "optb_last_roundtrip_kind": (ct.c_int, []),
    "optb_encode_host": (ct.c_int, [vp, LP, vp, vp, vp]),
    "optb_decode_host": (ct.c_int, [vp, LP, vp, vp, EP, vp]),
    "optb_sbs_plan": (ct.c_int, [f64p, ct.c_uint64, ct.c_uint64, u64p]),
    "optb_class_index_dev": (ct.c_int, [vp, vp, ct.c_uint64, ct.c_uint64, vp, vp, vp]),
    "optb_class_index_host": (ct.c_int, [vp, vp, ct.c_uint64, ct.c_uint64, vp, vp]),
    "optb_sbs_create":(ct.c_int, [vp, u64p, ct.c_uint64, ct.c_uint64, ct.c_uint64, u64p, vp,
                                   ct.c_int32, ct.POINTER(vp)]),
    "optb_sbs_destroy": (None, [vp]),
    "optb_sbs_clone": (ct.c_int, [vp, ct.POINTER(vp)]),
    "optb_sbs_next_dev": (ct.c_int, [vp, ct.c_uint64, ct.c_uint32, ct.c_uint32, vp, vp, vp]),
    "optb_sbs_next_host": (ct.c_int, [vp, ct.c_uint64, vp, vp]),
    "optb_sbs_batches_drawn": (ct.c_uint64, [vp]),
    "optb_sbs_set_force_serial": (ct.c_int, [vp, ct.c_int32]),
    "optb_sbs_plan_call": (ct.c_int, [ct.c_uint64, u64p, u64p, u64p, ct.c_uint64, ct.c_uint64, ct.c_uint64,
                                      ct.c_uint64, u64p, u64p, u64p, u64p, u64p]),
    "optb_sbs_set_profiling": (ct.c_int, [vp, ct.c_int32]),
    "optb_sbs_profile": (ct.c_int, [vp, fp, fp, fp]),
    "optb_gather_rows_dev": (ct.c_int, [vp, vp, ct.c_uint64, vp, ct.c_uint64, ct.c_int64, ct.c_uint64, vp,
                                        ct.c_uint64, vp]),
    "optb_inverse_perm_dev": (ct.c_int, [vp, vp, ct.c_uint64, vp, vp]),
    "optb_owner_labels_dev": (ct.c_int, [vp, vp, ct.c_uint64, ct.c_uint64, ct.c_uint32, vp, vp]),
    "optb_shard_row_ptrs_dev": (ct.c_int, [vp, vp, ct.c_uint64, vp, ct.c_uint32, ct.c_uint64, ct.c_uint64, vp,
                                           vp]),
    "optb_encode_rows_dev": (ct.c_int, [vp, LP, vp, ct.c_int32, vp, vp, vp]),
    "optb_roundtrip_rows_dev": (ct.c_int, [vp, LP, vp, ct.c_int32, vp, vp, EP, vp, vp]),
    "optb_ipc_export": (ct.c_int, [vp, vp, u64p]),
    "optb_ipc_open": (ct.c_int, [ct.c_int, vp, ct.c_uint64, ct.POINTER(vp)]),
    "optb_ipc_close": (ct.c_int, [vp, ct.c_uint64]),
    "optb_dump_dev": (ct.c_int, [vp, LP, vp, vp, ct.c_uint32, ct.c_uint32, ct.c_uint32, ct.c_char_p, ct.c_uint64]),
    "optb_load_dev": (ct.c_int, [vp, LP, ct.c_uint32, ct.c_uint32, ct.c_uint32, ct.c_char_p, ct.c_uint64, vp, vp]),
    "optb_load_records_dev": (ct.c_int, [vp, ct.c_char_p, ct.c_uint32, ct.c_uint32, ct.c_uint32, ct.c_uint32, vp,
                                         vp, ct.c_uint64, u64p]),
    "optb_pipeline_create":(ct.c_int, [vp, ct.POINTER(PipelineDesc), ct.POINTER(vp)]),
    "optb_pipeline_create_warm": (ct.c_int, [vp, LP, ct.c_uint32, ct.c_uint32, ct.c_uint32, ct.c_char_p,
                                             ct.c_uint64, EP, ct.c_int32, ct.POINTER(vp)]),
    "optb_pipeline_step": (ct.c_int, [vp, vp, vp]),
    "optb_pipeline_set_dataset": (ct.c_int, [vp, vp, ct.c_uint64]),
    "optb_pipeline_step_host": (ct.c_int, [vp, vp, ct.c_uint64, ct.c_uint64, vp, vp]),
    "optb_pipeline_host_wait": (ct.c_int, [vp, vp]),
    "optb_pipeline_draws": (ct.c_int, [vp, ct.c_uint64, ct.POINTER(vp), ct.POINTER(vp)]),
    "optb_pipeline_containers": (vp, [vp]),
    "optb_pipeline_timings": (ct.c_int, [vp, ct.c_uint64, fp, fp, fp]),
    "optb_pipeline_destroy": (None, [vp]),
    "optb_synth_pixels_dev":(ct.c_int, [vp, ct.c_uint64, ct.c_uint64, ct.c_uint64, ct.c_uint64, vp,
                                         ct.c_uint64, vp]),
}

for _name, (_res, _args) in SIGNATURES.items():
    _f = getattr(lib, _name)
    _f.restype, _f.argtypes = _res, _args

assert lib.optb_abi_version() == 1, "liboptb_cuda.so ABI mismatch"


def check(status: int) -> None:
    """Raise the errors.hpp-equivalent exception for a non-zero status."""
    if status:
        raise_for(status, lib.optb_last_error().decode())


_tls = threading.local()


def context(device: int = 0):
    """Per-thread, per-device optb_ctx (the reference functions are reentrant;
    one context per host thread keeps that property)."""
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    h = ctxs.get(device)
    if h is None:
        out = vp()
        check(lib.optb_ctx_create(device, ct.byref(out)))
        h = ctxs[device] = out.value
    return h


def launches(device: int = 0) -> int:
    return lib.optb_ctx_launches(context(device))
