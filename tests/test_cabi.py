"""CPU tests of the C ABI boundary (no GPU compute calls).

* liboptb_cuda.so loads and exports every function include/optb_cuda.h declares;
* the host-only entry points (metadata, layout validation, sampler::plan)
  return the reference's values and messages;
* the product package fails loudly when its CUDA library is missing.
"""
import ctypes as ct
import os
import re
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "optb_cuda.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^[A-Za-z_][\w\s\*]*?\b(optb_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_symbols_exported(pkg):
    names = declared_functions()
    assert len(names) >= 30
    lib = ct.CDLL(os.path.join(ROOT, "paper_2105_00619_b200", "liboptb_cuda.so"))
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    bound = set(pkg._lib.SIGNATURES)
    assert set(names) == bound, set(names) ^ bound


def test_nm_exports_are_plain_c():
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_2105_00619_b200", "liboptb_cuda.so")],
                         capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    for n in declared_functions():
        assert n in exported, n  # unmangled extern "C"


def test_metadata(pkg):
    C = pkg.codec
    assert [C.capacity(m) for m in range(5)] == [8, 16, 6, 9, 18]  # test_codec.cpp:37-46
    assert [C.container_value_bytes(m) for m in range(5)] == [8, 16, 8, 8, 16]
    assert [C.mode_name(m) for m in range(5)] == ["exact64", "exact128", "f64", "lossless64", "lossless128"]
    assert C.capacity_is_hard(0) and C.capacity_is_hard(4) and not C.capacity_is_hard(2)
    assert C.accept_limit(2) == 16
    assert C.offsets_stride(3, 3072, 9) == (9 * 3072 + 7) // 8 // 16 * 16 + (16 if (9 * 3072 + 7) // 8 % 16 else 0)
    L = C.layout(1, 16, 3072, 100, 3)
    assert C.layout_chunks(L) == 3 * 7 and C.container_bytes(L) == 21 * 3072 * 16
    assert pkg._lib.lib.optb_layout_rows(ct.byref(L)) == 300


def test_roundtrip_kind_constants(pkg):
    """codec.RT_KINDS mirrors the OPTB_RT_* kernel kinds of the header, and the
    byte accounting counts the container re-read only for the kernels that
    read it from HBM; no round trip has run in this (CPU) process."""
    src = open(HEADER).read()
    consts = {int(v): n for n, v in re.findall(r"#define OPTB_RT_(\w+) (\d+)", src)}
    C = pkg.codec
    assert {k: v.lower() for k, v in consts.items()} == C.RT_KINDS
    assert C.last_roundtrip_kind() == "none"
    L = C.layout(1, 16, 3072, 512, 97)
    rows, cb = 512 * 97, C.container_bytes(L)
    assert C.roundtrip_hbm_bytes(L, 1, True) == rows * 3072 * 2 + rows * 8 + 2 * cb  # "none": as two launches


def test_layout_check_messages(pkg):
    lib = pkg._lib.lib
    cases = [((0, 9, 10, 10, 1), 3, "encode: 9 images exceed exact64 capacity of 8"),
             ((2, 17, 10, 10, 1), 3, "encode: 17 images exceed f64 capacity of 16"),
             ((0, 0, 10, 10, 1), 1, "encode: batch must contain at least one image"),
             ((0, 8, 0, 10, 1), 2, "encode: image extents must be positive"),
             ((7, 8, 10, 10, 1), 1, "unknown codec mode"),
             ((2, 16, 10, 10, 1), 0, "")]
    for args, code, msg in cases:
        L = pkg._lib.Layout(*args)
        assert lib.optb_layout_check(ct.byref(L)) == code
        assert lib.optb_last_error().decode() == msg


def test_plan_host_entry(golden, pkg):
    meta, _ = golden
    for name, g in meta["sbs"]["plans"].items():
        assert pkg.sampler.plan(g["weights"], g["batch"], 1).counts == g["counts"], name
    with pytest.raises(pkg.errors.Error) as ei:
        pkg.sampler.plan([0.5, 0.4], 8, 1)
    assert str(ei.value) == meta["errors"]["plan_sum"]["msg"]
    for b in range(1, 65):  # test_sampler.cpp:46-53
        assert sum(pkg.sampler.plan([0.37, 0.21, 0.19, 0.23], b, 1).counts) == b


def test_missing_library_fails_loudly(tmp_path):
    dst = tmp_path / "paper_2105_00619_b200"
    shutil.copytree(os.path.join(ROOT, "paper_2105_00619_b200"), dst,
                    ignore=shutil.ignore_patterns("*.so", "csrc", "__pycache__"))
    r = subprocess.run([sys.executable, "-c", "import paper_2105_00619_b200"], cwd=tmp_path,
                       capture_output=True, text=True)
    assert r.returncode != 0 and "liboptb_cuda.so is missing" in r.stderr


def test_layout_arithmetic_matches_oracle(pkg, oracle_mod):
    """The C ABI's stream layout (chunks per batch as runner.cpp:77-90 cuts
    them, container and parity-plane bytes, the plane's 16-byte padded
    stride) equals the oracle's for every mode over a grid of ragged shapes
    -- the sizes every caller allocates from."""
    C, O = pkg.codec, oracle_mod
    for mode in range(5):
        cap = C.capacity(mode)
        for pc in sorted({1, 2, cap // 2 or 1, cap}):
            for P, B, nb in ((48, 37, 5), (3072, 512, 2), (108, 40, 3), (1024, 7, 1), (150528, 256, 1)):
                L = C.layout(mode, pc, P, B, nb)
                chunks = O.stream_chunks(B, nb, pc)
                assert C.layout_chunks(L) == chunks, (mode, pc, P, B, nb)
                assert C.container_bytes(L) == chunks * P * C.container_value_bytes(mode)
                ost = O.offsets_stride(mode, P, pc)
                assert C.offsets_stride(mode, P, pc) == ost
                assert C.offsets_bytes(L) == chunks * ost
