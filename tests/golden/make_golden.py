"""Generate the golden fixtures in tests/golden/ from the REFERENCE library.

Run here (where /root/reference exists and oracle/_ref/liboptb_ref.so was
built from its sources by oracle/Makefile):

    python tests/golden/make_golden.py

Every output array below is produced by the compiled reference
(optb_ref::codec / sampler / nn), not by the C restatement -- that is what
makes the fixtures an independent pin for both the oracle (CPU tests) and
the CUDA path (GPU tests).  Inputs are seeded numpy draws and are stored
next to the outputs so the fixtures are self-contained on the GPU box.
"""
from __future__ import annotations

import ctypes as ct
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
GAMMA = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1


def mix_inverse(z: int) -> int:
    """Inverse of the SplitMix64 finaliser (rng.hpp:17-20)."""
    def inv_xorshift(y, s):
        x = y
        for _ in range(64 // s + 1):
            x = y ^ (x >> s)
        return x & M64
    z = inv_xorshift(z, 31)
    z = (z * pow(0x94D049BB133111EB, -1, 1 << 64)) & M64
    z = inv_xorshift(z, 27)
    z = (z * pow(0xBF58476D1CE4E5B9, -1, 1 << 64)) & M64
    z = inv_xorshift(z, 30)
    return z


def ref_err(fn, *args):
    buf = ct.create_string_buffer(512)
    code = fn(*args, buf, 512)
    return code, buf.value.decode()


def codec_fixtures(rng):
    """Per mode: random small shapes (like test_codec.cpp:158-174) and CIFAR
    shapes at n = capacity and a partial n; planes/offsets/decodes from ref."""
    cases = []
    arrays = {}
    k = 0
    for mode in O.MODES:
        shapes = [(1, 1, 1), (2, 3, 1), (3, 3, 3), (4, 4, 3), (6, 6, 3), (32, 32, 3)]
        for shape in shapes:
            P = shape[0] * shape[1] * shape[2]
            for n in sorted({1, max(1, O.CAPACITY[mode] // 2), O.CAPACITY[mode], O.ACCEPT[mode]}):
                imgs = rng.integers(0, 256, size=(n, P), dtype=np.uint8)
                plane, offs = O.ref_encode(imgs, mode, shape)
                back = O.ref_decode(plane, offs, n, P, mode, shape)
                key = f"c{k}"
                arrays[key + "_in"] = imgs
                arrays[key + "_plane"] = plane
                if offs is not None:
                    arrays[key + "_offs"] = offs
                arrays[key + "_back"] = back
                cases.append({"key": key, "mode": mode, "n": n, "shape": list(shape)})
                k += 1
    # edge sets: all-0 and all-255 at capacity (max container)
    for mode in O.MODES:
        for val in (0, 255):
            n = O.CAPACITY[mode]
            imgs = np.full((n, 48), val, np.uint8)
            plane, offs = O.ref_encode(imgs, mode, (4, 4, 3))
            key = f"c{k}"
            arrays[key + "_in"] = imgs
            arrays[key + "_plane"] = plane
            if offs is not None:
                arrays[key + "_offs"] = offs
            arrays[key + "_back"] = O.ref_decode(plane, offs, n, 48, mode, (4, 4, 3))
            cases.append({"key": key, "mode": mode, "n": n, "shape": [4, 4, 3]})
            k += 1
    return cases, arrays


def stream_fixture(rng):
    """A gathered batch stream (runner.cpp:77-90): 2 batches of 40 rows drawn
    from a 96-row 16x16x3 dataset; per_chunk = capacity so batch 40 gives a
    partial last chunk for every mode; plus nn::decode_input fp32/fp16."""
    P = 768
    NB = 2
    ds = rng.integers(0, 256, size=(96, P), dtype=np.uint8)
    idx = rng.integers(0, 96, size=NB * 40).astype(np.int64)
    arrays = {"ds": ds, "idx": idx}
    meta = []
    for mode in O.MODES:
        cap = O.CAPACITY[mode]
        cpb = (40 + cap - 1) // cap
        planes, offs_all, ns = [], [], []
        for b in range(NB):
            for j in range(cpb):
                rows = idx[b * 40 + j * cap: b * 40 + min((j + 1) * cap, 40)]
                plane, offs = O.ref_encode(ds[rows], mode, (16, 16, 3))
                planes.append(plane)
                ost = O.offsets_stride(mode, P, cap)
                if ost:
                    o = np.zeros(ost, np.uint8)
                    o[: offs.size] = offs
                    offs_all.append(o)
                ns.append(len(rows))
        cont = np.concatenate(planes)
        offs_cat = np.concatenate(offs_all) if offs_all else None
        arrays[f"s{mode}_cont"] = cont
        if offs_cat is not None:
            arrays[f"s{mode}_offs"] = offs_cat
        # decode_input over all chunks of the stream (fp32 at 1/255, and fp16)
        nsa = np.array(ns, np.uint32)
        scale = np.float32(1.0) / np.float32(255.0)
        f32 = np.zeros((NB * 40, P), np.float32)
        f16 = np.zeros((NB * 40, P), np.uint16)
        ost = O.offsets_stride(mode, P, cap)
        for out, half in ((f32, 0), (f16, 1)):
            code, msg = ref_err(O.REF.ref_decode_input, mode, O.ptr(cont, O.u8p),
                                O.ptr(offs_cat, O.u8p), ost, O.ptr(nsa, O.u32p), len(ns), 16, 16, 3,
                                ct.c_float(scale), half, O.ptr(out))
            assert code == 0, msg
        arrays[f"s{mode}_f32"] = f32
        arrays[f"s{mode}_f16"] = f16
        meta.append({"mode": mode, "per_chunk": cap, "batch": 40, "n_batches": NB, "shape": [16, 16, 3]})
    return meta, arrays


def sbs_fixtures():
    out = {}
    arrays = {}
    # C2: CIFAR-100 labels e % 100, N = 50 000, uniform weights, B = 512, seed 1234
    labels = (np.arange(50000) % 100).astype(np.int32)
    off = np.zeros(101, np.uint64)
    mem = np.zeros(50000, np.int64)
    assert ref_err(O.REF.ref_class_index, O.ptr(labels, O.i32p), 50000, 100, O.ptr(off, O.u64p),
                   O.ptr(mem, O.i64p))[0] == 0
    w = np.full(100, 0.01)
    st = ct.c_int(0)
    buf = ct.create_string_buffer(512)
    h = O.REF.ref_cursor_create(O.ptr(w, O.f64p), 100, 512, 1234, O.ptr(off, O.u64p), O.ptr(mem, O.i64p),
                                ct.byref(st), buf, 512)
    assert st.value == 0
    ex = np.zeros(300 * 512, np.int64)
    cl = np.zeros(300 * 512, np.int32)
    O.REF.ref_cursor_next(h, 300, O.ptr(ex, O.i64p), O.ptr(cl, O.i32p))
    O.REF.ref_cursor_destroy(h)
    arrays["c2_examples"] = ex
    arrays["c2_classes"] = cl.astype(np.int16)
    out["c2"] = {"n": 50000, "classes": 100, "batch": 512, "seed": 1234, "batches": 300}

    # skewed [0.5, 0.25, 0.25], B = 16 over tiny classes incl. a
    # 7-example class drawn 8 per batch (several reshuffles inside one batch)
    sk_labels = np.array([0] * 7 + [1] * 11 + [2] * 3, np.int32)
    rng = np.random.default_rng(5)
    rng.shuffle(sk_labels)
    arrays["skew_labels"] = sk_labels
    off = np.zeros(4, np.uint64)
    mem = np.zeros(len(sk_labels), np.int64)
    assert ref_err(O.REF.ref_class_index, O.ptr(sk_labels, O.i32p), len(sk_labels), 3, O.ptr(off, O.u64p),
                   O.ptr(mem, O.i64p))[0] == 0
    w = np.array([0.5, 0.25, 0.25])
    h = O.REF.ref_cursor_create(O.ptr(w, O.f64p), 3, 16, 77, O.ptr(off, O.u64p), O.ptr(mem, O.i64p),
                                ct.byref(st), buf, 512)
    assert st.value == 0
    ex = np.zeros(50 * 16, np.int64)
    cl = np.zeros(50 * 16, np.int32)
    O.REF.ref_cursor_next(h, 50, O.ptr(ex, O.i64p), O.ptr(cl, O.i32p))
    O.REF.ref_cursor_destroy(h)
    arrays["skew_examples"] = ex
    arrays["skew_classes"] = cl
    out["skew"] = {"classes": 3, "weights": [0.5, 0.25, 0.25], "batch": 16, "seed": 77, "batches": 50}

    # Rejection sampling inside Fisher-Yates (rng.hpp:29-35).  For i = 3 the
    # only rejected 64-bit draw is 2^64 - 1; the seed is chosen by inverting
    # the SplitMix64 chain so that (a) the constructor's shuffle of class 0
    # (3 examples) and (b) the first lazy reshuffle of class 1 both hit it.
    # Class 1 has 3 examples and count 2, class 0 count 2, plus an empty class 2.
    s_bad = (mix_inverse(M64) - GAMMA) & M64  # state whose first draw is 2^64-1
    # ctor: event0 = class0 (m=3) at seed s0; want s0 = s_bad -> K0 = 3 (1 rejection)
    seed_a = s_bad
    arrays["rej_a_members"] = np.array([10, 11, 12, 20, 21, 22], np.int64)
    w_rej = np.array([0.5, 0.5, 0.0])
    off_rej = np.array([0, 3, 6, 6], np.uint64)
    h = O.REF.ref_cursor_create(O.ptr(w_rej, O.f64p), 3, 4, seed_a, O.ptr(off_rej, O.u64p),
                                O.ptr(arrays["rej_a_members"], O.i64p), ct.byref(st), buf, 512)
    assert st.value == 0, buf.value
    ex = np.zeros(40, np.int64)
    O.REF.ref_cursor_next(h, 10, O.ptr(ex, O.i64p), None)
    O.REF.ref_cursor_destroy(h)
    arrays["rej_a_examples"] = ex
    out["rej_a"] = {"seed": seed_a, "counts": [2, 2, 0], "class_offsets": [0, 3, 6, 6], "batch": 4,
                    "weights": [0.5, 0.5, 0.0], "batches": 10}

    # (b): event order: ctor c0 (m=3, K=2), ctor c1 (m=3, K=2), ctor c2 (m=0, K=0),
    # then batch 1 needs class 0 again after 2 draws -> pos 2<3 fine; batch 1
    # draws c0 at pos 2, then pos==3 -> lazy event of class 0 before its 2nd draw.
    # Put the rejection into that lazy event: invert the chain backwards.
    s3 = s_bad                                   # state at the lazy event
    s2 = (mix_inverse(s3) - 1 * GAMMA) & M64     # before ctor c2: K=0 -> s3 = mix(s2 + 1*g)
    s1 = (mix_inverse(s2) - 3 * GAMMA) & M64     # before ctor c1: K=2 -> s2 = mix(s1 + 3*g)
    s0 = (mix_inverse(s1) - 3 * GAMMA) & M64     # before ctor c0: K=2
    seed_b = s0
    h = O.REF.ref_cursor_create(O.ptr(w_rej, O.f64p), 3, 4, seed_b, O.ptr(off_rej, O.u64p),
                                O.ptr(arrays["rej_a_members"], O.i64p), ct.byref(st), buf, 512)
    assert st.value == 0, buf.value
    ex = np.zeros(40, np.int64)
    O.REF.ref_cursor_next(h, 10, O.ptr(ex, O.i64p), None)
    O.REF.ref_cursor_destroy(h)
    arrays["rej_b_examples"] = ex
    out["rej_b"] = {"seed": seed_b, "counts": [2, 2, 0], "class_offsets": [0, 3, 6, 6], "batch": 4,
                    "weights": [0.5, 0.5, 0.0], "batches": 10}

    # plan() count vectors (test_sampler.cpp:22-54) from the reference
    plans = {}
    for name, ws, b in [("half_quarters", [0.5, 0.25, 0.25], 16), ("single", [1.0], 13),
                        ("tenths", [0.1] * 10, 16), ("starved", [0.99, 0.01], 10),
                        ("uniform100_512", [0.01] * 100, 512), ("odd4_37", [0.37, 0.21, 0.19, 0.23], 37)]:
        wv = np.array(ws, np.float64)
        counts = np.zeros(len(ws), np.uint64)
        code, msg = ref_err(O.REF.ref_sbs_plan, O.ptr(wv, O.f64p), len(ws), b, 1, O.ptr(counts, O.u64p))
        assert code == 0, msg
        plans[name] = {"weights": ws, "batch": b, "counts": [int(c) for c in counts]}
    out["plans"] = plans
    return out, arrays


def error_fixtures():
    """Reference error codes + messages for the validation paths the
    reference tests assert on (test_codec.cpp:118-156, 102-116;
    test_sampler.cpp:56-64, 101-110)."""
    errs = {}
    buf_plane = np.zeros(16 * 64, np.uint8)
    offs = np.zeros(64, np.uint8)
    for mode in O.MODES:
        n = O.ACCEPT[mode] + 1
        imgs = np.zeros((n, 1), np.uint8)
        errs[f"capacity_{mode}"] = ref_err(O.REF.ref_encode, mode, O.ptr(imgs, O.u8p), n, 1, 1, 1,
                                           O.ptr(buf_plane, O.u8p), O.ptr(offs, O.u8p))
    # decode range errors: exact64 n=1 value 256; f64 n=1 value 256.0; lossless64 n=2 bit 14 set
    plane = np.zeros(16, np.uint8)
    plane[:8] = np.frombuffer(np.uint64(256).tobytes(), np.uint8)
    out = np.zeros(16, np.uint8)
    errs["range_exact64"] = ref_err(O.REF.ref_decode, 0, O.ptr(plane, O.u8p), None, 1, 1, 1, 1, O.ptr(out, O.u8p))
    plane[:8] = np.frombuffer(np.float64(256.0).tobytes(), np.uint8)
    errs["range_f64"] = ref_err(O.REF.ref_decode, 2, O.ptr(plane, O.u8p), None, 1, 1, 1, 1, O.ptr(out, O.u8p))
    plane[:8] = np.frombuffer(np.float64(-1.0).tobytes(), np.uint8)
    errs["range_f64_neg"] = ref_err(O.REF.ref_decode, 2, O.ptr(plane, O.u8p), None, 1, 1, 1, 1, O.ptr(out, O.u8p))
    plane[:8] = np.frombuffer(np.uint64(1 << 14).tobytes(), np.uint8)
    o1 = np.zeros(1, np.uint8)
    errs["range_lossless64"] = ref_err(O.REF.ref_decode, 3, O.ptr(plane, O.u8p), O.ptr(o1, O.u8p), 2, 1, 1, 1,
                                       O.ptr(out, O.u8p))
    # sampler
    counts = np.zeros(3, np.uint64)
    for name, ws, b in [("neg", [0.7, -0.2, 0.5], 8), ("sum", [0.5, 0.4], 8), ("batch0", [0.5, 0.5], 0)]:
        wv = np.array(ws, np.float64)
        errs[f"plan_{name}"] = ref_err(O.REF.ref_sbs_plan, O.ptr(wv, O.f64p), len(ws), b, 1, O.ptr(counts, O.u64p))
    lab = np.array([0, 3], np.int32)
    off = np.zeros(4, np.uint64)
    mem = np.zeros(2, np.int64)
    errs["label_range"] = ref_err(O.REF.ref_class_index, O.ptr(lab, O.i32p), 2, 3, O.ptr(off, O.u64p),
                                  O.ptr(mem, O.i64p))
    st = ct.c_int(0)
    buf = ct.create_string_buffer(512)
    w_e = np.array([0.5, 0.5])
    off_e = np.array([0, 2, 2], np.uint64)
    mem_e = np.array([0, 1], np.int64)
    O.REF.ref_cursor_create(O.ptr(w_e, O.f64p), 2, 4, 9, O.ptr(off_e, O.u64p), O.ptr(mem_e, O.i64p),
                            ct.byref(st), buf, 512)
    errs["empty_class"] = (st.value, buf.value.decode())
    return {k: {"code": v[0], "msg": v[1]} for k, v in errs.items()}


def optb_fixtures():
    """OPTB stream bytes (codec.cpp:283-317) for every mode at capacity."""
    arrays = {}
    rng = np.random.default_rng(17)
    for mode in O.MODES:
        n = O.CAPACITY[mode]
        imgs = rng.integers(0, 256, size=(n, 12), dtype=np.uint8)
        out = np.zeros(4096, np.uint8)
        ln = ct.c_size_t(0)
        code, msg = ref_err(O.REF.ref_write_optb, mode, O.ptr(imgs, O.u8p), n, 3, 2, 2, O.ptr(out, O.u8p), 4096,
                            ct.byref(ln))
        assert code == 0, msg
        arrays[f"optb{mode}_in"] = imgs
        arrays[f"optb{mode}_bytes"] = out[: ln.value]
    return arrays


def main():
    if not O.ref_available():
        sys.exit("oracle/_ref/liboptb_ref.so missing: run `make -f oracle/Makefile` where /root/reference exists")
    rng = np.random.default_rng(20210503)
    cases, a1 = codec_fixtures(rng)
    smeta, a2 = stream_fixture(rng)
    sbs, a3 = sbs_fixtures()
    a4 = optb_fixtures()
    errs = error_fixtures()
    np.savez_compressed(os.path.join(OUT, "codec.npz"), **a1)
    np.savez_compressed(os.path.join(OUT, "stream.npz"), **a2)
    np.savez_compressed(os.path.join(OUT, "sbs.npz"), **a3)
    np.savez_compressed(os.path.join(OUT, "optb.npz"), **a4)
    meta = {"generator": "tests/golden/make_golden.py (reference compiled from /root/reference/proj/src)",
            "codec_cases": cases, "streams": smeta, "sbs": sbs, "errors": errs,
            "scale_bits": "0x3b808081"}
    with open(os.path.join(OUT, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1)
    for fn in ("codec.npz", "stream.npz", "sbs.npz", "optb.npz", "golden.json"):
        print(fn, os.path.getsize(os.path.join(OUT, fn)))


if __name__ == "__main__":
    main()
