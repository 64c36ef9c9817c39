"""CPU tests: the oracle (oracle/optb_oracle.c) pinned against the reference.

1. every committed golden fixture (produced by the reference compiled from
   its own sources, tests/golden/make_golden.py) and the reference test
   suites' known answers (test_codec.cpp, test_sampler.cpp, test_tensor.cpp);
2. randomized differential runs against oracle/_ref (the compiled reference)
   when it is present.
"""
import numpy as np
import pytest


def test_codec_goldens(golden, oracle_mod):
    meta, arrays = golden
    O = oracle_mod
    a = arrays["codec"]
    for case in meta["codec_cases"]:
        k, mode, n = case["key"], case["mode"], case["n"]
        imgs = a[k + "_in"]
        plane, offs = O.encode(imgs, mode)
        assert np.array_equal(plane, a[k + "_plane"]), case
        if O.HAS_OFFSETS[mode]:
            assert np.array_equal(offs, a[k + "_offs"]), case
        back = O.decode(plane, offs, n, imgs.shape[1], mode)
        assert np.array_equal(back, a[k + "_back"]), case


def test_reference_known_answers(oracle_mod):
    O = oracle_mod
    plane, _ = O.encode(np.array([[3], [5]], np.uint8), O.EXACT64)
    assert int(plane.view(np.uint64)[0]) == 1283  # test_codec.cpp:48-54
    plane, offs = O.encode(np.array([[7], [4]], np.uint8), O.LOSSLESS64)
    assert int(plane.view(np.uint64)[0]) == 259 and offs[0] == 0x01  # :74-84
    assert O.decode(plane, offs, 2, 1, O.LOSSLESS64)[:, 0].tolist() == [7, 4]
    assert O.decode(np.frombuffer(np.uint64(1283).tobytes(), np.uint8), None, 2, 1, O.EXACT64)[:, 0].tolist() == [3, 5]
    with pytest.raises(O.OracleError, match="exceeds range of 1 packed"):
        O.decode(np.frombuffer(np.uint64(256).tobytes(), np.uint8), None, 1, 1, O.EXACT64)
    with pytest.raises(O.OracleError, match="out of range for 1 images"):
        O.decode(np.frombuffer(np.float64(256.0).tobytes(), np.uint8), None, 1, 1, O.F64)
    # roundtrip_error: f64 lossy at 16 (test_codec.cpp:193-202), exact within capacity
    rng = np.random.default_rng(5)
    assert O.roundtrip_error(rng.integers(0, 256, (16, 16), dtype=np.uint8), O.F64).max() > 0
    for mode in O.MODES:
        assert O.roundtrip_error(rng.integers(0, 256, (O.CAPACITY[mode], 9), dtype=np.uint8), mode).max() == 0


def test_capacity_messages(golden, oracle_mod):
    meta, _ = golden
    O = oracle_mod
    for mode in O.MODES:
        n = O.ACCEPT[mode] + 1
        with pytest.raises(O.OracleError) as ei:
            O.encode(np.zeros((n, 1), np.uint8), mode)
        assert str(ei.value) == meta["errors"][f"capacity_{mode}"]["msg"]
        assert ei.value.code == meta["errors"][f"capacity_{mode}"]["code"]


def test_stream_goldens(golden, oracle_mod):
    meta, arrays = golden
    O = oracle_mod
    a = arrays["stream"]
    scale = float(np.float32(1.0) / np.float32(255.0))
    for s in meta["streams"]:
        mode, pc, B, nb = s["mode"], s["per_chunk"], s["batch"], s["n_batches"]
        cont, offs = O.encode_stream(a["ds"], a["idx"], mode, pc, B, nb)
        assert np.array_equal(cont, a[f"s{mode}_cont"]), mode
        if offs is not None:
            assert np.array_equal(offs, a[f"s{mode}_offs"]), mode
        f32 = O.decode_stream(cont, offs, mode, pc, 768, B, nb, out_dtype=O.F32, scale=scale)
        assert np.array_equal(f32.view(np.uint32), a[f"s{mode}_f32"].view(np.uint32)), mode
        f16 = O.decode_stream(cont, offs, mode, pc, 768, B, nb, out_dtype=O.F16, scale=scale)
        assert np.array_equal(f16, a[f"s{mode}_f16"]), mode


def test_float_to_half_exhaustive_on_pixel_domain(oracle_mod):
    """test_tensor.cpp:20-73 semantics restricted to the values the decode
    epilogue produces: float_to_half(q * 1/255) == numpy RNE for all q."""
    O = oracle_mod
    s = np.float32(1.0) / np.float32(255.0)
    for q in range(256):
        v = np.float32(q) * s
        assert O.float_to_half(float(v)) == np.float16(v).view(np.uint16)
        f = np.array([v], np.float32).view(np.uint32).astype(np.uint64)[0]
        assert O.float_to_bf16(float(v)) == int((f + 0x7FFF + ((f >> 16) & 1)) >> 16)


def test_sbs_goldens(golden, oracle_mod):
    meta, arrays = golden
    O = oracle_mod
    a = arrays["sbs"]
    labels = (np.arange(50000) % 100).astype(np.int32)
    off, mem = O.class_index(labels, 100)
    cur = O.Cursor(O.sbs_plan([0.01] * 100, 512), off, mem, 512, 1234)
    ex, cl = cur.next(300)
    assert np.array_equal(ex, a["c2_examples"])
    assert np.array_equal(cl, a["c2_classes"].astype(np.int32))
    g = meta["sbs"]["skew"]
    off, mem = O.class_index(a["skew_labels"], 3)
    cur = O.Cursor(O.sbs_plan(g["weights"], 16), off, mem, 16, g["seed"])
    assert np.array_equal(cur.next(g["batches"])[0], a["skew_examples"])
    for case in ("rej_a", "rej_b"):
        g = meta["sbs"][case]
        cur = O.Cursor(np.array(g["counts"], np.uint64), np.array(g["class_offsets"], np.uint64),
                       a["rej_a_members"], g["batch"], g["seed"])
        assert np.array_equal(cur.next(g["batches"])[0], a[f"{case}_examples"]), case
    for name, p in meta["sbs"]["plans"].items():
        assert O.sbs_plan(p["weights"], p["batch"]).tolist() == p["counts"], name


def test_sampler_messages(golden, oracle_mod):
    meta, _ = golden
    O = oracle_mod
    errs = meta["errors"]
    for name, (w, b) in {"neg": ([0.7, -0.2, 0.5], 8), "sum": ([0.5, 0.4], 8), "batch0": ([0.5, 0.5], 0)}.items():
        with pytest.raises(O.OracleError) as ei:
            O.sbs_plan(w, b)
        assert str(ei.value) == errs[f"plan_{name}"]["msg"]
    with pytest.raises(O.OracleError) as ei:
        O.class_index(np.array([0, 3], np.int32), 3)
    assert str(ei.value) == errs["label_range"]["msg"]
    with pytest.raises(O.OracleError) as ei:
        O.Cursor(np.array([2, 2], np.uint64), np.array([0, 2, 2], np.uint64), np.array([0, 1]), 4, 9)
    assert str(ei.value) == errs["empty_class"]["msg"]


def test_splitmix_known_values(oracle_mod):
    """seed 0 gives e220a8397b1dcdaf, 6e789e6aa1b965f4, 06c45d188009454f."""
    import ctypes as ct
    O = oracle_mod
    st = ct.c_uint64(0)
    vals = [O.C.orc_next_u64(ct.byref(st)) for _ in range(3)]
    assert vals == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


@pytest.mark.skipif(not __import__("oracle").ref_available(), reason="oracle/_ref not built")
def test_differential_vs_compiled_reference(oracle_mod):
    """Randomized: oracle == reference for all modes, shapes, n (incl. lossy f64)."""
    O = oracle_mod
    rng = np.random.default_rng(0xACCE551)
    for mode in O.MODES:
        for _ in range(150):
            P = int(rng.integers(1, 200))
            n = int(rng.integers(1, O.ACCEPT[mode] + 1))
            imgs = rng.integers(0, 256, size=(n, P), dtype=np.uint8)
            if rng.random() < 0.2:
                imgs[:] = rng.choice([0, 255])
            p1, o1 = O.encode(imgs, mode)
            p2, o2 = O.ref_encode(imgs, mode)
            assert np.array_equal(p1, p2)
            if o1 is not None:
                assert np.array_equal(o1, o2)
            assert np.array_equal(O.decode(p1, o1, n, P, mode), O.ref_decode(p2, o2, n, P, mode))
    # random corrupt containers: same accept/reject decision and message
    for _ in range(300):
        mode = int(rng.integers(0, 5))
        n = int(rng.integers(1, O.ACCEPT[mode] + 1))
        P = int(rng.integers(1, 8))
        plane = rng.integers(0, 256, size=P * O.WC[mode], dtype=np.uint8)
        if mode == O.F64:
            plane = (rng.random(P) * 2.0 ** rng.integers(0, 130) - rng.integers(0, 2)).astype(np.float64).view(np.uint8)
        offs = rng.integers(0, 256, size=(n * P + 7) // 8, dtype=np.uint8) if O.HAS_OFFSETS[mode] else None
        r1 = r2 = None
        try:
            b1 = O.decode(plane, offs, n, P, mode)
        except O.OracleError as e:
            r1 = str(e)
        try:
            b2 = O.ref_decode(plane, offs, n, P, mode)
        except O.OracleError as e:
            r2 = str(e)
        assert r1 == r2
        if r1 is None:
            assert np.array_equal(b1, b2)
