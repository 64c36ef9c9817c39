"""Codec parity on the GPU, through the C ABI (liboptb_cuda.so).

Bar: bit-exact for packed words, parity planes and decoded pixels; float
epilogues bit-exact to the reference's binary32 / binary16 values (the
north_star allows <= 1 ulp fp32; we assert 0 ulp).  Checkers: the committed
reference fixtures (tests/golden, produced by the compiled reference) and the
C oracle (oracle/) on the same seeded inputs.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SCALE = np.float32(1.0) / np.float32(255.0)  # runner.hpp:22, bits 0x3b808081


def test_scale_bits():
    assert SCALE.view(np.uint32) == 0x3B808081


def test_golden_codec_cases(golden, pkg, torch_cuda):
    meta, arrays = golden
    C = pkg.codec
    a = arrays["codec"]
    for case in meta["codec_cases"]:
        k, mode, n = case["key"], case["mode"], case["n"]
        shape = C.ImageShape(*case["shape"])
        imgs = [C.Image(shape, a[k + "_in"][i]) for i in range(n)]
        enc = C.encode(imgs, mode)
        assert np.array_equal(enc.plane, a[k + "_plane"]), case
        if C.mode_has_offsets(mode):
            assert np.array_equal(enc.offsets, a[k + "_offs"]), case
        back = C.decode(enc)
        assert len(back) == n
        for i in range(n):
            assert np.array_equal(back[i].pixels, a[k + "_back"][i]), case


def test_reference_unit_goldens(pkg, torch_cuda):
    """test_codec.cpp:48-116 known answers."""
    C = pkg.codec
    one = C.ImageShape(1, 1, 1)
    px = lambda v: C.Image(one, np.array([v], np.uint8))  # noqa: E731
    enc = C.encode([px(3), px(5)], C.CodecMode.ExactInt64)
    assert enc.word(0) == 1283 and enc.packed.shape == (1,)
    zeros = [C.Image(C.ImageShape(2, 2, 1), np.zeros(4, np.uint8)) for _ in range(3)]
    assert all(v == 0 for v in C.encode(zeros, C.CodecMode.ExactInt128).packed.reshape(-1))
    enc = C.encode([px(7), px(4)], C.CodecMode.LosslessOffset64)
    assert enc.word(0) == 259 and enc.offset_bit(0, 0) and not enc.offset_bit(1, 0)
    back = C.decode(enc)
    assert back[0].pixels[0] == 7 and back[1].pixels[0] == 4
    e = C.EncodedBatch(C.CodecMode.ExactInt64, one, 2, np.frombuffer(np.uint64(1283).tobytes(), np.uint8).copy())
    b = C.decode(e)
    assert (b[0].pixels[0], b[1].pixels[0]) == (3, 5)
    e.n_images = 1
    e.plane = np.frombuffer(np.uint64(256).tobytes(), np.uint8).copy()
    with pytest.raises(pkg.errors.FormatError, match="exceeds range of 1 packed images"):
        C.decode(e)
    f = C.EncodedBatch(C.CodecMode.Float64Faithful, one, 1, np.frombuffer(np.float64(256.0).tobytes(), np.uint8).copy())
    with pytest.raises(pkg.errors.FormatError, match="out of range for 1 images"):
        C.decode(f)


def test_error_messages_match_reference(golden, pkg, torch_cuda):
    meta, _ = golden
    C, E = pkg.codec, pkg.errors
    errs = meta["errors"]
    one = C.ImageShape(1, 1, 1)
    for mode in range(5):
        n = C.accept_limit(mode) + 1
        imgs = [C.Image(one, np.zeros(1, np.uint8)) for _ in range(n)]
        with pytest.raises(E.CapacityError) as ei:
            C.encode(imgs, mode)
        assert str(ei.value) == errs[f"capacity_{mode}"]["msg"]
    cases = {"range_exact64": (0, np.uint64(256), 1), "range_f64": (2, np.float64(256.0), 1),
             "range_f64_neg": (2, np.float64(-1.0), 1), "range_lossless64": (3, np.uint64(1 << 14), 2)}
    for name, (mode, val, n) in cases.items():
        e = C.EncodedBatch(C.CodecMode(mode), one, n, np.frombuffer(val.tobytes(), np.uint8).copy(),
                           np.zeros(1, np.uint8) if C.mode_has_offsets(mode) else np.zeros(0, np.uint8))
        with pytest.raises(E.FormatError) as ei:
            C.decode(e)
        assert str(ei.value) == errs[name]["msg"]
    # shape validation (codec.cpp:86-93)
    imgs = [C.Image(C.ImageShape(2, 2, 1), np.zeros(4, np.uint8)), C.Image(C.ImageShape(2, 2, 3), np.zeros(12, np.uint8))]
    with pytest.raises(E.ShapeError):
        C.encode(imgs, 0)
    with pytest.raises(E.Error, match="at least one image"):
        C.encode([], 0)


def test_random_roundtrips_vs_oracle(pkg, oracle_mod, torch_cuda):
    """test_codec.cpp:158-174 style: random small shapes, n <= capacity, all modes."""
    C, O = pkg.codec, oracle_mod
    rng = np.random.default_rng(99)
    for mode in range(5):
        for _ in range(60):
            shape = C.ImageShape(int(rng.integers(1, 5)), int(rng.integers(1, 5)), int(rng.integers(1, 4)))
            n = int(rng.integers(1, C.accept_limit(mode) + 1))
            arr = rng.integers(0, 256, size=(n, shape.pixel_count()), dtype=np.uint8)
            enc = C.encode([C.Image(shape, arr[i]) for i in range(n)], mode)
            plane, offs = O.encode(arr, mode)
            assert np.array_equal(enc.plane, plane)
            if offs is not None:
                assert np.array_equal(enc.offsets, offs)
            back = np.stack([b.pixels for b in C.decode(enc)])
            assert np.array_equal(back, O.decode(plane, offs, n, shape.pixel_count(), mode))
            if n <= C.capacity(mode):
                assert np.array_equal(back, arr)


def _stream_case(pkg, torch, O, mode, per_chunk, P, B, nb, rng, gather=True, out_dtype=None):
    C = pkg.codec
    dev = torch.device("cuda", 0)
    n_ds = max(B * nb // 2, 1) if gather else B * nb
    ds = rng.integers(0, 256, size=(n_ds, P), dtype=np.uint8)
    idx = rng.integers(0, n_ds, size=B * nb).astype(np.int64) if gather else None
    L = C.layout(mode, per_chunk, P, B, nb)
    cont, offs = C.alloc_stream(L)
    ds_d = torch.from_numpy(ds).to(dev)
    idx_d = torch.from_numpy(idx).to(dev) if gather else None
    C.encode_dev(L, ds_d, cont, offs, row_index=idx_d)
    src = ds if not gather else None
    ref_cont, ref_offs = O.encode_stream(ds, idx, mode, per_chunk, B, nb)
    got = cont.cpu().numpy()[: ref_cont.size]
    assert np.array_equal(got, ref_cont), (mode, per_chunk, P, B, nb)
    if ref_offs is not None:
        assert np.array_equal(offs.cpu().numpy()[: ref_offs.size], ref_offs)
    rows = B * nb
    out = torch.empty((rows, P), dtype=torch.uint8, device=dev)
    C.decode_dev(L, cont, out, offsets=offs)
    C.sync()
    want = ds[idx] if gather else ds[:rows]
    if per_chunk <= C.capacity(mode):
        assert np.array_equal(out.cpu().numpy(), want)
    assert np.array_equal(out.cpu().numpy(), O.decode_stream(ref_cont, ref_offs, mode, per_chunk, P, B, nb))
    del src
    return L, cont, offs, ref_cont, ref_offs


def test_stream_golden_gather_and_epilogues(golden, pkg, torch_cuda):
    """runner.cpp:77-90 gather-encode + nn::decode_input (fp32) + MP fp16 tape."""
    torch = torch_cuda
    meta, arrays = golden
    C = pkg.codec
    a = arrays["stream"]
    dev = torch.device("cuda", 0)
    ds = torch.from_numpy(a["ds"]).to(dev)
    idx = torch.from_numpy(a["idx"]).to(dev)
    for s in meta["streams"]:
        mode, pc, B, nb = s["mode"], s["per_chunk"], s["batch"], s["n_batches"]
        P = 768
        L = C.layout(mode, pc, P, B, nb)
        cont, offs = C.alloc_stream(L)
        C.encode_dev(L, ds, cont, offs, row_index=idx)
        want = a[f"s{mode}_cont"]
        assert np.array_equal(cont.cpu().numpy()[: want.size], want), mode
        if C.mode_has_offsets(mode):
            wo = a[f"s{mode}_offs"]
            assert np.array_equal(offs.cpu().numpy()[: wo.size], wo), mode
        rows = B * nb
        for dt, key in ((torch.float32, "f32"), (torch.float16, "f16")):
            out = torch.empty((rows, P), dtype=dt, device=dev)
            C.decode_dev(L, cont, out, offsets=offs, scale=float(SCALE))
            C.sync()
            got = out.cpu().numpy()
            ref = a[f"s{mode}_{key}"]
            if key == "f32":
                assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), mode
            else:
                assert np.array_equal(got.view(np.uint16), ref), mode
        out = torch.empty((rows, P), dtype=torch.bfloat16, device=dev)
        C.decode_dev(L, cont, out, offsets=offs, scale=float(SCALE))
        C.sync()
        f32 = a[f"s{mode}_f32"].view(np.uint32).astype(np.uint64)
        bf = ((f32 + 0x7FFF + ((f32 >> 16) & 1)) >> 16).astype(np.uint16)
        assert np.array_equal(out.view(torch.int16).cpu().numpy().view(np.uint16), bf), mode


@pytest.mark.parametrize("mode,per_chunk,P,B,nb", [
    (0, 8, 3072, 128, 1),      # C1 CIFAR-10 exact64
    (1, 16, 3072, 512, 2),     # C2 shape, exact128
    (0, 2, 3072, 4096, 1),     # C3 sweep n=2
    (0, 4, 3072, 4096, 1),     # n=4
    (0, 8, 3072, 4096, 1),     # n=8
    (1, 16, 3072, 4096, 1),    # n=16
    (1, 16, 3072, 100, 3),     # partial last chunk (100 = 6*16 + 4)
    (0, 8, 48, 37, 5),         # P%16==0, tiny, partial chunks
    (3, 9, 3072, 512, 1),      # lossless64, P%32==0
    (4, 18, 3072, 512, 1),     # lossless128
    (2, 6, 3072, 256, 1),      # f64 exact range
    (2, 16, 3072, 64, 1),      # f64 lossy range
    (3, 9, 108, 40, 2),        # lossless, unaligned bit offsets
    (3, 5, 3072, 23, 2),       # lossless64 vector path, per_chunk < capacity, partial chunks
    (4, 11, 768, 50, 2),       # lossless128 vector path, per_chunk < capacity, partial chunks
    (4, 18, 1568, 36, 1),      # lossless128, P % 32 == 0 but odd group count per chunk
    (1, 16, 108, 40, 2),       # exact, P%16 != 0 (generic path)
    (0, 5, 27, 13, 3),         # odd everything
])
def test_stream_parity_vs_oracle(pkg, oracle_mod, torch_cuda, mode, per_chunk, P, B, nb):
    rng = np.random.default_rng(mode * 1000 + per_chunk * 7 + P + B + nb)
    _stream_case(pkg, torch_cuda, oracle_mod, mode, per_chunk, P, B, nb, rng, gather=True)
    _stream_case(pkg, torch_cuda, oracle_mod, mode, per_chunk, P, B, nb, rng, gather=False)


@pytest.mark.parametrize("mode,per_chunk,P,B,nb", [
    (1, 16, 3072, 512, 2),     # C2 shape, exact128 (fused launch)
    (0, 8, 3072, 128, 3),      # C1 exact64 (fused)
    (1, 16, 3072, 100, 3),     # partial last chunk, partial last tile
    (0, 5, 48, 37, 5),         # tiny P, per_chunk < capacity
    (2, 6, 3072, 256, 1),      # f64 narrow (fused)
    (2, 16, 3072, 64, 2),      # f64 lossy (fused, 16-image variant)
    (1, 16, 768, 1000, 1),     # items not a multiple of the warp tile
    (3, 9, 3072, 512, 1),      # lossless64 fused (P % 512 == 0)
    (4, 18, 3072, 100, 2),     # lossless128 fused, partial chunks
    (4, 11, 1024, 50, 2),      # lossless128 fused, per_chunk < capacity
    (3, 9, 768, 64, 2),        # lossless, P % 512 != 0: separate launches
    (1, 16, 108, 40, 2),       # generic path: separate launches
])
@pytest.mark.parametrize("dtype", ["uint8", "float32", "bfloat16"])
def test_roundtrip_dev_vs_oracle(pkg, oracle_mod, torch_cuda, mode, per_chunk, P, B, nb, dtype):
    """optb_roundtrip_dev (one launch where it applies) == oracle encode_stream
    + decode_stream: containers, parity planes and the decoded layer input."""
    torch, C, O = torch_cuda, pkg.codec, oracle_mod
    rng = np.random.default_rng(mode * 31 + per_chunk + P + B + nb)
    n_ds = max(B * nb // 2, 1)
    ds = rng.integers(0, 256, size=(n_ds, P), dtype=np.uint8)
    idx = rng.integers(0, n_ds, size=B * nb).astype(np.int64)
    L = C.layout(mode, per_chunk, P, B, nb)
    cont, offs = C.alloc_stream(L)
    dt = getattr(torch, dtype)
    out = torch.empty((B * nb, P), dtype=dt, device="cuda")
    C.roundtrip_dev(L, torch.from_numpy(ds).cuda(), cont, out, offsets=offs, row_index=torch.from_numpy(idx).cuda(),
                    scale=float(SCALE) if dtype != "uint8" else 1.0)
    C.sync()
    rc, ro = O.encode_stream(ds, idx, mode, per_chunk, B, nb)
    assert np.array_equal(cont.cpu().numpy()[: rc.size], rc)
    if ro is not None:
        assert np.array_equal(offs.cpu().numpy()[: ro.size], ro)
    kind = {"uint8": O.U8, "float32": O.F32, "bfloat16": O.BF16}[dtype]
    want = O.decode_stream(rc, ro, mode, per_chunk, P, B, nb, out_dtype=kind,
                           scale=float(SCALE) if dtype != "uint8" else 1.0)
    got = out.cpu()
    got = got.view(torch.int16).numpy() if dtype == "bfloat16" else got.numpy()
    assert np.array_equal(got.view(want.dtype), want)


@pytest.mark.parametrize("shape", ["deep", "wide"])
@pytest.mark.parametrize("P,B,nb", [(3072, 512, 2), (3072, 100, 3), (768, 1000, 1), (3056, 33, 5)])
def test_roundtrip_il_shapes_vs_oracle(pkg, oracle_mod, torch_cuda, monkeypatch, shape, P, B, nb):
    """exact128 -> u8 runs the interleaved kernel in its deep (5 warps x 4
    stages) or wide (8 x 2) shape by launch size; both shapes, forced, on
    small and ragged geometries (warps with 0, 1 or a partial tile) == oracle."""
    torch, C, O = torch_cuda, pkg.codec, oracle_mod
    monkeypatch.setenv("OPTB_IL_SHAPE", shape)
    rng = np.random.default_rng(P + B + nb)
    n_ds = B * nb
    ds = rng.integers(0, 256, size=(n_ds, P), dtype=np.uint8)
    idx = rng.integers(0, n_ds, size=B * nb).astype(np.int64)
    L = C.layout(1, 16, P, B, nb)
    cont, offs = C.alloc_stream(L)
    out = torch.empty((B * nb, P), dtype=torch.uint8, device="cuda")
    C.roundtrip_dev(L, torch.from_numpy(ds).cuda(), cont, out, offsets=offs, row_index=torch.from_numpy(idx).cuda())
    C.sync()
    rc, _ = O.encode_stream(ds, idx, 1, 16, B, nb)
    assert np.array_equal(cont.cpu().numpy()[: rc.size], rc)
    assert np.array_equal(out.cpu().numpy(), ds[idx])


def test_roundtrip_dev_is_one_launch(pkg, torch_cuda):
    """Vector geometries take the fused single launch -- the interleaved
    kernel, lossless included (P % 512 == 0); OPTB_IL_LOSSLESS=0 keeps the
    lossless modes on the phase-ordered kernel, with identical containers."""
    import os
    torch, C = torch_cuda, pkg.codec
    P, B, nb = 3072, 512, 2
    ds = torch.randint(0, 256, (B * nb, P), dtype=torch.uint8, device="cuda")
    for mode, pc, launches in ((1, 16, 1), (0, 8, 1), (2, 6, 1), (3, 9, 1), (4, 18, 1)):
        L = C.layout(mode, pc, P, B, nb)
        cont, offs = C.alloc_stream(L)
        out = torch.empty((B * nb, P), dtype=torch.uint8, device="cuda")
        C.sync()
        n0 = pkg._lib.launches(0)
        C.roundtrip_dev(L, ds, cont, out, offsets=offs)
        C.sync()
        assert pkg._lib.launches(0) - n0 == launches, mode
        assert C.last_roundtrip_kind() == "interleaved", mode
        if pc <= C.capacity(mode):
            assert torch.equal(out, ds)
        if mode >= 3:
            cont2, offs2 = C.alloc_stream(L)
            out2 = torch.empty_like(out)
            os.environ["OPTB_IL_LOSSLESS"] = "0"
            try:
                C.roundtrip_dev(L, ds, cont2, out2, offsets=offs2)
                C.sync()
                assert C.last_roundtrip_kind() == "phase_ordered", mode
            finally:
                os.environ.pop("OPTB_IL_LOSSLESS", None)
            assert torch.equal(cont2, cont) and torch.equal(offs2, offs) and torch.equal(out2, out), mode
    # off the vector path: two launches
    L = C.layout(1, 16, 108, 40, 2)
    cont, offs = C.alloc_stream(L)
    C.roundtrip_dev(L, torch.randint(0, 256, (80, 108), dtype=torch.uint8, device="cuda"), cont,
                    torch.empty((80, 108), dtype=torch.uint8, device="cuda"))
    C.sync()
    assert C.last_roundtrip_kind() == "split"


@pytest.mark.parametrize("mode,pc", [(3, 9), (4, 18), (2, 6), (0, 8), (1, 16)])
def test_roundtrip_dev_full_size_properties(pkg, torch_cuda, mode, pc):
    """C3-sized streams (65 536 CIFAR images, > L2): the fused launch's
    containers and parity planes equal optb_encode_dev's, and the decoded rows
    are the gathered rows (lossless at capacity) -- with every warp in either
    phase at once, so the phases' shared-memory rings must not overlap."""
    torch, C = torch_cuda, pkg.codec
    P, B, nb = 3072, 4096, 16
    rows = B * nb
    ds = torch.randint(0, 256, (rows, P), dtype=torch.uint8, device="cuda")
    idx = torch.randperm(rows, device="cuda")
    L = C.layout(mode, pc, P, B, nb)
    cont, offs = C.alloc_stream(L)
    out = torch.empty((rows, P), dtype=torch.uint8, device="cuda")
    C.roundtrip_dev(L, ds, cont, out, offsets=offs, row_index=idx)
    C.sync()
    assert torch.equal(out, ds[idx])
    cont2, offs2 = C.alloc_stream(L)
    C.encode_dev(L, ds, cont2, offs2, row_index=idx)
    C.sync()
    nbytes = C.container_bytes(L)
    assert torch.equal(cont[:nbytes], cont2[:nbytes])
    if offs is not None:
        ob = C.offsets_bytes(L)
        assert torch.equal(offs[:ob], offs2[:ob])


@pytest.mark.parametrize("mode,pc,P,B,nb,dtype", [
    (1, 16, 3056, 4001, 16, "uint8"),    # deep interleaved shape: partial chunks, partial last tile
    (1, 16, 3072, 4096, 16, "bfloat16"),  # wide shape, float epilogue, full size
    (0, 8, 3056, 4001, 16, "uint8"),
    (2, 16, 3056, 4001, 16, "uint8"),
])
def test_roundtrip_dev_full_size_ragged(pkg, torch_cuda, mode, pc, P, B, nb, dtype):
    """Interleaved round trip at full size with ragged geometry (P / 16 odd,
    a one-image last chunk per batch, a partial last warp tile): the fused
    launch's containers equal optb_encode_dev's and its decoded rows equal
    optb_decode_dev's on those containers (the split launches are checked
    against the oracle above)."""
    torch, C = torch_cuda, pkg.codec
    rows = B * nb
    ds = torch.randint(0, 256, (rows, P), dtype=torch.uint8, device="cuda")
    idx = torch.randint(0, rows, (rows,), device="cuda")
    L = C.layout(mode, pc, P, B, nb)
    dt = getattr(torch, dtype)
    sc = float(SCALE) if dtype != "uint8" else 1.0
    cont, offs = C.alloc_stream(L)
    out = torch.empty((rows, P), dtype=dt, device="cuda")
    C.roundtrip_dev(L, ds, cont, out, offsets=offs, row_index=idx, scale=sc)
    cont2, offs2 = C.alloc_stream(L)
    C.encode_dev(L, ds, cont2, offs2, row_index=idx)
    out2 = torch.empty_like(out)
    C.decode_dev(L, cont2, out2, offsets=offs2, scale=sc)
    C.sync()
    nbytes = C.container_bytes(L)
    assert torch.equal(cont[:nbytes], cont2[:nbytes])
    assert torch.equal(out.view(torch.uint8), out2.view(torch.uint8))
    if dtype == "uint8" and pc <= C.capacity(mode):
        assert torch.equal(out, ds[idx])


@pytest.mark.parametrize("mode", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("dtype", ["float32", "float16", "bfloat16"])
def test_float_epilogue_vs_oracle(pkg, oracle_mod, torch_cuda, mode, dtype):
    torch = torch_cuda
    C, O = pkg.codec, oracle_mod
    rng = np.random.default_rng(7 + mode)
    P, B, nb = 3072, 64, 2
    pc = C.capacity(mode)
    L, cont, offs, rc, ro = _stream_case(pkg, torch, O, mode, pc, P, B, nb, rng)
    dt = getattr(torch, dtype)
    out = torch.empty((B * nb, P), dtype=dt, device="cuda")
    C.decode_dev(L, cont, out, offsets=offs, scale=float(SCALE))
    C.sync()
    kind = {"float32": O.F32, "float16": O.F16, "bfloat16": O.BF16}[dtype]
    ref = O.decode_stream(rc, ro, mode, pc, P, B, nb, out_dtype=kind, scale=float(SCALE))
    got = out.cpu()
    got = got.numpy().view(np.uint32) if dtype == "float32" else got.view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(got, ref.view(got.dtype))


@pytest.mark.parametrize("dtype", ["float32", "float16", "bfloat16"])
def test_epilogue_scale_edges_vs_oracle(pkg, oracle_mod, torch_cuda, dtype):
    """The float epilogue's fast form (FFMA identity for 0 < s < 2^100) and its
    plain-FMUL fallback agree bit for bit with the reference product on edge
    scales: negative, +-0, subnormal, overflowing, the 2^100 boundary; also
    per-class tables mixing both forms."""
    torch, C, O = torch_cuda, pkg.codec, oracle_mod
    rng = np.random.default_rng(17)
    P, B, nb = 768, 32, 2
    L, cont, offs, rc, ro = _stream_case(pkg, torch, O, 1, 16, P, B, nb, rng)
    dt = getattr(torch, dtype)
    kind = {"float32": O.F32, "float16": O.F16, "bfloat16": O.BF16}[dtype]
    f32 = lambda v: float(np.float32(v))  # noqa: E731
    scales = [f32(1 / 255), -f32(1 / 255), 0.0, -0.0, f32(1e-42), f32(3e38), f32(2.0 ** 100),
              float(np.nextafter(np.float32(2.0 ** 100), np.float32(0))), f32(0.75), f32(1.0)]
    for sc in scales:
        out = torch.empty((B * nb, P), dtype=dt, device="cuda")
        C.decode_dev(L, cont, out, scale=sc)
        C.sync()
        want = O.decode_stream(rc, ro, 1, 16, P, B, nb, out_dtype=kind, scale=sc)
        got = out.cpu()
        got = got.numpy().view(np.uint32) if dtype == "float32" else got.view(torch.int16).numpy().view(np.uint16)
        assert np.array_equal(got, want.view(got.dtype)), sc
    row_class = rng.integers(0, len(scales), size=B * nb).astype(np.int32)
    cs = np.array(scales, np.float32)
    cb = rng.uniform(-2, 2, len(scales)).astype(np.float32)
    out = torch.empty((B * nb, P), dtype=dt, device="cuda")
    C.decode_dev(L, cont, out, class_scale=torch.from_numpy(cs).cuda(), class_bias=torch.from_numpy(cb).cuda(),
                 row_class=torch.from_numpy(row_class).cuda())
    C.sync()
    want = O.decode_stream(rc, ro, 1, 16, P, B, nb, out_dtype=kind, scale=1.0, class_scale=cs, class_bias=cb,
                           row_class=row_class)
    got = out.cpu()
    got = got.numpy().view(np.uint32) if dtype == "float32" else got.view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(got, want.view(got.dtype))


def test_per_class_epilogue(pkg, oracle_mod, torch_cuda):
    """Per-class preprocessing table (the GPU form of sampler.hpp:39-40's hook):
    identity table == plain epilogue; random table == oracle."""
    torch = torch_cuda
    C, O = pkg.codec, oracle_mod
    rng = np.random.default_rng(3)
    P, B, nb = 3072, 96, 2
    L, cont, offs, rc, ro = _stream_case(pkg, torch, O, 1, 16, P, B, nb, rng)
    rows = B * nb
    row_class = rng.integers(0, 10, size=rows).astype(np.int32)
    rc_d = torch.from_numpy(row_class).cuda()
    plain = torch.empty((rows, P), dtype=torch.float32, device="cuda")
    C.decode_dev(L, cont, plain, scale=float(SCALE))
    ident = torch.empty_like(plain)
    C.decode_dev(L, cont, ident, class_scale=torch.full((10,), float(SCALE), device="cuda"),
                 class_bias=torch.zeros(10, device="cuda"), row_class=rc_d)
    C.sync()
    assert torch.equal(plain.view(torch.int32), ident.view(torch.int32))
    cs = rng.uniform(0.001, 0.01, 10).astype(np.float32)
    cb = rng.uniform(-1, 1, 10).astype(np.float32)
    got = torch.empty_like(plain)
    C.decode_dev(L, cont, got, class_scale=torch.from_numpy(cs).cuda(), class_bias=torch.from_numpy(cb).cuda(),
                 row_class=rc_d)
    C.sync()
    ref = O.decode_stream(rc, ro, 1, 16, P, B, nb, out_dtype=O.F32, scale=1.0, class_scale=cs, class_bias=cb,
                          row_class=row_class)
    assert np.array_equal(got.cpu().numpy().view(np.uint32), ref.view(np.uint32))


def test_unaligned_pointers_and_strides(pkg, oracle_mod, torch_cuda):
    """Generic path: dataset rows at an odd stride and 1-byte-misaligned base."""
    torch = torch_cuda
    C, O = pkg.codec, oracle_mod
    rng = np.random.default_rng(11)
    P, B, nb, stride = 3072, 32, 2, 3077
    raw = torch.from_numpy(rng.integers(0, 256, size=(64 * stride + 1,), dtype=np.uint8)).cuda()
    ds = raw[1:].view(64, stride)[:, :P]
    idx = rng.integers(0, 64, size=B * nb).astype(np.int64)
    L = C.layout(0, 8, P, B, nb)
    cont, offs = C.alloc_stream(L)
    C.encode_dev(L, ds, cont, offs, row_index=torch.from_numpy(idx).cuda())
    ref, _ = O.encode_stream(ds.cpu().numpy(), idx, 0, 8, B, nb)
    assert np.array_equal(cont.cpu().numpy()[: ref.size], ref)
    big = torch.zeros((B * nb, P + 5), dtype=torch.uint8, device="cuda")
    C.decode_dev(L, cont, big[:, :P], offsets=offs)
    C.sync()
    assert np.array_equal(big[:, :P].cpu().numpy(), ds.cpu().numpy()[idx])
    assert int(big[:, P:].sum()) == 0


def test_f64_decode_arbitrary_containers_vs_oracle(pkg, oracle_mod, torch_cuda):
    """f64 decode on arbitrary (also fractional, huge and lossy) binary64
    containers equals the oracle's fmod peel (codec.cpp:159-178)."""
    torch = torch_cuda
    C, O = pkg.codec, oracle_mod
    rng = np.random.default_rng(64)
    for n in (1, 3, 6, 7, 9, 12, 16):
        P = 96
        vals = rng.random(P) * 2.0 ** rng.integers(0, 8 * n + 1, size=P)
        vals[::7] = np.floor(vals[::7])
        vals[5] = -0.0
        if n > 6:  # lossy range: no range check, huge / infinite sums peel too
            vals[3], vals[4] = np.inf, 1e300
        plane = vals.astype(np.float64).view(np.uint8)
        try:
            want = O.decode(plane, None, n, P, O.F64)
        except O.OracleError:
            want = None
        L = C.layout(2, n, P, n, 1)
        out = torch.empty((n, P), dtype=torch.uint8, device="cuda")
        C.decode_dev(L, torch.from_numpy(plane.copy()).cuda(), out)
        if want is None:
            with pytest.raises(pkg.errors.FormatError):
                C.sync()
        else:
            C.sync()
            assert np.array_equal(out.cpu().numpy(), want), n


def test_device_range_check_reports_first_chunk(pkg, torch_cuda):
    """A corrupted container in a multi-chunk stream -> FormatError naming the
    n of the first offending chunk (codec.cpp:191-194; nn.cpp decodes in order)."""
    torch = torch_cuda
    C, E = pkg.codec, pkg.errors
    P, B = 48, 20  # exact64, per_chunk 8 -> chunks of 8, 8, 4 per batch
    L = C.layout(0, 8, P, B, 2)
    cont = torch.zeros(C.container_bytes(L), dtype=torch.uint8, device="cuda")
    out = torch.empty((B * 2, P), dtype=torch.uint8, device="cuda")
    C.decode_dev(L, cont, out)
    C.sync()
    cont.view(torch.int64)[P * 2 + 5] = 1 << 40  # chunk 2 (n=4): byte 5 set
    cont.view(torch.int64)[P * 5 + 1] = 1 << 40  # chunk 5 (n=4) as well
    C.decode_dev(L, cont, out)
    with pytest.raises(E.FormatError, match="^decode: container value exceeds range of 4 packed images$"):
        C.sync()
    C.sync()  # latch cleared


def test_full_size_c4_bf16_roundtrip(pkg, torch_cuda):
    """BASELINE C4 at full size (256 x 224x224x3, exact128, bf16 epilogue):
    size-independent properties -- decode(encode(x)) == x and the bf16 output
    equals the 256-entry table RNE_bf16(RN(q * 1/255)) indexed by x."""
    torch = torch_cuda
    C = pkg.codec
    P, B = 224 * 224 * 3, 256
    g = torch.Generator(device="cuda").manual_seed(4)
    x = torch.randint(0, 256, (B, P), dtype=torch.uint8, device="cuda", generator=g)
    L = C.layout(1, 16, P, B, 1)
    cont, _ = C.alloc_stream(L)
    C.encode_dev(L, x, cont)
    back = torch.empty_like(x)
    C.decode_dev(L, cont, back)
    out = torch.empty((B, P), dtype=torch.bfloat16, device="cuda")
    C.decode_dev(L, cont, out, scale=float(SCALE))
    C.sync()
    assert torch.equal(back, x)
    table = (torch.arange(256, dtype=torch.float32) * torch.tensor(SCALE)).to(torch.bfloat16).cuda()
    assert torch.equal(out.view(torch.int16), table[x.long()].view(torch.int16))
    # container = byte transpose of the raw batch (test_codec.cpp:218-230)
    w = cont.view(16, P, 16)  # [chunk][pixel][image byte]
    assert torch.equal(w[3, :, 5], x[3 * 16 + 5])


def test_edge_values_and_empty(pkg, oracle_mod, torch_cuda):
    torch = torch_cuda
    C, O = pkg.codec, oracle_mod
    for mode in range(5):
        for v in (0, 255):
            n = C.capacity(mode)
            arr = np.full((n, 3072), v, np.uint8)
            L = C.layout(mode, n, 3072, n, 1)
            cont, offs = C.encode_host(L, arr)
            plane, po = O.encode(arr, mode)
            assert np.array_equal(cont, plane)
            if po is not None:
                assert np.array_equal(offs[: po.size], po)
            assert np.array_equal(C.decode_host(L, cont, offs), arr)
    # zero batches: no-op, no error
    L = C.layout(1, 16, 3072, 512, 0)
    cont = torch.zeros(16, dtype=torch.uint8, device="cuda")
    C.encode_dev(L, torch.zeros((1, 3072), dtype=torch.uint8, device="cuda"), cont)
    C.sync()


def test_host_api_multi_slice(pkg, oracle_mod, torch_cuda):
    """optb_encode_host / optb_decode_host over a stream larger than one
    staging slice (pinned and pageable host buffers)."""
    torch = torch_cuda
    C, O = pkg.codec, oracle_mod
    rng = np.random.default_rng(5)
    P, B, nb = 3072, 512, 24  # 37.7 MB > one 32 MiB slice
    imgs = rng.integers(0, 256, size=(B * nb, P), dtype=np.uint8)
    L = C.layout(1, 16, P, B, nb)
    cont, _ = C.encode_host(L, imgs)
    ref, _ = O.encode_stream(imgs, None, 1, 16, B, nb)
    assert np.array_equal(cont, ref)
    pinned = torch.from_numpy(cont).pin_memory().numpy()
    back = C.decode_host(L, pinned)
    assert np.array_equal(back, imgs)
    f = C.decode_host(L, cont, dtype=C.F32, scale=float(SCALE))
    assert np.array_equal(f, imgs.astype(np.float32) * SCALE)
    # ImageNet-shaped: slices inside one batch
    P2, B2 = 224 * 224 * 3, 64
    im2 = rng.integers(0, 256, size=(B2, P2), dtype=np.uint8)
    L2 = C.layout(1, 16, P2, B2, 1)
    c2, _ = C.encode_host(L2, im2)
    assert np.array_equal(C.decode_host(L2, c2), im2)
