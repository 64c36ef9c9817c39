"""BASELINE configurations at full size, compared element for element with
the C oracle (oracle/optb_oracle.c, pinned against the reference's own
fixtures in test_oracle.py):

* C4  ImageNet 256 x 224x224x3, exact128 (16 -> 1), fused launch -> bf16
      and -> u8, gathered rows (codec.cpp:106-208, nn.cpp:153-192);
* C3  the packing-ratio sweep n = 2 / 4 / 8 / 16 (plus the lossless and f64
      capacities) on 4096-image batches, fused and split launches;
* C5  SBS over 2^20 labels for 2300 batches, across the first lazy reshuffle
      of every class (sampler.cpp:84-104).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SCALE = float(np.float32(1.0) / np.float32(255.0))


def _bits(t, torch):
    return t.view(torch.int16).cpu().numpy().view(np.uint16) if t.element_size() == 2 else t.cpu().numpy()


@pytest.mark.parametrize("dtype", ["bfloat16", "uint8"])
def test_c4_full_size_fused_vs_oracle(pkg, oracle_mod, torch_cuda, dtype):
    torch, C, O = torch_cuda, pkg.codec, oracle_mod
    P, B = 224 * 224 * 3, 256
    rng = np.random.default_rng(44)
    pool = rng.integers(0, 256, size=(B + 37, P), dtype=np.uint8)
    idx = rng.permutation(B + 37)[:B].astype(np.int64)  # SBS-style gathered rows
    L = C.layout(1, 16, P, B, 1)
    src = torch.from_numpy(pool).cuda()
    cont, _ = C.alloc_stream(L)
    dt = getattr(torch, dtype)
    out = torch.empty((B, P), dtype=dt, device="cuda")
    C.roundtrip_dev(L, src, cont, out, row_index=torch.from_numpy(idx).cuda(), scale=SCALE)
    C.sync()
    want_c, _ = O.encode_stream(pool, idx, 1, 16, B, 1)
    got_c = cont.cpu().numpy()[: want_c.size]
    assert np.array_equal(got_c, want_c)
    kind = O.BF16 if dtype == "bfloat16" else O.U8
    want = O.decode_stream(want_c, None, 1, 16, P, B, 1, out_dtype=kind, scale=SCALE)
    assert np.array_equal(_bits(out, torch).view(want.dtype), want)
    # the split launches agree with the fused one
    out2 = torch.empty_like(out)
    C.decode_dev(L, cont, out2, scale=SCALE)
    C.sync()
    assert torch.equal(out2.view(torch.uint8), out.view(torch.uint8))


@pytest.mark.parametrize("mode,n", [(0, 2), (0, 4), (0, 8), (1, 16), (3, 9), (4, 18), (2, 6)])
@pytest.mark.parametrize("dtype", ["uint8", "float32"])
def test_c3_sweep_full_size_vs_oracle(pkg, oracle_mod, torch_cuda, mode, n, dtype):
    torch, C, O = torch_cuda, pkg.codec, oracle_mod
    P, B = 3072, 4096
    x = O.synth_pixels(3 + n, 0, B, P)
    L = C.layout(mode, n, P, B, 1)
    xs = torch.from_numpy(x).cuda()
    dt = getattr(torch, dtype)
    cont, offs = C.alloc_stream(L)
    out = torch.empty((B, P), dtype=dt, device="cuda")
    C.roundtrip_dev(L, xs, cont, out, offsets=offs, scale=SCALE)
    C.sync()
    want_c, want_o = O.encode_stream(x, None, mode, n, B, 1)
    assert np.array_equal(cont.cpu().numpy()[: want_c.size], want_c)
    if want_o is not None:
        assert np.array_equal(offs.cpu().numpy()[: want_o.size], want_o)
    kind = O.F32 if dtype == "float32" else O.U8
    want = O.decode_stream(want_c, want_o, mode, n, P, B, 1, out_dtype=kind, scale=SCALE)
    assert np.array_equal(out.cpu().numpy().view(want.dtype), want)
    # split launches
    cont2, offs2 = C.alloc_stream(L)
    C.encode_dev(L, xs, cont2, offs2)
    out2 = torch.empty_like(out)
    C.decode_dev(L, cont2, out2, offsets=offs2, scale=SCALE)
    C.sync()
    assert np.array_equal(cont2.cpu().numpy()[: want_c.size], want_c)
    assert np.array_equal(out2.cpu().numpy().view(want.dtype), want)


def test_c5_sbs_across_lazy_reshuffles_vs_oracle(pkg, oracle_mod, torch_cuda):
    """2^20 labels over 100 classes (10 485 or 10 486 per class), B = 512:
    classes 0-11 draw 6 per batch and reshuffle after ~1748 batches, the rest
    draw 5 and reshuffle after ~2097 -- 2300 batches cross both, in calls of
    different sizes (parallel Fisher-Yates + compose at m ~ 10.5 k)."""
    torch, S, O = torch_cuda, pkg.sampler, oracle_mod
    n = 1 << 20
    labels = (np.arange(n) % 100).astype(np.int32)
    p = S.plan([0.01] * 100, 512, 1234)
    offs, mem = S.class_index_dev(torch.from_numpy(labels).cuda(), 100)
    cur = S.BatchCursor.from_device_index(p, offs, mem)
    ro, rm = O.class_index(labels, 100)
    oc = O.Cursor(O.sbs_plan([0.01] * 100, 512), ro, rm, 512, 1234)
    for nb in (700, 1000, 64, 536):  # 2300 batches
        ex, cl = cur.next_dev(nb)
        rex, rcl = oc.next(nb)
        assert np.array_equal(ex.cpu().numpy(), rex), nb
        assert np.array_equal(cl.cpu().numpy(), rcl), nb
    assert cur.batches_drawn() == 2300


def test_c5_sbs_sharded_calls_vs_oracle(pkg, oracle_mod, torch_cuda):
    """The pipeline's form at C5 scale: one call per epoch (2048 batches),
    shard 3 of 8 -- the rank's batches of the global stream across the first
    lazy reshuffle."""
    torch, S, O = torch_cuda, pkg.sampler, oracle_mod
    n, G, r = 1 << 20, 8, 3
    labels = (np.arange(n) % 100).astype(np.int32)
    p = S.plan([0.01] * 100, 512, 1234)
    offs, mem = S.class_index_dev(torch.from_numpy(labels).cuda(), 100)
    cur = S.BatchCursor.from_device_index(p, offs, mem)
    ro, rm = O.class_index(labels, 100)
    oc = O.Cursor(O.sbs_plan([0.01] * 100, 512), ro, rm, 512, 1234)
    for _ in range(2):
        ex, _ = cur.next_dev(2048, shard=r, n_shards=G)
        rex, _ = oc.next(2048)
        assert np.array_equal(ex.cpu().numpy(), rex.reshape(2048, 512)[r::G].reshape(-1))
