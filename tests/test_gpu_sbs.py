"""Selective batch sampling parity on the GPU, through the C ABI.

Bar: the example index sequence is identical to the reference BatchCursor's
(sampler.cpp:67-104) -- checked against committed reference fixtures
(including two engineered rejection-sampling events) and the C oracle.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cursor(pkg, weights, batch, seed, labels=None, by_class=None, n_classes=None):
    S = pkg.sampler
    p = S.plan(weights, batch, seed)
    if by_class is None:
        by_class = S.ClassIndex.from_labels(labels, n_classes or len(weights)).by_class
    return S.BatchCursor(p, S.ClassIndex(by_class))


def test_plan_counts_golden(golden, pkg, torch_cuda):
    meta, _ = golden
    for name, g in meta["sbs"]["plans"].items():
        assert pkg.sampler.plan(g["weights"], g["batch"], 1).counts == g["counts"], name


def test_plan_validation_messages(golden, pkg, torch_cuda):
    meta, _ = golden
    S, E = pkg.sampler, pkg.errors
    errs = meta["errors"]
    for name, (w, b) in {"neg": ([0.7, -0.2, 0.5], 8), "sum": ([0.5, 0.4], 8), "batch0": ([0.5, 0.5], 0)}.items():
        with pytest.raises(E.Error) as ei:
            S.plan(w, b, 1)
        assert str(ei.value) == errs[f"plan_{name}"]["msg"]
    with pytest.raises(E.Error):
        S.plan([], 8, 1)
    S.plan([0.5, 0.5 + 5e-10], 8, 1)  # within tolerance (test_sampler.cpp:63)


def test_class_index_vs_oracle(pkg, oracle_mod, torch_cuda, golden):
    S = pkg.sampler
    rng = np.random.default_rng(1)
    for n, C in [(6, 3), (1000, 7), (50000, 100), (300000, 1000), (5000, 1)]:
        labels = rng.integers(0, C, size=n).astype(np.int32)
        offs, mem = S.class_index_dev(labels, C)
        ro, rm = oracle_mod.class_index(labels, C)
        assert np.array_equal(offs.cpu().numpy().astype(np.uint64), ro)
        assert np.array_equal(mem.cpu().numpy(), rm)
    idx = S.ClassIndex.from_labels([0, 1, 0, 2, 1, 0], 3)  # test_sampler.cpp:66-73
    assert idx.by_class == [[0, 2, 5], [1, 4], [3]]
    with pytest.raises(pkg.errors.Error) as ei:
        S.ClassIndex.from_labels([0, 3], 3)
    assert str(ei.value) == golden[0]["errors"]["label_range"]["msg"]


def test_c2_stream_golden(golden, pkg, torch_cuda):
    """CIFAR-100 (labels e % 100, N=50 000), uniform weights, B=512, seed 1234:
    300 batches, drawn in calls of varying size (generation pool across calls)."""
    torch = torch_cuda
    meta, arrays = golden
    a = arrays["sbs"]
    labels = (np.arange(50000) % 100).astype(np.int32)
    S = pkg.sampler
    p = S.plan([0.01] * 100, 512, 1234)
    offs, mem = S.class_index_dev(labels, 100)
    cur = S.BatchCursor.from_device_index(p, offs, mem)
    got = []
    for n in (1, 7, 97, 3, 150, 42):
        ex, cl = cur.next_dev(n)
        got.append(ex.cpu().numpy())
        if n == 97:
            assert np.array_equal(cl.cpu().numpy(), np.repeat(np.arange(100), p.counts).astype(np.int32).tolist() * 97)
    got = np.concatenate(got)
    assert np.array_equal(got, a["c2_examples"])
    assert list(got[:8]) == [49700, 4400, 38800, 38700, 5000, 25800, 33401, 41901]  # SURVEY §8(a) probe
    torch.cuda.synchronize()


@pytest.mark.parametrize("case", ["skew", "rej_a", "rej_b"])
@pytest.mark.parametrize("serial", [False, True])
def test_small_streams_golden(golden, pkg, torch_cuda, case, serial):
    meta, arrays = golden
    a = arrays["sbs"]
    g = meta["sbs"][case]
    S = pkg.sampler
    if case == "skew":
        cur = _cursor(pkg, g["weights"], g["batch"], g["seed"], labels=a["skew_labels"])
        want = a["skew_examples"]
    else:
        o = g["class_offsets"]
        m = a["rej_a_members"].tolist()
        by_class = [m[o[c]:o[c + 1]] for c in range(3)]
        cur = S.BatchCursor(S.plan(g["weights"], g["batch"], g["seed"]), S.ClassIndex(by_class))
        want = a[f"{case}_examples"]
    cur.set_force_serial(serial)
    got = np.concatenate([cur.next_arrays(1)[0] if i % 2 else cur.next_arrays(3)[0] for i in range(g["batches"] // 4 * 2)]
                         + [cur.next_arrays(g["batches"] - (g["batches"] // 4) * 4)[0]])
    assert np.array_equal(got, want[: got.size])


def test_stream_vs_oracle_random(pkg, oracle_mod, torch_cuda):
    """Random class sizes (incl. size-1 and empty classes), skewed weights."""
    S, O = pkg.sampler, oracle_mod
    rng = np.random.default_rng(2024)
    for trial in range(6):
        C = int(rng.integers(2, 40))
        sizes = rng.integers(0, 60, size=C)
        sizes[0] = max(sizes[0], 1)
        w = rng.random(C) * (sizes > 0)
        w = w / w.sum()
        B = int(rng.integers(1, 200))
        counts = O.sbs_plan(w, B)
        by_class, e = [], 0
        for c in range(C):
            by_class.append(list(range(e, e + int(sizes[c]))))
            e += int(sizes[c])
        seed = int(rng.integers(0, 2**63))
        off = np.zeros(C + 1, np.uint64)
        off[1:] = np.cumsum(sizes)
        mem = np.arange(e, dtype=np.int64)
        oc = O.Cursor(counts, off, mem, B, seed)
        cur = S.BatchCursor(S.SamplerPlan(list(w), B, [int(x) for x in counts], seed), S.ClassIndex(by_class))
        for n in (1, 5, 13):
            ex, cl = cur.next_arrays(n)
            rex, rcl = oc.next(n)
            assert np.array_equal(ex, rex), trial
            assert np.array_equal(cl, rcl), trial


def test_sharded_union_equals_stream(pkg, torch_cuda):
    """optb_sbs_next_dev(shard, n_shards): G independent cursors (one per
    simulated rank) reproduce the single stream with no communication."""
    S = pkg.sampler
    labels = (np.arange(20000) % 10).astype(np.int32)
    p = S.plan([0.1] * 10, 128, 77)
    offs, mem = S.class_index_dev(labels, 10)
    single = S.BatchCursor.from_device_index(p, offs, mem)
    full = np.concatenate([single.next_dev(40)[0].cpu().numpy(), single.next_dev(40)[0].cpu().numpy()])
    full = full.reshape(80, 128)
    for G in (2, 4, 8):
        parts = {}
        for r in range(G):
            cur = S.BatchCursor.from_device_index(p, offs, mem)
            mine = []
            for call in range(2):
                ex, _ = cur.next_dev(40, shard=r, n_shards=G)
                mine.append(ex.cpu().numpy().reshape(-1, 128))
            parts[r] = mine
        for call in range(2):
            for r in range(G):
                rows = full[call * 40 + r: (call + 1) * 40: G]
                assert np.array_equal(parts[r][call], rows), (G, r, call)


def test_hook_and_composition(pkg, torch_cuda):
    """test_sampler.cpp:75-147: composition, hook order, seeds, coverage, errors."""
    S, E = pkg.sampler, pkg.errors
    two = S.ClassIndex([[0, 1, 2], [3, 4]])
    cur = S.BatchCursor(S.plan([0.5, 0.5], 4, 9), two)
    for _ in range(20):
        batch = cur.next()
        assert len(batch) == 4
        assert sum(d.cls == 0 for d in batch) == 2
        assert all((d.example <= 2) == (d.cls == 0) for d in batch)
    calls = []
    cur = S.BatchCursor(S.plan([0.5, 0.5], 4, 9), two)
    cur.set_preprocess_hook(lambda c, e: calls.append((c, e)))
    batch = cur.next()
    assert calls == [(d.cls, d.example) for d in batch]

    def stream(seed):
        c = S.BatchCursor(S.plan([0.5, 0.5], 4, seed), S.ClassIndex([[0, 1, 2], [3, 4]]))
        return [d.example for _ in range(10) for d in c.next()]
    assert stream(42) == stream(42) and stream(42) != stream(43)
    cov = S.BatchCursor(S.plan([1.0], 2, 5), S.ClassIndex([[10, 11, 12, 13, 14, 15, 16]]))
    assert len({d.example for _ in range(4) for d in cov.next()}) == 7
    with pytest.raises(E.Error, match="class 1"):
        S.BatchCursor(S.plan([0.5, 0.5], 4, 9), S.ClassIndex([[0, 1], []]))
    S.BatchCursor(S.plan([1.0, 0.0], 4, 9), S.ClassIndex([[0, 1], []]))
    with pytest.raises(E.Error, match="index has 2 classes, plan has 3"):
        S.BatchCursor(S.plan([0.5, 0.25, 0.25], 4, 9), two)


def test_c5_scale_stream_vs_oracle(pkg, oracle_mod, torch_cuda):
    """C5-sized labels (2^20 examples, 100 classes), B=512: 64 batches."""
    S, O = pkg.sampler, oracle_mod
    n = 1 << 20
    labels = (np.arange(n) % 100).astype(np.int32)
    p = S.plan([0.01] * 100, 512, 1234)
    offs, mem = S.class_index_dev(labels, 100)
    cur = S.BatchCursor.from_device_index(p, offs, mem)
    ex, _ = cur.next_dev(64)
    ro, rm = O.class_index(labels, 100)
    oc = O.Cursor(O.sbs_plan([0.01] * 100, 512), ro, rm, 512, 1234)
    rex, _ = oc.next(64)
    assert np.array_equal(ex.cpu().numpy(), rex)


@pytest.mark.parametrize("case", ["rej_a", "rej_b"])
def test_rejection_with_calls_in_flight(golden, pkg, torch_cuda, case):
    """Device draws enqueued back to back with no host synchronisation: when a
    call hits a rejection, the calls already enqueued behind it were planned
    from the host's (now stale) chain walk -- the device detects the mismatch
    and redoes them serially from its own chain state, and the host resyncs
    its mirror once it sees the divergence.  The stream equals the reference's."""
    torch = torch_cuda
    meta, arrays = golden
    a = arrays["sbs"]
    g = meta["sbs"][case]
    S = pkg.sampler
    o = g["class_offsets"]
    m = a["rej_a_members"].tolist()
    by_class = [m[o[c]:o[c + 1]] for c in range(3)]
    want = a[f"{case}_examples"]
    cur = S.BatchCursor(S.plan(g["weights"], g["batch"], g["seed"]), S.ClassIndex(by_class))
    outs, drawn = [], 0
    while drawn + 2 <= g["batches"]:
        ex, _ = cur.next_dev(2)
        outs.append(ex.clone())
        drawn += 2
    torch.cuda.synchronize()
    got = torch.cat(outs).cpu().numpy()
    assert np.array_equal(got, want[: got.size])
    # and the cursor keeps going correctly afterwards
    rest = g["batches"] - drawn
    if rest:
        ex, _ = cur.next_dev(rest)
        torch.cuda.synchronize()
        assert np.array_equal(ex.cpu().numpy(), want[got.size: got.size + ex.numel()])


def test_cursor_copy_forks_identical_stream(pkg, oracle_mod, torch_cuda):
    """A copy of a cursor (optb_sbs_clone; the reference class is copyable,
    sampler.hpp:45-68) continues the identical stream independently -- taken
    mid-stream, with device calls still in flight, across lazy reshuffles."""
    import copy
    torch, S, O = torch_cuda, pkg.sampler, oracle_mod
    n = 3000
    labels = (np.arange(n) % 7).astype(np.int32)
    p = S.plan([1 / 7] * 7, 64, 77)
    offs, mem = S.class_index_dev(torch.from_numpy(labels).cuda(), 7)
    cur = S.BatchCursor.from_device_index(p, offs, mem)
    ro, rm = O.class_index(labels, 7)
    oc = O.Cursor(O.sbs_plan([1 / 7] * 7, 64), ro, rm, 64, 77)
    ex, _ = cur.next_dev(30)           # in flight when the copy is taken
    twin = copy.copy(cur)
    rex, _ = oc.next(30)
    assert np.array_equal(ex.cpu().numpy(), rex)
    want, _ = oc.next(90)              # 90 more batches: several reshuffles of every class
    a, _ = cur.next_dev(90)
    b, _ = twin.next_dev(45)
    b2, _ = twin.next_dev(45)
    assert np.array_equal(a.cpu().numpy(), want)
    assert np.array_equal(torch.cat([b, b2]).cpu().numpy(), want)
    assert twin.batches_drawn() == cur.batches_drawn() == 120
