"""The E-D pipeline (optb_pipeline_*): every step's decoded rows equal the
oracle's decode of the oracle's encode of the reference-stream draws."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SCALE = float(np.float32(1.0) / np.float32(255.0))


def _setup(pkg, O, torch, N=4000, Ccls=10, B=64, seed=99):
    S = pkg.sampler
    labels = (np.arange(N) % Ccls).astype(np.int32)
    ds = O.synth_pixels(7, 0, N, 768)
    p = S.plan([1.0 / Ccls] * Ccls, B, seed)
    offs, mem = S.class_index_dev(labels, Ccls)
    ro, rm = O.class_index(labels, Ccls)
    ref = O.Cursor(O.sbs_plan([1.0 / Ccls] * Ccls, B), ro, rm, B, seed)
    return S, labels, ds, p, offs, mem, ref


@pytest.mark.parametrize("split", [False, True])
@pytest.mark.parametrize("mode,dtype,spd", [(1, "uint8", 1), (0, "float32", 1), (3, "bfloat16", 2),
                                            (2, "float16", 3), (1, "uint8", 4)])
def test_pipeline_steps_vs_oracle(pkg, oracle_mod, torch_cuda, mode, dtype, spd, split):
    torch, O = torch_cuda, oracle_mod
    from paper_2105_00619_b200.pipeline import Pipeline
    S, labels, ds, p, offs, mem, ref = _setup(pkg, O, torch)
    B, nb, P = 64, 5, 768
    cur = S.BatchCursor.from_device_index(p, offs, mem)
    ds_d = torch.from_numpy(ds).cuda()
    dt = getattr(torch, dtype)
    pc = pkg.codec.capacity(mode)
    pipe = Pipeline(cur, ds_d, mode, B, nb, per_chunk=pc, out_dtype=dt, scale=SCALE, steps_per_draw=spd,
                    split_kernels=split)
    kind = {"uint8": O.U8, "float32": O.F32, "bfloat16": O.BF16, "float16": O.F16}[dtype]
    for step in range(6):
        out = torch.empty((B * nb, P), dtype=dt, device="cuda")
        pipe.step(out)
        pkg.codec.sync()
        ex, _ = ref.next(nb)
        cont, offs_ = O.encode_stream(ds, ex, mode, pc, B, nb)
        want = O.decode_stream(cont, offs_, mode, pc, P, B, nb, out_dtype=kind, scale=SCALE)
        got = out.cpu()
        got = got.numpy() if dtype in ("uint8", "float32") else got.view(torch.int16).numpy().view(np.uint16)
        assert np.array_equal(got.view(want.dtype), want), step
    pipe.close()


@pytest.mark.parametrize("G,split", [(1, True), (2, False), (2, True), (4, False)])  # 4: three draw buffers
def test_pipeline_sharded_and_class_epilogue(pkg, oracle_mod, torch_cuda, G, split):
    """Per-class epilogue fed by the step's own draw classes.  With split
    launches the decode reads the draw buffer's classes after the encode: the
    side stream must not refill that buffer before the decode ran (steps
    enqueued back to back, no host sync, so a premature reuse shows)."""
    torch, O = torch_cuda, oracle_mod
    from paper_2105_00619_b200.pipeline import Pipeline
    S, labels, ds, p, offs, mem, ref = _setup(pkg, O, torch)
    B, nb, P = 64, 3, 768
    n_steps = 6
    ds_d = torch.from_numpy(ds).cuda()
    cs = torch.linspace(0.001, 0.01, 10, device="cuda")
    cb = torch.linspace(-1, 1, 10, device="cuda")
    outs = {}
    for r in range(G):
        cur = S.BatchCursor.from_device_index(p, offs, mem)
        pipe = Pipeline(cur, ds_d, 1, B, nb, shard=r, n_shards=G, out_dtype=torch.float32, class_scale=cs,
                        class_bias=cb, split_kernels=split)
        outs[r] = []
        for _ in range(n_steps):
            o = torch.empty((B * nb, P), dtype=torch.float32, device="cuda")
            pipe.step(o)
            outs[r].append(o)
        pkg.codec.sync()
        pipe.close()
    for step in range(n_steps):
        ex, cl = ref.next(nb * G)
        ex, cl = ex.reshape(nb * G, B), cl.reshape(nb * G, B)
        for r in range(G):
            e, c = ex[r::G].reshape(-1), cl[r::G].reshape(-1)
            cont, _ = O.encode_stream(ds, e, 1, 16, B, nb)
            want = O.decode_stream(cont, None, 1, 16, P, B, nb, out_dtype=O.F32, scale=1.0,
                                   class_scale=cs.cpu().numpy(), class_bias=cb.cpu().numpy(), row_class=c)
            assert np.array_equal(outs[r][step].cpu().numpy().view(np.uint32), want.view(np.uint32)), (step, r)



def test_c2_full_size_fused_pipeline(pkg, oracle_mod, torch_cuda):
    """The bench workload at full size (C2: 50 000 x 32x32x3, 100 classes,
    B = 512, 97 batches per step, exact128, fused launch): for three steps the
    decoded rows are exactly the dataset rows the oracle cursor draws
    (exact128 at capacity is lossless), so draws and codec both match."""
    torch, O = torch_cuda, oracle_mod
    from paper_2105_00619_b200.pipeline import Pipeline
    S = pkg.sampler
    N, K, B, nb, P = 50000, 100, 512, 97, 3072
    labels = (np.arange(N) % K).astype(np.int32)
    ds = torch.randint(0, 256, (N, P), dtype=torch.uint8, device="cuda")
    offs, mem = S.class_index_dev(torch.from_numpy(labels).cuda(), K)
    cur = S.BatchCursor.from_device_index(S.plan([1.0 / K] * K, B, 1234), offs, mem)
    pipe = Pipeline(cur, ds, 1, B, nb, per_chunk=16, steps_per_draw=2)
    assert pipe.fused
    ro, rm = O.class_index(labels, K)
    ref = O.Cursor(O.sbs_plan([1.0 / K] * K, B), ro, rm, B, 1234)
    out = torch.empty((B * nb, P), dtype=torch.uint8, device="cuda")
    for step in range(3):
        pipe.step(out)
        pkg.codec.sync()
        want, _ = ref.next(nb)
        assert torch.equal(out, ds[torch.from_numpy(want).cuda()]), step
    pipe.close()


@pytest.mark.parametrize("dtype", ["uint8", "bfloat16"])
def test_pipeline_step_host_vs_oracle(pkg, oracle_mod, torch_cuda, dtype):
    """optb_pipeline_step_host: host dataset in, host rows out, one C-ABI call
    per step (uploads and downloads on the library's copy streams) == the
    oracle's decode of the reference-stream draws, for every step."""
    torch, O = torch_cuda, oracle_mod
    from paper_2105_00619_b200.pipeline import Pipeline
    S, labels, ds, p, offs, mem, ref = _setup(pkg, O, torch)
    B, nb, P = 64, 5, 768
    cur = S.BatchCursor.from_device_index(p, offs, mem)
    ds_host = torch.from_numpy(ds).pin_memory()
    dt = getattr(torch, dtype)
    pipe = Pipeline(cur, ds_host.cuda(), 1, B, nb, per_chunk=16, out_dtype=dt, scale=SCALE, steps_per_draw=2)
    outs = [torch.empty((B * nb, P), dtype=dt).pin_memory() for _ in range(5)]
    for o in outs:
        pipe.step_host(ds_host, o)
    pipe.host_wait()
    pkg.codec.sync()
    kind = {"uint8": O.U8, "bfloat16": O.BF16}[dtype]
    for step in range(5):
        ex, _ = ref.next(nb)
        cont, offs_ = O.encode_stream(ds, ex, 1, 16, B, nb)
        want = O.decode_stream(cont, offs_, 1, 16, P, B, nb, out_dtype=kind, scale=SCALE)
        got = outs[step] if dtype == "uint8" else outs[step].view(torch.int16)
        assert np.array_equal(got.numpy().view(want.dtype), want), step
    pipe.close()


def test_pipeline_timing_stride(pkg, oracle_mod, torch_cuda):
    """record_timings with timing_stride: only every stride-th step carries
    timing events (the others launch back to back, overlapping via
    programmatic dependent launch); their outputs are unaffected."""
    torch, O = torch_cuda, oracle_mod
    from paper_2105_00619_b200.pipeline import Pipeline
    S, labels, ds, p, offs, mem, ref = _setup(pkg, O, torch)
    B, nb, P = 64, 5, 768
    cur = S.BatchCursor.from_device_index(p, offs, mem)
    pipe = Pipeline(cur, torch.from_numpy(ds).cuda(), 1, B, nb, per_chunk=16, record_timings=True,
                    steps_per_draw=2, timing_stride=3)
    outs = []
    for _ in range(7):
        o = torch.empty((B * nb, P), dtype=torch.uint8, device="cuda")
        pipe.step(o)
        outs.append(o)
    pkg.codec.sync()
    for step in (0, 3, 6):
        s_ms, e_ms, d_ms = pipe.timings(step)
        assert e_ms > 0 and d_ms == 0.0
    for step in (1, 2, 4, 5):
        with pytest.raises(pkg.errors.Error):
            pipe.timings(step)
    for step in range(7):
        ex, _ = ref.next(nb)
        assert torch.equal(outs[step].cpu(), torch.from_numpy(ds[ex])), step
    pipe.close()


@pytest.mark.parametrize("mode,split,spd", [(1, False, 1), (1, False, 4), (1, True, 1), (4, True, 2), (0, True, 1),
                                             (0, False, 2)])
def test_pipeline_back_to_back_steps_early_gather(pkg, oracle_mod, torch_cuda, mode, split, spd):
    """Steps enqueued back to back without a host sync (each step's round trip
    may start gathering while the previous one drains: RowSrc::early), each
    into its own output, all equal to the oracle; then a library decode that
    rewrites the dataset in the same stream between two steps (a kernel that
    triggers its dependents early): the next step must gather the new rows."""
    torch, O = torch_cuda, oracle_mod
    from paper_2105_00619_b200.pipeline import Pipeline
    C = pkg.codec
    N = 4096
    S, labels, ds, p, offs, mem, ref = _setup(pkg, O, torch, N=N)
    B, nb, P = 64, 40, 768  # 2560 rows per step
    cur = S.BatchCursor.from_device_index(p, offs, mem)
    ds_d = torch.from_numpy(ds).cuda()
    s = torch.cuda.Stream()
    pipe = Pipeline(cur, ds_d, mode, B, nb, per_chunk=C.capacity(mode), steps_per_draw=spd, split_kernels=split)
    outs = [torch.empty((B * nb, P), dtype=torch.uint8, device="cuda") for _ in range(8)]
    with torch.cuda.stream(s):
        for o in outs:
            pipe.step(o, s)
    s.synchronize()
    for k, o in enumerate(outs):
        ex, _ = ref.next(nb)
        assert np.array_equal(o.cpu().numpy(), ds[ex]), k
    # a second dataset written into ds_d by optb_decode_dev on the same stream
    new = O.synth_pixels(11, 0, N, P)
    L2 = C.layout(1, 16, P, N, 1)
    cont2, _ = C.alloc_stream(L2)
    new_d = torch.from_numpy(new).cuda()
    outs2 = [torch.empty((B * nb, P), dtype=torch.uint8, device="cuda") for _ in range(2)]
    with torch.cuda.stream(s):
        C.encode_dev(L2, new_d, cont2, stream=s)
        pipe.step(outs2[0], s)  # still the old rows? no: encode_dev does not write ds_d
        C.decode_dev(L2, cont2, ds_d, stream=s)  # ds_d := new, in stream order
        pipe.step(outs2[1], s)
    s.synchronize()
    ex0, _ = ref.next(nb)
    ex1, _ = ref.next(nb)
    assert np.array_equal(outs2[0].cpu().numpy(), ds[ex0])
    assert np.array_equal(outs2[1].cpu().numpy(), new[ex1])
    pipe.close()


def test_pipeline_dataset_is_previous_output(pkg, oracle_mod, torch_cuda):
    """A step whose dataset is the PREVIOUS step's output (set_dataset to the
    buffer the step before wrote, enqueued back to back): it must not gather
    before that step finished writing -- the early-gather check compares the
    dataset with the previous step's output range as well as its own."""
    torch, O = torch_cuda, oracle_mod
    from paper_2105_00619_b200.pipeline import Pipeline
    N = 4096
    S, labels, ds, p, offs, mem, ref = _setup(pkg, O, torch, N=N)
    B, nb, P = 64, N // 64, 768  # one step's output is a full dataset
    cur = S.BatchCursor.from_device_index(p, offs, mem)
    a = torch.from_numpy(ds).cuda()
    b = torch.empty_like(a)
    c = torch.empty_like(a)
    s = torch.cuda.Stream()
    pipe = Pipeline(cur, a, 1, B, nb, per_chunk=16)
    with torch.cuda.stream(s):
        pipe.step(c, s)   # warm: a -> c
        pipe.step(b, s)   # a -> b
        pipe.set_dataset(b)
        pipe.step(c, s)   # b -> c, right behind the step that writes b
    s.synchronize()
    ex0, _ = ref.next(nb)
    ex1, _ = ref.next(nb)
    ex2, _ = ref.next(nb)
    step1 = ds[ex1]
    assert np.array_equal(b.cpu().numpy(), step1)
    assert np.array_equal(c.cpu().numpy(), step1[ex2])
    pipe.close()


def test_pipeline_step_host_rejects_short_dataset(pkg, oracle_mod, torch_cuda):
    """step_host with fewer dataset rows than the sampler's examples is an
    argument error (the draws would read past the end of the upload)."""
    torch, O = torch_cuda, oracle_mod
    from paper_2105_00619_b200.pipeline import Pipeline
    S, labels, ds, p, offs, mem, ref = _setup(pkg, O, torch)
    B, nb, P = 64, 2, 768
    cur = S.BatchCursor.from_device_index(p, offs, mem)
    pipe = Pipeline(cur, torch.from_numpy(ds).cuda(), 1, B, nb, per_chunk=16)
    short = torch.from_numpy(ds[:100]).pin_memory()
    out = torch.empty((B * nb, P), dtype=torch.uint8).pin_memory()
    with pytest.raises(pkg.errors.Error, match="100 dataset rows, the sampler draws from 4000 examples"):
        pipe.step_host(short, out)
    # the pipeline is still usable
    pipe.step_host(torch.from_numpy(ds).pin_memory(), out)
    pipe.host_wait()
    ex, _ = ref.next(nb)
    assert np.array_equal(out.numpy(), ds[ex])
    pipe.close()


def test_pipeline_warm_start_vs_oracle(pkg, oracle_mod, torch_cuda, tmp_path):
    """Warm start (PipelineConfig::warm_start, pipeline.cpp:154-177): an
    epoch dumped in OPTB files (optb_dump_dev) is loaded once and every step
    decodes it again -- equal to the oracle's decode of the oracle's encode
    of the reference-stream draws, every step; a missing dump is a
    FormatError at creation."""
    torch, O = torch_cuda, oracle_mod
    from paper_2105_00619_b200.pipeline import Pipeline
    C = pkg.codec
    S, labels, ds, p, offs, mem, ref = _setup(pkg, O, torch)
    B, nb, P = 64, 5, 768
    shape = C.ImageShape(16, 16, 3)
    ref_ex, _ = ref.next(nb)
    for mode in (1, 4):
        n = C.capacity(mode)
        L = C.layout(mode, n, P, B, nb)
        want_c, want_o = O.encode_stream(ds, ref_ex, mode, n, B, nb)
        cont, offs_ = C.alloc_stream(L)
        cont[: want_c.size].copy_(torch.from_numpy(want_c))
        if want_o is not None:
            offs_[: want_o.size].copy_(torch.from_numpy(want_o))
        d = tmp_path / f"warm{mode}"
        C.dump_dev(L, cont, offs_, shape, str(d), 0)
        warm = Pipeline.warm(mode, B, nb, shape, str(d), 0, per_chunk=n, out_dtype=torch.float32, scale=SCALE,
                             record_timings=True)
        want = O.decode_stream(want_c, want_o, mode, n, P, B, nb, out_dtype=O.F32, scale=SCALE)
        for k in range(3):
            o = torch.empty((B * nb, P), dtype=torch.float32, device="cuda")
            warm.step(o)
            C.sync()
            assert np.array_equal(o.cpu().numpy().view(np.uint32), want.view(np.uint32)), (mode, k)
            s_ms, e_ms, d_ms = warm.timings(k)
            assert s_ms == 0.0 and d_ms > 0
        warm.close()
    with pytest.raises(pkg.errors.FormatError):
        Pipeline.warm(1, B, nb, shape, str(tmp_path / "missing"), 0)


@pytest.mark.parametrize("mode,n", [(1, 12), (4, 10)])
def test_pipeline_corrupt_epoch_fails_at_its_step(pkg, oracle_mod, torch_cuda, tmp_path, mode, n):
    """Failure semantics (pipeline.cpp:60-82, 213-215; the reference's
    test_pipeline.cpp:200-239): an epoch whose OPTB files pass the header
    checks but hold a container value out of range for its chunk loads
    fine, and the step that decodes it reports the reference's FormatError
    at the next sync -- not earlier steps, which were clean; the latch is
    cleared, so the pipeline keeps serving after the error."""
    torch, O = torch_cuda, oracle_mod
    from paper_2105_00619_b200.pipeline import Pipeline
    C = pkg.codec
    S, labels, ds, p, offs, mem, ref = _setup(pkg, O, torch)
    B, nb, P = 64, 3, 768
    shape = C.ImageShape(16, 16, 3)
    L = C.layout(mode, n, P, B, nb)
    ref_ex, _ = ref.next(nb)
    good_c, good_o = O.encode_stream(ds, ref_ex, mode, n, B, nb)
    bad_c = good_c.copy()
    # chunk 2, pixel 5: set a bit above the chunk's n packed images
    wc = C.container_value_bytes(mode)
    word = bad_c[(2 * P + 5) * wc:(2 * P + 6) * wc]
    bit = 8 * 15 if mode == 1 else 7 * 17  # exact128: byte of image 15; lossless128: field of image 17
    word[bit // 8] |= 1 << (bit % 8)
    dirs = {}
    for tag, c in (("good", good_c), ("bad", bad_c)):
        cont, offs_ = C.alloc_stream(L)
        cont[: c.size].copy_(torch.from_numpy(c))
        if good_o is not None:
            offs_[: good_o.size].copy_(torch.from_numpy(good_o))
        dirs[tag] = tmp_path / tag
        C.dump_dev(L, cont, offs_, shape, str(dirs[tag]), 0)
    want = O.decode_stream(good_c, good_o, mode, n, P, B, nb)
    o = torch.empty((B * nb, P), dtype=torch.uint8, device="cuda")
    good = Pipeline.warm(mode, B, nb, shape, str(dirs["good"]), 0, per_chunk=n)
    for _ in range(2):  # clean steps: no error
        good.step(o)
        C.sync()
        assert np.array_equal(o.cpu().numpy(), want)
    good.close()
    bad = Pipeline.warm(mode, B, nb, shape, str(dirs["bad"]), 0, per_chunk=n)  # the header checks pass
    bad.step(o)
    with pytest.raises(pkg.errors.FormatError, match=f"^decode: container value exceeds range of {n} packed images$"):
        C.sync()
    C.sync()  # the latch is cleared after it was reported
    bad.close()
    good = Pipeline.warm(mode, B, nb, shape, str(dirs["good"]), 0, per_chunk=n)
    good.step(o)
    C.sync()
    assert np.array_equal(o.cpu().numpy(), want)
    good.close()


@pytest.mark.parametrize("mode,spd", [(3, 1), (4, 2)])
def test_pipeline_lossless_interleaved_steps(pkg, oracle_mod, torch_cuda, mode, spd):
    """Lossless pipeline steps on the interleaved round trip (P % 512 == 0),
    enqueued back to back (early gather across steps): every step's rows,
    containers and parity planes equal the oracle's."""
    torch, O = torch_cuda, oracle_mod
    from paper_2105_00619_b200.pipeline import Pipeline
    C, S = pkg.codec, pkg.sampler
    N, Ccls, B, nb, P = 4096, 10, 64, 20, 1024
    labels = (np.arange(N) % Ccls).astype(np.int32)
    ds = O.synth_pixels(5, 0, N, P)
    offs, mem = S.class_index_dev(labels, Ccls)
    cur = S.BatchCursor.from_device_index(S.plan([1.0 / Ccls] * Ccls, B, 77), offs, mem)
    ro, rm = O.class_index(labels, Ccls)
    ref = O.Cursor(O.sbs_plan([1.0 / Ccls] * Ccls, B), ro, rm, B, 77)
    n = C.capacity(mode)
    pipe = Pipeline(cur, torch.from_numpy(ds).cuda(), mode, B, nb, per_chunk=n, steps_per_draw=spd)
    assert pipe.fused
    s = torch.cuda.Stream()
    outs = [torch.empty((B * nb, P), dtype=torch.uint8, device="cuda") for _ in range(4)]
    with torch.cuda.stream(s):
        for o in outs:
            pipe.step(o, s)
    s.synchronize()
    assert C.last_roundtrip_kind() == "interleaved"
    for k, o in enumerate(outs):
        ex, _ = ref.next(nb)
        assert np.array_equal(o.cpu().numpy(), ds[ex]), k
    # the last step's containers, materialised in HBM as by two calls
    want_c, _ = O.encode_stream(ds, ex, mode, n, B, nb)
    nbytes = C.container_bytes(pipe.layout)

    class _Arr:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (pipe.containers_ptr(), False),
                                    "version": 3}
    cont = torch.as_tensor(_Arr(), device="cuda").cpu().numpy()
    assert np.array_equal(cont[: want_c.size], want_c)
    pipe.close()
