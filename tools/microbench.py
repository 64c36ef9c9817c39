"""Kernel-level timing of the C2 workload pieces in isolation (CUDA events).

    python tools/microbench.py

Prints a JSON dict: encode / decode / sbs / pipeline-step times in us and
the algorithmic GB/s of encode and decode, each measured as back-to-back
launches (no other work in flight).
"""
import ctypes as ct
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timeit(fn, stream, reps=20, warm=5):
    import torch
    for _ in range(warm):
        fn()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    evs[0].record(stream)
    for i in range(reps):
        fn()
        evs[i + 1].record(stream)
    evs[-1].synchronize()
    return [evs[i].elapsed_time(evs[i + 1]) * 1e3 for i in range(reps)]


def main():
    import torch

    import paper_2105_00619_b200 as pkg
    from paper_2105_00619_b200.pipeline import Pipeline
    C, S = pkg.codec, pkg.sampler
    dev = torch.device("cuda", 0)
    N, P, B, NB, K = 50000, 3072, 512, 97, 100
    s = torch.cuda.Stream(dev)
    res = {}
    with torch.cuda.stream(s):
        ds = torch.randint(0, 256, (N, P), dtype=torch.uint8, device=dev)
        labels = torch.arange(N, device=dev, dtype=torch.int32) % K
        plan = S.plan([1.0 / K] * K, B, 1234)
        offs, mem = S.class_index_dev(labels, K)
        cur = S.BatchCursor.from_device_index(plan, offs, mem)
        rows = B * NB
        ex, cl = cur.next_dev(NB)
        for mode in (1, 0):
            pc = C.capacity(mode)
            L = C.layout(mode, pc, P, B, NB)
            cont, _ = C.alloc_stream(L)
            out = torch.empty((rows, P), dtype=torch.uint8, device=dev)
            outf = torch.empty((rows, P), dtype=torch.float32, device=dev)
            outb = torch.empty((rows, P), dtype=torch.bfloat16, device=dev)
            cb = C.container_bytes(L)
            t_enc = timeit(lambda: C.encode_dev(L, ds, cont, row_index=ex, stream=s), s)
            t_encs = timeit(lambda: C.encode_dev(L, ds[:rows], cont, stream=s), s)
            t_dec = timeit(lambda: C.decode_dev(L, cont, out, stream=s), s)
            t_decf = timeit(lambda: C.decode_dev(L, cont, outf, scale=1 / 255, stream=s), s)
            t_decb = timeit(lambda: C.decode_dev(L, cont, outb, scale=1 / 255, stream=s), s)
            t_rt = timeit(lambda: C.roundtrip_dev(L, ds, cont, out, row_index=ex, stream=s), s)
            bases = torch.tensor([ds.data_ptr()], dtype=torch.int64, device=dev)
            ptrs = C.shard_row_ptrs_dev(ex, bases, N, P, stream=s)
            t_rtp = timeit(lambda: C.roundtrip_rows_dev(L, ptrs, cont, out, stream=s), s)
            m = C.mode_name(mode)
            for name, t, byts in (("roundtrip_gather_u8", t_rt, 2 * (rows * P + cb) + rows * 8),
                                  ("roundtrip_rowptrs_u8", t_rtp, 2 * (rows * P + cb) + rows * 8),
                                  ("encode_gather", t_enc, rows * P + cb + rows * 8),
                                  ("encode_seq", t_encs, rows * P + cb),
                                  ("decode_u8", t_dec, cb + rows * P),
                                  ("decode_f32", t_decf, cb + rows * P * 4),
                                  ("decode_bf16", t_decb, cb + rows * P * 2)):
                us = statistics.median(t)
                res[f"{m}.{name}"] = {"us": round(us, 2), "GBps": round(byts / us / 1e3, 1)}
        ex_b = torch.empty(rows, dtype=torch.int64, device=dev)
        cl_b = torch.empty(rows, dtype=torch.int32, device=dev)
        t_sbs = timeit(lambda: cur.next_dev(NB, examples=ex_b, classes=cl_b, stream=s), s)
        res["sbs_next_97"] = {"us": round(statistics.median(t_sbs), 2)}
        copy_src = torch.empty(rows * P, dtype=torch.uint8, device=dev)
        copy_dst = torch.empty_like(copy_src)
        t_cp = timeit(lambda: copy_dst.copy_(copy_src), s)
        res["torch_copy_152MB"] = {"us": round(statistics.median(t_cp), 2),
                                   "GBps": round(2 * rows * P / statistics.median(t_cp) / 1e3, 1)}
        lib = pkg._lib.lib
        prof = lambda: [ct.c_float() for _ in range(3)]  # noqa: E731
        pkg._lib.check(lib.optb_sbs_set_profiling(cur._h, 1))
        cur.next_dev(NB, examples=ex_b, classes=cl_b, stream=s)
        p3 = prof()
        pkg._lib.check(lib.optb_sbs_profile(cur._h, *[ct.byref(x) for x in p3]))
        res["sbs_alone_phases_us"] = [round(x.value * 1e3, 1) for x in p3]
        out = torch.empty((rows, P), dtype=torch.uint8, device=dev)
        for spd in (2, 4):
            for split in (False, True):
                pipe = Pipeline(cur, ds, 1, B, NB, steps_per_draw=spd, split_kernels=split)
                t_pipe = timeit(lambda: pipe.step(out, s), s, reps=32)
                res[f"pipeline_step_spd{spd}{'_split' if split else ''}"] = {"us": round(statistics.mean(t_pipe), 2)}
                pipe.close()
        pipe = Pipeline(cur, ds, 1, B, NB)
        t_pipe = timeit(lambda: pipe.step(out, s), s, reps=30)
        res["pipeline_step"] = {"us": round(statistics.mean(t_pipe), 2)}
        p3 = prof()
        pkg._lib.check(lib.optb_sbs_profile(cur._h, *[ct.byref(x) for x in p3]))
        res["sbs_in_pipeline_phases_us"] = [round(x.value * 1e3, 1) for x in p3]
        import time
        t0 = time.perf_counter()
        for _ in range(50):
            cur.next_dev(NB, examples=ex_b, classes=cl_b, stream=s)
        t_host = (time.perf_counter() - t0) / 50 * 1e6
        s.synchronize()
        res["sbs_host_us_per_call"] = round(t_host, 1)
        pipe.close()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
