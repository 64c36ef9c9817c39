"""All BASELINE.json configurations on one B200 (secondary to bench.py's C2 headline).

    python tools/configs_bench.py [--cpu]

Per config: device-resident encode+decode throughput (images/s), algorithmic
GB/s of each kernel and its fraction of the measured HBM peak, plus (with
--cpu) the reference CPU path (oracle/_ref, all host threads) on a bounded
sample of the same config.  Working sets exceed L2 (the configs are
replicated into >= 1 GB streams where a single batch would fit in L2).

  C1  CIFAR-10  128 x 32x32x3, exact64 (8 -> 1), decode -> u8 and -> fp32
  C3  4096 x 32x32x3, n = 2 / 4 / 8 (exact64) and 16 (exact128); lossless64/128; f64 n=6
  C4  ImageNet 256 x 224x224x3, exact128 (16 -> 1), fused decode -> bf16
  C5  2^20-image stream, SBS (100 classes, B=512) + exact128, one GPU's shard
Prints one JSON object.
"""
import argparse
import ctypes as ct
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timeit(fn, stream, reps=10, warm=3):
    import torch
    for _ in range(warm):
        fn()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    evs[0].record(stream)
    for i in range(reps):
        fn()
        evs[i + 1].record(stream)
    evs[-1].synchronize()
    return statistics.median(evs[i].elapsed_time(evs[i + 1]) for i in range(reps)) / 1e3


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:  # noqa: BLE001
        return 6650.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cpu", action="store_true")
    args = ap.parse_args()
    import torch

    import paper_2105_00619_b200 as pkg
    from paper_2105_00619_b200.pipeline import Pipeline
    C, S = pkg.codec, pkg.sampler
    dev = torch.device("cuda", 0)
    s = torch.cuda.Stream(dev)
    pk = peak()
    res = {"peak_gbs": pk}

    def codec_case(name, mode, per_chunk, P, B, nb, out_dtype=torch.uint8, scale=1.0, gather=False):
        L = C.layout(mode, per_chunk, P, B, nb)
        rows = B * nb
        with torch.cuda.stream(s):
            src = torch.randint(0, 256, (rows, P), dtype=torch.uint8, device=dev)
            idx = torch.randperm(rows, device=dev) if gather else None
            cont, offs = C.alloc_stream(L)
            out = torch.empty((rows, P), dtype=out_dtype, device=dev)
            t_enc = timeit(lambda: C.encode_dev(L, src, cont, offs, row_index=idx, stream=s), s)
            t_dec = timeit(lambda: C.decode_dev(L, cont, out, offsets=offs, scale=scale, stream=s), s)
            # optb_roundtrip_dev: one fused launch on the vector path
            t_rt = timeit(lambda: C.roundtrip_dev(L, src, cont, out, offsets=offs, row_index=idx, scale=scale,
                                                  stream=s), s)
            C.sync(0, s)
            rt_kind = C.last_roundtrip_kind()
            rt_b = C.roundtrip_hbm_bytes(L, out.element_size(), gather)
        cb, ob = C.container_bytes(L), C.offsets_bytes(L)
        es = out.element_size()
        enc_b = rows * P + cb + ob + (rows * 8 if gather else 0)
        dec_b = cb + ob + rows * P * es
        r = {"mode": C.mode_name(mode), "per_chunk": per_chunk, "images": rows, "P": P,
             "out": str(out_dtype).replace("torch.", ""),
             "images_per_s": round(rows / (t_enc + t_dec), 1),
             "encode_us": round(t_enc * 1e6, 1), "decode_us": round(t_dec * 1e6, 1),
             "encode_gbs": round(enc_b / t_enc / 1e9, 1), "decode_gbs": round(dec_b / t_dec / 1e9, 1),
             "encode_frac": round(enc_b / t_enc / 1e9 / pk, 3), "decode_frac": round(dec_b / t_dec / 1e9 / pk, 3),
             "roundtrip_us": round(t_rt * 1e6, 1), "roundtrip_images_per_s": round(rows / t_rt, 1),
             "roundtrip_fused": P % 16 == 0 and (mode in (0, 1, 2) or P % 512 == 0)}
        # interleaved fused kernel (exact / f64): the container re-read is an
        # L2 hit, the HBM bytes are rows in + containers and rows out
        r.update({"roundtrip_kernel": rt_kind, "roundtrip_hbm_bytes": rt_b,
                  "roundtrip_frac": round(rt_b / t_rt / 1e9 / pk, 3)})
        res[name] = r
        del src, cont, out

    # C1: 128-image CIFAR-10 batches, streamed as 512 batches per launch (1.6 GB round trip)
    codec_case("C1_exact64_u8", 0, 8, 3072, 128, 512)
    codec_case("C1_exact64_f32", 0, 8, 3072, 128, 512, torch.float32, 1 / 255)
    # C3 sweep: 4096-image batches x 16
    for n in (2, 4, 8):
        codec_case(f"C3_n{n}_exact64", 0, n, 3072, 4096, 16)
    codec_case("C3_n16_exact128", 1, 16, 3072, 4096, 16)
    codec_case("C3_n9_lossless64", 3, 9, 3072, 4096, 16)
    codec_case("C3_n18_lossless128", 4, 18, 3072, 4096, 16)
    codec_case("C3_n6_f64", 2, 6, 3072, 4096, 16)
    # C4: ImageNet 256 x 224x224x3, exact128, fused bf16 -- a stream of 8
    # batches per launch (2.5 GB round trip), and one batch per launch
    # rotating over 8 distinct batches (each launch's 154 MB working set was
    # evicted from L2 by the seven before it)
    IMG = 224 * 224 * 3
    codec_case("C4_exact128_bf16", 1, 16, IMG, 256, 8, torch.bfloat16, 1 / 255)
    codec_case("C4_exact128_u8", 1, 16, IMG, 256, 8)
    L4 = C.layout(1, 16, IMG, 256, 1)
    with torch.cuda.stream(s):
        bat = [(torch.randint(0, 256, (256, IMG), dtype=torch.uint8, device=dev), *C.alloc_stream(L4),
                torch.empty((256, IMG), dtype=torch.bfloat16, device=dev)) for _ in range(8)]
        k = [0]

        def one(fused):
            x, cont, _, out = bat[k[0] % 8]
            k[0] += 1
            if fused:
                C.roundtrip_dev(L4, x, cont, out, scale=1 / 255, stream=s)
            else:
                C.encode_dev(L4, x, cont, stream=s)
                C.decode_dev(L4, cont, out, scale=1 / 255, stream=s)
        t_split = timeit(lambda: one(False), s, reps=16, warm=8)
        t_fused = timeit(lambda: one(True), s, reps=16, warm=8)
        C.sync(0, s)
        k4 = C.last_roundtrip_kind()
        b4 = C.roundtrip_hbm_bytes(L4, 2, False)
    b4_split = 256 * IMG * 5  # rows read + containers written and read back + bf16 out
    res["C4_per_batch_bf16"] = {"images_per_launch": 256, "split_us": round(t_split * 1e6, 1),
                                "fused_us": round(t_fused * 1e6, 1),
                                "images_per_s_split": round(256 / t_split, 1),
                                "images_per_s_fused": round(256 / t_fused, 1),
                                "fused_kernel": k4,
                                "split_frac": round(b4_split / t_split / 1e9 / pk, 3),
                                "fused_frac": round(b4 / t_fused / 1e9 / pk, 3)}
    del bat

    # C5: 2^20-image stream, SBS + gather-encode + decode (one GPU's shard = whole stream here)
    N, K, B, NB = 1 << 20, 100, 512, 256
    with torch.cuda.stream(s):
        ds = torch.empty((N, 3072), dtype=torch.uint8, device=dev)
        ctx = pkg._lib.context(0)
        pkg._lib.check(pkg._lib.lib.optb_synth_pixels_dev(ctx, 7, 0, N, 3072, ct.c_void_p(ds.data_ptr()), 3072,
                                                          ct.c_void_p(s.cuda_stream)))
        labels = torch.arange(N, device=dev, dtype=torch.int32) % K
        t0 = time.perf_counter()
        offs, mem = S.class_index_dev(labels, K)
        t_ci = time.perf_counter() - t0
        cur = S.BatchCursor.from_device_index(S.plan([1.0 / K] * K, B, 1234), offs, mem)
        pipe = Pipeline(cur, ds, 1, B, NB, steps_per_draw=2)
        out = torch.empty((B * NB, 3072), dtype=torch.uint8, device=dev)
        t_step = timeit(lambda: pipe.step(out, s), s, reps=10, warm=4)
        pipe.close()
    res["C5_sbs_exact128_1gpu"] = {"images_per_step": B * NB, "images_per_s": round(B * NB / t_step, 1),
                                   "step_ms": round(t_step * 1e3, 3), "class_index_2^20_ms_incl_sync": round(t_ci * 1e3, 2)}
    del ds

    if args.cpu:
        import oracle as O
        threads = os.cpu_count() or 1
        if O.ref_available():
            R = O.REF
            cpu = {}
            for name, mode, n, P, B in (("C1_exact64", 0, 8, 3072, 128), ("C3_n16_exact128", 1, 16, 3072, 4096),
                                        ("C4_exact128", 1, 16, 150528, 256)):
                nb = max(threads, 4)
                rows = B * nb if B * nb * P < (1 << 31) else B * 2
                nb = rows // B
                ds = np.random.default_rng(0).integers(0, 256, size=(rows, P), dtype=np.uint8)
                h = R.ref_dataset_create(O.ptr(ds, O.u8p), rows, 1, P, 1)
                ex = np.arange(rows, dtype=np.int64)
                chk = ct.c_uint64()
                secs = R.ref_bench_roundtrip(h, mode, O.ptr(ex, O.i64p), nb, B, threads, 0, ct.byref(chk))
                R.ref_dataset_destroy(h)
                cpu[name] = {"images_per_s": round(rows / secs, 1), "threads": threads, "sample_images": rows}
            res["cpu_reference"] = cpu
    print(json.dumps(res))


if __name__ == "__main__":
    main()
