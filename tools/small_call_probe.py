"""Latency anatomy of the drop-in's per-chunk host calls (codec::encode /
codec::decode of one 16-image CIFAR chunk -> optb_encode_host /
optb_decode_host): host wall time per call, and the CUPTI timeline
(torch.profiler) of the H2D, kernel and D2H each call issues.

    python tools/small_call_probe.py
"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    from torch.profiler import ProfilerActivity, profile

    import paper_2105_00619_b200 as pkg
    C = pkg.codec
    res = {}
    for mode, n in ((1, 16), (0, 8), (3, 9)):
        L = C.layout(mode, n, 3072, n, 1)
        imgs = np.random.default_rng(0).integers(0, 256, size=(n, 3072), dtype=np.uint8)
        cont, offs = C.encode_host(L, imgs)
        for _ in range(20):
            C.encode_host(L, imgs)
            C.decode_host(L, cont, offs)
        te, td = [], []
        for _ in range(200):
            t0 = time.perf_counter()
            C.encode_host(L, imgs)
            t1 = time.perf_counter()
            C.decode_host(L, cont, offs)
            td.append(time.perf_counter() - t1)
            te.append(t1 - t0)
        res[C.mode_name(mode)] = {"encode_us": round(statistics.median(te) * 1e6, 2),
                                  "decode_us": round(statistics.median(td) * 1e6, 2)}
    L = C.layout(1, 16, 3072, 16, 1)
    imgs = np.random.default_rng(0).integers(0, 256, size=(16, 3072), dtype=np.uint8)
    cont, offs = C.encode_host(L, imgs)
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for _ in range(5):
            C.encode_host(L, imgs)
            C.decode_host(L, cont, offs)
    prof.export_chrome_trace("/tmp/small_trace.json")
    tr = json.load(open("/tmp/small_trace.json"))
    evs = [e for e in tr["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset",
                                                                                  "cuda_runtime", "cuda_driver")]
    t_min = min(e["ts"] for e in evs)
    res["timeline_us"] = [[round(e["ts"] - t_min, 1), round(e["dur"], 1), e["cat"], e["name"][:50]]
                          for e in sorted(evs, key=lambda e: e["ts"])][-60:]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
