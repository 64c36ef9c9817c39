"""SBS call cost against call size (the shim's ring refills and the C5
pipeline's one-epoch calls): host time of optb_sbs_next_host / next_dev and
the device phases (upload, reshuffle K9+K8, gather K10) per call.

    python tools/sbs_scale_probe.py
"""
import ctypes as ct
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch

    import paper_2105_00619_b200 as pkg
    S, lib = pkg.sampler, pkg._lib.lib
    dev = torch.device("cuda", 0)
    out = {}
    for N in (50000, 1 << 20):
        labels = torch.arange(N, device=dev, dtype=torch.int32) % 100
        offs, mem = S.class_index_dev(labels, 100)
        # the shim's refill sequence: next_host(4), (8), (16), ...
        cur = S.BatchCursor.from_device_index(S.plan([0.01] * 100, 512, 1234), offs, mem)
        seq = []
        k = 4
        while k <= 2048:
            ex = np.zeros(k * 512, np.int64)
            cl = np.zeros(k * 512, np.int32)
            t0 = time.perf_counter()
            pkg._lib.check(lib.optb_sbs_next_host(cur._h, k, ct.c_void_p(ex.ctypes.data), ct.c_void_p(cl.ctypes.data)))
            seq.append([k, round((time.perf_counter() - t0) * 1e3, 3)])
            k *= 2
        out[f"N{N}_next_host_refills_ms"] = seq
        # steady calls of fixed size with device-phase profiling
        for n, G in ((1, 1), (16, 1), (97, 1), (2048, 1), (2048 * 8, 8)):
            cur = S.BatchCursor.from_device_index(S.plan([0.01] * 100, 512, 1234), offs, mem)
            pkg._lib.check(lib.optb_sbs_set_profiling(cur._h, 1))
            rows = (n // G) * 512
            exd = torch.empty(rows, dtype=torch.int64, device=dev)
            cld = torch.empty(rows, dtype=torch.int32, device=dev)
            host, ph = [], []
            for it in range(6):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                cur.next_dev(n, 0, G, exd, cld)
                torch.cuda.synchronize()
                host.append((time.perf_counter() - t0) * 1e3)
                p3 = [ct.c_float() for _ in range(3)]
                pkg._lib.check(lib.optb_sbs_profile(cur._h, *[ct.byref(x) for x in p3]))
                ph.append([x.value for x in p3])
            out[f"N{N}_n{n}_G{G}"] = {"host_ms_first": round(host[0], 3), "host_ms_median": round(statistics.median(host[2:]), 3),
                                      "upload_reshuffle_gather_ms": [round(statistics.median(p[i] for p in ph[2:]), 4)
                                                                     for i in range(3)]}
            print(f"N{N}_n{n}_G{G}", out[f"N{N}_n{n}_G{G}"], flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
