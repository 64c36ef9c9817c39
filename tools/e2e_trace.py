"""CUPTI timeline (torch.profiler) of bench.py's e2e leg: optb_pipeline_step_host
at the headline (C5) size, every memcpy and kernel the library issues on its
internal streams, with start / end offsets in ms.

    python tools/e2e_trace.py [--steps 5] [--rows N]

Prints one JSON object: per stream, the [start, end, name, bytes] of each
activity, plus the host time of every step_host call.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--rows", type=int, default=1 << 20)
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    import paper_2105_00619_b200 as pkg
    from paper_2105_00619_b200.pipeline import Pipeline
    S = pkg.sampler
    dev = torch.device("cuda", 0)
    N, P, B, K = args.rows, 3072, 512, 100
    NB = N // B
    ds = torch.randint(0, 256, (N, P), dtype=torch.uint8, device=dev)
    ds_host = ds.cpu().pin_memory()
    labels = torch.arange(N, device=dev, dtype=torch.int32) % K
    offs, mem = S.class_index_dev(labels, K)
    cur = S.BatchCursor.from_device_index(S.plan([1.0 / K] * K, B, 1234), offs, mem)
    pipe = Pipeline(cur, ds, 1, B, NB)
    outs = [torch.empty((NB * B, P), dtype=torch.uint8).pin_memory() for _ in range(2)]
    stream = torch.cuda.Stream(dev)
    for k in range(2):
        pipe.step_host(ds_host, outs[k % 2], stream)
    pipe.host_wait()
    torch.cuda.synchronize()
    host = []
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        t0 = time.perf_counter()
        for k in range(args.steps):
            a = time.perf_counter()
            pipe.step_host(ds_host, outs[k % 2], stream)
            host.append([round((a - t0) * 1e3, 3), round((time.perf_counter() - t0) * 1e3, 3)])
        pipe.host_wait()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    path = "/tmp/e2e_trace.json"
    prof.export_chrome_trace(path)
    with open(path) as f:
        tr = json.load(f)
    evs = [e for e in tr["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    t_min = min(e["ts"] for e in evs) if evs else 0
    by_stream = {}
    for e in sorted(evs, key=lambda e: e["ts"]):
        sid = str(e.get("args", {}).get("stream", e.get("tid")))
        by_stream.setdefault(sid, []).append([round((e["ts"] - t_min) / 1e3, 3), round((e["ts"] + e["dur"] - t_min) / 1e3, 3),
                                              e["name"][:60], e.get("args", {}).get("bytes")])
    print(json.dumps({"wall_ms_per_step": round(wall / args.steps * 1e3, 3), "host_calls_ms": host,
                      "streams": by_stream}))
    pipe.close()


if __name__ == "__main__":
    main()
