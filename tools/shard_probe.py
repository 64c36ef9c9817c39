"""One rank's share of an N-GPU run, on one GPU: the C2 pipeline with
shard 0 of n_shards (every rank draws the whole stream and keeps its
batches), for n_shards = 1, 2, 4, 8 -- device time per step, host enqueue
time per step, and the side-stream SBS time per call.

    python tools/shard_probe.py
"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2105_00619_b200 as pkg
    from paper_2105_00619_b200.pipeline import Pipeline
    S = pkg.sampler
    dev = torch.device("cuda", 0)
    N, P, B, NB, K = 50000, 3072, 512, 97, 100
    ds = torch.randint(0, 256, (N, P), dtype=torch.uint8, device=dev)
    labels = torch.arange(N, device=dev, dtype=torch.int32) % K
    offs, mem = S.class_index_dev(labels, K)
    out = torch.empty((B * NB, P), dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream(dev)
    res = {}
    for G in (1, 2, 4, 8):
        for spd in (2, 4):
            cur = S.BatchCursor.from_device_index(S.plan([1.0 / K] * K, B, 1234), offs, mem)
            pipe = Pipeline(cur, ds, 1, B, NB, shard=0, n_shards=G, steps_per_draw=spd, record_timings=True)
            for _ in range(2 * spd + 2):
                pipe.step(out, s)
            torch.cuda.synchronize()
            steps = 8 * spd
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            t0 = time.perf_counter()
            for _ in range(steps):
                pipe.step(out, s)
            th = (time.perf_counter() - t0) / steps * 1e6
            e1.record(s)
            e1.synchronize()
            ms = e0.elapsed_time(e1) / steps
            tim = [pipe.timings(k) for k in range(pipe.steps - steps, pipe.steps)]
            res[f"G{G}_spd{spd}"] = {"step_us": round(ms * 1e3, 1), "host_us_per_step": round(th, 1),
                                     "sbs_side_us_per_step": round(statistics.mean(t[0] for t in tim) * 1e3, 1),
                                     "roundtrip_us": round(statistics.mean(t[1] for t in tim) * 1e3, 1)}
            pipe.close()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
