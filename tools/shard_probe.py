"""One rank's share of an N-GPU run, on one GPU: the pipeline with shard 0
of n_shards (every rank draws the whole stream and keeps its batches), for
n_shards = 1, 2, 4, 8 -- device time per step (events around the timed
steps only), host enqueue time per step.  --c5: the headline C5 stream (2^20
images, one epoch = 2048 batches per rank per step, one sampler call per
step); default the C2 stream (50 000 images, 97 batches per step).

    python tools/shard_probe.py [--c5]
"""
import json
import os
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
    c5 = "--c5" in sys.argv
    N, P, B, K = (1 << 20) if c5 else 50000, 3072, 512, 100
    NB = N // B
    ds = torch.randint(0, 256, (N, P), dtype=torch.uint8, device=dev)
    labels = torch.arange(N, device=dev, dtype=torch.int32) % K
    offs, mem = S.class_index_dev(labels, K)
    out = torch.empty((B * NB, P), dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream(dev)
    res = {}
    for G in (1, 2, 4, 8):
        for spd in ((1,) if c5 else (2, 4)):
            cur = S.BatchCursor.from_device_index(S.plan([1.0 / K] * K, B, 1234), offs, mem)
            pipe = Pipeline(cur, ds, 1, B, NB, shard=0, n_shards=G, steps_per_draw=spd)
            for _ in range(2 * spd + 2):
                pipe.step(out, s)
            torch.cuda.synchronize()
            steps = 10 if c5 else 8 * spd
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            t0 = time.perf_counter()
            for _ in range(steps):
                pipe.step(out, s)
            th = (time.perf_counter() - t0) / steps * 1e6
            e1.record(s)
            e1.synchronize()
            ms = e0.elapsed_time(e1) / steps
            res[f"G{G}_spd{spd}"] = {"step_us": round(ms * 1e3, 1), "host_us_per_step": round(th, 1)}
            pipe.close()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
