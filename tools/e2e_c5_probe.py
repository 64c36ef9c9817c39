"""Where the C5 e2e leg loses against the PCIe bidirectional ceiling.

    python tools/e2e_c5_probe.py [--steps 10,30]

Times, on the bench's C5 buffers (3.2 GB pinned dataset up, 3.2 GB decoded
rows down per step):
  raw_both     : one H2D and one D2H copy at once, no dependencies (ceiling)
  raw_pattern  : the leg's dependency pattern with copies only -- H2D(k) on
                 the up stream, D2H(k) after H2D(k) on the down stream,
                 double-buffered -- per step, for each K
  raw_chunked  : the same with each copy split into C pieces, the D2H piece j
                 waiting only for H2D piece j (finer interleave of directions)
  raw_split    : C pieces each way, the step's D2H waiting for its whole H2D
                 (the leg's real dependency: the kernel needs every row)
  step_host    : optb_pipeline_step_host, for each K
Prints one JSON line.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", default="10,30")
    ap.add_argument("--chunks", default="4,16")
    ap.add_argument("--skip-pipeline", action="store_true")
    args = ap.parse_args()
    import torch

    import bench
    dev = torch.device("cuda", 0)
    N, P = bench.N_EXAMPLES, bench.P
    nbytes = N * P
    host_in = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    host_in.copy_(torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device=dev).cpu())
    host_out = [torch.empty(nbytes, dtype=torch.uint8).pin_memory() for _ in range(2)]
    d_in = [torch.empty(nbytes, dtype=torch.uint8, device=dev) for _ in range(2)]
    d_out = [torch.empty(nbytes, dtype=torch.uint8, device=dev) for _ in range(2)]
    up, down = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    res = {"bytes_each_way": nbytes}

    def ev():
        return torch.cuda.Event(enable_timing=True)

    # ceiling: both directions at once
    for _ in range(2):
        e0, e1, e2 = ev(), ev(), ev()
        torch.cuda.synchronize()
        e0.record(up)
        down.wait_event(e0)
        with torch.cuda.stream(up):
            d_in[0].copy_(host_in, non_blocking=True)
        with torch.cuda.stream(down):
            host_out[0].copy_(d_out[0], non_blocking=True)
        e1.record(up)
        e2.record(down)
        torch.cuda.synchronize()
        t = max(e0.elapsed_time(e1), e0.elapsed_time(e2))
    res["raw_both_ms"] = round(t, 2)
    res["raw_both_gbs"] = round(2 * nbytes / t / 1e6, 1)
    for name, d, h in (("h2d", d_in[0], host_in), ("d2h", host_out[0], d_out[0])):
        e0, e1 = ev(), ev()
        torch.cuda.synchronize()
        e0.record(up)
        with torch.cuda.stream(up):
            d.copy_(h, non_blocking=True)
        e1.record(up)
        torch.cuda.synchronize()
        res[f"raw_{name}_gbs"] = round(nbytes / e0.elapsed_time(e1) / 1e6, 1)

    def pattern(K, C, lockstep=True):
        per = (nbytes + C - 1) // C
        origin, end = ev(), ev()
        # the leg's events: used[b] = "kernel" k done (after H2D(k) and
        # D2H(k-2)); H2D(k+2) waits for it, D2H(k) follows it
        used = [torch.cuda.Event(), torch.cuda.Event()]
        down_done = [torch.cuda.Event(), torch.cuda.Event()]
        cs = torch.cuda.Stream(dev)
        torch.cuda.synchronize()
        origin.record(up)
        down.wait_event(origin)
        cs.wait_event(origin)
        for k in range(K):
            b = k % 2
            if k >= 2:
                up.wait_event(used[b])
            pieces = []
            for j in range(0, nbytes, per):
                with torch.cuda.stream(up):
                    d_in[b][j:j + per].copy_(host_in[j:j + per], non_blocking=True)
                e = torch.cuda.Event()
                e.record(up)
                pieces.append((j, e))
            cs.wait_event(pieces[-1][1])
            if k >= 2:
                cs.wait_event(down_done[b])
            used[b].record(cs)
            for j, e in pieces:
                down.wait_event(e if lockstep else pieces[-1][1])
                with torch.cuda.stream(down):
                    host_out[b][j:j + per].copy_(d_out[b][j:j + per], non_blocking=True)
            down_done[b].record(down)
        end.record(down)
        up_end = ev()
        up_end.record(up)
        torch.cuda.synchronize()
        return max(origin.elapsed_time(end), origin.elapsed_time(up_end)) / K

    steps = [int(s) for s in args.steps.split(",")]
    for K in steps:
        res[f"raw_pattern_K{K}_ms"] = round(pattern(K, 1), 2)
        for C in [int(c) for c in args.chunks.split(",")]:
            res[f"raw_chunked{C}_K{K}_ms"] = round(pattern(K, C), 2)
            res[f"raw_split{C}_K{K}_ms"] = round(pattern(K, C, lockstep=False), 2)
    del d_out
    if not args.skip_pipeline:
        import paper_2105_00619_b200 as pkg
        from paper_2105_00619_b200.pipeline import Pipeline
        S = pkg.sampler
        del d_in
        torch.cuda.empty_cache()
        ds = torch.empty((N, P), dtype=torch.uint8, device=dev)
        ds.view(-1).copy_(host_in)
        ds_host = host_in.view(N, P)
        labels = torch.arange(N, device=dev, dtype=torch.int32) % bench.N_CLASSES
        offs, mem = S.class_index_dev(labels, bench.N_CLASSES)
        cur = S.BatchCursor.from_device_index(S.plan([1.0 / bench.N_CLASSES] * bench.N_CLASSES, bench.BATCH,
                                                     bench.SEED), offs, mem)
        pipe = Pipeline(cur, ds, bench.MODE, bench.BATCH, bench.BATCHES_PER_STEP, per_chunk=bench.PER_CHUNK)
        del ds
        torch.cuda.empty_cache()
        stream = torch.cuda.Stream(dev)
        outs = [h.view(N, P) for h in host_out]
        kk = [0]

        def step():
            pipe.step_host(ds_host, outs[kk[0] % 2], stream)
            kk[0] += 1
        with torch.cuda.stream(stream):
            for _ in range(2):
                step()
            pipe.host_wait(stream)
            torch.cuda.synchronize()
            for K in steps:
                e0, e1 = ev(), ev()
                e0.record(stream)
                for _ in range(K):
                    step()
                pipe.host_wait(stream)
                e1.record(stream)
                torch.cuda.synchronize()
                res[f"step_host_K{K}_ms"] = round(e0.elapsed_time(e1) / K, 2)
        pipe.close()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
