"""Timeline of bench.py's e2e leg (host buffers in and out every step).

    python tools/e2e_probe.py [--steps 8]

Runs the same double-buffered loop as bench.run_e2e -- bulk H2D of the
epoch's pinned dataset (copy stream), optb_pipeline_step (compute stream),
D2H of the decoded rows (copy stream) -- with CUDA events around every
copy and step, and prints per-step durations and start offsets (ms), so
the achieved overlap can be compared with the PCIe bound.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--d2h-chunks", type=int, default=1)
    args = ap.parse_args()
    import torch

    import bench
    import paper_2105_00619_b200 as pkg
    from paper_2105_00619_b200.pipeline import Pipeline
    S = pkg.sampler
    dev = torch.device("cuda", 0)
    N, P, B, NB, K = bench.N_EXAMPLES, bench.P, bench.BATCH, bench.BATCHES_PER_STEP, bench.N_CLASSES
    rows = B * NB
    stream = torch.cuda.Stream(dev)
    copy_in, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ds = torch.randint(0, 256, (N, P), dtype=torch.uint8, device=dev)
    ds_host = ds.cpu().pin_memory()
    labels = torch.arange(N, device=dev, dtype=torch.int32) % K
    offs, mem = S.class_index_dev(labels, K)
    cur = S.BatchCursor.from_device_index(S.plan([1.0 / K] * K, B, 1234), offs, mem)
    ds_devs = [torch.empty_like(ds) for _ in range(2)]
    pipe = Pipeline(cur, ds_devs[0], 1, B, NB, steps_per_draw=2)
    outs = [torch.empty((rows, P), dtype=torch.uint8, device=dev) for _ in range(2)]
    out_hosts = [torch.empty((rows, P), dtype=torch.uint8).pin_memory() for _ in range(2)]
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    n = args.steps + 2
    h0, h1, c0, c1, d0, d1 = ([E() for _ in range(n + 1)] for _ in range(6))
    enc_done = [torch.cuda.Event(), torch.cuda.Event()]
    up_done = [torch.cuda.Event(), torch.cuda.Event()]
    down_done = [torch.cuda.Event(), torch.cuda.Event()]
    origin = E()

    def upload(k):
        b = k % 2
        if k >= 2:
            copy_in.wait_event(enc_done[b])
        with torch.cuda.stream(copy_in):
            h0[k].record(copy_in)
            ds_devs[b].copy_(ds_host, non_blocking=True)
            h1[k].record(copy_in)
        up_done[b].record(copy_in)

    origin.record(stream)
    torch.cuda.synchronize()
    for k in range(n):
        b = k % 2
        if k == 0:
            upload(0)
        upload(k + 1) if k + 1 < n + 1 else None
        stream.wait_event(up_done[b])
        pipe.set_dataset(ds_devs[b])
        if k >= 2:
            stream.wait_event(down_done[b])
        c0[k].record(stream)
        pipe.step(outs[b], stream)
        c1[k].record(stream)
        enc_done[b].record(stream)
        d2h.wait_event(enc_done[b])
        with torch.cuda.stream(d2h):
            d0[k].record(d2h)
            per = (rows + args.d2h_chunks - 1) // args.d2h_chunks
            for j in range(0, rows, per):
                out_hosts[b][j:j + per].copy_(outs[b][j:j + per], non_blocking=True)
            d1[k].record(d2h)
        down_done[b].record(d2h)
    torch.cuda.synchronize()
    res = []
    for k in range(2, n):
        res.append({"step": k,
                    "h2d_next": [round(origin.elapsed_time(h0[k + 1]), 3), round(h0[k + 1].elapsed_time(h1[k + 1]), 3)],
                    "compute": [round(origin.elapsed_time(c0[k]), 3), round(c0[k].elapsed_time(c1[k]), 3)],
                    "d2h": [round(origin.elapsed_time(d0[k]), 3), round(d0[k].elapsed_time(d1[k]), 3)]})
    per_step = (origin.elapsed_time(d1[n - 1]) - origin.elapsed_time(d1[2])) / (n - 3)
    print(json.dumps({"ms_per_step": round(per_step, 3), "timeline_ms [start, duration]": res}))
    pipe.close()


if __name__ == "__main__":
    main()
