"""Host cost of one enqueue, per API call (no GPU wait in between).

    python tools/launch_probe.py

Times, on the host, back-to-back async calls of optb_roundtrip_dev (C2
layout), optb_encode_dev, optb_decode_dev, the pipeline step (steps_per_draw
1 and 4) and a bare torch kernel launch for scale; each the median of 5
runs of 200 calls, after warm-up, with the device drained between runs.
"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2105_00619_b200 as pkg  # noqa: E402
from paper_2105_00619_b200.pipeline import Pipeline  # noqa: E402

C, S = pkg.codec, pkg.sampler
dev = torch.device("cuda", 0)
s = torch.cuda.Stream(dev)
N, P, B, NB, K = 50000, 3072, 512, 97, 100


def host_us(fn, n=200, runs=5):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    res = []
    for _ in range(runs):
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        res.append((time.perf_counter() - t0) / n * 1e6)
        torch.cuda.synchronize()
    return round(statistics.median(res), 2)


ds = torch.randint(0, 256, (N, P), dtype=torch.uint8, device=dev)
L = C.layout(1, 16, P, B, NB)
rows = B * NB
idx = torch.randint(0, N, (rows,), device=dev)
cont, offs = C.alloc_stream(L)
out = torch.empty((rows, P), dtype=torch.uint8, device=dev)
x = torch.empty(16, device=dev)
res = {"torch_add_": host_us(lambda: x.add_(1.0)),
       "roundtrip_dev": host_us(lambda: C.roundtrip_dev(L, ds, cont, out, row_index=idx, stream=s)),
       "encode_dev": host_us(lambda: C.encode_dev(L, ds, cont, row_index=idx, stream=s)),
       "decode_dev": host_us(lambda: C.decode_dev(L, cont, out, stream=s))}
labels = torch.arange(N, device=dev, dtype=torch.int32) % K
co, cm = S.class_index_dev(labels, K)
for spd in (1, 4):
    cur = S.BatchCursor.from_device_index(S.plan([1.0 / K] * K, B, 1234), co, cm)
    pipe = Pipeline(cur, ds, 1, B, NB, steps_per_draw=spd)
    res[f"pipeline_step_spd{spd}"] = host_us(lambda: pipe.step(out, s))
    pipe.close()
print(json.dumps(res))
