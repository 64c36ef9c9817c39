"""Fused exact128 round trip around the C2 size: is the uneven last round of
tiles (49 664 images = 15.73 tiles per warp per phase) a measurable cost?

    python tools/bal_probe.py

Times optb_roundtrip_dev for stream sizes with 14.25 .. 16.1 tiles per warp
(15.0 = perfectly balanced) and prints the fraction of the measured peak.
"""
import sys, os, statistics, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_2105_00619_b200 as pkg
C = pkg.codec
dev = torch.device("cuda", 0)
s = torch.cuda.Stream()
P = 3072
res = {}
for rows in (44992, 46176, 47360, 48544, 49664, 49728, 50912):
    B = 16; nb = rows // 16
    L = C.layout(1, 16, P, B, nb)
    with torch.cuda.stream(s):
        src = torch.randint(0, 256, (rows, P), dtype=torch.uint8, device=dev)
        idx = torch.randperm(rows, device=dev)
        cont, offs = C.alloc_stream(L)
        out = torch.empty((rows, P), dtype=torch.uint8, device=dev)
        for _ in range(3):
            C.roundtrip_dev(L, src, cont, out, row_index=idx, stream=s)
        ts = []
        for rep in range(3):
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(11)]
            evs[0].record(s)
            for i in range(10):
                C.roundtrip_dev(L, src, cont, out, row_index=idx, stream=s)
                evs[i + 1].record(s)
            evs[-1].synchronize()
            ts += [evs[i].elapsed_time(evs[i + 1]) for i in range(10)]
        t = statistics.median(ts) / 1e3
    b = 2 * (rows * P + C.container_bytes(L)) + rows * 8
    tiles = rows // 16 * 6
    res[rows] = {"us": round(t * 1e6, 2), "frac": round(b / t / 1e9 / 6444.1, 4), "tiles_per_warp": round(tiles / 1184, 3),
                 "us_per_kimg": round(t * 1e6 / rows * 1000, 4)}
    del src, idx, cont, out
print(json.dumps(res, indent=0))
