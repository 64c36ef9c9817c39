"""Fused round-trip efficiency against launch size (tiles per warp).

    python tools/gran_probe.py

Times optb_roundtrip_dev (gather, u8 out) back to back for exact128 and
exact64 CIFAR streams of 32K..256K images and prints the fraction of the
measured HBM peak with the tiles each warp processes per phase.  A linear
fit t = fixed + rows * marginal separates the per-launch fixed cost (ramp,
phase switch, tail) from the marginal bandwidth.
"""
import sys, os, statistics, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_2105_00619_b200 as pkg
C = pkg.codec
dev = torch.device("cuda", 0)
s = torch.cuda.Stream()
res = {}
P = 3072
for mode, pc in ((1, 16), (0, 8)):
    for rows in (32768, 65536, 131072, 262144):
        B = 4096; nb = rows // B
        L = C.layout(mode, pc, P, B, nb)
        with torch.cuda.stream(s):
            src = torch.randint(0, 256, (rows, P), dtype=torch.uint8, device=dev)
            idx = torch.randperm(rows, device=dev)
            cont, offs = C.alloc_stream(L)
            out = torch.empty((rows, P), dtype=torch.uint8, device=dev)
            for _ in range(3):
                C.roundtrip_dev(L, src, cont, out, row_index=idx, stream=s)
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(11)]
            evs[0].record(s)
            for i in range(10):
                C.roundtrip_dev(L, src, cont, out, row_index=idx, stream=s)
                evs[i + 1].record(s)
            evs[-1].synchronize()
            t = statistics.median(evs[i].elapsed_time(evs[i + 1]) for i in range(10)) / 1e3
        b = 2 * (rows * P + C.container_bytes(L)) + rows * 8
        tiles = C.container_bytes(L) // (512 * (16 if mode == 1 else 8))
        res[f"mode{mode}_rows{rows}"] = {"us": round(t * 1e6, 1), "frac": round(b / t / 1e9 / 6444.1, 3),
                                          "tiles_per_warp": round(tiles / 1184, 1)}
        del src, idx, cont, out
print(json.dumps(res))
