"""Fused round trip: interleaved (deep / wide shape) vs phase-ordered kernel
against launch size, exact128, u8 and bf16 outputs.

    python tools/il_probe.py

Each size rotates over enough distinct (rows, containers, output) sets that
every launch finds its inputs evicted from L2 (>= 400 MB per rotation), like
the C4 per-batch case.  Prints us per launch and the tiles per warp of the
wide shape (1184 warps).
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2105_00619_b200 as pkg  # noqa: E402

C = pkg.codec
dev = torch.device("cuda", 0)
s = torch.cuda.Stream()
P = 3072
res = {}
for dt in (torch.uint8, torch.bfloat16):
    for rows in (2048, 4096, 8192, 12288, 16384, 24576, 32768, 49152, 65536):
        B = min(rows, 4096)
        nb = rows // B
        L = C.layout(1, 16, P, B, nb)
        per = rows * P * (2 + dt.itemsize)
        k = max(2, -(-400_000_000 // per))
        with torch.cuda.stream(s):
            sets = []
            for _ in range(k):
                cont, offs = C.alloc_stream(L)
                sets.append((torch.randint(0, 256, (rows, P), dtype=torch.uint8, device=dev), cont,
                             torch.empty((rows, P), dtype=dt, device=dev)))
        tiles_per_warp = rows / 16 * (P // 16) / 32 / 1184
        r = {"tiles_per_warp_wide": round(tiles_per_warp, 2)}
        for name, env in (("phase", {"OPTB_RT_INTERLEAVE": "0"}),
                          ("il_wide", {"OPTB_IL_SHAPE": "wide", "OPTB_IL_BULK": "1"}),
                          ("il_wide_lane_st", {"OPTB_IL_SHAPE": "wide", "OPTB_IL_BULK": "0"}),
                          ("il_deep", {"OPTB_IL_SHAPE": "deep"}), ("default", {})):
            for kk in ("OPTB_RT_INTERLEAVE", "OPTB_IL_SHAPE", "OPTB_IL_BULK"):
                os.environ.pop(kk, None)
            os.environ.update(env)
            if name == "il_deep" and dt != torch.uint8:
                continue
            with torch.cuda.stream(s):
                for i in range(2 * k):
                    x, cont, out = sets[i % k]
                    C.roundtrip_dev(L, x, cont, out, scale=1 / 255 if dt != torch.uint8 else 1.0, stream=s)
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                n = max(8, 2 * k)
                ev[0].record(s)
                for i in range(n):
                    x, cont, out = sets[i % k]
                    C.roundtrip_dev(L, x, cont, out, scale=1 / 255 if dt != torch.uint8 else 1.0, stream=s)
                ev[1].record(s)
                ev[1].synchronize()
            r[name + "_us"] = round(ev[0].elapsed_time(ev[1]) / n * 1e3, 1)
        for kk in ("OPTB_RT_INTERLEAVE", "OPTB_IL_SHAPE", "OPTB_IL_BULK"):
            os.environ.pop(kk, None)
        r["default_kernel"] = C.last_roundtrip_kind()
        res[f"{str(dt).replace('torch.', '')}_{rows}"] = r
        del sets
        print(json.dumps({f"{str(dt).replace('torch.', '')}_{rows}": r}), flush=True)
