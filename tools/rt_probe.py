"""One fused round trip per mode on a C3-sized stream (for ncu captures).

    python tools/rt_probe.py MODE PER_CHUNK [ROWS] [REPS]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2105_00619_b200 as pkg
    C = pkg.codec
    mode, pc = int(sys.argv[1]), int(sys.argv[2])
    rows = int(sys.argv[3]) if len(sys.argv) > 3 else 65536
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    P, B = 3072, 4096
    L = C.layout(mode, pc, P, B, rows // B)
    src = torch.randint(0, 256, (rows, P), dtype=torch.uint8, device="cuda")
    idx = torch.randperm(rows, device="cuda")
    cont, offs = C.alloc_stream(L)
    out = torch.empty((rows, P), dtype=torch.uint8, device="cuda")
    for _ in range(reps):
        C.roundtrip_dev(L, src, cont, out, offsets=offs, row_index=idx)
    C.sync()


if __name__ == "__main__":
    main()
