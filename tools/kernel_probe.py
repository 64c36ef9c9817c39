"""Run one codec configuration a few times (for ncu captures of a single kernel pair).

    python tools/kernel_probe.py MODE PER_CHUNK P BATCH N_BATCHES [OUT_DTYPE] [REPS] [fused]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2105_00619_b200 as pkg
    C = pkg.codec
    mode, pc, P, B, nb = (int(x) for x in sys.argv[1:6])
    dt = getattr(torch, sys.argv[6]) if len(sys.argv) > 6 else torch.uint8
    reps = int(sys.argv[7]) if len(sys.argv) > 7 else 3
    L = C.layout(mode, pc, P, B, nb)
    x = torch.randint(0, 256, (B * nb, P), dtype=torch.uint8, device="cuda")
    cont, offs = C.alloc_stream(L)
    out = torch.empty((B * nb, P), dtype=dt, device="cuda")
    fused = len(sys.argv) > 8 and sys.argv[8] == "fused"
    for _ in range(reps):
        if fused:
            C.roundtrip_dev(L, x, cont, out, offsets=offs, scale=1 / 255)
        else:
            C.encode_dev(L, x, cont, offs)
            C.decode_dev(L, cont, out, offsets=offs, scale=1 / 255)
    C.sync()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
