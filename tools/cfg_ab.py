"""A/B timing of a subset of bench.py's configuration sub-keys.

    python tools/cfg_ab.py C3_n9 C3_n18 [--reps N]

Runs bench.config_suite restricted to the named cases (substring match) and
prints one JSON object per case: fused / split images/s, encode / decode
fractions of the measured peak, the kernel that ran and the check.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    import paper_2105_00619_b200 as pkg
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    reps = 1
    if "--reps" in sys.argv:
        reps = int(sys.argv[sys.argv.index("--reps") + 1])
        args = [a for a in args if a != str(reps)]
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    peak, _ = bench.measured_peak()
    for r in range(reps):
        res = bench.config_suite(torch, pkg, dev, stream, peak, only=args or None)
        for k, v in res.items():
            keep = {x: v.get(x) for x in ("value", "kernel", "roundtrip_us", "hbm_frac", "encode_us", "decode_us",
                                          "encode_frac", "decode_frac", "check", "ms_per_step")}
            print(json.dumps({"case": k, "rep": r, **keep}), flush=True)


if __name__ == "__main__":
    main()
