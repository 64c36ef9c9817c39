"""bench.py's config suite (C1-C4, C2) under the current environment, one
compact JSON line: images/s and HBM fractions per config.  For A/B runs of
the OPTB_* switches:

    OPTB_ENCODE_BULK=0 python tools/ab_env.py [name-substring ...]
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
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    peak, _ = bench.measured_peak()
    res = bench.config_suite(torch, pkg, dev, stream, peak)
    keys = sys.argv[1:]
    out = {k: {kk: v.get(kk) for kk in ("value", "kernel", "hbm_frac", "encode_us", "decode_us", "encode_frac",
                                         "decode_frac", "check")}
           for k, v in res.items() if not keys or any(s in k for s in keys)}
    env = {k: v for k, v in os.environ.items() if k.startswith("OPTB_")}
    print(json.dumps({"env": env, "configs": out}))


if __name__ == "__main__":
    main()
