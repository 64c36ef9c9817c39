import sys, time, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_2105_00619_b200 as pkg
from paper_2105_00619_b200.pipeline import Pipeline
S = pkg.sampler
dev = torch.device("cuda", 0)
N, P, B, NB, K = 50000, 3072, 512, 97, 100
ds = torch.randint(0, 256, (N, P), dtype=torch.uint8, device=dev)
labels = torch.arange(N, device=dev, dtype=torch.int32) % K
offs, mem = S.class_index_dev(labels, K)
for spd in (1, 2, 4):
    cur = S.BatchCursor.from_device_index(S.plan([1.0 / K] * K, B, 1234), offs, mem)
    pipe = Pipeline(cur, ds, 1, B, NB, steps_per_draw=spd)
    out = torch.empty((B * NB, P), dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    for _ in range(8):
        pipe.step(out, s)
    torch.cuda.synchronize()
    res = []
    for rep in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(6):
            pipe.step(out, s)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        res.append((t1 - t0) / 6 * 1e6)
    print("spd", spd, "host us/step", [round(x, 1) for x in res])
    pipe.close()
