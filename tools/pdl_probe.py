import sys, os, statistics
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_2105_00619_b200 as pkg
from paper_2105_00619_b200.pipeline import Pipeline
C, S = pkg.codec, pkg.sampler
dev = torch.device("cuda", 0)
N, P, B, NB, K = 50000, 3072, 512, 97, 100
ds = torch.randint(0, 256, (N, P), dtype=torch.uint8, device=dev)
labels = torch.arange(N, device=dev, dtype=torch.int32) % K
offs, mem = S.class_index_dev(labels, K)
out = torch.empty((B * NB, P), dtype=torch.uint8, device=dev)
s = torch.cuda.Stream()
res = []
for rep in range(3):
    cur = S.BatchCursor.from_device_index(S.plan([1.0 / K] * K, B, 1234), offs, mem)
    pipe = Pipeline(cur, ds, 1, B, NB, steps_per_draw=4, record_timings=False)
    for _ in range(12): pipe.step(out, s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(200): pipe.step(out, s)
    e1.record(s); e1.synchronize()
    res.append(e0.elapsed_time(e1) / 200 * 1e3)
    pipe.close()
L = C.layout(1, 16, P, B, NB)
cont, _ = C.alloc_stream(L)
idx = torch.randperm(N, device=dev)[: B * NB]
for _ in range(5): C.roundtrip_dev(L, ds, cont, out, row_index=idx, stream=s)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(200): C.roundtrip_dev(L, ds, cont, out, row_index=idx, stream=s)
e1.record(s); e1.synchronize()
print("PDL", os.environ.get("OPTB_PDL", "0"), "pipeline us/step", [round(x, 2) for x in res], "bare roundtrip us", round(e0.elapsed_time(e1) / 200 * 1e3, 2))
