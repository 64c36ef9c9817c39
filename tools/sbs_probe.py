import sys, os, time, ctypes as ct, statistics
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_2105_00619_b200 as pkg
S = pkg.sampler
lib = pkg._lib.lib
dev = torch.device("cuda", 0)
N, B, NB, K = 50000, 512, 97, 100
labels = torch.arange(N, device=dev, dtype=torch.int32) % K
offs, mem = S.class_index_dev(labels, K)
for G in (1, 8):
    for spd in (1, 2):
        cur = S.BatchCursor.from_device_index(S.plan([1.0 / K] * K, B, 1234), offs, mem)
        pkg._lib.check(lib.optb_sbs_set_profiling(cur._h, 1))
        ex = torch.empty(NB * B * spd, dtype=torch.int64, device=dev)
        cl = torch.empty(NB * B * spd, dtype=torch.int32, device=dev)
        for _ in range(3):
            cur.next_dev(NB * G * spd, 0, G, ex, cl)
        torch.cuda.synchronize()
        ph, host = [], []
        for _ in range(10):
            t0 = time.perf_counter()
            cur.next_dev(NB * G * spd, 0, G, ex, cl)
            host.append((time.perf_counter() - t0) * 1e6)
            torch.cuda.synchronize()
            p3 = [ct.c_float() for _ in range(3)]
            pkg._lib.check(lib.optb_sbs_profile(cur._h, *[ct.byref(x) for x in p3]))
            ph.append([x.value * 1e3 for x in p3])
        print("G", G, "spd", spd, "host us", round(statistics.median(host), 1),
              "upload/reshuffle/gather us", [round(statistics.median(p[i] for p in ph), 1) for i in range(3)])
