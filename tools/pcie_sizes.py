import torch, time, json
dev = torch.device("cuda", 0)
res = {}
for nb in (153_600_000, 805_306_368, 3_221_225_472):
    h_in = torch.empty(nb, dtype=torch.uint8).pin_memory(); h_out = torch.empty(nb, dtype=torch.uint8).pin_memory()
    h_in.fill_(1); h_out.fill_(2)
    d_a = torch.empty(nb, dtype=torch.uint8, device=dev); d_b = torch.empty(nb, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    def t(fn, reps=3):
        fn(); torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps): fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / reps
    up = t(lambda: d_a.copy_(h_in, non_blocking=True))
    dn = t(lambda: h_out.copy_(d_b, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
    bi = t(both)
    res[nb] = {"h2d_gbs": nb/up/1e9, "d2h_gbs": nb/dn/1e9, "bidir_gbs": 2*nb/bi/1e9}
    print(nb, res[nb], flush=True)
    del h_in, h_out, d_a, d_b
