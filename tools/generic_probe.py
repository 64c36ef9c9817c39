import sys, json, torch
sys.path.insert(0, "/root/repo")
import bench, paper_2105_00619_b200 as pkg
C = pkg.codec
dev = torch.device("cuda", 0); s = torch.cuda.Stream(dev)
peak, _ = bench.measured_peak()
for (mode, pc, P, B, nb) in ((1, 16, 154587, 256, 2), (1, 16, 150528, 256, 2), (0, 8, 3000, 4096, 16), (0, 8, 3072, 4096, 16)):
    L = C.layout(mode, pc, P, B, nb)
    rows = B * nb
    with torch.cuda.stream(s):
        src = torch.randint(0, 256, (rows, P), dtype=torch.uint8, device=dev)
        cont, offs = C.alloc_stream(L)
        out = torch.empty((rows, P), dtype=torch.uint8, device=dev)
        te = bench.b2b_time(torch, lambda: C.encode_dev(L, src, cont, offs, stream=s), s, 10)
        td = bench.b2b_time(torch, lambda: C.decode_dev(L, cont, out, offsets=offs, stream=s), s, 10)
        tr = bench.b2b_time(torch, lambda: C.roundtrip_dev(L, src, cont, out, offsets=offs, stream=s), s, 10)
        C.sync(0, s)
        ok = bool(torch.equal(out, src))
    cb = C.container_bytes(L)
    print(json.dumps({"P": P, "mode": mode, "enc_frac": round((rows*P+cb)/te/1e9/peak, 3), "dec_frac": round((rows*P+cb)/td/1e9/peak, 3),
                      "rt_us": round(tr*1e6, 1), "kind": C.last_roundtrip_kind(), "ok": ok}))
