"""One launch of every kernel family on its BASELINE configuration, for an
`ncu --set full` capture (the per-kernel counters behind DESIGN.md §4):

    ncu --set full --clock-control none --import-source on -o k \
        python tools/ncu_kernels.py
    python tools/ncu_summary.py --full k.ncu-rep r02

Cases (each launched twice; ncu replays every launch with a cold L2):
  C5  pipeline step (SBS kernels + k_roundtrip_il<exact128,u8>) at 2^20 images
  C1  exact64 fused -> u8 / fp32
  C3  lossless64 n=9 / lossless128 n=18 / f64 n=6: encode, decode, fused
  C3L lossless64 / lossless128: split encode + decode only
  C3LF lossless64 / lossless128: fused round trips only
  C3FF f64 (n=6) / exact64 (n=8): fused round trips only
  C3S exact128 (n=16) / f64 (n=6): split encode + decode only
  C1S exact64 -> u8 / fp32 and C4 exact128 -> bf16 (8 batches): split only
  C4  ImageNet exact128: fused -> bf16, split encode + decode -> bf16
  K7  class index over 2^20 labels
  io  record loader (CHW -> HWC), 4096 CIFAR records
"""
import ctypes as ct
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import paper_2105_00619_b200 as pkg
    from paper_2105_00619_b200.pipeline import Pipeline
    C, S = pkg.codec, pkg.sampler
    dev = torch.device("cuda", 0)
    s = torch.cuda.Stream(dev)
    scale = float(np.float32(1.0) / np.float32(255.0))
    only = set(sys.argv[1:])

    def want(tag):
        return not only or tag in only

    with torch.cuda.stream(s):
        if want("C5"):
            N = 1 << 20
            ds = torch.empty((N, 3072), dtype=torch.uint8, device=dev)
            ctx = pkg._lib.context(0)
            pkg._lib.check(pkg._lib.lib.optb_synth_pixels_dev(ctx, 7, 0, N, 3072, ct.c_void_p(ds.data_ptr()), 3072,
                                                              ct.c_void_p(s.cuda_stream)))
            labels = torch.arange(N, device=dev, dtype=torch.int32) % 100
            offs, mem = S.class_index_dev(labels, 100)
            cur = S.BatchCursor.from_device_index(S.plan([0.01] * 100, 512, 1234), offs, mem)
            pipe = Pipeline(cur, ds, 1, 512, N // 512)
            out = torch.empty((N, 3072), dtype=torch.uint8, device=dev)
            for _ in range(2):
                pipe.step(out, s)
            C.sync(0, s)
            pipe.close()
            del ds, out
            torch.cuda.empty_cache()

        def codec(mode, n, P, B, nb, dt=torch.uint8, fused=True, split=True):
            L = C.layout(mode, n, P, B, nb)
            x = torch.randint(0, 256, (B * nb, P), dtype=torch.uint8, device=dev)
            cont, offs_ = C.alloc_stream(L)
            out = torch.empty((B * nb, P), dtype=dt, device=dev)
            for _ in range(2):
                if fused:
                    C.roundtrip_dev(L, x, cont, out, offsets=offs_, scale=scale, stream=s)
                if split:
                    C.encode_dev(L, x, cont, offs_, stream=s)
                    C.decode_dev(L, cont, out, offsets=offs_, scale=scale, stream=s)
            C.sync(0, s)
            del x, cont, out

        if want("C1"):
            codec(0, 8, 3072, 128, 512, fused=True, split=False)
            codec(0, 8, 3072, 128, 512, torch.float32, fused=True, split=False)
        if want("C3"):
            codec(3, 9, 3072, 4096, 16)
            codec(4, 18, 3072, 4096, 16)
            codec(2, 6, 3072, 4096, 16)
        if want("C1S"):  # exact64 split encode + decode (u8, fp32) and the C4 bf16 split pair
            codec(0, 8, 3072, 128, 512, fused=False)
            codec(0, 8, 3072, 128, 512, torch.float32, fused=False)
            codec(1, 16, 224 * 224 * 3, 256, 8, torch.bfloat16, fused=False)
        if want("C3S"):  # exact128 / f64 split encode + decode only (source-level captures)
            codec(1, 16, 3072, 4096, 16, fused=False)
            codec(2, 6, 3072, 4096, 16, fused=False)
        if want("C3FF"):  # f64 and exact64 fused round trips only (source-level captures)
            codec(2, 6, 3072, 4096, 16, split=False)
            codec(0, 8, 3072, 4096, 16, split=False)
        if want("C3LF"):  # lossless fused round trips only (source-level captures)
            codec(3, 9, 3072, 4096, 16, split=False)
            codec(4, 18, 3072, 4096, 16, split=False)
        if want("C3L"):  # lossless split kernels only (source-level captures)
            codec(3, 9, 3072, 4096, 16, fused=False)
            codec(4, 18, 3072, 4096, 16, fused=False)
        if want("C4"):
            codec(1, 16, 224 * 224 * 3, 256, 1, torch.bfloat16)
        if want("K7"):
            labels = torch.arange(1 << 20, device=dev, dtype=torch.int32) % 100
            for _ in range(2):
                S.class_index_dev(labels, 100)
            C.sync(0, s)
        if want("io"):
            rec = np.random.default_rng(0).integers(0, 256, size=(4096, 3073), dtype=np.uint8)
            rec[:, 0] %= 10
            with tempfile.NamedTemporaryFile(suffix=".bin") as f:
                f.write(rec.tobytes())
                f.flush()
                for _ in range(2):
                    C.load_records_dev(f.name, C.ImageShape(32, 32, 3), 10, max_records=4096)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
