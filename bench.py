"""Benchmark: images/s encode+decode (and achieved HBM GB/s vs peak) per BASELINE.json.

Headline workload (BASELINE.json configs[4], "C5"): a 2^20-image synthetic
CIFAR-shaped stream (1 048 576 x 32x32x3 u8 = 3.2 GB, labels e % 100)
resident in HBM on every GPU; selective batch sampling with uniform weights
over 100 classes, batch 512, seed 1234; every step is one epoch of the
reference's draw stream per GPU (floor(2^20 / 512) = 2048 batches): SBS draws
(side stream) -> gather-encode of the drawn rows into exact128 containers ->
decode back to u8 rows, one fused launch per step (optb_pipeline_step).
Containers are materialised in HBM.  N GPUs: one process per GPU, each keeps
the global stream's batches t % N == rank (weak scaling, no collective on the
data path).  C1-C4 and the round-1 C2 headline are reported as sub-keys
under "configs".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--gpus N > 1 without a torchrun environment re-launches itself under
torch.distributed.run with N ranks.  Rank 0 prints one JSON line.
`--impl reference` times the reference's own CPU implementation
(oracle/_ref, compiled from /root/reference's sources) on the host cores over
a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_EXAMPLES = 1 << 20           # C5: 2^20-image stream
N_CLASSES = 100
BATCH = 512
SEED = 1234
DATA_SEED = 7                  # RunConfig::data_seed (runner.hpp:34)
P = 32 * 32 * 3
BATCHES_PER_STEP = N_EXAMPLES // BATCH  # 2048: one epoch per GPU (runner.cpp:52-57)
MODE = 1                       # ExactInt128, the reference default (runner.hpp:52)
PER_CHUNK = 16
METRIC = "images/sec encode+decode (and achieved HBM GB/s vs peak) at 1/2/4/8 B200"
UNIT = "images/s"


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def config(world):
    return {"workload": "C5: 2^20-image CIFAR-shaped stream (1048576 x 32x32x3 u8, 3.2 GB) in HBM per GPU, SBS "
                        "(uniform 100 classes, B=512, seed 1234) + exact128 gather-encode + decode to u8; one step = "
                        "one epoch = 2048 batches per GPU",
            "global_batch": BATCH, "batches_per_step_per_gpu": BATCHES_PER_STEP, "mode": "exact128",
            "per_chunk": PER_CHUNK, "image": [32, 32, 3], "decode_out": "u8", "dataset_images": N_EXAMPLES,
            "parallelism": f"independent batch shards x{world} (t % N == rank), no data-path collective",
            "l2": "inputs larger than L2: 3.2 GB dataset (25x the 126 MB L2); every step streams 3.2 GB of "
                  "gathered rows in and 3.2 GB of containers + 3.2 GB of decoded rows out",
            "pipeline": "native optb_pipeline: the next epoch's SBS draws on a side stream overlap the current "
                        "step's gather-encode + decode, one optb_roundtrip_dev launch per step (each warp "
                        "stores an encoded tile into the HBM container stream and decodes it one tile later, "
                        "reading it back while it is still in L2)"}


# ---------------------------------------------------------------- collectives
# Control-plane collectives of the run (barriers, the max over ranks of the
# device times): NCCL with one process per GPU, gloo when ranks share a GPU
# (then the per-rank times are summed so the whole-job rate is never overstated).
COLL = {"group": None, "device": None, "op": None}


def coll_barrier(dist):
    g = COLL["group"]
    if g is not None:
        dist.barrier(group=g, device_ids=[COLL["device"].index])
    else:
        dist.barrier()


def coll_reduce_ms(torch, dist, ms):
    t = torch.tensor([float(ms)], device=COLL["device"])
    dist.all_reduce(t, op=COLL["op"], group=COLL["group"])
    return float(t.item())


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clocks and throttle reasons with NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001
            self.nv, self.err = None, str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.001)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "")}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kname):
    """dram read+write bytes per launch of `kname` from the committed ncu
    --set full summary (profiles/ncu_summary.json), with the capture's tag."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
    except Exception:  # noqa: BLE001
        return None, None
    # keys are "<case>:<kernel>" (tools/ncu_cases.sh; the headline kernel is
    # captured at C5) or bare kernel names; ncu names carry every template argument
    ks = sorted(d.get("kernels", {}).items(), key=lambda kv: not kv[0].startswith("C5:"))
    for kn, kv in ks:
        kn = kn.split(":", 1)[1] if ":" in kn.split("<")[0] else kn
        if kn == kname or kn.startswith(kname[:-1] + ","):
            return kv.get("dram_bytes_per_launch"), d.get("tag")
    return None, None


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# ---------------------------------------------------------------- reference side (checker + CPU baseline)
# Everything below that touches oracle/ is the CHECKER and the CPU BASELINE:
# the reference library compiled from its own sources (oracle/_ref), or the C
# restatement when it was not built.  It never runs inside a timed GPU region.
class RefStream:
    """The reference BatchCursor over the headline stream (checker): yields
    this rank's draws of step k, in order."""

    def __init__(self, labels, world, rank):
        import ctypes as ct

        import oracle as O
        self.O, self.ct, self.world, self.rank = O, ct, world, rank
        self.off = np.zeros(N_CLASSES + 1, np.uint64)
        self.mem = np.zeros(len(labels), np.int64)
        if O.ref_available():
            R = O.REF
            buf = ct.create_string_buffer(512)
            R.ref_class_index(O.ptr(labels, O.i32p), len(labels), N_CLASSES, O.ptr(self.off, O.u64p),
                              O.ptr(self.mem, O.i64p), buf, 512)
            w = np.full(N_CLASSES, 1.0 / N_CLASSES)
            st = ct.c_int(0)
            self.h = R.ref_cursor_create(O.ptr(w, O.f64p), N_CLASSES, BATCH, SEED, O.ptr(self.off, O.u64p),
                                         O.ptr(self.mem, O.i64p), ct.byref(st), buf, 512)
            self.kind = "reference"
        else:
            self.off, self.mem = O.class_index(labels, N_CLASSES)
            self.cur = O.Cursor(O.sbs_plan([1.0 / N_CLASSES] * N_CLASSES, BATCH), self.off, self.mem, BATCH, SEED)
            self.h, self.kind = None, "port"
        self.steps = 0

    def next_batches(self, n):
        if self.h is not None:
            ex = np.zeros(n * BATCH, np.int64)
            self.O.REF.ref_cursor_next(self.h, n, self.O.ptr(ex, self.O.i64p), None)
            return ex
        return self.cur.next(n)[0]

    def step(self, batches_per_rank):
        ex = self.next_batches(batches_per_rank * self.world).reshape(-1, BATCH)
        self.steps += 1
        return np.ascontiguousarray(ex[self.rank::self.world].reshape(-1))

    def close(self):
        if self.h is not None:
            self.O.REF.ref_cursor_destroy(self.h)
            self.h = None


class RefBaseline:
    """The reference CPU path (oracle/_ref = the reference compiled from its
    own sources; else the C oracle port) on the headline stream: per sample,
    BatchCursor::next draws, then per batch image_of gather + codec::encode
    per 16-image chunk + codec::decode, batches split over `threads` host
    threads (the functions are reentrant)."""

    def __init__(self, ds, labels):
        import oracle as O
        self.O, self.ds, self.labels = O, ds, labels
        if O.ref_available():
            self.rs = RefStream(labels, 1, 0)
            self.dsh = O.REF.ref_dataset_create(O.ptr(ds, O.u8p), ds.shape[0], 32, 32, 3)
            self.kind = "reference"
        else:
            off, mem = O.class_index(labels, N_CLASSES)
            self.cur = O.Cursor(O.sbs_plan([1.0 / N_CLASSES] * N_CLASSES, BATCH), off, mem, BATCH, SEED)
            self.dsh, self.kind = None, "port"

    def rate(self, n_batches: int, threads: int):
        import ctypes as ct
        O = self.O
        t0 = time.perf_counter()
        if self.dsh is not None:
            ex = np.zeros(n_batches * BATCH, np.int64)
            O.REF.ref_cursor_next(self.rs.h, n_batches, O.ptr(ex, O.i64p), None)
            t_sbs = time.perf_counter() - t0
            chk = ct.c_uint64(0)
            secs = O.REF.ref_bench_roundtrip(self.dsh, MODE, O.ptr(ex, O.i64p), n_batches, BATCH, threads, 0,
                                             ct.byref(chk)) + t_sbs
        else:
            threads = 1
            ex, _ = self.cur.next(n_batches)
            cont, _ = O.encode_stream(self.ds, ex, MODE, PER_CHUNK, BATCH, n_batches)
            O.decode_stream(cont, None, MODE, PER_CHUNK, P, BATCH, n_batches)
            secs = time.perf_counter() - t0
        sample = (f"{n_batches} batches x {BATCH} images of the C5 stream (BatchCursor::next draws + image_of "
                  f"gather + codec::encode/decode per 16-image chunk), {threads} host threads")
        return n_batches * BATCH / secs, sample, threads

    def close(self):
        if self.dsh is not None:
            self.O.REF.ref_dataset_destroy(self.dsh)
            self.rs.close()
            self.dsh = None


def host_dataset():
    import oracle as O
    labels = (np.arange(N_EXAMPLES) % N_CLASSES).astype(np.int32)
    return O.synth_pixels(DATA_SEED, 0, N_EXAMPLES, P), labels


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    ds, labels = host_dataset()
    rb = RefBaseline(ds, labels)
    sample_batches = max(threads * 2, 8)
    for _ in range(args.warmup):
        rb.rate(sample_batches, threads)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v, sample, used = rb.rate(sample_batches, threads)
        vals.append(v)
    wall = time.perf_counter() - t0
    rb.close()
    v = statistics.median(vals)
    line = {"metric": METRIC, "value": round(v, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(wall / args.steps * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": config(world), "impl": "reference",
            "cpu_baseline": {"value": round(v, 1), "unit": UNIT, "cores": used, "kind": rb.kind,
                             "sample": sample + f", median of {args.steps} steps", "cpu_model": cpu_model()},
            "e2e": {"value": round(v, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- launcher
def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn(args):
    """--gpus N > 1 outside torchrun: re-launch this script with N ranks, one
    per GPU, and pass rank 0's line through."""
    import torch
    n_dev = torch.cuda.device_count()
    if n_dev < args.gpus and not args.oversubscribe:
        print(f"bench.py: --gpus {args.gpus} but only {n_dev} GPU(s) visible", file=sys.stderr, flush=True)
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    print("bench.py: launching " + " ".join(cmd[2:6]), file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def b2b_time(torch, fn, stream, reps, warm=3):
    """Per-launch time of `reps` back-to-back calls: CUDA events only around
    the whole run (an event between two launches would stop them from
    overlapping ramp and drain)."""
    for _ in range(warm):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


# ---------------------------------------------------------------- the other BASELINE configs
def config_suite(torch, pkg, dev, stream, peak, quick=False, only=None):
    """C1-C4 (and C2 with SBS) on this GPU: the fused round trip
    (optb_roundtrip_dev) and the separate encode / decode launches, each
    timed back to back over a working set larger than L2.  Fractions: HBM
    bytes of the kernel that ran (interleaved: the container re-read is an L2
    hit) and the SURVEY 8(d) bytes (all encode + decode bytes) over the
    measured copy peak."""
    from paper_2105_00619_b200.pipeline import Pipeline
    C, S = pkg.codec, pkg.sampler
    res = {}
    reps = 5 if quick else 10

    def case(name, mode, per_chunk, Pp, B, nb, out_dtype=None, scale=1.0, rotate=1):
        if only and not any(o in name for o in only):
            return
        out_dtype = out_dtype or torch.uint8
        L = C.layout(mode, per_chunk, Pp, B, nb)
        rows = B * nb
        with torch.cuda.stream(stream):
            bufs = []
            for _ in range(rotate):
                src = torch.randint(0, 256, (rows, Pp), dtype=torch.uint8, device=dev)
                cont, offs = C.alloc_stream(L, dev.index)
                out = torch.empty((rows, Pp), dtype=out_dtype, device=dev)
                bufs.append((src, cont, offs, out))
            k = [0]

            def pick():
                b = bufs[k[0] % rotate]
                k[0] += 1
                return b

            def rt():
                src, cont, offs, out = pick()
                C.roundtrip_dev(L, src, cont, out, offsets=offs, scale=scale, stream=stream)

            def enc():
                src, cont, offs, _ = pick()
                C.encode_dev(L, src, cont, offs, stream=stream)

            def dec():
                _, cont, offs, out = pick()
                C.decode_dev(L, cont, out, offsets=offs, scale=scale, stream=stream)
            t_rt = b2b_time(torch, rt, stream, reps * rotate)
            C.sync(dev.index, stream)
            kind = C.last_roundtrip_kind()
            rt_b = C.roundtrip_hbm_bytes(L, out.element_size(), False)
            t_enc = b2b_time(torch, enc, stream, reps * rotate)
            t_dec = b2b_time(torch, dec, stream, reps * rotate)
            C.sync(dev.index, stream)
            # check: the fused round trip reproduces the input (every mode is
            # exact below its exact capacity; checker only, outside the timing)
            src, cont, offs, out = bufs[0]
            C.roundtrip_dev(L, src, cont, out, offsets=offs, scale=1.0, stream=stream)
            C.sync(dev.index, stream)
            ok = bool(torch.equal(out.to(torch.float32) if out.dtype != torch.uint8 else out,
                                  src.to(torch.float32) if out.dtype != torch.uint8 else src))
        cb, ob = C.container_bytes(L), C.offsets_bytes(L)
        es = out.element_size()
        enc_b = rows * Pp + cb + ob
        dec_b = cb + ob + rows * Pp * es
        s8d = enc_b + dec_b
        res[name] = {"mode": C.mode_name(mode), "per_chunk": per_chunk, "images_per_launch": rows, "P": Pp,
                     "out": str(out_dtype).replace("torch.", ""), "value": round(rows / t_rt, 1), "unit": UNIT,
                     "kernel": kind, "roundtrip_us": round(t_rt * 1e6, 2),
                     "hbm_bytes_per_launch": rt_b, "hbm_frac": round(rt_b / t_rt / 1e9 / peak, 4),
                     "survey_8d_bytes_per_launch": s8d, "survey_8d_frac": round(s8d / t_rt / 1e9 / peak, 4),
                     "encode_us": round(t_enc * 1e6, 2), "decode_us": round(t_dec * 1e6, 2),
                     "encode_frac": round(enc_b / t_enc / 1e9 / peak, 4),
                     "decode_frac": round(dec_b / t_dec / 1e9 / peak, 4),
                     "split_value": round(rows / (t_enc + t_dec), 1), "check": ok}
        del bufs
        torch.cuda.empty_cache()

    scale = float(np.float32(1.0) / np.float32(255.0))
    # C1: CIFAR-10 batches of 128, exact64 (8 -> 1), streamed 512 batches per launch
    case("C1_exact64_u8", 0, 8, 3072, 128, 512)
    case("C1_exact64_f32", 0, 8, 3072, 128, 512, torch.float32, scale)
    # C3: packing-ratio sweep on batches of 4096, 16 batches per launch
    for n in (2, 4, 8):
        case(f"C3_n{n}_exact64", 0, n, 3072, 4096, 16)
    case("C3_n16_exact128", 1, 16, 3072, 4096, 16)
    if not quick:
        case("C3_n9_lossless64", 3, 9, 3072, 4096, 16)
        case("C3_n18_lossless128", 4, 18, 3072, 4096, 16)
        case("C3_n6_f64", 2, 6, 3072, 4096, 16)
    # C4: ImageNet 256 x 224x224x3, 16x packing, fused decode -> bf16: one
    # 256-image batch per launch rotating over 8 batches (each launch's
    # 154 MB working set was evicted by the seven before it), and 8 batches
    # per launch
    IMG = 224 * 224 * 3
    case("C4_exact128_bf16", 1, 16, IMG, 256, 1, torch.bfloat16, scale, rotate=8)
    case("C4_exact128_bf16_8batches", 1, 16, IMG, 256, 8, torch.bfloat16, scale)
    if not quick:
        case("C4_exact128_u8_8batches", 1, 16, IMG, 256, 8)

    # C2: the CIFAR-100 workload with SBS (the round-1 headline): 50 000
    # images, one epoch = 97 batches per step, draws 4 epochs per sampler call
    N2, nb2 = 50000, 50000 // BATCH
    if only and not any(o in "C2_sbs" for o in only):
        return res
    with torch.cuda.stream(stream):
        ctx = pkg._lib.context(dev.index)
        import ctypes as ct
        ds2 = torch.empty((N2, P), dtype=torch.uint8, device=dev)
        pkg._lib.check(pkg._lib.lib.optb_synth_pixels_dev(ctx, DATA_SEED, 0, N2, P, ct.c_void_p(ds2.data_ptr()), P,
                                                          ct.c_void_p(stream.cuda_stream)))
        lab2 = torch.arange(N2, device=dev, dtype=torch.int32) % N_CLASSES
        offs2, mem2 = S.class_index_dev(lab2, N_CLASSES, device=dev.index)
        out2 = torch.empty((nb2 * BATCH, P), dtype=torch.uint8, device=dev)
        for mode, pc, key in ((1, 16, "C2_sbs_exact128_u8"), (0, 8, "C2_sbs_exact64_u8")):
            cur2 = S.BatchCursor.from_device_index(S.plan([1.0 / N_CLASSES] * N_CLASSES, BATCH, SEED), offs2, mem2,
                                                   device=dev.index)
            pipe2 = Pipeline(cur2, ds2, mode, BATCH, nb2, per_chunk=pc, device=dev.index, steps_per_draw=4)
            t2 = b2b_time(torch, lambda: pipe2.step(out2, stream), stream, 40 if quick else 100, warm=8)
            C.sync(dev.index, stream)
            kind = C.last_roundtrip_kind()
            L2 = pipe2.layout
            rows2 = nb2 * BATCH
            cb2 = C.container_bytes(L2)
            hbm2 = 2 * rows2 * P + rows2 * 8 + cb2 + (0 if kind.startswith("interleaved") else cb2)
            s8d2 = 2 * rows2 * P + rows2 * 8 + 2 * cb2
            res[key] = {"mode": C.mode_name(mode), "per_chunk": pc, "images_per_step": rows2,
                        "value": round(rows2 / t2, 1), "unit": UNIT, "ms_per_step": round(t2 * 1e3, 4),
                        "kernel": kind, "hbm_bytes_per_step": hbm2, "hbm_frac": round(hbm2 / t2 / 1e9 / peak, 4),
                        "survey_8d_frac": round(s8d2 / t2 / 1e9 / peak, 4),
                        "note": "50000-image dataset (1.2x L2), 97 batches per step, SBS 4 epochs per sampler call"}
            pipe2.close()
        del ds2, out2
        torch.cuda.empty_cache()
    return res


# ---------------------------------------------------------------- e2e
def run_e2e(args, torch, dist, S, Pipeline, ds, offs, mem, stream, dev, rank, world, rows, images_per_step,
            ref_rows):
    """End to end through the C ABI with HOST buffers, every step:
    optb_pipeline_step_host -- ONE call per step: the epoch's pinned host
    dataset is uploaded into one of two device buffers (copy engine), the step
    runs, the decoded rows are downloaded into pinned host memory (second copy
    engine); consecutive calls overlap both PCIe directions and the kernels.
    `ref_rows(k)` gives the reference cursor's rows of step k (checker)."""
    ds_host = ds.cpu().pin_memory()
    plan2 = S.plan([1.0 / N_CLASSES] * N_CLASSES, BATCH, SEED)
    cur2 = S.BatchCursor.from_device_index(plan2, offs, mem, device=dev.index)
    pipe2 = Pipeline(cur2, ds, MODE, BATCH, BATCHES_PER_STEP, per_chunk=PER_CHUNK, shard=rank, n_shards=world,
                     device=dev.index)
    out_hosts = [torch.empty((rows, P), dtype=torch.uint8).pin_memory() for _ in range(2)]
    k = [0]

    def step():
        pipe2.step_host(ds_host, out_hosts[k[0] % 2], stream)
        k[0] += 1

    with torch.cuda.stream(stream):
        for _ in range(2):
            step()
        pipe2.host_wait(stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            coll_barrier(dist)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            step()
        pipe2.host_wait(stream)
        e1.record(stream)
        e1.synchronize()
        torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / args.e2e_steps
    last = k[0] - 1
    want = ref_rows(last)
    ok = None if want is None else bool(torch.equal(out_hosts[last % 2], ds_host[torch.from_numpy(want)]))
    pipe2.close()
    if world > 1:
        ms = coll_reduce_ms(torch, dist, ms)
    h2d, d2h = ds_host.numel(), rows * P
    # the PCIe ceiling on this box, same buffers and sizes, right after the
    # leg: one direction at a time and both at once (two copy engines)
    pcie = None
    try:
        d_a = torch.empty(h2d, dtype=torch.uint8, device=dev)
        d_b = torch.empty(d2h, dtype=torch.uint8, device=dev)
        hv_in, hv_out = ds_host.view(-1), out_hosts[0].view(-1)
        s_up, s_dn = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

        def timed(fn, reps=2):
            fn()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            for _ in range(reps):
                fn()
            torch.cuda.synchronize(dev)
            return (time.perf_counter() - t0) / reps

        def up():
            with torch.cuda.stream(s_up):
                d_a.copy_(hv_in, non_blocking=True)

        def down():
            with torch.cuda.stream(s_dn):
                hv_out.copy_(d_b, non_blocking=True)

        def both():
            up()
            down()
        t_up, t_dn, t_bi = timed(up), timed(down), timed(both)
        bidir = (h2d + d2h) / t_bi / 1e9
        pcie = {"h2d_gbs": round(h2d / t_up / 1e9, 1), "d2h_gbs": round(d2h / t_dn / 1e9, 1),
                "bidir_gbs": round(bidir, 1),
                "e2e_frac_of_bidir": round((h2d + d2h) / (ms / 1e3) / 1e9 / bidir, 3),
                "how": "torch copies of the leg's own pinned buffers (3.2 GB each way), measured after the leg"}
        del d_a, d_b
    except Exception as ex:  # noqa: BLE001
        pcie = {"error": f"{type(ex).__name__}: {ex}"[:200]}
    del out_hosts, ds_host
    return {"value": round(images_per_step / (ms / 1e3), 1), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": round(ms, 3),
            "pcie_gbs_achieved": round((h2d + d2h) / (ms / 1e3) / 1e9, 1), "pcie_ceiling": pcie, "check": ok,
            "check_against": "rank 0: the decoded rows of the last step == dataset rows the reference cursor draws",
            "path": ("optb_pipeline_step_host, one C-ABI call per step: bulk H2D of the epoch's pinned host dataset "
                     "(3.2 GB) into one of two device buffers (copy engine) -> SBS draws + fused "
                     "gather-encode-decode -> D2H of the decoded rows (3.2 GB) to pinned host (second copy engine); "
                     "consecutive steps overlap both PCIe directions and the kernels")}


# ---------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=30)
    ap.add_argument("--sharded-steps", type=int, default=3,
                    help="N > 1 only: steps of the dataset-sharded variants")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the C1-C4 / C2 sub-keys")
    ap.add_argument("--no-check", action="store_true", help="skip the reference check of the last step")
    ap.add_argument("--probe-steps", type=int, default=6,
                    help="steps of the per-kernel timing pass (events around every launch)")
    ap.add_argument("--oversubscribe", action="store_true",
                    help="allow --gpus N above the visible GPU count (ranks share GPUs: a smoke run of the N-rank "
                         "path; device times are summed)")
    ap.add_argument("--split-kernels", action="store_true",
                    help="headline with separate encode / decode launches instead of the fused round trip")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(args)

    import ctypes as ct

    import torch
    import torch.distributed as dist

    import paper_2105_00619_b200 as pkg
    from paper_2105_00619_b200.pipeline import Pipeline
    C, S = pkg.codec, pkg.sampler
    rank, world, local = env_rank()
    if world != args.gpus and rank == 0:
        print(f"bench.py: WORLD_SIZE={world} overrides --gpus {args.gpus}", file=sys.stderr, flush=True)
    n_dev = torch.cuda.device_count()
    local = local % n_dev
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    oversub = False
    if world > 1:
        # Rendezvous over gloo, then compare the ranks' GPU UUIDs: one process
        # per GPU runs every collective of the run over NCCL; ranks sharing a
        # GPU (a smoke run on one device) keep gloo -- NCCL refuses that.
        dist.init_process_group("gloo")
        uuids = [None] * world
        dist.all_gather_object(uuids, str(torch.cuda.get_device_properties(local).uuid))
        oversub = len(set(uuids)) < world
        COLL["group"] = None if oversub else dist.new_group(backend="nccl")
        COLL["device"] = torch.device("cpu") if oversub else dev
        COLL["op"] = dist.ReduceOp.SUM if oversub else dist.ReduceOp.MAX
        if not oversub:
            coll_barrier(dist)  # first NCCL collective: the communicator is up
        print(f"bench.py: rank {rank}/{world} on cuda:{local} ({uuids[rank]}), control plane "
              f"{'gloo (GPUs shared)' if oversub else 'NCCL'}", file=sys.stderr, flush=True)
    peak, peak_kind = measured_peak()

    stream = torch.cuda.Stream(dev)
    rows = BATCH * BATCHES_PER_STEP
    with torch.cuda.stream(stream):
        ctx = pkg._lib.context(local)
        ds = torch.empty((N_EXAMPLES, P), dtype=torch.uint8, device=dev)
        pkg._lib.check(pkg._lib.lib.optb_synth_pixels_dev(ctx, DATA_SEED, 0, N_EXAMPLES, P, ct.c_void_p(ds.data_ptr()),
                                                          P, ct.c_void_p(stream.cuda_stream)))
        labels = torch.arange(N_EXAMPLES, device=dev, dtype=torch.int32) % N_CLASSES
        plan = S.plan([1.0 / N_CLASSES] * N_CLASSES, BATCH, SEED)
        offs, mem = S.class_index_dev(labels, N_CLASSES, device=local)
        cur = S.BatchCursor.from_device_index(plan, offs, mem, device=local)
        out = torch.empty((rows, P), dtype=torch.uint8, device=dev)
    torch.cuda.synchronize(dev)

    # ---- headline: K back-to-back pipeline steps, CUDA events only around
    # the whole timed region (an event between two round trips would stop
    # the next one from overlapping its launch ramp with this one's drain)
    pipe = Pipeline(cur, ds, MODE, BATCH, BATCHES_PER_STEP, per_chunk=PER_CHUNK, shard=rank, n_shards=world,
                    device=local, split_kernels=args.split_kernels)
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            pipe.step(out, stream)
        C.sync(local, stream)
        torch.cuda.synchronize(dev)
        launches0 = pkg._lib.launches(local)
        if world > 1:
            coll_barrier(dist)
        torch.cuda.synchronize(dev)
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            t_wall0 = time.perf_counter()
            start.record(stream)
            for _ in range(args.steps):
                pipe.step(out, stream)
            end.record(stream)
            t_enqueue = time.perf_counter() - t_wall0
            end.synchronize()
            t_wall = time.perf_counter() - t_wall0
        torch.cuda.synchronize(dev)
        if world > 1:
            coll_barrier(dist)
        C.sync(local, stream)
        launches = pkg._lib.launches(local) - launches0
    rt_kind = C.last_roundtrip_kind()
    fused = pipe.fused
    cont_bytes = C.container_bytes(pipe.layout)
    ms = start.elapsed_time(end) / args.steps
    ms_local = ms
    if world > 1:
        ms = coll_reduce_ms(torch, dist, ms)
    images_per_step = rows * world
    value = images_per_step / (ms / 1e3)

    # ---- check (reference cursor = checker, outside every timed region):
    # the last timed step's decoded rows are the dataset rows the reference
    # cursor draws, and its containers are their exact128 packing (at
    # capacity: the [16][P] -> [P][16] byte transpose of each chunk)
    ref = None
    check = None
    if rank == 0 and not args.no_check:
        try:
            ref = RefStream(labels.cpu().numpy(), world, rank)
            for _ in range(args.warmup + args.steps - 1):
                ref.step(BATCHES_PER_STEP)
            want = torch.from_numpy(ref.step(BATCHES_PER_STEP)).to(dev)
            rows_ok = bool(torch.equal(out, ds[want]))
            cont = _dev_bytes(torch, pipe.containers_ptr(), cont_bytes, dev)
            packed = ds[want].view(-1, PER_CHUNK, P).transpose(1, 2).contiguous().view(-1)
            cont_ok = bool(torch.equal(cont, packed))
            check = {"ok": rows_ok and cont_ok, "decoded_rows": rows_ok, "containers": cont_ok,
                     "against": f"{ref.kind} BatchCursor (oracle/_ref = the reference compiled from its sources) "
                                "draws of the last timed step, rank 0's batches"}
            del cont, packed, want
        except Exception as ex:  # noqa: BLE001
            check = {"ok": False, "error": f"{type(ex).__name__}: {ex}"[:300]}

    # ---- per-kernel durations: a separate pass with events around every
    # launch (isolated launches, no overlap with their neighbours)
    probe = Pipeline(S.BatchCursor.from_device_index(plan, offs, mem, device=local), ds, MODE, BATCH,
                     BATCHES_PER_STEP, per_chunk=PER_CHUNK, shard=rank, n_shards=world, device=local,
                     record_timings=True, split_kernels=args.split_kernels)
    with torch.cuda.stream(stream):
        for _ in range(2 + args.probe_steps):
            probe.step(out, stream)
        C.sync(local, stream)
    tim = [probe.timings(k) for k in range(2, 2 + args.probe_steps)]
    probe.close()
    t_sbs = statistics.mean(t[0] for t in tim)
    t_k1 = statistics.mean(t[1] for t in tim)
    t_k2 = statistics.mean(t[2] for t in tim)

    # ---- roofline of the dominant kernel.  The timed region runs nothing
    # but the step's launches on this stream (the draws are on the side
    # stream), so the kernel's average launch duration over the timed region
    # is the region time / K.
    interleaved = fused and rt_kind.startswith("interleaved")
    gathered = rows * P + rows * 8      # gathered rows + row ids in
    if fused:
        kname = "k_roundtrip_il<exact128,u8>" if interleaved else "k_roundtrip_vec<exact128,u8>"
        kbytes = gathered + cont_bytes + rows * P + (0 if interleaved else cont_bytes)
        k_ms_region = ms_local
    else:
        kname, kbytes = "k_encode_bulk<exact128>", gathered + cont_bytes
        k_ms_region = ms_local * t_k1 / (t_k1 + t_k2)
    s8d_bytes = gathered + 2 * cont_bytes + rows * P
    achieved = kbytes / (k_ms_region / 1e3) / 1e9
    traffic, traffic_tag = ncu_traffic(kname)
    roofline = {"bound": "hbm", "kernel": kname, "kernel_kind": rt_kind,
                "launch_timing": "CUDA events around the timed region on the launching stream, which runs only "
                                 "this kernel (one launch per step, back to back): region time / K",
                "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
                "peak_source": peak_kind, "traffic": traffic, "traffic_source": f"profiles/ncu_summary.json ({traffic_tag})",
                "frac_of_spec_8tbs": round(achieved / 8000.0, 4),
                "algorithmic_bytes_per_launch": kbytes,
                "algorithmic_bytes_note": ("compulsory HBM bytes: 3072 B gathered row + 8 B row id in, 3072 B "
                                           "container + 3072 B decoded row out per image; the container re-read "
                                           "is served from L2" if interleaved else "every encode + decode byte"),
                "survey_8d_bytes_per_launch": s8d_bytes,
                "survey_8d_gbs": round(s8d_bytes / (k_ms_region / 1e3) / 1e9, 1),
                "isolated_launch_ms": round(t_k1, 4),
                "isolated_launch_frac": round(kbytes / (t_k1 / 1e3) / 1e9 / peak, 4),
                "sbs_side_stream_ms_per_step": round(t_sbs, 4),
                "host_enqueue_us_per_step": round(t_enqueue / args.steps * 1e6, 1)}
    if not fused:
        roofline["decode_isolated_ms"] = round(t_k2, 4)

    configs = None
    if not args.no_configs and rank == 0:
        configs = config_suite(torch, pkg, dev, stream, peak, quick=world > 1)

    e2e = None
    if args.e2e_steps > 0:
        def ref_rows(k):
            if ref is None:
                return None
            r2 = RefStream(labels.cpu().numpy(), world, rank)
            for _ in range(k):
                r2.step(BATCHES_PER_STEP)
            w = r2.step(BATCHES_PER_STEP)
            r2.close()
            return w
        pipe.close()
        pipe = None
        torch.cuda.empty_cache()
        e2e = run_e2e(args, torch, dist, S, Pipeline, ds, offs, mem, stream, dev, rank, world, rows,
                      images_per_step, ref_rows)

    # ---- N > 1: the optional dataset-sharded variants (each rank holds 1/N
    # of the dataset), reported separately from the headline
    sharded = None
    if world > 1 and args.sharded_steps > 0:
        sharded = run_sharded(args, torch, dist, S, ds, offs, mem, out, stream, dev, rank, world, oversub,
                              images_per_step)

    cpu = shim_api = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # the CPU baseline runs at N = 1 only
        threads = os.cpu_count() or 1
        ds_h, lab_h = host_dataset()
        rb = RefBaseline(ds_h, lab_h)
        runs = [rb.rate(max(threads * 2, 8), threads) for _ in range(3)]
        runs1 = [rb.rate(4, 1) for _ in range(3)]
        rb.close()
        v, sample, used = sorted(runs)[1]
        v1, sample1, _ = sorted(runs1)[1]
        cpu = {"value": round(v, 1), "unit": UNIT, "cores": used, "kind": rb.kind, "sample": sample + ", median of 3",
               "single_thread": {"value": round(v1, 1), "cores": 1, "sample": sample1 + ", median of 3"},
               "cpu_model": cpu_model(), "nproc": os.cpu_count()}
        del ds_h
        shim_api = run_shim_api()

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "u8", "data": "synthetic (counter-based SplitMix64 pixels, seed 7)",
                "config": config(world), "roofline": roofline, "check": check, "cpu_baseline": cpu, "e2e": e2e,
                "configs": configs, "shim_api": shim_api, "sharded_dataset": sharded, "clocks": clk.summary(),
                "gpu_launches": int(launches), "wall_s_timed": round(t_wall, 4),
                "timing": "CUDA events on the launching stream around the K timed steps only; max over ranks"}
        if oversub:
            line["oversubscribed"] = f"{world} ranks on {n_dev} GPU(s): per-rank device times summed"
        print(json.dumps(line), flush=True)
    if pipe is not None:
        pipe.close()
    if ref is not None:
        ref.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_shim_api(n_batches=200):
    """The reference runner's call pattern through the unchanged C++ API
    (tools/shim_api_bench.cpp: one BatchCursor::next per batch, image_of +
    codec::encode per 16-image chunk, codec::decode per chunk; C2 stream, one
    host thread) built twice: against the drop-in shim (GPU underneath) and
    against the reference itself (oracle/_ref/ref_api_bench, compiled from
    its sources).  Same stream, same checksum."""
    res = {}
    for key, path in (("drop_in", os.path.join(ROOT, "paper_2105_00619_b200", "optb_shim_api_bench")),
                      ("reference", os.path.join(ROOT, "oracle", "_ref", "ref_api_bench"))):
        if not os.path.exists(path):
            res[key] = {"unavailable": f"{os.path.relpath(path, ROOT)} not built"}
            continue
        try:
            r = subprocess.run([path, "50000", str(n_batches)], capture_output=True, text=True, timeout=300)
            res[key] = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception as ex:  # noqa: BLE001
            res[key] = {"unavailable": f"{type(ex).__name__}: {ex}"[:200]}
    d, r = res.get("drop_in", {}), res.get("reference", {})
    if "images_per_s" in d and "images_per_s" in r:
        res["speedup"] = round(d["images_per_s"] / r["images_per_s"], 3)
        res["same_stream"] = d.get("checksum") == r.get("checksum")
    return res


def _dev_bytes(torch, ptr, n, dev):
    """A uint8 view of n device bytes at ptr (library-owned memory)."""
    class _Arr:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "|u1", "data": (ptr, False), "version": 3}
    return torch.as_tensor(_Arr(), device=dev)


def run_sharded(args, torch, dist, S, ds, offs, mem, out, stream, dev, rank, world, oversub, images_per_step):
    """Dataset-sharded global gather (optional).  "peer": the
    shards are mapped over CUDA IPC and the fused round-trip kernel gathers
    each drawn row from the GPU that owns it (NVLink peer loads), device-timed
    with CUDA events, max over ranks.  "a2a": the drawn rows cross ranks in
    one NCCL all-to-all per step (host-driven, wall clock)."""
    from paper_2105_00619_b200.sharded import PeerShardedGather, ShardedGather
    per = (N_EXAMPLES + world - 1) // world
    res = {}
    with torch.cuda.stream(stream):
        local_rows = ds[rank * per:(rank + 1) * per].clone()
    try:
        with torch.cuda.stream(stream):
            cur4 = S.BatchCursor.from_device_index(S.plan([1.0 / N_CLASSES] * N_CLASSES, BATCH, SEED), offs, mem,
                                                   device=dev.index)
            pg = PeerShardedGather(cur4, local_rows, N_EXAMPLES, rank, world, BATCH, BATCHES_PER_STEP,
                                   device=dev.index)
            for _ in range(args.warmup):
                pg.step(out, stream)
            torch.cuda.synchronize(dev)
            coll_barrier(dist)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.sharded_steps):
                pg.step(out, stream)
            e1.record(stream)
            e1.synchronize()
            pms = e0.elapsed_time(e1) / args.sharded_steps
            cur6 = S.BatchCursor.from_device_index(S.plan([1.0 / N_CLASSES] * N_CLASSES, BATCH, SEED), offs, mem,
                                                   device=dev.index)
            for _ in range(args.warmup + args.sharded_steps):
                ex6, _ = cur6.next_dev(BATCHES_PER_STEP * world, shard=rank, n_shards=world)
            pok = bool(torch.equal(out, ds[ex6]))
            remote = int(((ex6 // per) != rank).sum())
            pg.close()
            pms = coll_reduce_ms(torch, dist, pms)
        res["peer"] = {"value": round(images_per_step / (pms / 1e3), 1), "unit": UNIT, "ms_per_step": round(pms, 3),
                       "exchange": "CUDA IPC-mapped shards read by the fused gather-encode-decode kernel "
                                   "(optb_roundtrip_rows_dev)" + (" -- ranks share one GPU" if oversub else
                                                                  " over NVLink / NVSwitch"),
                       "rows_from_peers_per_step_rank0": remote, "check": pok,
                       "timing": "CUDA events on the launching stream, max over ranks"}
    except Exception as ex:  # noqa: BLE001
        res["peer"] = {"unavailable": f"{type(ex).__name__}: {ex}"[:300]}
    try:
        with torch.cuda.stream(stream):
            cur4 = S.BatchCursor.from_device_index(S.plan([1.0 / N_CLASSES] * N_CLASSES, BATCH, SEED), offs, mem,
                                                   device=dev.index)
            sg = ShardedGather(cur4, local_rows, N_EXAMPLES, rank, world, BATCH, BATCHES_PER_STEP,
                               device=dev.index, exchange="gloo" if oversub else "nccl", group=COLL["group"])
            sg.step(out)
            torch.cuda.synchronize(dev)
            coll_barrier(dist)
            t0 = time.perf_counter()
            for _ in range(args.sharded_steps):
                sg.step(out)
            torch.cuda.synchronize(dev)
            sms = (time.perf_counter() - t0) / args.sharded_steps * 1e3
            sms = coll_reduce_ms(torch, dist, sms)
        res["a2a"] = {"value": round(images_per_step / (sms / 1e3), 1), "unit": UNIT, "ms_per_step": round(sms, 3),
                      "exchange": "gloo (ranks share a GPU)" if oversub else "nccl all_to_all_single",
                      "timing": "host wall clock around synchronised steps (the exchange is host-driven)"}
    except Exception as ex:  # noqa: BLE001
        res["a2a"] = {"unavailable": f"{type(ex).__name__}: {ex}"[:300]}
    return res


if __name__ == "__main__":
    sys.exit(main())
