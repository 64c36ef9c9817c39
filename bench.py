"""Benchmark: images/s encode+decode (and achieved HBM GB/s vs peak) per BASELINE.json.

Workload (BASELINE.json configs[1], "C2"): CIFAR-100-shaped synthetic dataset
(50 000 x 32x32x3 u8, labels e % 100) resident in HBM; selective batch
sampling with uniform weights over 100 classes, batch 512, seed 1234; every
step is one epoch of the reference's draw stream (floor(50000/512) = 97
batches per GPU): SBS draws (optb_sbs_next_dev) -> gather-encode of the
drawn rows into exact128 containers (optb_encode_dev) -> decode of every
container back to u8 rows (optb_decode_dev).  Containers are materialised in
HBM between the kernels.  N GPUs: one process per GPU, each draws the global
stream's batches t % N == rank (weak scaling, no collective on the data path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Rank 0 prints one JSON line.  `--impl reference` times the reference's own
CPU implementation (oracle/_ref, compiled from /root/reference's sources)
on the host cores over a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_EXAMPLES = 50000
N_CLASSES = 100
BATCH = 512
SEED = 1234
DATA_SEED = 7  # RunConfig::data_seed (runner.hpp:34)
P = 32 * 32 * 3
BATCHES_PER_STEP = N_EXAMPLES // BATCH  # 97: one epoch (runner.cpp:52-57)
MODE = 1  # ExactInt128, the reference default (runner.hpp:52)
TIMING_STRIDE = 8  # per-kernel timing events on every 8th step of the timed loops
PER_CHUNK = 16
METRIC = "images/sec encode+decode (and achieved HBM GB/s vs peak) at 1/2/4/8 B200"
UNIT = "images/s"


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def config(world, steps_per_draw=4):
    return {"workload": "C2: CIFAR-100-shaped 50000x32x32x3 u8 dataset in HBM, SBS (uniform 100 classes, "
                        "B=512, seed 1234) + exact128 gather-encode + decode to u8; 1 epoch = 97 batches "
                        "per GPU per step",
            "global_batch": BATCH, "batches_per_step_per_gpu": BATCHES_PER_STEP, "mode": "exact128",
            "per_chunk": PER_CHUNK, "image": [32, 32, 3], "decode_out": "u8",
            "parallelism": f"independent batch shards x{world} (t % N == rank)",
            "l2": "inputs larger than L2: 153.6 MB dataset (> 126 MB L2), and every step streams 152.6 MB of "
                  "containers + 152.6 MB of decoded rows through it",
            "pipeline": "native optb_pipeline: SBS draws for the next steps on a side stream overlap the "
                        "current step's gather-encode + decode, one optb_roundtrip_dev launch per step (every warp "
                        "stores each encoded tile into the HBM container stream and decodes it one tile later, "
                        "reading it back while it is still in L2); steps_per_draw epochs per sampler call",
            "steps_per_draw": steps_per_draw}


# ---------------------------------------------------------------- collectives
# The run's control-plane collectives (barriers, the max-over-ranks of device
# times): NCCL with one process per GPU, gloo when ranks share a GPU (then the
# per-rank times are summed so the whole-job rate is never overstated).
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


def ncu_traffic():
    """dram read+write bytes per launch of the roofline kernel from the
    committed ncu --set full summary (profiles/ncu_summary.json), if any."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d
    except Exception:  # noqa: BLE001
        return None


# ---------------------------------------------------------------- reference arm
def reference_rate(n_batches_sample: int, threads: int, repeats: int = 1):
    """Time the reference CPU path (oracle/_ref = the reference compiled from
    its own sources; else the C oracle port) on a bounded sample: SBS draws
    with the reference BatchCursor, then per batch image_of gather +
    codec::encode per chunk + codec::decode per chunk, batches split over
    `threads` host threads.  Returns (images/s, kind, sample description)."""
    import ctypes as ct

    import oracle as O
    labels = (np.arange(N_EXAMPLES) % N_CLASSES).astype(np.int32)
    ds = O.synth_pixels(DATA_SEED, 0, N_EXAMPLES, P)
    rates = []
    if O.ref_available():
        R = O.REF
        off = np.zeros(N_CLASSES + 1, np.uint64)
        mem = np.zeros(N_EXAMPLES, np.int64)
        buf = ct.create_string_buffer(512)
        R.ref_class_index(O.ptr(labels, O.i32p), N_EXAMPLES, N_CLASSES, O.ptr(off, O.u64p), O.ptr(mem, O.i64p),
                          buf, 512)
        w = np.full(N_CLASSES, 1.0 / N_CLASSES)
        st = ct.c_int(0)
        h = R.ref_cursor_create(O.ptr(w, O.f64p), N_CLASSES, BATCH, SEED, O.ptr(off, O.u64p), O.ptr(mem, O.i64p),
                                ct.byref(st), buf, 512)
        dsh = R.ref_dataset_create(O.ptr(ds, O.u8p), N_EXAMPLES, 32, 32, 3)
        ex = np.zeros(n_batches_sample * BATCH, np.int64)
        chk = ct.c_uint64(0)
        for _ in range(repeats):
            t0 = time.perf_counter()
            R.ref_cursor_next(h, n_batches_sample, O.ptr(ex, O.i64p), None)
            t_sbs = time.perf_counter() - t0
            secs = R.ref_bench_roundtrip(dsh, MODE, O.ptr(ex, O.i64p), n_batches_sample, BATCH, threads, 0,
                                         ct.byref(chk))
            rates.append(n_batches_sample * BATCH / (secs + t_sbs))
        R.ref_dataset_destroy(dsh)
        R.ref_cursor_destroy(h)
        kind = "reference"
    else:
        off, mem = O.class_index(labels, N_CLASSES)
        cur = O.Cursor(O.sbs_plan([1.0 / N_CLASSES] * N_CLASSES, BATCH), off, mem, BATCH, SEED)
        for _ in range(repeats):
            t0 = time.perf_counter()
            ex, _ = cur.next(n_batches_sample)
            cont, _ = O.encode_stream(ds, ex, MODE, PER_CHUNK, BATCH, n_batches_sample)
            O.decode_stream(cont, None, MODE, PER_CHUNK, P, BATCH, n_batches_sample)
            rates.append(n_batches_sample * BATCH / (time.perf_counter() - t0))
        kind, threads = "port", 1
    sample = (f"{n_batches_sample} batches x {BATCH} images of the C2 stream (SBS draws + image_of gather + "
              f"codec::encode/decode per 16-image chunk), {threads} host threads, median of {repeats}")
    return statistics.median(rates), kind, sample, threads


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    sample_batches = max(threads * 2, 8)
    for _ in range(args.warmup):
        reference_rate(sample_batches, threads, 1)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v, kind, sample, used = reference_rate(sample_batches, threads, 1)
        vals.append(v)
    wall = time.perf_counter() - t0
    v = statistics.median(vals)
    line = {"metric": METRIC, "value": round(v, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(wall / args.steps * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": config(world, args.steps_per_draw), "impl": "reference",
            "cpu_baseline": {"value": round(v, 1), "unit": UNIT, "cores": used, "kind": kind, "sample": sample},
            "e2e": {"value": round(v, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0

def run_e2e(args, torch, dist, S, Pipeline, ds, offs, mem, stream, dev, rank, world, rows, images_per_step, red_dev):
    """End-to-end steps with host buffers in and out (see main).  Two legs:
    optb_pipeline_step_host -- ONE C-ABI call per step: the epoch's pinned host
    dataset is uploaded into one of two device buffers (copy engine), the step
    runs, the decoded rows are downloaded into pinned host memory (second copy
    engine); consecutive calls overlap both PCIe directions and the kernels --
    and a zero-copy leg in which the gather kernel reads the drawn rows
    straight from pinned host memory."""
    out_shape = (rows, P)
    oversub = red_dev.type == "cpu"  # ranks share GPUs: per-rank times summed
    ds_host = ds.cpu().pin_memory()
    d2h = torch.cuda.Stream(dev)
    plan2 = S.plan([1.0 / N_CLASSES] * N_CLASSES, BATCH, SEED)
    results = []
    for zero_copy in (False, True):
        cur2 = S.BatchCursor.from_device_index(plan2, offs, mem, device=dev.index)
        pipe2 = Pipeline(cur2, ds_host if zero_copy else ds, MODE, BATCH, BATCHES_PER_STEP,
                         per_chunk=PER_CHUNK, shard=rank, n_shards=world, device=dev.index,
                         steps_per_draw=args.steps_per_draw)
        outs = [torch.empty(out_shape, dtype=torch.uint8, device=dev) for _ in range(2)]
        out_hosts = [torch.empty(out_shape, dtype=torch.uint8).pin_memory() for _ in range(2)]
        ev = lambda: torch.cuda.Event()  # noqa: E731
        dec_done, down_done = [ev(), ev()], [ev(), ev()]
        k_state = [0]

        def step():
            k = k_state[0]
            b = k % 2
            if not zero_copy:
                pipe2.step_host(ds_host, out_hosts[b], stream)
            else:
                if k >= 2:
                    stream.wait_event(down_done[b])
                pipe2.step(outs[b], stream)
                dec_done[b].record(stream)
                d2h.wait_event(dec_done[b])
                with torch.cuda.stream(d2h):
                    out_hosts[b].copy_(outs[b], non_blocking=True)
                down_done[b].record(d2h)
            k_state[0] += 1

        def wait_all():
            if not zero_copy:
                pipe2.host_wait(stream)
            else:
                stream.wait_event(down_done[(k_state[0] - 1) % 2])

        with torch.cuda.stream(stream):
            for _ in range(max(4, args.warmup)):  # includes the sampler's generation-pool growth
                step()
            wait_all()
            torch.cuda.synchronize(dev)
            if world > 1:
                coll_barrier(dist)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.e2e_steps):
                step()
            wait_all()
            e1.record(stream)
            e1.synchronize()
            torch.cuda.synchronize(dev)
            ms = e0.elapsed_time(e1) / args.e2e_steps
            cur3 = S.BatchCursor.from_device_index(plan2, offs, mem, device=dev.index)
            for _ in range(k_state[0]):
                ex3, _ = cur3.next_dev(BATCHES_PER_STEP * world, shard=rank, n_shards=world)
            ok = bool(torch.equal(out_hosts[(k_state[0] - 1) % 2], ds_host[ex3.cpu()]))
            pipe2.close()
        if world > 1:
            ms = coll_reduce_ms(torch, dist, ms)
        h2d_bytes = rows * P if zero_copy else ds_host.numel()
        results.append({"value": round(images_per_step / (ms / 1e3), 1), "unit": UNIT,
                        "h2d_bytes_per_step": int(h2d_bytes), "d2h_bytes_per_step": rows * P,
                        "ms_per_step": round(ms, 3), "check": ok,
                        "path": ("pinned host dataset read zero-copy by the gather-encode kernel -> decode -> "
                                 "D2H of the decoded rows (copy stream, double-buffered)") if zero_copy else
                                ("optb_pipeline_step_host, one C-ABI call per step: bulk H2D of the epoch's pinned "
                                 "host dataset into one of two device buffers (copy engine) -> SBS draws + fused "
                                 "gather-encode-decode -> D2H of the decoded rows to pinned host (second copy "
                                 "engine); consecutive steps overlap both PCIe directions")})
    return results[0], results[1]


# ---------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--sharded-steps", type=int, default=3,
                    help="N > 1 only: steps of the dataset-sharded (all-to-all) variant")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--split-steps", type=int, default=50,
                    help="steps of the same pipeline with separate encode / decode launches (per-kernel view)")
    ap.add_argument("--split-kernels", action="store_true",
                    help="headline with separate encode / decode launches instead of the fused round trip")
    ap.add_argument("--steps-per-draw", type=int, default=4,
                    help="epochs of SBS draws computed per sampler call (amortises its fixed cost)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import ctypes as ct

    import torch
    import torch.distributed as dist

    import paper_2105_00619_b200 as pkg
    from paper_2105_00619_b200.pipeline import Pipeline
    C, S = pkg.codec, pkg.sampler
    rank, world, local = env_rank()
    n_dev = torch.cuda.device_count()
    local = local % n_dev
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    oversub = False
    if world > 1:
        # Rendezvous over gloo, then compare the ranks' GPU UUIDs: one process
        # per GPU (however the launcher maps devices) runs every collective of
        # the run over NCCL; ranks sharing a GPU (a smoke run of the sharded
        # path on one device) keep gloo -- NCCL refuses two ranks per GPU.
        dist.init_process_group("gloo")
        uuids = [None] * world
        dist.all_gather_object(uuids, str(torch.cuda.get_device_properties(local).uuid))
        oversub = len(set(uuids)) < world
        COLL["group"] = None if oversub else dist.new_group(backend="nccl")
        COLL["device"] = torch.device("cpu") if oversub else dev
        COLL["op"] = dist.ReduceOp.SUM if oversub else dist.ReduceOp.MAX
    red_dev = torch.device("cpu") if oversub else dev

    stream = torch.cuda.Stream(dev, priority=int(os.environ.get("OPTB_BENCH_PRIO", "0")))
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
    # The native E-D pipeline (optb_pipeline_*): per step, SBS draws of step
    # k+1 on a side stream overlap gather-encode + decode of step k.
    tstride = TIMING_STRIDE if args.steps >= 4 * TIMING_STRIDE else 1  # short runs: every step
    # per-kernel timing events on every TIMING_STRIDE-th step only: an event
    # between two round-trip launches stops the second from overlapping its
    # launch ramp with the first one's drain (programmatic dependent launch)
    pipe = Pipeline(cur, ds, MODE, BATCH, BATCHES_PER_STEP, per_chunk=PER_CHUNK, shard=rank, n_shards=world,
                    device=local, record_timings=True, steps_per_draw=args.steps_per_draw,
                    split_kernels=args.split_kernels, timing_stride=tstride)
    L = pipe.layout

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
        if world > 1:
            coll_barrier(dist)
        C.sync(local, stream)
        launches = pkg._lib.launches(local) - launches0
    # per-kernel durations of the last (up to 60) timed steps -- the
    # pipeline keeps a 64-step ring of timing events
    timed = [k for k in range(args.warmup, args.warmup + args.steps) if k % tstride == 0][-60:]
    tim = [pipe.timings(k) for k in timed]
    t_sbs, t_enc, t_dec = [t[0] for t in tim], [t[1] for t in tim], [t[2] for t in tim]
    ms = start.elapsed_time(end) / args.steps
    if world > 1:
        # one GPU per rank: max over ranks.  Oversubscribed smoke runs (ranks
        # share a GPU, whose timed regions may or may not overlap): the sum,
        # so the whole-job rate is never overstated.
        ms = coll_reduce_ms(torch, dist, ms)
    images_per_step = rows * world
    value = images_per_step / (ms / 1e3)

    # roofline for the dominant kernel (per-launch algorithmic bytes / launch time)
    enc_ms, dec_ms = statistics.mean(t_enc), statistics.mean(t_dec)
    cont_bytes = C.container_bytes(L)
    enc_bytes = rows * P + cont_bytes + rows * 8  # gathered rows + containers + row index
    dec_bytes = cont_bytes + rows * P
    peak, peak_kind = measured_peak()
    fused = pipe.fused
    if fused and statistics.mean(t_dec) > 0.005:
        raise RuntimeError("pipeline reported separate decode launches on the fused path")
    # The fused launch for exact128 is the interleaved kernel (k_roundtrip_il;
    # the library reports which kernel the last step ran): each container
    # tile is read back while still in L2, so its HBM bytes are the
    # compulsory ones -- gathered rows + row ids in, containers + decoded rows
    # out.  The SURVEY 8(d) figure (which also counts the container re-read)
    # is reported beside it.
    rt_kind = C.last_roundtrip_kind()
    interleaved = fused and rt_kind.startswith("interleaved")
    l2_bytes = 0
    if interleaved:
        kname, kms, kbytes = "k_roundtrip_il<exact128,u8>", enc_ms, enc_bytes + rows * P
        l2_bytes = cont_bytes
    elif fused:  # phase-ordered: every byte of encode + decode is an HBM byte
        kname, kms, kbytes = "k_roundtrip_vec<exact128,u8>", enc_ms, enc_bytes + dec_bytes
    elif enc_ms >= dec_ms:
        kname, kms, kbytes = "k_encode_vec<exact128>", enc_ms, enc_bytes
    else:
        kname, kms, kbytes = "k_decode_vec<exact128,u8>", dec_ms, dec_bytes
    achieved = kbytes / (kms / 1e3) / 1e9
    nsum = ncu_traffic()
    traffic = None
    if nsum:  # ncu names carry every template argument: match on the prefix
        for kn, kv in nsum.get("kernels", {}).items():
            if kn == kname or kn.startswith(kname[:-1] + ","):
                traffic = kv.get("dram_bytes_per_launch")
                break
    roofline = {"bound": "hbm", "kernel": kname, "kernel_kind": rt_kind,
                "launch_timing": ("CUDA events on the launching stream around every %d-th timed step's launch; "
                                  "those launches cannot overlap their neighbours (an event sits between), so this "
                                  "is the isolated launch duration -- back-to-back steps overlap ramp and tail "
                                  "(step_gbs)" % tstride),
                "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "peak_source": peak_kind, "traffic": traffic,
                "frac_of_spec_8tbs": round(achieved / 8000.0, 4),
                "algorithmic_bytes_per_launch": kbytes,
                "l2_served_bytes_per_launch": l2_bytes,
                "survey_8d_bytes_per_launch": kbytes + l2_bytes,
                "survey_8d_gbs": round((kbytes + l2_bytes) / (kms / 1e3) / 1e9, 1),
                "host_enqueue_us_per_step": round(t_enqueue / args.steps * 1e6, 1),
                "kernels_ms": ({"sbs_side_stream": round(statistics.mean(t_sbs), 4),
                                "roundtrip": round(enc_ms, 4)} if fused else
                               {"sbs_side_stream": round(statistics.mean(t_sbs), 4), "encode": round(enc_ms, 4),
                                "decode": round(dec_ms, 4)}),
                "step_gbs": round((kbytes if fused else enc_bytes + dec_bytes) / (ms / 1e3) / 1e9, 1),
                "step_frac": round((kbytes if fused else enc_bytes + dec_bytes) / (ms / 1e3) / 1e9 / peak, 4)}
    if not fused:
        roofline["encode_gbs"] = round(enc_bytes / (enc_ms / 1e3) / 1e9, 1)
        roofline["decode_gbs"] = round(dec_bytes / (dec_ms / 1e3) / 1e9, 1)
    # the same pipeline with separate encode / decode launches per step
    # (optb_encode_dev + optb_decode_dev), for the per-kernel view
    split = None
    if fused and args.split_steps > 0:
        with torch.cuda.stream(stream):
            cur5 = S.BatchCursor.from_device_index(S.plan([1.0 / N_CLASSES] * N_CLASSES, BATCH, SEED), offs, mem,
                                                   device=local)
            pipe5 = Pipeline(cur5, ds, MODE, BATCH, BATCHES_PER_STEP, per_chunk=PER_CHUNK, shard=rank,
                             n_shards=world, device=local, record_timings=True, steps_per_draw=args.steps_per_draw,
                             split_kernels=True)
            for _ in range(args.warmup):
                pipe5.step(out, stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.split_steps):
                pipe5.step(out, stream)
            e1.record(stream)
            e1.synchronize()
            sms_ = e0.elapsed_time(e1) / args.split_steps
            if world > 1:
                sms_ = coll_reduce_ms(torch, dist, sms_)
            tim5 = [pipe5.timings(k) for k in range(max(args.warmup, args.warmup + args.split_steps - 60),
                                                     args.warmup + args.split_steps)]
            pipe5.close()
        e5, d5 = statistics.mean(t[1] for t in tim5), statistics.mean(t[2] for t in tim5)
        split = {"ms_per_step": round(sms_, 4), "value": round(images_per_step / (sms_ / 1e3), 1),
                 "encode_ms": round(e5, 4), "decode_ms": round(d5, 4),
                 "encode_gbs": round(enc_bytes / (e5 / 1e3) / 1e9, 1),
                 "decode_gbs": round(dec_bytes / (d5 / 1e3) / 1e9, 1)}

    # e2e: host buffers in and out, every step.  The epoch's input rows live
    # in pinned host memory; each step uploads the dataset epoch with one bulk
    # H2D copy (copy engine) into one of two device buffers while the previous
    # step computes, gathers / encodes / decodes from it, and copies the
    # decoded rows back to pinned host memory on a D2H stream (double-buffered,
    # so both PCIe directions and the kernels overlap).  The zero-copy variant
    # (the gather kernel reads the drawn rows straight from pinned memory) is
    # reported alongside.
    e2e = e2e_zc = None
    if args.e2e_steps > 0:
        e2e, e2e_zc = run_e2e(args, torch, dist, S, Pipeline, ds, offs, mem, stream, dev, rank, world, rows,
                              images_per_step, red_dev)
        # this box's pinned-memory PCIe bandwidth (same-size copies, same
        # run): the e2e leg is transfer-bound, so its bound is what these allow
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import pcie_probe
        pc = pcie_probe.measure(torch, BATCH * BATCHES_PER_STEP * P)
        bound_ms = max(e2e["h2d_bytes_per_step"] / pc["h2d_gbs"], e2e["d2h_bytes_per_step"] / pc["d2h_gbs"],
                       (e2e["h2d_bytes_per_step"] + e2e["d2h_bytes_per_step"]) / pc["bidir_gbs"]) / 1e6
        # (the probe's copies run once, after the e2e leg: a frac slightly
        # above 1 means the link was a little faster during the leg)
        e2e["pcie"] = dict(pc, bound_ms_per_step=round(bound_ms, 3),
                           frac_of_pcie_bound=round(bound_ms / e2e["ms_per_step"], 3))
    # The same workload in exact64 (8 images per 64-bit word; SURVEY §8:
    # BASELINE.json does not name C2's mode -- the headline uses the
    # reference default exact128, this is the other exact mode)
    exact64 = None
    if args.split_steps > 0:
        with torch.cuda.stream(stream):
            cur7 = S.BatchCursor.from_device_index(S.plan([1.0 / N_CLASSES] * N_CLASSES, BATCH, SEED), offs, mem,
                                                   device=local)
            t7 = TIMING_STRIDE if args.split_steps >= 4 * TIMING_STRIDE else 1
            pipe7 = Pipeline(cur7, ds, 0, BATCH, BATCHES_PER_STEP, per_chunk=8, shard=rank, n_shards=world,
                             device=local, record_timings=True, steps_per_draw=args.steps_per_draw,
                             timing_stride=t7)
            for _ in range(args.warmup):
                pipe7.step(out, stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.split_steps):
                pipe7.step(out, stream)
            e1.record(stream)
            e1.synchronize()
            ms7 = e0.elapsed_time(e1) / args.split_steps
            if world > 1:
                ms7 = coll_reduce_ms(torch, dist, ms7)
            k7 = statistics.mean(pipe7.timings(k)[1] for k in range(args.warmup, args.warmup + args.split_steps)
                                 if k % t7 == 0)
            il7 = C.last_roundtrip_kind().startswith("interleaved")
            pipe7.close()
        cb7 = C.container_bytes(C.layout(0, 8, P, BATCH, BATCHES_PER_STEP))
        # HBM bytes: rows in, containers out, rows out (+ the container
        # re-read for the phase-ordered kernel; interleaved: an L2 hit)
        b7 = 2 * rows * P + cb7 + rows * 8 + (0 if il7 else cb7)
        exact64 = {"mode": "exact64", "per_chunk": 8, "ms_per_step": round(ms7, 4),
                   "kernel": "k_roundtrip_il<exact64,u8>" if il7 else "k_roundtrip_vec<exact64,u8>",
                   "value": round(images_per_step / (ms7 / 1e3), 1), "kernel_ms": round(k7, 4),
                   "kernel_gbs": round(b7 / (k7 / 1e3) / 1e9, 1), "kernel_frac": round(b7 / (k7 / 1e3) / 1e9 / peak, 4)}

    # N > 1: the optional dataset-sharded variants (each rank holds 1/N of the
    # dataset), reported separately from the headline.  "peer": the shards are
    # mapped over CUDA IPC and the fused roundtrip kernel gathers each drawn
    # row from the GPU that owns it (NVLink peer loads), device-timed with
    # CUDA events, max over ranks.  "a2a": drawn rows cross ranks in one
    # all-to-all per step (host-driven, wall clock around synchronised steps).
    sharded = sharded_a2a = None
    if world > 1 and args.sharded_steps > 0:
        from paper_2105_00619_b200.sharded import PeerShardedGather, ShardedGather
        per = (N_EXAMPLES + world - 1) // world
        # optional legs: a failure (e.g. peers not mappable when each process
        # sees one GPU) is reported in the line instead of ending the run
        with torch.cuda.stream(stream):
            local_rows = ds[rank * per:(rank + 1) * per].clone()
        try:
            with torch.cuda.stream(stream):
                cur4 = S.BatchCursor.from_device_index(S.plan([1.0 / N_CLASSES] * N_CLASSES, BATCH, SEED), offs, mem,
                                                       device=local)
                pg = PeerShardedGather(cur4, local_rows, N_EXAMPLES, rank, world, BATCH, BATCHES_PER_STEP,
                                       device=local)
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
                # check the last step against the replicated dataset
                cur6 = S.BatchCursor.from_device_index(S.plan([1.0 / N_CLASSES] * N_CLASSES, BATCH, SEED), offs, mem,
                                                       device=local)
                for _ in range(args.warmup + args.sharded_steps):
                    ex6, _ = cur6.next_dev(BATCHES_PER_STEP * world, shard=rank, n_shards=world)
                pok = bool(torch.equal(out, ds[ex6]))
                remote = int(((ex6 // per) != rank).sum())
                pg.close()
                pms = coll_reduce_ms(torch, dist, pms)
            sharded = {"value": round(images_per_step / (pms / 1e3), 1), "unit": UNIT, "ms_per_step": round(pms, 3),
                       "exchange": "peer memory: CUDA IPC-mapped shards read by the fused gather-encode-decode kernel "
                                   "(optb_roundtrip_rows_dev)" + (" -- ranks share one GPU (smoke run)" if oversub else
                                                                 " over NVLink / NVSwitch"),
                       "rows_from_peers_per_step_rank0": remote, "bytes_from_peers_per_step_rank0": remote * P,
                       "check": pok, "timing": "CUDA events on the launching stream, max over ranks (sum when ranks share a GPU)"}
        except Exception as ex:  # noqa: BLE001
            sharded = {"unavailable": f"{type(ex).__name__}: {ex}"[:300]}
        try:
            with torch.cuda.stream(stream):
                cur4 = S.BatchCursor.from_device_index(S.plan([1.0 / N_CLASSES] * N_CLASSES, BATCH, SEED), offs, mem,
                                                       device=local)
                sg = ShardedGather(cur4, local_rows, N_EXAMPLES, rank, world, BATCH, BATCHES_PER_STEP, device=local,
                                   exchange="gloo" if oversub else "nccl", group=COLL["group"])
                sg.step(out)
                torch.cuda.synchronize(dev)
                coll_barrier(dist)
                t0 = time.perf_counter()
                moved = 0
                for _ in range(args.sharded_steps):
                    _, recv = sg.step(out)
                    moved += (sum(recv) - recv[rank]) * P
                torch.cuda.synchronize(dev)
                sms = (time.perf_counter() - t0) / args.sharded_steps * 1e3
                sms = coll_reduce_ms(torch, dist, sms)
            sharded_a2a = {"value": round(images_per_step / (sms / 1e3), 1), "unit": UNIT, "ms_per_step": round(sms, 3),
                           "exchange": "gloo (oversubscribed smoke run)" if oversub else "nccl all_to_all_single",
                           "bytes_exchanged_per_step_rank0": int(moved / args.sharded_steps),
                           "timing": "host wall clock around synchronised steps (the exchange is host-driven)"}

        except Exception as ex:  # noqa: BLE001
            sharded_a2a = {"unavailable": f"{type(ex).__name__}: {ex}"[:300]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # the CPU baseline runs at N = 1 only
        threads = os.cpu_count() or 1
        v, kind, sample, used = reference_rate(max(threads * 2, 8), threads, 3)
        cpu = {"value": round(v, 1), "unit": UNIT, "cores": used, "kind": kind, "sample": sample}

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "u8", "data": "synthetic", "config": config(world, args.steps_per_draw),
                "roofline": roofline, "split_kernels": split, "exact64": exact64, "cpu_baseline": cpu, "e2e": e2e,
                "e2e_zero_copy": e2e_zc,
                "sharded_dataset": sharded, "sharded_dataset_a2a": sharded_a2a, "clocks": clk.summary(),
                "gpu_launches": int(launches), "wall_s_timed": round(t_wall, 4)}
        if oversub:
            line["oversubscribed"] = f"{world} ranks on {n_dev} GPU(s): per-rank device times summed"
        print(json.dumps(line), flush=True)
    pipe.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
