"""Summarise ncu captures into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py gpurun_out/launches3.csv gpurun_out/prof3.ncu-rep [more.ncu-rep ...] r01

Writes profiles/<tag>_launches.csv (kernel, duration per launch: the
`--metrics gpu__time_duration.sum` launch list) and profiles/ncu_summary.json
(per-kernel metrics of the `--set full` capture, dram read+write bytes per
launch = the bench's `roofline.traffic`).
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEEP = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__shared_mem_per_block_dynamic"]
MODES = {"0": "exact64", "1": "exact128", "2": "f64", "3": "lossless64", "4": "lossless128"}
OUTS = {"0": "u8", "1": "f32", "2": "f16", "3": "bf16"}


def short(name):
    n = name.split("(")[0].replace("void ", "").replace("optb_b200::", "").replace("<unnamed>::", "")
    n = n.replace("unnamed>::", "").strip()
    if "<" in n:
        base, args = n.split("<", 1)
        args = [a.strip().replace("(int)", "").replace("(bool)", "") for a in args.rstrip(">").split(",")]
        tf = {"1": "true", "0": "false"}
        if base in ("k_encode_vec", "k_encode_bulk"):  # <MODE, PTRS[, DEEP]>
            args = [MODES.get(args[0], args[0])] + [tf.get(a, a) for a in args[1:]]
        elif base in ("k_decode_vec", "k_encode_generic", "k_decode_generic", "k_roundtrip_vec", "k_roundtrip_il"):
            args = [MODES.get(args[0], args[0])] + [OUTS.get(a, a) for a in args[1:2]] + \
                   [tf.get(a, a) for a in args[2:]]
        n = f"{base}<{','.join(args)}>"
    return n


def launches(path, tag):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                out.append((int(d["ID"]), short(d["Kernel Name"]), float(d["Metric Value"])))
    dst = os.path.join(ROOT, "profiles", f"{tag}_launches.csv")
    with open(dst, "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised replay:\n"
                "# compare shares of the step, not absolutes); bench.py --steps 4 --warmup 3 --e2e-steps 0 "
                "--split-steps 4 --no-cpu-baseline\n")
        f.write("id,kernel,duration_ns\n")
        for i, k, t in out:
            f.write(f"{i},{k},{t:.0f}\n")
    return out


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    kern = {}
    for r in rows[2:]:
        d, u = dict(zip(hdr, r)), dict(zip(hdr, units))
        m = {}
        for k in KEEP:
            if k in d and d[k] != "":
                v, unit = float(d[k].replace(",", "")), u[k]
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit)
                if scale:
                    v, unit = v * scale, "byte"
                m[k] = {"value": v, "unit": unit}
        rb = m.get("dram__bytes_read.sum", {}).get("value", 0.0)
        wb = m.get("dram__bytes_write.sum", {}).get("value", 0.0)
        kern.setdefault(short(d["Kernel Name"]), {"metrics": m, "dram_bytes_per_launch": rb + wb})
    return kern


def main():
    lcsv, tag, reps = sys.argv[1], sys.argv[-1], sys.argv[2:-1]
    out = launches(lcsv, tag)
    kern = {}
    for rep in reps:
        kern.update(full(rep))
    rows, P = 97 * 512, 3072
    summ = {"source": f"ncu --set full --clock-control none --import-source on on bench.py (tag {tag}, B200)",
            "note": "ncu flushes caches before each replayed kernel; writes still dirty in L2 at kernel end are "
                    "not counted in dram__bytes_write, so traffic is below the algorithmic bytes for the "
                    "write-heavy kernels",
            "algorithmic_bytes_per_launch": {"k_encode_vec<exact128,false>": rows * P * 2 + rows * 8,
                                             "k_encode_bulk<exact128,false,true>": rows * P * 2 + rows * 8,
                                             "k_decode_vec<exact128,u8,true,true>": rows * P * 2,
                                             "k_roundtrip_il<exact128,u8,false,false,true,true>": rows * P * 3 + rows * 8,
                                             "k_decode_vec<exact128,u8,true>": rows * P * 2,
                                             "k_roundtrip_vec<exact128,u8,false,false>": rows * P * 4 + rows * 8,
                                             # interleaved: the container re-read is an L2 hit
                                             "k_roundtrip_il<exact128,u8,false,false>": rows * P * 3 + rows * 8},
            "kernels": kern}
    json.dump(summ, open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w"), indent=1)
    step = {}
    # the last draw call of the fused pipeline in the launch list: its SBS
    # launches and the roundtrip launches (steps_per_draw of them) they fed
    is_rt = [k.startswith(("k_roundtrip_vec<exact128", "k_roundtrip_il<exact128")) for _, k, _ in out]
    last_rt = max(i for i, r in enumerate(is_rt) if r)
    lo = last_rt
    while lo > 0 and is_rt[lo - 1]:
        lo -= 1
    while lo > 0 and not is_rt[lo - 1]:
        lo -= 1
    for _, k, t in out[lo:last_rt + 1]:
        step[k] = step.get(k, 0) + t
    tot = sum(step.values())
    for k, t in sorted(step.items(), key=lambda x: -x[1]):
        print(f"{k:40s} {t / 1e3:8.1f} us  {100 * t / tot:5.1f} %")
    for k, v in kern.items():
        print(k, v["dram_bytes_per_launch"], v["metrics"].get("gpu__time_duration.sum"))


if __name__ == "__main__":
    main()
