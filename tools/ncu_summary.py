"""Summarise ncu captures into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py [--launches gpurun_out/launches.csv] gpurun_out/k.ncu-rep [more.ncu-rep ...] r02

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
# plus every metric with one of these prefixes (stall sampling, pipe usage)
KEEP_PREFIX = ("smsp__pcsamp_warps_issue_stalled_", "sm__inst_executed_pipe_", "smsp__issue_active.avg.pct",
               "sm__pipe_alu_cycles_active.avg.pct", "sm__pipe_fma_cycles_active.avg.pct",
               "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "dram__throughput.avg.pct")
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
                "# compare shares of the step, not absolutes)\n")
        f.write("id,kernel,duration_ns\n")
        for i, k, t in out:
            f.write(f"{i},{k},{t:.0f}\n")
    return out


def full(path):
    """Per-kernel metrics of one capture: an .ncu-rep (exported here) or its
    `--page raw --csv` export (tools/ncu_cases.sh)."""
    if path.endswith(".csv"):
        raw = open(path).read()
    else:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = [r for r in csv.reader(raw.splitlines())]
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    rows = rows[start:]
    hdr, units = rows[0], rows[1]
    kern = {}
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        d, u = dict(zip(hdr, r)), dict(zip(hdr, units))
        m = {}
        names = KEEP + [k for k in hdr if k.startswith(KEEP_PREFIX) and k not in KEEP]
        for k in names:
            if k in d and d[k] not in ("", "0", "n/a"):
                try:
                    v, unit = float(d[k].replace(",", "")), u[k]
                except ValueError:
                    continue
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit)
                if scale:
                    v, unit = v * scale, "byte"
                m[k] = {"value": v, "unit": unit}
        rb = m.get("dram__bytes_read.sum", {}).get("value", 0.0)
        wb = m.get("dram__bytes_write.sum", {}).get("value", 0.0)
        kern[short(d["Kernel Name"])] = {"metrics": m, "dram_bytes_per_launch": rb + wb}
    return kern


def main():
    """ncu_summary.py [--launches LIST.csv] REP.ncu-rep [REP ...] TAG"""
    args = sys.argv[1:]
    lcsv = None
    if args and args[0] == "--launches":
        lcsv, args = args[1], args[2:]
    tag, reps = args[-1], args[:-1]
    raw_dir = None
    if reps and reps[0] == "--raw":  # a tools/ncu_cases.sh directory: <case>.raw.csv per case
        raw_dir = reps[1]
        reps = [os.path.join(raw_dir, f) for f in sorted(os.listdir(raw_dir)) if f.endswith(".raw.csv")]
    if lcsv:
        out = launches(lcsv, tag)
        tot = sum(t for _, _, t in out) or 1.0
        per = {}
        for _, k, t in out:
            per[k] = per.get(k, 0.0) + t
        for k, t in sorted(per.items(), key=lambda x: -x[1])[:20]:
            print(f"{k:60s} {t / 1e3:10.1f} us  {100 * t / tot:5.1f} %")
    kern = {}
    for rep in reps:
        case = os.path.basename(rep).split(".")[0] + ":" if raw_dir else ""
        for k, v in full(rep).items():
            kern[case + k] = v  # the last capture of a kernel wins (the warmed launch)
    summ = {"source": f"ncu --set full --clock-control none --import-source on (tag {tag}, B200)",
            "tag": tag,
            "note": "ncu flushes caches before each replayed kernel; writes still dirty in L2 at kernel end are "
                    "not counted in dram__bytes_write, so traffic is below the algorithmic bytes for the "
                    "write-heavy kernels",
            "kernels": kern}
    json.dump(summ, open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w"), indent=1)
    for k, v in kern.items():
        t = v["metrics"].get("gpu__time_duration.sum", {})
        print(f"{k:70s} dram {v['dram_bytes_per_launch'] / 1e6:9.2f} MB  {t.get('value')} {t.get('unit')}")


if __name__ == "__main__":
    main()
