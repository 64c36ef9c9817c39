"""Per-source-line view of an ncu SASS source page (run here, on the CPU box).

    python tools/ncu_source_lines.py SOURCE.csv OBJ.o CSV_NAME MANGLED [UNITS] > out.json

SOURCE.csv: `ncu -i rep --page source --csv --print-source sass` of a capture
(tools/ncu_cases.sh / ncu_c5_source.sh); OBJ.o: the object the kernel was
compiled into (build/codec_vN.o; its cubin's line table maps each SASS
address to codec_impl.cuh:line); CSV_NAME picks the source-page section
(first kernel whose demangled name contains it), MANGLED the same
instantiation's cubin section (a substring of its mangled name).  UNITS divides the counts (e.g. the launch's
tile count, for per-tile figures).  Prints totals and the top lines by
executed instructions, warp-stall samples and excess shared wavefronts.
"""
import collections
import csv
import json
import os
import re
import subprocess
import sys
import tempfile

COLS = ["Instructions Executed", "Warp Stall Sampling (All Samples)", "L1 Wavefronts Shared",
        "L1 Wavefronts Shared Ideal", "L1 Wavefronts Shared Excessive", "L1 Conflicts Shared N-Way"]


def line_map(obj, kernel_substr):
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True, check=True)
        cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
        txt = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
    amap, cur, on = {}, None, False
    for ln in txt.splitlines():
        if ln.startswith(".text."):
            if on:
                break
            on = kernel_substr in ln
            continue
        if not on:
            continue
        m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', ln)
        if m:
            cur = f"{m.group(1)}:{m.group(2)}"
            continue
        m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+", ln)
        if m:
            amap[int(m.group(1), 16)] = cur
    return amap


def main():
    src, obj, cname, ksub = sys.argv[1:5]
    units = float(sys.argv[5]) if len(sys.argv) > 5 else 1.0
    rows = list(csv.reader(open(src)))
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
    sec = next((a, b) for a, b in zip(starts, starts[1:] + [len(rows)]) if cname in rows[a][1])
    name = rows[sec[0]][1]
    hdr = rows[sec[0] + 1]
    H = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[sec[0] + 2:sec[1]] if len(r) == len(hdr)]
    amap = line_map(obj, ksub)
    base = int(data[0][H["Address"]], 16)
    agg = collections.defaultdict(collections.Counter)
    ops = collections.defaultdict(collections.Counter)
    tot = collections.Counter()
    for r in data:
        ln = amap.get(int(r[H["Address"]], 16) - base, "?")
        op = re.sub(r"^@!?U?P\w+\s+", "", r[H["Source"]].strip()).split(" ")[0]
        for c in COLS:
            try:
                v = float(r[H[c]] or 0) if c in H else 0.0
            except ValueError:
                v = 0.0
            agg[ln][c] += v
            tot[c] += v
        ops[ln][op] += float(r[H["Instructions Executed"]] or 0)

    def top(col, n=15):
        out = []
        for k, v in sorted(agg.items(), key=lambda x: -x[1][col])[:n]:
            out.append({"line": k, **{c: round(v[c] / units, 2) for c in COLS},
                        "ops": {o: round(c / units, 1) for o, c in ops[k].most_common(4)}})
        return out
    print(json.dumps({"kernel": name, "units": units, "totals_per_unit": {c: round(tot[c] / units, 2) for c in COLS},
                      "totals": dict(tot), "top_by_instructions": top("Instructions Executed"),
                      "top_by_stall_samples": top("Warp Stall Sampling (All Samples)"),
                      "top_by_excess_shared_wavefronts": top("L1 Wavefronts Shared Excessive", 5)}, indent=1))


if __name__ == "__main__":
    main()
