"""Summarise ncu outputs into profiles/: launch-list CSV -> per-kernel shares,
full .ncu-rep -> key metrics + top stall sites.  Usage:
    python tools/ncu_summary.py launches <launches.csv> <out.md> [skip_fraction]
    python tools/ncu_summary.py full <rep.ncu-rep> <out.md>
"""
import collections
import csv
import io
import re
import subprocess
import sys


def launches(path, out, skip=0.0):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if r and r[0] == "ID":
            hdr, start = r, i + 1
            break
    ki, vi, gi, bi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size"), hdr.index("Block Size")
    mi, ui = hdr.index("Metric Name"), hdr.index("Metric Unit")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    data = [(re.sub(r"\(.*", "", r[ki]).replace("void ", ""), r[gi], r[bi],
             float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-3))
            for r in rows[start:] if len(r) > vi and r[mi] == "gpu__time_duration.sum"]
    data = data[int(len(data) * skip):]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, g, b, v in data:
        agg[(n, g, b)][0] += 1
        agg[(n, g, b)][1] += v
    tot = sum(a[1] for a in agg.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list summary ({len(data)} launches, gpu__time_duration.sum, "
                f"--clock-control none; serialized, so compare SHARES)\n\n")
        f.write(f"source: `{path}`\n\n| kernel | grid | block | launches | us/launch | total us | share |\n|---|---|---|---|---|---|---|\n")
        for (n, g, b), (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"| `{n[:70]}` | {g} | {b} | {c} | {t / c:.2f} | {t:.1f} | {100 * t / tot:.1f}% |\n")


def full(rep, out):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(det)))
    h = r[0]
    mi, vi, ui, si, ki = (h.index(x) for x in ("Metric Name", "Metric Value", "Metric Unit", "Section Name", "Kernel Name"))
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    rawv = {k: f"{v} {u}" for k, u, v in zip(rr[0], rr[1], rr[2])} if len(rr) > 2 else {}
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                         text=True).stdout
    s = list(csv.reader(io.StringIO(src)))
    with open(out, "w") as f:
        f.write(f"# ncu --set full: `{r[1][ki][:120]}`\n\nreport: `{rep}`\n\n| section | metric | value | unit |\n|---|---|---|---|\n")
        for x in r[1:]:
            if x[si] in ("GPU Speed Of Light Throughput", "Launch Statistics", "Occupancy", "Memory Workload Analysis"):
                f.write(f"| {x[si]} | {x[mi]} | {x[vi]} | {x[ui]} |\n")
        f.write("\n## raw counters\n\n")
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                  "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                  "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread"):
            for key in rawv:
                if key.startswith(k):
                    f.write(f"- `{key}` = {rawv[key]}\n")
        if len(s) > 2:
            hh = s[1]
            sti, ii = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed")
            rows = [(x[0], x[1], float(x[sti] or 0), float(x[ii] or 0)) for x in s[2:] if len(x) > ii]
            tot = sum(x[2] for x in rows) or 1
            f.write("\n## top stall sites (SASS)\n\n| share | executed | instruction |\n|---|---|---|\n")
            for a, t, smp, n in sorted(rows, key=lambda x: -x[2])[:20]:
                f.write(f"| {100 * smp / tot:.1f}% | {n:.0f} | `{t[:90]}` |\n")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3], float(sys.argv[4]) if len(sys.argv) > 4 else 0.0)
    else:
        full(sys.argv[2], sys.argv[3])
