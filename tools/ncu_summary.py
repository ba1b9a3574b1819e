"""Summarise ncu outputs into profiles/: launch-list CSV -> per-kernel shares,
full .ncu-rep -> key metrics + top stall sites.  Usage:
    python tools/ncu_summary.py launches <launches.csv> <out.md> [skip_fraction]
    python tools/ncu_summary.py full <rep.ncu-rep> <out.md>
    python tools/ncu_summary.py traffic <decode.csv> <scoring.csv> <out.json>   (bench.py roofline.traffic)
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
    mi, ui, ii = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("ID")
    tscale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    bscale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    per = collections.OrderedDict()  # launch id -> {name, grid, block, t, dram}
    for r in rows[start:]:
        if len(r) <= vi:
            continue
        e = per.setdefault(r[ii], {"n": re.sub(r"\(.*", "", r[ki].replace("(anonymous namespace)::", "")).replace("void ", ""),
                                   "g": r[gi], "b": r[bi], "t": 0.0, "dram": 0.0, "has_dram": False})
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            e["t"] = v * tscale.get(r[ui], 1e-3)
        elif r[mi].startswith("dram__bytes_"):
            e["dram"] += v * bscale.get(r[ui], 1.0)
            e["has_dram"] = True
    data = list(per.values())
    data = data[int(len(data) * skip):]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    has_dram = any(x["has_dram"] for x in data)
    for x in data:
        a = agg[(x["n"], x["g"], x["b"])]
        a[0] += 1
        a[1] += x["t"]
        a[2] += x["dram"]
    tot = sum(a[1] for a in agg.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list summary ({len(data)} launches, gpu__time_duration.sum"
                f"{' + dram__bytes_{read,write}.sum' if has_dram else ''}, --clock-control none; "
                f"serialized, so compare SHARES)\n\n")
        f.write(f"source: `{path}`\n\n| kernel | grid | block | launches | us/launch | total us | share |"
                f"{' DRAM MB/launch |' if has_dram else ''}\n|---|---|---|---|---|---|---|{'---|' if has_dram else ''}\n")
        for (n, g, b), (c, t, d) in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"| `{n[:70]}` | {g} | {b} | {c} | {t / c:.2f} | {t:.1f} | {100 * t / tot:.1f}% |"
                    f"{f' {d / c / 1e6:.2f} |' if has_dram else ''}\n")
    return agg


def full(rep, out):
    """rep: a .ncu-rep, or the prefix of its exported pages (<prefix>_details.csv,
    <prefix>_raw.csv, <prefix>_source.csv: profile_round2.sh exports them on the box)."""
    if not rep.endswith(".ncu-rep"):
        return full_csv(rep, out)
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
        cs = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                            capture_output=True, text=True).stdout
        cur, hdr, lines = None, None, []
        for x in csv.reader(io.StringIO(cs)):
            if len(x) >= 2 and x[0] == "File Path":
                cur = x[1].split("/")[-1]
            elif len(x) > 2 and x[0] == "Line No":
                hdr = x
            elif hdr and len(x) > 5 and x[0]:
                try:
                    lines.append((float(x[4] or 0), cur, x[0], x[1].strip()))
                except ValueError:
                    pass
        tot = sum(x[0] for x in lines) or 1
        if lines:
            f.write("\n## top stall sites (CUDA source lines)\n\n| share | line | source |\n|---|---|---|\n")
            for smp, fn, ln, src_ in sorted(lines, reverse=True)[:20]:
                f.write(f"| {100 * smp / tot:.1f}% | {fn}:{ln} | `{src_[:90]}` |\n")


def full_csv(prefix, out):
    r = list(csv.reader(open(prefix + "_details.csv")))
    h = r[0]
    mi, vi, ui, si, ki = (h.index(x) for x in ("Metric Name", "Metric Value", "Metric Unit", "Section Name", "Kernel Name"))
    rr = [x for x in csv.reader(open(prefix + "_raw.csv")) if x]
    rawv = {k: f"{v} {u}" for k, u, v in zip(rr[0], rr[1], rr[2])} if len(rr) > 2 else {}
    with open(out, "w") as f:
        f.write(f"# ncu --set full: `{r[1][ki][:120]}`\n\nexported pages: `{prefix}_{{details,raw,source}}.csv`\n\n"
                "| section | metric | value | unit |\n|---|---|---|---|\n")
        for x in r[1:]:
            if x[si] in ("GPU Speed Of Light Throughput", "Launch Statistics", "Occupancy", "Memory Workload Analysis",
                         "Compute Workload Analysis"):
                f.write(f"| {x[si]} | {x[mi]} | {x[vi]} | {x[ui]} |\n")
        f.write("\n## raw counters\n\n")
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                  "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                  "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread"):
            for key in rawv:
                if key.startswith(k):
                    f.write(f"- `{key}` = {rawv[key]}\n")
        try:
            s = list(csv.reader(open(prefix + "_source.csv")))
        except OSError:
            s = []
        if len(s) > 2:
            hh = s[1]
            sti, ii = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed")
            rows = [(x[0], x[1], float(x[sti] or 0), float(x[ii] or 0)) for x in s[2:] if len(x) > ii]
            tot = sum(x[2] for x in rows) or 1
            f.write("\n## top stall sites (SASS)\n\n| share | executed | instruction |\n|---|---|---|\n")
            for a, t, smp, n in sorted(rows, key=lambda x: -x[2])[:20]:
                f.write(f"| {100 * smp / tot:.1f}% | {n:.0f} | `{t.strip()[:90]}` |\n")


CLASSES = (("gemm_decode_kernel", "gemm_decode"), ("attn_decode", "decode_attention"), ("sampler", "sampler"),
           ("layernorm", "layernorm"), ("gemm_tc", "gemm_tc"), ("logprob_gather", "logprob_gather"))


def traffic(dec_csv, score_csv, out):
    """Mean DRAM bytes (read + write) per launch for each bench kernel class."""
    import json
    import os
    tot = collections.defaultdict(lambda: [0, 0.0])
    for path in (dec_csv, score_csv):
        agg = launches(path, os.devnull)
        for (n, _, _), (c, _, d) in agg.items():
            for key, cls in CLASSES:
                if key in n:
                    tot[cls][0] += c
                    tot[cls][1] += d
    doc = {"source": f"{dec_csv} + {score_csv} (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                     "dram__bytes_write.sum; decode list with --cache-control none, steady state of "
                     "tools/profile_decode.py --new 88)",
           "bytes_per_launch": {k: v[1] / v[0] for k, v in tot.items() if v[0]}}
    with open(out, "w") as f:
        json.dump(doc, f, indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "traffic":
        traffic(sys.argv[2], sys.argv[3], sys.argv[4])
    elif sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3], float(sys.argv[4]) if len(sys.argv) > 4 else 0.0)
    else:
        full(sys.argv[2], sys.argv[3])
