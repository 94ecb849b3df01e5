"""Summarise an ncu capture of the persistent ADMM kernel into profiles/.

usage: python tools/ncu_summary.py <report.ncu-rep> <launches.csv> <tag> [shape]

Writes profiles/<tag>.md (human summary: key counters, stall split by
barrier-delimited SASS region) and merges the per-launch DRAM traffic into
profiles/ncu_traffic.json (read by bench.py for roofline.traffic).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed_pipe_fp64.sum"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6,
        "usecond": 1e3, "msecond": 1e6, "nsecond": 1}


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def raw_metrics(rep):
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            try:
                out[k] = (float(vals[i].replace(",", "")), units[i])
            except ValueError:
                out[k] = (vals[i], units[i])
    return out


def sass_regions(rep):
    text = ncu("-i", rep, "--page", "source", "--csv", "--print-source", "sass")
    rows = list(csv.reader(io.StringIO(text)))
    hdr = rows[1]
    data = rows[2:]
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_src = hdr.index("Source")
    tot = sum(float(r[i_s] or 0) for r in data) or 1.0
    regions, acc, start = [], 0.0, 0
    for k, r in enumerate(data):
        acc += float(r[i_s] or 0)
        s = r[i_src]
        if "BAR." in s or "EXIT" in s or k == len(data) - 1:
            if acc / tot >= 0.005:
                regions.append((start, k, 100.0 * acc / tot, s.strip()[:48]))
            acc, start = 0.0, k + 1
    top = sorted(((float(r[i_s] or 0) / tot * 100, k, r[i_src].strip()[:60]) for k, r in enumerate(data)),
                 reverse=True)[:12]
    return regions, top


def launches(path):
    out = []
    with open(path) as fh:
        for r in csv.reader(l for l in fh if not l.startswith("==")):
            if len(r) > 14 and r[12] == "gpu__time_duration.sum":
                out.append((r[4], float(r[14].replace(",", ""))))
    return out


def main():
    rep, lcsv, tag = sys.argv[1:4]
    shape = sys.argv[4] if len(sys.argv) > 4 else "ieee8500"
    m = raw_metrics(rep)
    regions, top = sass_regions(rep)
    ls = launches(lcsv) if os.path.exists(lcsv) else []
    dram = None
    if "dram__bytes_read.sum" in m and "dram__bytes_write.sum" in m:
        dram = (m["dram__bytes_read.sum"][0] * UNIT.get(m["dram__bytes_read.sum"][1], 1) +
                m["dram__bytes_write.sum"][0] * UNIT.get(m["dram__bytes_write.sum"][1], 1))
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    lines = [f"# ncu summary `{tag}` ({shape})", "",
             f"report: `{os.path.basename(rep)}` (`ncu --set full --clock-control none --import-source on`, one launch)", "",
             "| metric | value | unit |", "|---|---|---|"]
    for k, (v, u) in m.items():
        lines.append(f"| {k} | {v} | {u} |")
    lines += ["", f"DRAM bytes per launch (read+write): {dram:.0f}" if dram else "", "",
              "## Launch list (`--metrics gpu__time_duration.sum`, cold, serialised)", "",
              "| kernel | ns |", "|---|---|"]
    for name, t in ls:
        lines.append(f"| {name} | {t:.0f} |")
    lines += ["", "## Warp-stall samples by barrier-delimited SASS region", "",
              "| SASS rows | share | region ends at |", "|---|---|---|"]
    for a, b, share, s in regions:
        lines.append(f"| {a}-{b} | {share:.1f}% | `{s}` |")
    lines += ["", "## Hottest SASS instructions", "", "| share | row | instruction |", "|---|---|---|"]
    for share, k, s in top:
        lines.append(f"| {share:.1f}% | {k} | `{s}` |")
    with open(os.path.join(ROOT, "profiles", f"{tag}.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    cur = {}
    if os.path.exists(tp):
        with open(tp) as fh:
            cur = json.load(fh)
    if dram is not None:
        cur[shape] = dram
        with open(tp, "w") as fh:
            json.dump(cur, fh, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
