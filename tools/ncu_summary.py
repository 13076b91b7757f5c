#!/usr/bin/env python
"""Summarise gpurun_out ncu artefacts into a markdown file under profiles/.

    python tools/ncu_summary.py --tag r01d --out profiles/r01_words.md

Reads gpurun_out/launches_words_<tag>.csv (gpu__time_duration launch list,
cold-cache and serialised: compare shares, not absolutes) and
gpurun_out/prof_*_<tag>.ncu-rep (one `--set full` capture of the top kernel).
"""

from __future__ import annotations

import argparse
import collections
import csv
import glob
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots active %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads / warp instr"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers / thread"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("dram__bytes_read.sum", "DRAM bytes read"),
    ("dram__bytes_write.sum", "DRAM bytes written"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("lts__t_bytes.sum", "L2 bytes (all requests)"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % of peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1tex throughput % of peak"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe % (dup check)"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
]


def launch_table(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        name = r[ki].split("(")[0].replace("void ", "").strip()
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}[r[ui]]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v * scale
    tot = sum(v[1] for v in agg.values())
    lines = ["| kernel | launches | total ms | share |", "|---|---:|---:|---:|"]
    for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1])[:14]:
        lines.append(f"| `{k[:70]}` | {n} | {ms:.3f} | {ms / tot:.3f} |")
    lines.append(f"| **total** | {sum(v[0] for v in agg.values())} | {tot:.3f} | 1.000 |")
    return "\n".join(lines)


def raw_csv(path):
    """The raw metrics page of a capture: the .ncu-rep, or its shrunk
    <name>.raw.csv.gz (tools/ncu_shrink.sh)."""
    if path.endswith(".raw.csv.gz"):
        import gzip
        return gzip.open(path, "rt").read()
    return subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout


def full_capture(path):
    raw = raw_csv(path)
    r = list(csv.reader(io.StringIO(raw)))
    h, v = r[0], r[2] if len(r) > 2 else r[1]
    units = r[1] if len(r) > 2 else [""] * len(h)
    name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
    lines = [f"kernel: `{name[:120]}`", "", "| metric | value | unit |", "|---|---:|---|"]
    for m, label in METRICS:
        if m in h:
            lines.append(f"| {label} (`{m}`) | {v[h.index(m)]} | {units[h.index(m)]} |")
    st = [(x, float(v[h.index(x)])) for x in h
          if x.startswith("smsp__average_warps_issue_stalled") and x.endswith("per_issue_active.ratio")]
    lines += ["", "top stall reasons (warps stalled per issued instruction):", "",
              "| reason | ratio |", "|---|---:|"]
    for x, y in sorted(st, key=lambda t: -t[1])[:6]:
        lines.append(f"| {x.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} | {y:.3f} |")
    return "\n".join(lines)


def capture_traffic(path):
    """(kernel short name, dram read + write bytes) of a --set full capture."""
    raw = raw_csv(path)
    r = list(csv.reader(io.StringIO(raw)))
    h, v = r[0], r[2] if len(r) > 2 else r[1]
    units = r[1] if len(r) > 2 else [""] * len(h)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    tot = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        if m in h:
            tot += float(v[h.index(m)].replace(",", "")) * scale.get(units[h.index(m)], 1)
    name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
    short = name.split("(")[0].replace("void ", "").split("<")[0].split("::")[-1].strip()
    return short, int(tot)


def source_hotspots(src_gz, top=12):
    """Per-CUDA-line stall samples and executed instructions from the shrunk
    source page (<name>.src.csv.gz, --print-source cuda,sass)."""
    import gzip
    rows = list(csv.reader(io.StringIO(gzip.open(src_gz, "rt").read())))
    lines = []
    fname = "?"
    for r in rows:
        if r and r[0] == "File Path" and len(r) > 1:
            fname = os.path.basename(r[1])
        elif r and r[0].strip().isdigit():
            try:
                lines.append((f"{fname}:{int(r[0])}", float(r[4]), float(r[7]), r[1].strip()[:90]))
            except (ValueError, IndexError):
                pass
    ts = sum(x[1] for x in lines) or 1.0
    ti = sum(x[2] for x in lines) or 1.0
    out = ["| file:line | stall samples | instructions | source |", "|---|---:|---:|---|"]
    for ln, st, ins, src in sorted(lines, key=lambda x: -x[1])[:top]:
        out.append(f"| {ln} | {100 * st / ts:.1f}% | {100 * ins / ti:.1f}% | `{src.replace('|', '\\|')}` |")
    return "\n".join(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--workload", default="words")
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    parts = [f"# ncu summary {a.title or a.tag} ({a.workload})", ""]
    bench = os.path.join(OUT, f"bench_{a.workload}_{a.tag}.json")
    if os.path.exists(bench):
        d = json.loads(open(bench).read().strip().splitlines()[-1])
        d.pop("profile", None)
        parts += ["## bench line (same box, same build)", "", "```json", json.dumps(d, indent=1), "```", ""]
    lp = os.path.join(OUT, f"launches_{a.workload}_{a.tag}.csv")
    if os.path.exists(lp):
        parts += ["## launch list (ncu --metrics gpu__time_duration.sum --clock-control none; cold, serialised;"
                  " shares are what to compare)", "", launch_table(lp), ""]
    for rep in sorted(glob.glob(os.path.join(OUT, f"prof_*{a.workload}*_{a.tag}.ncu-rep"))
                    + sorted(glob.glob(os.path.join(OUT, f"prof_*{a.workload}*_{a.tag}.raw.csv.gz")))):
        parts += [f"## full capture `{os.path.basename(rep)}` (ncu --set full --clock-control none)", "",
                  full_capture(rep), ""]
        src = rep.replace(".raw.csv.gz", ".src.csv.gz")
        if src != rep and os.path.exists(src):
            parts += ["source hot spots (share of stall samples, share of executed warp instructions):", "",
                      source_hotspots(src), ""]
        # roofline.traffic source for bench.py: DRAM bytes per launch of the captured kernel
        kname, tb = capture_traffic(rep)
        tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        tab = json.load(open(tpath)) if os.path.exists(tpath) else {}
        tab[f"{a.workload}:{kname}"] = {"dram_bytes_per_launch": tb, "capture": os.path.basename(rep),
                                        "note": "dram__bytes_read.sum + dram__bytes_write.sum, one launch, "
                                                "ncu --set full --clock-control none"}
        json.dump(tab, open(tpath, "w"), indent=1, sort_keys=True)
    os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
    open(a.out, "w").write("\n".join(parts))
    print(a.out)


if __name__ == "__main__":
    main()
