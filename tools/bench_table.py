#!/usr/bin/env python
"""Collect bench.py JSON lines (gpurun_out/bench_<workload>_<tag>.json) into
one markdown file under profiles/: a summary table plus every line verbatim.

    python tools/bench_table.py --tag r01f --out profiles/r01_bench.md
"""

from __future__ import annotations

import argparse
import glob
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    rows, raw = [], []
    for p in sorted(glob.glob(os.path.join(OUT, f"bench_*_{a.tag}.json"))):
        name = os.path.basename(p)[len("bench_"):-len(f"_{a.tag}.json")]
        lines = [l for l in open(p).read().strip().splitlines() if l.startswith("{")]
        if not lines:
            continue
        d = json.loads(lines[-1])
        d.pop("profile", None)
        raw.append((name, d))
        rf = d.get("roofline") or {}
        cb = d.get("cpu_baseline") or {}
        e2e = d.get("e2e") or {}
        rows.append("| {} | {} | {} | {} | {} | {} | {} | {} |".format(
            name, d.get("value"), d.get("unit"), e2e.get("value"), d.get("ms_per_step"),
            f"{rf.get('kernel')} {rf.get('achieved')}/{rf.get('peak')} {rf.get('unit')} = {rf.get('frac')}" if rf else "",
            f"{cb.get('value')} {cb.get('unit')} ({cb.get('kind')}, {cb.get('cores')} cores)" if cb else "",
            (d.get("clocks") or {}).get("sm_mhz")))
    parts = [f"# bench lines, tag {a.tag} (B200, one GPU)", "",
             "| run | value | unit | e2e | ms/step | roofline (dominant kernel) | cpu baseline | SM MHz |",
             "|---|---:|---|---:|---:|---|---|---:|", *rows, ""]
    for name, d in raw:
        parts += [f"## {name}", "", "```json", json.dumps(d, indent=1), "```", ""]
    open(a.out, "w").write("\n".join(parts))
    print(a.out)


if __name__ == "__main__":
    main()
