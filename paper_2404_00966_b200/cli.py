"""`query` harness over GTSI snapshots (reference cli.py:147-246, SURVEY.md
§8(f) f3): answer a workload's R / K lines from a snapshot on the device.

    python -m paper_2404_00966_b200.cli query --snapshot S --workload W
           [--out results.jsonl] [--batch-sizes 128,1024] [--check]
           [--no-prune] [--memory-units U] [--json]

Workload lines (reference io.py:217-263): `R <radius> <payload>`,
`K <k> <payload>`; `#` comments and blank lines are skipped; vector payloads
are whitespace-separated floats, string payloads one token.  Results are
JSON lines {query_index, kind, answers[{id, distance}], verified_count,
pruned_nodes} (io.py:279-295); the run report goes to stderr.  --check
re-answers every query with pruning disabled -- the exhaustive scan of every
live entry (the reference's pruning-off mode, search.py:338-355) -- and exits
2 if any answer differs.  Exit codes: 0 ok, 1 usage / validation / format
errors, 2 answers disagreeing with the exhaustive scan, 3 I/O failures.
"""

from __future__ import annotations

import argparse
import json
import sys
import time

import numpy as np

EXIT_OK, EXIT_USAGE, EXIT_MISMATCH, EXIT_IO = 0, 1, 2, 3


class WorkloadFormatError(ValueError):
    """Malformed workload line."""


class AnswerMismatch(RuntimeError):
    """Pruned answers differ from the exhaustive scan."""


def parse_workload(path, metric):
    """(kind, value, payload) per R / K line; I / D lines are rejected here
    (the reference routes them to `update`)."""
    ops = []
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, raw in enumerate(fh, start=1):
            toks = raw.split()
            if not toks or toks[0].startswith("#"):
                continue
            tag = toks[0]
            if tag in ("I", "D"):
                raise WorkloadFormatError(f"line {lineno}: query accepts only R and K lines; use update")
            if tag not in ("R", "K"):
                raise WorkloadFormatError(f"line {lineno}: unknown op tag {tag!r}")
            if len(toks) < 3:
                raise WorkloadFormatError(f"line {lineno}: {tag} needs a value and a payload")
            try:
                value = float(toks[1]) if tag == "R" else int(toks[1])
            except ValueError:
                raise WorkloadFormatError(f"line {lineno}: bad value {toks[1]!r}") from None
            if (tag == "R" and value < 0) or (tag == "K" and value < 1):
                raise WorkloadFormatError(f"line {lineno}: {'radius must be >= 0' if tag == 'R' else 'k must be >= 1'}")
            if metric == "edit":
                if len(toks) != 3:
                    raise WorkloadFormatError(f"line {lineno}: expected one string payload token")
                payload = toks[2]
            else:
                try:
                    payload = np.array([float(t) for t in toks[2:]], dtype=np.float64)
                except ValueError:
                    raise WorkloadFormatError(f"line {lineno}: not a number in the payload") from None
            ops.append(("range" if tag == "R" else "knn", value, payload))
    return ops


def _answer(searcher, ops, base):
    """One batch: its R lines as one range batch, its K lines as one kNN batch."""
    out = {}
    for kind, call in (("range", searcher.range_batch_array), ("knn", searcher.knn_batch_array)):
        sel = [i for i, op in enumerate(ops) if op[0] == kind]
        if not sel:
            continue
        res = call([ops[i][2] for i in sel], [ops[i][1] for i in sel])
        for t, i in enumerate(sel):
            a, b = res.offsets[t], res.offsets[t + 1]
            out[i] = {"query_index": base + i, "kind": kind,
                      "answers": [{"id": int(x), "distance": float(d)} for x, d in zip(res.ids[a:b], res.dis[a:b])],
                      "verified_count": int(res.stats.verified[t]), "pruned_nodes": int(res.stats.pruned_nodes[t])}
    return [out[i] for i in sorted(out)]


def cmd_query(args):
    from .search import BatchSearcher
    from .snapshot import load_snapshot
    tree = load_snapshot(args.snapshot)
    ops = parse_workload(args.workload, tree.dataset.metric)
    try:
        sizes = [int(b) for b in args.batch_sizes.split(",") if b]
    except ValueError:
        raise ValueError(f"bad batch size list {args.batch_sizes!r}") from None
    if not sizes or any(b < 1 for b in sizes):
        raise ValueError("batch sizes must be positive integers")
    searcher = BatchSearcher(tree, memory_units=args.memory_units, pruning=not args.no_prune)
    timings, records = [], []
    for bs in sizes:
        records = []
        t0 = time.perf_counter()
        for lo in range(0, len(ops), bs):
            records.extend(_answer(searcher, ops[lo:lo + bs], lo))
        sec = time.perf_counter() - t0
        timings.append({"batch_size": bs, "queries": len(ops), "seconds": round(sec, 6),
                        "qps": round(len(ops) / sec, 3) if sec > 0 else None})
    if args.check:
        scan = BatchSearcher(tree, memory_units=args.memory_units, pruning=False)
        want = []
        for lo in range(0, len(ops), max(sizes)):
            want.extend(_answer(scan, ops[lo:lo + max(sizes)], lo))
        for g, w in zip(records, want):
            if g["answers"] != w["answers"]:
                raise AnswerMismatch(f"query {g['query_index']} ({g['kind']}) disagrees with the exhaustive scan")
    fh = open(args.out, "w", encoding="utf-8") if args.out else sys.stdout
    try:
        for rec in records:
            fh.write(json.dumps(rec, separators=(", ", ": ")) + "\n")
    finally:
        if args.out:
            fh.close()
    report = {"command": "query", "snapshot": args.snapshot, "queries": len(ops), "pruning": not args.no_prune,
              "checked": bool(args.check), "total_verified": sum(r["verified_count"] for r in records),
              "total_pruned_nodes": sum(r["pruned_nodes"] for r in records), "timings": timings}
    if args.json:
        print(json.dumps(report, separators=(", ", ": ")), file=sys.stderr)
    else:
        for k, v in report.items():
            print(f"{k}: {v}", file=sys.stderr)
    return EXIT_OK


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        self.exit(EXIT_USAGE, f"{self.prog}: error: {message}\n")


def _parser():
    top = _Parser(prog="gts-b200", description=__doc__.split("\n\n")[0])
    top.add_argument("--memory-units", type=int, default=None, help="search-time row budget")
    top.add_argument("--json", action="store_true", help="emit the report as JSON")
    sub = top.add_subparsers(dest="command", required=True)
    p = sub.add_parser("query", help="answer R/K workload lines from a snapshot")
    p.add_argument("--snapshot", required=True)
    p.add_argument("--workload", required=True)
    p.add_argument("--out", help="results path (default stdout)")
    p.add_argument("--batch-sizes", default="128", help="comma list; one timing row each")
    p.add_argument("--check", action="store_true", help="verify against the exhaustive (pruning-off) scan")
    p.add_argument("--no-prune", action="store_true", help="verify every live entry")
    return top


def main(argv=None):
    from .metrics import MetricMismatchError
    from .runtime import BudgetError
    from .snapshot import SnapshotFormatError
    try:
        args = _parser().parse_args(argv)
    except SystemExit as exc:
        return int(exc.code or 0)
    try:
        return cmd_query(args)
    except AnswerMismatch as exc:
        print(f"gts-b200: reference mismatch: {exc}", file=sys.stderr)
        return EXIT_MISMATCH
    except (WorkloadFormatError, SnapshotFormatError, MetricMismatchError, BudgetError, ValueError) as exc:
        print(f"gts-b200: error: {exc}", file=sys.stderr)
        return EXIT_USAGE
    except OSError as exc:
        print(f"gts-b200: i/o error: {exc}", file=sys.stderr)
        return EXIT_IO


if __name__ == "__main__":
    sys.exit(main())
