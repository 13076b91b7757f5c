"""`query` harness (paper_2404_00966_b200/cli.py; reference cli.py:147-246):
exit codes 0 / 1 / 2 / 3 and JSON-lines results.  Usage, format and I/O
failures are host-side (CPU); answering and --check need the device."""

import json
import os
import shutil
import subprocess
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

SNAP = os.path.join(GOLDEN, "snap_l2.gtsi")


def run(*args):
    p = subprocess.run([sys.executable, "-m", "paper_2404_00966_b200.cli", *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    return p.returncode, p.stdout, p.stderr


def test_usage_format_and_io_errors(tmp_path):
    assert run("query")[0] == 1                                   # missing required arguments
    assert run("bogus")[0] == 1
    wl = tmp_path / "w.txt"
    assert run("query", "--snapshot", str(tmp_path / "nope.gtsi"), "--workload", str(wl))[0] == 3
    for bad in ("X 1 0.5 0.5", "R -1 0.5 0.5", "K 0 0.5 0.5", "R 1", "I 7 0.1 0.2", "R 0.1 a b"):
        wl.write_text(f"# comment\n\n{bad}\n")
        code, _, err = run("query", "--snapshot", SNAP, "--workload", str(wl))
        assert code == 1, (bad, err)
    wl.write_text("R 0.1 0.5 0.5\n")
    assert run("query", "--snapshot", SNAP, "--workload", str(wl), "--batch-sizes", "0")[0] == 1
    bad_snap = tmp_path / "bad.gtsi"
    bad_snap.write_bytes(b"GTSX" + b"\0" * 60)
    assert run("query", "--snapshot", str(bad_snap), "--workload", str(wl))[0] == 1


@pytest.mark.gpu
def test_query_answers_check_and_mismatch(tmp_path):
    from oracle import oracle as O
    import paper_2404_00966_b200 as P
    tree = P.load_snapshot(SNAP)
    mat = tree.dataset.mat
    rng = np.random.default_rng(0)
    lines, want_ops = [], []
    for i in range(40):
        q = mat[int(rng.integers(0, mat.shape[0]))] + rng.normal(0, 0.01, mat.shape[1])
        if i % 2:
            lines.append("R 0.15 " + " ".join(repr(float(x)) for x in q))
            want_ops.append(("range", 0.15, q))
        else:
            lines.append("K 7 " + " ".join(repr(float(x)) for x in q))
            want_ops.append(("knn", 7, q))
    wl = tmp_path / "w.txt"
    wl.write_text("\n".join(lines) + "\n")
    out = tmp_path / "r.jsonl"
    code, _, err = run("--json", "query", "--snapshot", SNAP, "--workload", str(wl), "--out", str(out), "--check",
                       "--batch-sizes", "7,40")
    assert code == 0, err
    recs = [json.loads(l) for l in out.read_text().splitlines()]
    assert [r["query_index"] for r in recs] == list(range(40))
    od = O.Payloads(O.L2, vec=mat, ids=tree.dataset.ids)
    for r, (kind, v, q) in zip(recs, want_ops):
        oq = O.Payloads(O.L2, vec=q[None])
        w = (O.brute(od, oq, O.RANGE, radii=np.array([v])) if kind == "range"
             else O.brute(od, oq, O.KNN, ks=np.array([v]))).answers()[0]
        assert r["kind"] == kind
        assert [a["id"] for a in r["answers"]] == w[0].tolist()
        assert [a["distance"] for a in r["answers"]] == w[1].tolist()
    assert json.loads(err.strip().splitlines()[-1])["checked"] is True
    # a poisoned snapshot (node ranges that exclude their entries) prunes true
    # answers: --check exits 2 (reference test_cli.py:239-255)
    t2 = P.load_snapshot(SNAP)
    t2.min_dis[2:] = t2.max_dis[2:] + 10.0
    t2.max_dis[2:] = t2.min_dis[2:] + 1.0
    poisoned = tmp_path / "p.gtsi"
    P.save_snapshot(t2, str(poisoned))
    code, _, err = run("query", "--snapshot", str(poisoned), "--workload", str(wl), "--check")
    assert code == 2, err
