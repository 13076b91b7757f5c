"""Time the unmodified Python reference (metrictree, /root/reference) on the
bench's words workload, to anchor bench.py's C-oracle CPU baseline to the
real package.  Runs in the build container (the
reference does not travel to the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \
        python tools/python_reference_words.py > profiles/r02_python_reference.json

Same collection and query batch as bench.py --workload words (seeds 12 / 13);
a bounded sample of the batch (range r=1 and kNN k=10), one worker
(ParallelRuntime(workers=1): the reference is GIL-bound)."""

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import metrictree as M  # noqa: E402

w = bench.WORKLOADS["words"]
codes, off = bench.gen_strings(w["n"], 12, w["min_len"], w["max_len"], w["alphabet"])
qc, qo = bench.string_queries(codes, off, w["nq"], 13, w["alphabet"])
strs = ["".join(map(chr, codes[off[i]:off[i + 1]])) for i in range(w["n"])]
qs = ["".join(map(chr, qc[qo[i]:qo[i + 1]])) for i in range(w["nq"])]
t0 = time.perf_counter()
tree = M.build(M.Dataset.from_strings(strs, "edit"), M.TreeConfig(20, 0))
build_s = time.perf_counter() - t0
rt = M.ParallelRuntime(workers=1) if hasattr(M, "ParallelRuntime") else None
eng = M.BatchSearcher(tree, runtime=rt)
sample = [qs[i] for i in range(0, w["nq"], w["nq"] // 16)]
eng.range_batch(sample[:2], 1.0)   # numba JIT warm-up
t0 = time.perf_counter()
eng.range_batch(sample, 1.0)
t_range = time.perf_counter() - t0
t0 = time.perf_counter()
eng.knn_batch(sample, 10)
t_knn = time.perf_counter() - t0
n = len(sample)
print(json.dumps({
    "what": "unmodified Python reference (metrictree BatchSearcher, 1 worker) on bench.py's words workload",
    "host": f"build container, {os.cpu_count()} cores (not the GPU box)",
    "n": w["n"], "sample_queries": n, "build_s": round(build_s, 1),
    "range_qps": round(n / t_range, 3), "knn_qps": round(n / t_knn, 3),
    "mixed_qps": round(2 * n / (t_range + t_knn), 3),
}))
