"""A/B: the tensor-core L2 paths (barrier-free k_leafgroup_mma3, the default;
block-barrier k_leafgroup_mma2 in both shapes; single-stage k_leafgroup_mma)
and the CUDA-core path give identical answers and identical verified counts
(GTS_NO_MMA selects the CUDA-core path at index creation, GTS_MMA_V2 /
GTS_MMA_SHAPE / GTS_MMA_V1 the older kernels; each variant runs in its own
process)."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SCRIPT = r"""
import json, sys, numpy as np
sys.path.insert(0, %r)
import paper_2404_00966_b200 as P
rng = np.random.default_rng(0)
mat = P.generate_clustered(20000, 128, 40, seed=3, spread=0.05).astype(np.float32).astype(np.float64)
q = (mat[rng.integers(0, 20000, 300)] + rng.normal(0, 0.01, (300, 128))).astype(np.float32).astype(np.float64)
t = P.build(P.Dataset.from_vectors(mat, P.L2), P.TreeConfig(20, 0))
e = P.BatchSearcher(t)
a, s = e.range_batch(list(q), 0.6)
k, _ = e.knn_batch(list(q), 10)
print(json.dumps({"r": [x[0].tolist() for x in a], "rd": [x[1].tolist() for x in a],
                  "k": [x[0].tolist() for x in k], "kd": [x[1].tolist() for x in k],
                  "ver": s.verified.tolist()}))
""" % ROOT


def run(env_extra):
    env = dict(os.environ, **env_extra)
    out = subprocess.run([sys.executable, "-c", SCRIPT], capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_mma_equals_cuda_core_path():
    a = run({})                          # k_leafgroup_mma3 + k_recheck (default)
    b = run({"GTS_NO_MMA": "1"})         # CUDA-core k_leafgroup_vec
    c = run({"GTS_MMA_V1": "1"})         # single-stage k_leafgroup_mma, inline recheck
    d = run({"GTS_MMA_V2": "1"})         # k_leafgroup_mma2, one CTA per SM
    e = run({"GTS_MMA_V2": "1", "GTS_MMA_SHAPE": "256"})   # k_leafgroup_mma2, two CTAs per SM
    for x in (b, c, d, e):
        assert a["r"] == x["r"] and a["rd"] == x["rd"]
        assert a["k"] == x["k"] and a["kd"] == x["kd"]
        assert a["ver"] == x["ver"]
