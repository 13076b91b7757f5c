"""Row grouping at the sizes where the block-private counting sort runs
(group_rows: >= 65,536 frontier rows and <= 40k nodes; smaller batches use
the per-row-atomic kernels, which the other parity tests cover).  Answers of
the grouped vector kernels (k_leafgroup_mma3 fed by bulk-copied leaf tiles
for 128-d L2, k_leafgroup_tile for 32-d L1) against oracle brute force.
"""

import numpy as np
import pytest

import paper_2404_00966_b200 as P
from oracle import oracle as O
from test_gpu_parity import check_against_oracle, f32

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("metric,dim", [(P.L2, 128), (P.L1, 32)])
def test_block_private_grouping_at_scale(metric, dim):
    rng = np.random.default_rng(41)
    n, nq = 20_000, 1_000
    mat = f32(P.generate_clustered(n, dim, 5, seed=42, spread=0.05))
    ds = P.Dataset.from_vectors(mat, metric)
    tree = P.build(ds, P.TreeConfig(20, 0))
    q = f32(mat[rng.integers(0, n, nq)] + rng.normal(0, 0.02, (nq, dim)))
    code = O.L2 if metric == P.L2 else O.L1
    radii = rng.uniform(0.6, 1.0, nq) if metric == P.L2 else rng.uniform(1.5, 3.0, nq)
    check_against_oracle(ds, tree, list(q), O.Payloads(code, vec=mat), O.Payloads(code, vec=q),
                         radii, rng.integers(1, 60, nq), threads=16)
