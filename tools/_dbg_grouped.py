import os, sys, numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import paper_2404_00966_b200 as P
from oracle import oracle as O
from test_gpu_parity import string_queries
rng = np.random.default_rng(10)
alpha = "ACGT"
strs = P.generate_sequences(3000, seed=11, min_len=20, max_len=40, alphabet=alpha)
si = P.StreamingIndex(P.Dataset.from_strings(strs, P.EDIT), P.TreeConfig(8, 0), cache_capacity=64)
live = dict(enumerate(strs)); next_id = 3000; deleted = set()
for step in range(6):
    for oid in rng.choice(sorted(live), 40, replace=False):
        si.delete(int(oid)); del live[int(oid)]; deleted.add(int(oid))
    for _ in range(30):
        s = "".join(alpha[i] for i in rng.integers(0, 4, int(rng.integers(20, 41))))
        si.insert(next_id, s); live[next_id] = s; next_id += 1
    q = string_queries(list(live.values()), 10, rng, alpha)
    os.environ.pop("GTS_EDIT_GROUPED", None)
    a0, _ = si.query_range(q, 8.0)
    os.environ["GTS_EDIT_GROUPED"] = "1"
    a1, _ = si.query_range(q, 8.0)
    print("step", step, "rebuilds", si.rebuild_count, "placed", si.placed_count() if callable(getattr(si, "placed_count", None)) else "?", "pending", len(si.pending))
    for qi, (x, y) in enumerate(zip(a0, a1)):
        if not np.array_equal(x[0], y[0]):
            ex = set(y[0].tolist()) - set(x[0].tolist()); mi = set(x[0].tolist()) - set(y[0].tolist())
            print("  q", qi, "len", len(q[qi]), "extra", [(i, i in deleted, O.edit(q[qi], strs[i] if i < 3000 else live.get(i, "?"))) for i in ex],
                  "missing", [(i, i in deleted, O.edit(q[qi], live[i])) for i in mi])
