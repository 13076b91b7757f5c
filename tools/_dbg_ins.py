import os, sys, numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
os.environ["GTS_TRACE"] = "1"
import paper_2404_00966_b200 as P
from test_gpu_updates import make
rng = np.random.default_rng(3)
metric, payloads, new = make("dna", 12000, rng)
si = P.StreamingIndex(P.Dataset.from_strings(payloads, metric), P.TreeConfig(20, 0), cache_capacity=5000)
print("levels", si.tree.levels, file=sys.stderr)
live = {i: payloads[i] for i in range(12000)}
dels = [int(i) for i in rng.choice(sorted(live), 150, replace=False)]
ins = [(oid, new()) for oid in dels[:60]] + [(12000 + k, new()) for k in range(300)]
si.batch_update(inserts=ins, deletes=dels)
print("placed", si.placed_count, "pending", len(si.pending), file=sys.stderr)
