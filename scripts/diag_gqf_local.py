import os, sys, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
os.environ["FK_GQF_SMALL"] = "0"; os.environ["FK_GQF_TRACE"] = "1"
from paper_2212_09005_b200 import Gqf
rng = np.random.default_rng(48)
q = 22
base = rng.integers(0, 2 ** 62, int(0.6 * (1 << q)), dtype=np.uint64)
g = Gqf(q=q, r=8, seed=3)
g.bulk_insert(base)
for step in range(4):
    keys = rng.integers(0, 2 ** 62, int(rng.integers(5, 100)), dtype=np.uint64)
    cur = g._cur
    if step % 2: g.insert_many(keys)
    else: g.bulk_insert(keys)
    print("step", step, "in place:", g._cur is cur, file=sys.stderr)
