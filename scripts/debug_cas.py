"""Concurrent-mode FULL investigation (debug only)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from conftest import counter_keys
from paper_2212_09005_b200 import Tcf
from paper_2212_09005_b200.hashing import fingerprint_many, potc_pair_many
n = int(0.9 * 2 ** 20)
keys = counter_keys(1, n)
fps = fingerprint_many(keys, 0)
b1, b2 = potc_pair_many(fps, 2 ** 16)
for g in (1, 2, 4):
    for rep in range(5):
        f = Tcf(num_blocks=2 ** 16, group_width=g, mode="concurrent")
        codes = f.insert_many(keys)
        bad = np.flatnonzero(codes == 3)
        if len(bad):
            blk = f._blocks.reshape(-1, 16)
            bk = f._backing
            i = bad[0]
            print("g", g, "rep", rep, "FULL", len(bad), "first", i, "b1 used", (blk[b1[i]] > 1).sum(),
                  "b2 used", (blk[b2[i]] > 1).sum(), "backing used", (bk > 1).sum(), "of", len(bk),
                  "counters", f.counters, "codes hist", np.bincount(codes, minlength=4).tolist())
        else:
            print("g", g, "rep", rep, "ok", np.bincount(codes, minlength=4).tolist())
