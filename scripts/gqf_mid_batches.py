#!/usr/bin/env python
"""Mid-size GQF batches at q = 28 (half load): per batch size, the time of
one bulk insert and one bulk delete on each apply path -- the region-local
in-place apply (default), the whole-table rebuild (FK_GQF_LOCAL=0) and the
small-batch region path (FK_GQF_SMALL default, where it applies).  One JSON
line per (size, path)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2212_09005_b200 import Gqf
    q = int(sys.argv[1]) if len(sys.argv) > 1 else 28
    rng = np.random.default_rng(1)
    base = torch.from_numpy(rng.integers(0, 2 ** 62, (1 << q) // 2, dtype=np.uint64).view(np.int64)).cuda()
    g = Gqf(q=q, r=8)
    g.bulk_insert(base)
    torch.cuda.synchronize()
    paths = {"local": {"FK_GQF_SMALL": "0", "FK_GQF_LOCAL": "1"},
             "rebuild": {"FK_GQF_SMALL": "0", "FK_GQF_LOCAL": "0"},
             "small": {"FK_GQF_LOCAL": "0"}}
    for size in (100, 1000, 4000, 16000):
        keys = torch.from_numpy(rng.integers(0, 2 ** 62, size, dtype=np.uint64).view(np.int64)).cuda()
        for name, env in paths.items():
            for k in ("FK_GQF_SMALL", "FK_GQF_LOCAL"):
                os.environ.pop(k, None)
            os.environ.update(env)
            ins, dels = [], []
            for rep in range(4):
                a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                a.record()
                g.bulk_insert(keys)
                b.record()
                g.bulk_delete(keys)
                c.record()
                c.synchronize()
                if rep:
                    ins.append(a.elapsed_time(b))
                    dels.append(b.elapsed_time(c))
            print(json.dumps({"q": q, "batch": size, "path": name, "insert_ms": float(np.median(ins)),
                              "delete_ms": float(np.median(dels))}), flush=True)


if __name__ == "__main__":
    main()
