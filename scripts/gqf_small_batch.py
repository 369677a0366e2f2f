#!/usr/bin/env python
"""Latency of small GQF insert batches into a large table (q=28, half full):
the region-local path (default) vs the full canonical rebuild
(FK_GQF_SMALL=0).  One JSON line per (path, batch size)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2212_09005_b200 import Gqf
    from paper_2212_09005_b200.workloads import counter_stream_device
    q = int(sys.argv[1]) if len(sys.argv) > 1 else 28
    g = Gqf(q=q, r=8)
    g.bulk_insert(counter_stream_device(1, 5, int(0.5 * (1 << q))))
    for limit in ("0", None):
        if limit is None:
            os.environ.pop("FK_GQF_SMALL", None)
        else:
            os.environ["FK_GQF_SMALL"] = limit
        for bs in (1, 100, 1000, 10000):
            keys = counter_stream_device(7, 9, bs * 10)
            torch.cuda.synchronize()
            t = time.perf_counter()
            for i in range(10):
                g.insert_many(keys[i * bs:(i + 1) * bs])
            torch.cuda.synchronize()
            ms = (time.perf_counter() - t) / 10 * 1e3
            torch.cuda.synchronize()
            t = time.perf_counter()
            for i in range(10):
                g.bulk_delete(keys[i * bs:(i + 1) * bs])
            torch.cuda.synchronize()
            dms = (time.perf_counter() - t) / 10 * 1e3
            print(json.dumps({"q": q, "path": "full rebuild" if limit == "0" else "region-local",
                              "batch": bs, "insert_ms_per_call": ms, "delete_ms_per_call": dms}), flush=True)


if __name__ == "__main__":
    main()
