"""Per-op end-to-end time of the C3 point-TCF ops from pinned host keys
(the bench's e2e step, op by op), against the measured H2D ceiling."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2212_09005_b200 import Tcf  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    ls = 28
    n = int(0.9 * (1 << ls))
    keys = bench.device_keys(torch, 1, bench.TAG_UNIFORM, n, dev)
    hk = torch.empty(n, dtype=torch.int64, pin_memory=True)
    hk.copy_(keys.cpu())
    f = Tcf(num_blocks=(1 << ls) // 16, mode="ordered")
    res = {}
    for rep in range(3):
        f._reset()
        for name, fn in (("insert", f.insert_many), ("query", f.query_many), ("delete", f.delete_many)):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn(hk)
            torch.cuda.synchronize()
            res.setdefault(name, []).append((time.perf_counter() - t0) * 1e3)
    out = {k: round(min(v), 2) for k, v in res.items()}
    out["h2d_ms_at_55GBs"] = round(8 * n / 55.5e9 * 1e3, 2)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
