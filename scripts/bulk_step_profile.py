"""Per-kernel GPU time of one configs[0] bulk-TCF step (insert, pos/neg
query, delete) next to each op's event time: the gap is launch and host
synchronisation overhead inside the op (not a bench)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import bench
from paper_2212_09005_b200 import BulkTcf

dev = torch.device("cuda", 0)
n = int(0.9 * (1 << 20))
keys = bench.device_keys(torch, 1, bench.TAG_UNIFORM, n, dev)
negs = bench.device_keys(torch, 2, bench.TAG_FPR, n, dev)
f = BulkTcf(num_blocks=(1 << 20) // 128)
ops = [("insert", lambda: f.insert_batch(keys)), ("query_pos", lambda: f.query_batch(keys)),
       ("query_neg", lambda: f.query_batch(negs)), ("delete", lambda: f.delete_batch(keys))]
for _ in range(5):
    f._reset()
    for _, fn in ops:
        fn()
torch.cuda.synchronize()
for name, fn in ops:
    f._reset()
    for pname, pfn in ops:
        if pname == name:
            break
        pfn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
    busy = 0.0
    rows = []
    for ev in prof.key_averages():
        t = ev.device_time_total
        if t > 0:
            busy += t
            rows.append((t, ev.count, ev.key[:70]))
    print("%s: event %.1f us, kernels %.1f us, launches %d" % (name, e0.elapsed_time(e1) * 1e3, busy,
                                                               sum(r[1] for r in rows)))
    for t, c, k in sorted(rows, reverse=True)[:8]:
        print("    %8.1f us  x%-3d %s" % (t, c, k))
