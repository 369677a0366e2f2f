import sys, os, time
sys.path.insert(0, os.getcwd())
import torch, bench
from paper_2212_09005_b200 import BulkTcf
dev = torch.device("cuda", 0)
n = int(0.9 * (1 << 20))
keys = bench.device_keys(torch, 1, bench.TAG_UNIFORM, n, dev)
negs = bench.device_keys(torch, 2, bench.TAG_FPR, n, dev)
f = BulkTcf(num_blocks=(1 << 20) // 128)
f.insert_batch(keys)
torch.cuda.synchronize()
for name, fn in [("query", lambda: f.query_batch(keys)), ("query_neg", lambda: f.query_batch(negs))]:
    for _ in range(5): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    for _ in range(100): fn()
    e1.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(name, "event ms/op %.4f" % (e0.elapsed_time(e1) / 100), "host ms/op %.4f" % ((t1 - t0) * 10))
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(20): fn()
        torch.cuda.synchronize()
    for ev in prof.key_averages():
        if ev.device_type is not None and "k_" in ev.key:
            print("   ", ev.key[:50], "avg us %.1f" % (ev.device_time_total / max(1, ev.count)), ev.count)
# time one host call without GPU work
t0 = time.perf_counter()
for _ in range(100): f._t.before_device_op()
print("before_device_op us", (time.perf_counter() - t0) * 1e4)
