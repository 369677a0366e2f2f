"""Live kernel timeline of one op of a bench workload (CUPTI through
torch.profiler: kernels run back to back on the stream, not serialised as
under ncu), with the idle gaps between them -- where launch latency and host
synchronisation go.

    python scripts/timeline.py bulk_tcf insert [out.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    workload, op = sys.argv[1], sys.argv[2]
    out = sys.argv[3] if len(sys.argv) > 3 else None
    a = argparse.Namespace(workload=workload, log_slots=28, log_slots_set=False, load=0.9)
    filt, ops, x, desc, _ = bench._workload_setup(a, 0, 1, torch.device("cuda", 0), torch)
    names = [nm for nm, _, _ in ops]
    k = names.index(op)
    for _ in range(3):
        filt._reset()
        for _, fn, _ in ops:
            fn(x)
    filt._reset()
    for _, fn, _ in ops[:k]:
        fn(x)
    torch.cuda.synchronize()
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        ops[k][1](x)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda e: e.time_range.start)
    rows, t0, prev_end = [], None, None
    for e in evs:
        s, en = e.time_range.start, e.time_range.end
        if t0 is None:
            t0 = s
        rows.append({"name": e.name[:90], "start_us": s - t0, "dur_us": en - s,
                     "gap_us": 0 if prev_end is None else s - prev_end})
        prev_end = en if prev_end is None else max(prev_end, en)
    total = prev_end - t0 if rows else 0
    busy = sum(r["dur_us"] for r in rows)
    res = {"workload": workload, "op": op, "span_us": total, "busy_us": busy, "kernels": len(rows), "rows": rows}
    print("%s %s: span %.1f us, kernels busy %.1f us, %d device activities" % (workload, op, total, busy, len(rows)))
    for r in rows:
        print("  +%8.1f  gap %7.1f  dur %8.1f  %s" % (r["start_us"], r["gap_us"], r["dur_us"], r["name"]))
    if out:
        json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
