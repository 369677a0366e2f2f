"""One op of a secondary workload between cudaProfilerStart/Stop, for ncu
(`--profile-from-start off`): every kernel the op launches is captured, so
the DRAM bytes of the whole op (the pipeline the bench's roofline names)
can be summed.  Not a bench: run under ncu only.

    ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,\
gpu__time_duration.sum,lts__t_sectors.sum,lts__t_requests.sum --csv --log-file X.csv \
        python scripts/prof_workloads.py gqf_kmer bulk_insert
    python scripts/prof_workloads.py --summarize X.csv gqf_kmer bulk_insert profiles/r2e_gqf_kmer_bulk_insert_dram.json
"""
import argparse
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(workload, op):
    import torch
    import bench
    a = argparse.Namespace(workload=workload, log_slots=28, log_slots_set=False, load=0.9)
    filt, ops, x, desc, _ = bench._workload_setup(a, 0, 1, torch.device("cuda", 0), torch)
    names = [nm for nm, _, _ in ops]
    k = names.index(op)
    for _ in range(2):  # warm-up (scratch pools, CUB temp sizes)
        filt._reset()
        for _, fn, _ in ops:
            fn(x)
    filt._reset()
    for _, fn, _ in ops[:k]:
        fn(x)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    ops[k][1](x)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(json.dumps({"workload": workload, "op": op, "items": ops[k][2], "desc": desc}))


def summarize(path, workload, op, items, out):
    lines = open(path).read().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    hdr, data = rows[0], rows[1:]
    ki, mi, vi, ui, ii = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                          hdr.index("Metric Unit"), hdr.index("ID"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "sector": 1,
             "request": 1, "": 1}
    per = collections.OrderedDict()
    for r in data:
        if len(r) <= vi:
            continue
        key = (r[ii], r[ki].split("(")[0][:100])
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
        per.setdefault(key, {})[r[mi]] = v
    kern = collections.OrderedDict()
    for (_, name), m in per.items():
        d = kern.setdefault(name, collections.Counter())
        d["launches"] += 1
        for k, v in m.items():
            d[k] += v
    tot = collections.Counter()
    for d in kern.values():
        tot.update(d)
    dram = tot["dram__bytes_read.sum"] + tot["dram__bytes_write.sum"]
    res = {"workload": workload, "op": op, "items": items, "dram_bytes": dram, "dram_bytes_per_item": dram / items,
           "time_ns_serialised": tot["gpu__time_duration.sum"],
           "l2_sectors": tot.get("lts__t_sectors.sum"), "l2_requests": tot.get("lts__t_requests.sum"),
           "source": os.path.relpath(path, ROOT),
           "how": "ncu --profile-from-start off over one call of the op (scripts/prof_workloads.py); sums over "
                  "every kernel of the op; times are ncu's serialised cold-cache durations",
           "kernels": [{"kernel": k, "launches": int(d["launches"]), "dram_bytes": d["dram__bytes_read.sum"] +
                        d["dram__bytes_write.sum"], "time_ns": d["gpu__time_duration.sum"],
                        "share": d["gpu__time_duration.sum"] / max(1.0, tot["gpu__time_duration.sum"])}
                       for k, d in sorted(kern.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"])]}
    json.dump(res, open(out, "w"), indent=1)
    print("%s %s: %.1f B/item DRAM, %d kernels" % (workload, op, dram / items, len(kern)))
    for k in res["kernels"][:10]:
        print("  %5.1f%% %8.1f us  %6.1f MB  %s" % (100 * k["share"], k["time_ns"] / 1e3, k["dram_bytes"] / 1e6,
                                                    k["kernel"][:80]))


if __name__ == "__main__":
    if sys.argv[1] == "--summarize":
        summarize(sys.argv[2], sys.argv[3], sys.argv[4], int(sys.argv[5]), sys.argv[6])
    else:
        run(sys.argv[1], sys.argv[2])
