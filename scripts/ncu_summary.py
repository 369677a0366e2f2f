"""Summarise ncu output for profiles/ (run here, on the .ncu-rep / csv that
gpurun brought back in gpurun_out/).

  python scripts/ncu_summary.py full  gpurun_out/x.ncu-rep  profiles/x.json
  python scripts/ncu_summary.py launches gpurun_out/launches.csv profiles/x_launches.json

`full` keeps, per captured kernel, the counters the roofline claims rest on:
duration, DRAM bytes read/written, L1/L2 sectors requested and looked up,
L2 hit rate, cross-die (ltcfabric) sectors, DRAM / SM throughput.
`launches` aggregates a `--metrics gpu__time_duration.sum` launch list into
per-kernel count / total / mean time and each kernel's share of the step.
"""

import collections
import csv
import io
import json
import subprocess
import sys

FULL_METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__sectors_read.sum",
    "dram__bytes_read.sum.per_second",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
    "lrc__lts2lrc_sectors_op_read.sum",
    "lts__t_sectors_srcunit_tex_op_read.sum",
    "lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum",
    "lts__t_sectors_srcunit_ltcfabric.sum",
    "lts__t_sector_hit_rate.pct",
    "lts__t_sector_op_read_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__grid_size",
    "launch__block_size",
    "launch__registers_per_thread",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
]


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        k = {"kernel": r[hdr.index("Kernel Name")][:160]}
        for m in FULL_METRICS:
            if m in hdr:
                i = hdr.index(m)
                v = r[i].replace(",", "")
                try:
                    v = float(v)
                except ValueError:
                    pass
                k[m] = {"value": v, "unit": units[i]}
        res.append(k)
    json.dump({"source": rep, "kernels": res}, open(out, "w"), indent=1)
    for k in res:
        print(k["kernel"][:70], {m.split(".")[0][-28:]: k[m]["value"] for m in FULL_METRICS[:3] if m in k})


def launches(path, out):
    lines = open(path).read().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    hdr, data = rows[0], rows[1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in data:
        if len(r) <= vi:
            continue
        name = r[ki]
        short = name.split("(")[0][:120]
        v = float(r[vi].replace(",", ""))
        if r[ui] == "us":
            v *= 1e3
        elif r[ui] == "ms":
            v *= 1e6
        agg.setdefault(short, []).append(v)
    total = sum(sum(v) for v in agg.values())
    res = [{"kernel": k, "launches": len(v), "total_ms": sum(v) / 1e6, "mean_ms": sum(v) / len(v) / 1e6,
            "share": sum(v) / total} for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]))]
    json.dump({"source": path, "total_ms": total / 1e6, "kernels": res}, open(out, "w"), indent=1)
    for k in res[:12]:
        print("%4d %9.3f ms  %5.1f%%  %s" % (k["launches"], k["total_ms"], 100 * k["share"], k["kernel"][:90]))


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
