#!/usr/bin/env python
"""Benchmark: point TCF insert/query/delete ops/s at 0.9 load on B200.

Workload (BASELINE.json configs[2], "C3"): a point two-choice filter with
2^28 slots per GPU (num_blocks = 2^24, B = 16, 16-bit tags, 1% backing),
uniform 64-bit keys (the reference's counter_stream).  One step =
  reset table -> insert 0.9*2^28 keys -> query them (positive) ->
  query 0.9*2^28 fresh keys (negative) -> delete the inserted keys
so a step is 4 * 241,591,910 = 966,367,640 ops per GPU.  `value` is whole-job
ops/s over all ranks with keys already resident in HBM; `e2e` is the same
step through the public API from pinned host buffers (H2D of every key batch
and D2H of every result inside the timed region).  Inputs (1.9 GB key
arrays) and the 512 MiB table are larger than the 126 MB L2, so no flush is
needed between steps.

Multi-GPU (torchrun, one rank per GPU): weak scaling -- each rank owns a
2^28-slot sub-filter; keys are generated per rank and routed by the top
log2(N) fingerprint bits with an NCCL all-to-all.

`--impl reference` times the reference's own compiled kernels
(oracle/_ref, built from /root/reference/pkg/src/filterkit/_ckernels.pyx)
on the host's cores for the same metric.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "insert/query/delete ops/sec at 0.9 load (1/2/4/8 B200) + % HBM random-access roofline"
UNIT = "ops/s"
TAG_UNIFORM = 0x5851F42D4C957F2D
TAG_FPR = 0xB504F32D4F2D8C21

# Algorithmic bytes per op at 0.9 load: 8-B key, 32-B block
# sectors (b2 read on 26.0% of inserts, 14.37% of positive queries), one
# dirty 32-B sector written back per insert/delete, 1-B result.
BYTES_PER_OP = {
    "insert": 8 + 32 * (1 + 0.260) + 32 + 1,       # 81.3
    "query_pos": 8 + 32 * (1 + 0.1437) + 1,         # 45.6
    "query_neg": 8 + 64 + 1,                        # 73
    "delete": 8 + 32 * (1 + 0.1437) + 32 + 1,       # 77.6
}


# Random 32-B sectors per op (table blocks; the 5 MiB backing table is
# L2-resident): b2 read on 26.0% of inserts / 14.37% of positive queries and
# deletes, both blocks on every negative query.
SECTORS_PER_OP = {"insert": 1.260, "query_pos": 1.1437, "query_neg": 2.0, "delete": 1.1437}
# Insert/delete write one sector back: the first block touched is a random
# read-modify-write, the rest (b2 on 26.0% of inserts / 14.37% of deletes)
# plain random reads.  (rmw, extra reads) per op:
RMW_PER_OP = {"insert": (1.0, 0.260), "delete": (1.0, 0.1437), "query_pos": (0.0, 1.1437), "query_neg": (0.0, 2.0)}

# bytes each secondary-workload op returns to the host per item (e2e D2H):
# counts 8 B, found / removed flags 1 B; inserts return only failed keys
RESULT_BYTES = {"count": 8, "bulk_delete": 1, "query_pos": 1, "query_neg": 1, "delete": 1}

KERNEL_OF = {
    ("ordered", "insert"): "k_tcf_ordered1<KB=2,OP=insert> (one-barrier, u16, B=16, G=1)",
    ("ordered", "delete"): "k_tcf_ordered1<KB=2,OP=delete> (one-barrier, u16, B=16, G=1)",
    ("concurrent", "insert"): "k_tcf_insert_cas<u16,G=1,B=16>",
    ("concurrent", "delete"): "k_tcf_delete_cas<u16,G=1,B=16>",
}
for _m in ("ordered", "concurrent"):
    KERNEL_OF[(_m, "query_pos")] = KERNEL_OF[(_m, "query_neg")] = "k_tcf_query<u16,G=1,B=16>"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region.
    start() launches the sampler ahead of the warm-up (nvidia-smi takes a
    moment to produce its first row); `with sampler:` marks the timed
    window, and summary() keeps the rows that arrived inside it."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None
        self.t0 = self.t1 = None

    def start(self):
        if self.proc is None:
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                     "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self.thread = threading.Thread(target=self._read, daemon=True)
                self.thread.start()
            except OSError:
                self.proc = None
        return self

    def __enter__(self):
        self.start()
        self.t0 = time.monotonic()
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append((time.monotonic(), parts))

    def __exit__(self, *exc):
        self.t1 = time.monotonic()
        time.sleep(0.15)  # the row covering the window's end
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = [r for t, r in self.rows if self.t0 is not None and self.t0 <= t <= (self.t1 or t) + 0.12]
        window = "timed region"
        if not rows:
            rows, window = [r for _, r in self.rows], "whole run (no row inside the timed region)"
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "window": window}


def max_over_ranks(torch, value, dev):
    """Max of a float over the ranks (device tensor on NCCL, host on gloo)."""
    import torch.distributed as dist
    on = dev if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(value)], device=on, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def counter_stream(seed, tag, n):
    from paper_2212_09005_b200.workloads import counter_stream as cs
    return cs(seed, tag, n)


def device_keys(torch, seed, tag, n, device):
    """Same keys as counter_stream, generated on the device by the
    fk_counter_stream kernel (setup, not timed)."""
    from paper_2212_09005_b200.workloads import counter_stream_device
    return counter_stream_device(seed, tag, n, device)


def random_sector_ceiling(torch, filt, stream, reps=3):
    """Random 32-byte sector loads over the filter's own block table, same
    hash stream and load width as the kernels (fk_sector_gather), timed with
    CUDA events on the launching stream: the achievable random-access rate
    the per-op `frac_of_random_sector_ceiling` figures are against."""
    from paper_2212_09005_b200 import _lib
    lib = _lib.load()
    tab = filt._t.dev["blocks"]
    sink = torch.zeros(32, dtype=torch.int32, device=tab.device)
    n = 1 << 28
    sp = ctypes.c_void_p(stream.cuda_stream)
    _lib.check(lib.fk_sector_gather(_lib.dptr(tab), tab.numel(), n, 1, _lib.dptr(sink), sp), "gather")
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for r in range(reps):
        _lib.check(lib.fk_sector_gather(_lib.dptr(tab), tab.numel(), n, 2 + r, _lib.dptr(sink), sp), "gather")
    b.record(stream)
    b.synchronize()
    ms = a.elapsed_time(b) / reps
    sps = n / (ms / 1e3)
    # read-modify-write ceiling on a scratch table of the same size
    scratch = torch.zeros_like(tab)
    _lib.check(lib.fk_sector_rmw(_lib.dptr(scratch), scratch.numel(), n, 1, sp), "rmw")
    a.record(stream)
    for r in range(reps):
        _lib.check(lib.fk_sector_rmw(_lib.dptr(scratch), scratch.numel(), n, 2 + r, sp), "rmw")
    b.record(stream)
    b.synchronize()
    rmw = n / (a.elapsed_time(b) / reps / 1e3)
    del scratch
    return {"sectors_per_s": sps, "useful_gbs": 32 * sps / 1e9, "rmw_sectors_per_s": rmw,
            "table_bytes": tab.numel(),
            "how": "fk_sector_gather: %d random 32-B sector loads (ld.global.v8) over the %d MiB block table; "
                   "fk_sector_rmw: the same stream as load + 16-bit store back (the insert/delete pattern) on a "
                   "scratch table of the same size; mean of %d, CUDA events" % (n, tab.numel() >> 20, reps)}


def op_ceiling(op, ceiling):
    """Achievable ops/s of `op` if every access ran at the measured random
    ceilings: 1 read-modify-write and/or extra random sector reads per op."""
    rmw, reads = RMW_PER_OP[op]
    return 1.0 / (rmw / ceiling["rmw_sectors_per_s"] + reads / ceiling["sectors_per_s"])


def _newest_first(paths):
    """Committed captures, newest session tag first (r2x2_ after r2x_: the
    tag before the first underscore, compared as a string)."""
    return sorted(paths, key=lambda p: os.path.basename(p).split("_")[0], reverse=True)


def ncu_traffic(mode, op, n):
    """DRAM bytes (read + write) per launch of the dominant kernel from the
    committed ncu --set full summary (profiles/)."""
    import glob
    want = {"insert": "OP=insert", "delete": "OP=delete"}.get(op)
    for path in _newest_first(glob.glob(os.path.join(ROOT, "profiles", "*tcf_point_%s_full.json" % mode))):
        d = json.load(open(path))
        ks = d["kernels"]
        idx = {"insert": 0, "query_pos": 1, "query_neg": 2, "delete": 3}.get(op)
        if idx is None or idx >= len(ks):
            continue
        k = ks[idx]
        rd = k["dram__bytes_read.sum"]["value"] * _unit(k["dram__bytes_read.sum"]["unit"])
        wr = k["dram__bytes_write.sum"]["value"] * _unit(k["dram__bytes_write.sum"]["unit"])
        return {"bytes_per_launch": rd + wr, "bytes_per_op": (rd + wr) / n,
                "source": os.path.relpath(path, ROOT) + " :: " + k["kernel"][:60]}
    return None


def _unit(u):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)


def count_launches(torch, step):
    """Kernels launched by one untimed step, counted with the CUDA profiler
    (activity trace) -- ours are the fk:: kernels and the CUB algorithms
    compiled into libfkb200.so."""
    try:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step()
            torch.cuda.synchronize()
        names = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
        return sum(1 for nm in names if "fk::" in nm or "cub::" in nm or nm.startswith("k_"))
    except Exception:  # profiler unavailable: report unknown rather than guess
        return None


def zipf_queries(torch, filt, keys, stream, s=1.5, reps=3):
    """Skewed lookups on the filled table (secondary numbers, not in `value`):
    positive queries whose key ranks follow the reference's bounded Zipf(s)
    sampler (fk/workloads.py:81-118) over the inserted keys, 2^24 host draws
    tiled to one query per inserted key.  Hot keys' blocks stay in L2."""
    from paper_2212_09005_b200.workloads import zipf_bounded
    n = keys.numel()
    rng = np.random.default_rng(12345)
    ranks = zipf_bounded(rng, s, n, 1 << 24) - 1
    perm = torch.from_numpy(ranks).to(keys.device)
    idx = perm.repeat((n + perm.numel() - 1) // perm.numel())[:n]
    q = keys[idx]
    filt.query_many(q)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        found = filt.query_many(q)
    b.record(stream)
    b.synchronize()
    ms = a.elapsed_time(b) / reps
    return {"ops_per_s": n / (ms / 1e3), "ms": ms, "zipf_s": s, "all_found": bool(found.all()),
            "how": "query_many of %d keys with Zipf(%.1f) ranks over the inserted keys" % (n, s)}


def zipf_inserts(torch, f, keys, stream, s=1.5, reps=2):
    """Zipfian 64-bit keys into a fresh table (north star: "uniform and
    Zipfian 64-bit keys"): one insert per inserted-key slot of the uniform
    run, the key drawn with the reference's bounded Zipf(s) ranks over the
    uniform keys (fk/workloads.py:81-118; 2^24 host draws tiled), so the hot
    keys repeat millions of times, fill their two blocks and backing chain,
    and the rest come back FULL.  Concurrent mode only: the ordered mode
    serialises every copy of a key on its blocks (one round each) by design."""
    from paper_2212_09005_b200.workloads import zipf_bounded
    n = keys.numel()
    rng = np.random.default_rng(54321)
    ranks = torch.from_numpy(zipf_bounded(rng, s, n, 1 << 24) - 1).to(keys.device)
    q = keys[ranks.repeat((n + ranks.numel() - 1) // ranks.numel())[:n]]
    ms = []
    for _ in range(reps + 1):
        f._reset()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        codes = f.insert_many(q)
        b.record(stream)
        b.synchronize()
        ms.append(a.elapsed_time(b))
    ms = float(np.mean(ms[1:]))
    hist = torch.bincount(codes.to(torch.int64), minlength=4).tolist()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    found = f.query_many(q)
    b.record(stream)
    b.synchronize()
    qms = a.elapsed_time(b)
    return {"insert_ops_per_s": n / (ms / 1e3), "insert_ms": ms, "query_ops_per_s": n / (qms / 1e3),
            "query_ms": qms, "zipf_s": s, "distinct_keys": int(torch.unique(q).numel()),
            "codes": {"primary": hist[0], "secondary": hist[1], "backing": hist[2], "full": hist[3]},
            "all_found": bool(found.all()),
            "how": "concurrent-mode insert_many of %d keys with Zipf(%.1f) ranks over the uniform keys, then "
                   "query_many of the same stream" % (n, s)}


def concurrent_mode(torch, nb, args, keys, negs, stream, ceiling=None, steps=2):
    """The paper's free-threaded CAS mode on the same workload (secondary
    numbers; not bit-identical to the sequential reference)."""
    from paper_2212_09005_b200 import Tcf
    f = Tcf(num_blocks=nb, group_width=args.group_width, mode="concurrent")
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    res = {}
    n = keys.numel()
    for s in range(steps + 1):
        f._reset()
        evs[0].record(stream)
        f.insert_many(keys)
        evs[1].record(stream)
        f.query_many(keys)
        evs[2].record(stream)
        f.query_many(negs)
        evs[3].record(stream)
        f.delete_many(keys)
        evs[4].record(stream)
        torch.cuda.synchronize()
        if s:
            for i, op in enumerate(("insert", "query_pos", "query_neg", "delete")):
                res.setdefault(op, []).append(evs[i].elapsed_time(evs[i + 1]))
    out = {op: {"ops_per_s": n / (np.mean(v) / 1e3), "ms": float(np.mean(v))} for op, v in res.items()}
    if ceiling:
        for op in out:
            out[op]["frac_of_random_access_ceiling"] = out[op]["ops_per_s"] / op_ceiling(op, ceiling)
    out["step_ops_per_s"] = 4 * n / (sum(np.mean(v) for v in res.values()) / 1e3)
    out["zipf_inserts"] = zipf_inserts(torch, f, keys, stream)
    del f
    torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args, rank, world, local_rank):
    import torch
    from paper_2212_09005_b200 import Tcf

    local_rank %= torch.cuda.device_count()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    log_slots = args.log_slots
    nb = (1 << log_slots) // 16
    n = int(args.load * (1 << log_slots))
    dist = None
    if world > 1:
        import torch.distributed as dist
    # per-rank disjoint key streams
    keys = device_keys(torch, 1 + 1000 * rank, TAG_UNIFORM, n, dev)
    negs = device_keys(torch, 2 + 1000 * rank, TAG_FPR, n, dev)

    if world > 1:
        from paper_2212_09005_b200.sharding import ShardedTcf
        filt = ShardedTcf(num_blocks=nb * world, group_width=args.group_width, mode=args.mode)
    else:
        filt = Tcf(num_blocks=nb, group_width=args.group_width, mode=args.mode)

    ops = ("insert", "query_pos", "query_neg", "delete")
    stream = torch.cuda.current_stream()

    def step(ev=None):
        filt._reset()
        if ev:
            ev[0].record(stream)
        codes = filt.insert_many(keys)
        if ev:
            ev[1].record(stream)
        fpos = filt.query_many(keys)
        if ev:
            ev[2].record(stream)
        fneg = filt.query_many(negs)
        if ev:
            ev[3].record(stream)
        rem = filt.delete_many(keys)
        if ev:
            ev[4].record(stream)
        return codes, fpos, fneg, rem

    clk = ClockSampler(local_rank).start()  # running before the timed region starts
    for _ in range(args.warmup):
        codes, fpos, fneg, rem = step()
    torch.cuda.synchronize()
    # sanity (outside timing): nothing FULL, no false negatives
    n_full = int((codes == 3).sum())
    n_fn = int((~fpos).sum())
    fpr = float(fneg.float().mean())
    n_rem = int(rem.sum())

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with clk:
        t0.record(stream)
        for s in range(args.steps):
            step(evs[s])
        t1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms_total = t0.elapsed_time(t1)
    per_op_ms = {op: float(np.mean([evs[s][i].elapsed_time(evs[s][i + 1]) for s in range(args.steps)]))
                 for i, op in enumerate(ops)}
    if dist:
        ms_total = max_over_ranks(torch, ms_total, dev)
    ms_step = ms_total / args.steps
    total_ops = 4 * n * world
    value = total_ops / (ms_step / 1e3)

    # ---- end to end through the public API from pinned host memory ----------
    e2e = None
    if not args.no_e2e:
        hk = torch.empty(n, dtype=torch.int64, pin_memory=True)
        hn = torch.empty(n, dtype=torch.int64, pin_memory=True)
        hk.copy_(keys.cpu())
        hn.copy_(negs.cpu())
        e2e_steps = max(1, min(args.steps, 3))

        def e2e_step():
            filt._reset()
            c = filt.insert_many(hk)
            fp_ = filt.query_many(hk)
            fn_ = filt.query_many(hn)
            r = filt.delete_many(hk)
            return c, fp_, fn_, r
        e2e_step()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        ts = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        te = (time.perf_counter() - ts) / e2e_steps
        if dist:
            te = max_over_ranks(torch, te, dev)
        e2e = {"value": total_ops / te, "unit": UNIT, "h2d_bytes_per_step": 4 * 8 * n,
               "d2h_bytes_per_step": 4 * n, "ms_per_step": te * 1e3}
        del hk, hn

    peak, peak_kind = peaks()
    dom = max(per_op_ms, key=per_op_ms.get)
    local = filt._local if world > 1 else filt
    ceiling = random_sector_ceiling(torch, local, stream)
    per_op = {}
    for op in ops:
        rate = n / (per_op_ms[op] / 1e3)
        gbs = BYTES_PER_OP[op] * rate / 1e9
        per_op[op] = {"ops_per_s": rate, "ms": per_op_ms[op], "achieved_gbs": gbs,
                      "frac_of_%s_hbm" % peak_kind: gbs / peak,
                      "random_sectors_per_op": SECTORS_PER_OP[op],
                      "frac_of_random_sector_ceiling": SECTORS_PER_OP[op] * rate / ceiling["sectors_per_s"],
                      "random_access_ceiling_ops_per_s": op_ceiling(op, ceiling),
                      "frac_of_random_access_ceiling": rate / op_ceiling(op, ceiling)}
    achieved = BYTES_PER_OP[dom] * n / (per_op_ms[dom] / 1e3) / 1e9
    traffic = ncu_traffic(args.mode, dom, n)
    launches = count_launches(torch, step) if not args.no_launch_count else None
    conc = None
    zq = None
    if world == 1 and not args.no_concurrent:
        filt._reset()
        filt.insert_many(keys)
        zq = zipf_queries(torch, filt, keys, stream)
    if args.mode == "ordered" and not args.no_concurrent and world == 1:
        conc = concurrent_mode(torch, nb, args, keys, negs, stream, ceiling)
    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u16", "data": "synthetic",
        "config": {"workload": "C3: point TCF, 2^%d slots/GPU (nb=2^%d x B=16, 16-bit tags, 1%% backing), "
                               "uniform 64-bit keys, insert+pos query+neg query+delete at %.2f load"
                               % (log_slots, log_slots - 4, args.load),
                   "keys_per_op_per_gpu": n, "mode": args.mode, "group_width": args.group_width,
                   "l2": (("inputs (%.1f GB keys) and table (%d MiB) exceed the 126 MB L2; no flush"
                           if (1 << log_slots) * 2 > (126 << 20) else
                           "inputs %.1f GB; the %d MiB table is L2-resident (an L2-resident configuration, "
                           "not the headline)") % (8 * n / 1e9, (1 << log_slots) * 2 >> 20)),
                   "parallelism": ("hash-prefix shards x%d, %s" % (
                       world, "peer-memory exchange (fk_shard_dispatch/combine)"
                       if type(filt._router).__name__ == "_PeerRouter" and not filt._router.fallback
                       else "all-to-all exchange")) if world > 1 else "single GPU"},
        "per_op": per_op,
        "roofline": {"bound": "hbm", "kernel": KERNEL_OF[(args.mode, dom)], "op": dom, "achieved": achieved,
                     "peak": peak, "unit": "GB/s", "frac": achieved / peak, "peak_kind": peak_kind,
                     "bytes_per_op": BYTES_PER_OP[dom], "traffic": traffic["bytes_per_launch"] if traffic else None,
                     "traffic_bytes_per_op": traffic["bytes_per_op"] if traffic else None,
                     "traffic_source": traffic["source"] if traffic else None},
        "random_access_roofline": ceiling,
        "e2e": e2e,
        "gpu_launches": launches * args.steps if launches is not None else None,
        "gpu_launches_per_step": launches,
        "clocks": clk.summary(),
        "checks": {"full_codes": n_full, "false_negatives": n_fn, "neg_fpr": fpr, "removed": n_rem},
    }
    if conc:
        result["concurrent_mode"] = conc
    if zq:
        result["zipf_queries"] = zq
    if rank == 0 and world == 1 and not args.no_cpu:
        result["cpu_baseline"] = cpu_baseline(log_slots, args.load)
    return result if rank == 0 else None


# ---------------------------------------------------------------------------
# secondary workloads: bulk TCF (configs[0] shape) and GQF (configs[1], C2)
# ---------------------------------------------------------------------------

def _workload_setup(args, rank, world, dev, torch):
    """-> (filter, {op: (fn(dev_inputs), n_items)}, inputs, describe, cpu_fn)."""
    seed = 1 + 1000 * rank
    if args.workload == "bulk_tcf":
        from paper_2212_09005_b200 import BulkTcf
        from paper_2212_09005_b200.sharding import ShardedBulkTcf
        log_slots = args.log_slots if args.log_slots_set else 20
        nb = (1 << log_slots) // 128
        n = int(args.load * (1 << log_slots))
        filt = ShardedBulkTcf(num_blocks=nb * world) if world > 1 else BulkTcf(num_blocks=nb)
        keys = device_keys(torch, seed, TAG_UNIFORM, n, dev)
        negs = device_keys(torch, seed + 1, TAG_FPR, n, dev)
        ops = [("insert", lambda x: filt.insert_batch(x["keys"]), n),
               ("query_pos", lambda x: filt.query_batch(x["keys"]), n),
               ("query_neg", lambda x: filt.query_batch(x["negs"]), n),
               ("delete", lambda x: filt.delete_batch(x["keys"]), n)]
        desc = ("configs[0] shape: bulk TCF, 2^%d slots/GPU (nb=2^%d x B=128, 16-bit tags, 1%% backing), uniform "
                "64-bit keys, one insert_batch to %.2f load + pos/neg query_batch + delete_batch"
                % (log_slots, log_slots - 7, args.load))
        return filt, ops, {"keys": keys, "negs": negs}, desc, ("bulk_tcf", log_slots, args.load)
    from paper_2212_09005_b200 import Gqf
    from paper_2212_09005_b200.sharding import ShardedGqf
    from paper_2212_09005_b200.workloads import WorkloadSpec, gen_keys
    if args.workload == "gqf_kmer":
        # C4: Zipfian k-mer-like counting at load factor args.load
        q = args.log_slots if args.log_slots_set else 28
        w = kmer_zipf_workload(torch, q, args.load, seed, dev)
        filt = ShardedGqf(q=q + (world.bit_length() - 1)) if world > 1 else Gqf(q=q)
        x = {"occ": w["occ"], "uniq": w["uniq"]}
        ops = [("bulk_insert", lambda d: filt.bulk_insert(d["occ"]), w["n_occ"]),
               ("count", lambda d: filt.count_many(d["uniq"]), w["n_distinct"]),
               ("bulk_delete", lambda d: filt.bulk_delete(d["uniq"]), w["n_distinct"])]
        desc = ("C4: GQF q=%d r=8 per GPU, k-mer-like keys: %d distinct with Zipf(%.1f) multiplicities on "
                "[1, %d] (%d occurrences, shuffled), sized for load factor %.2f; naive bulk_insert of every "
                "occurrence + count_many(distinct) + bulk_delete(distinct, all copies)"
                % (q, w["n_distinct"], w["s"], w["cmax"], w["n_occ"], args.load))
        return filt, ops, x, desc, ("gqf_kmer", q, args.load)
    # GQF, C2: duplicate-heavy ur_count keys (counts U{1..100}), naive bulk insert
    q = args.log_slots if args.log_slots_set else 22
    occ = gen_keys(WorkloadSpec("ur_count", n=int(args.load * (1 << q)) // 4, seed=seed))
    uniq = np.unique(occ)
    filt = ShardedGqf(q=q + (world.bit_length() - 1)) if world > 1 else Gqf(q=q)
    x = {"occ": torch.from_numpy(occ.view(np.int64)).to(dev), "uniq": torch.from_numpy(uniq.view(np.int64)).to(dev)}
    ops = [("bulk_insert", lambda d: filt.bulk_insert(d["occ"]), len(occ)),
           ("count", lambda d: filt.count_many(d["uniq"]), len(uniq)),
           ("bulk_delete", lambda d: filt.bulk_delete(d["uniq"]), len(uniq))]
    desc = ("C2: GQF q=%d r=8 per GPU, ur_count keys (%d distinct x U{1..100} = %d occurrences), naive bulk_insert "
            "of every occurrence + count_many(distinct) + bulk_delete(distinct, all copies)" % (q, len(uniq), len(occ)))
    return filt, ops, x, desc, ("gqf", q, args.load)


def _expected_group_len(counts, r, rng):
    """Mean slots per distinct fingerprint under the count-group codec
    (fk/countgroups.py:28-52) for uniformly random remainders."""
    rem = rng.integers(0, 1 << r, len(counts))
    c = counts.astype(np.int64)
    base = (1 << r) - 1
    v = np.where(rem > 0, (c - 2) // np.maximum(rem, 1), 0)
    nd = np.zeros_like(v)
    t = v.copy()
    while (t > 0).any():
        nd += t > 0
        t //= base
    ln = np.where((rem == 0) | (c <= 2), c, 3 + nd)
    return float(ln.mean())


def _kmer_counts(q, alpha, seed, s, cmax, r):
    from paper_2212_09005_b200.workloads import zipf_bounded
    rng = np.random.default_rng(0x5EED0000 + seed)
    mean_len = _expected_group_len(zipf_bounded(rng, s, cmax, 1 << 20), r, rng)
    d = max(1, int(alpha * (1 << q) / mean_len))
    return zipf_bounded(rng, s, cmax, d), mean_len


def kmer_zipf_host(q, alpha, seed, s=1.5, cmax=100, r=8):
    """Host twin of kmer_zipf_workload (same distinct keys and multiplicities;
    host shuffle) for the CPU baseline sample."""
    from paper_2212_09005_b200.workloads import TAG_BASES
    counts, _ = _kmer_counts(q, alpha, seed, s, cmax, r)
    uniq = counter_stream(seed, TAG_BASES, len(counts))
    occ = np.repeat(uniq, counts)
    np.random.default_rng(seed).shuffle(occ)
    return occ, uniq


def kmer_zipf_workload(torch, q, alpha, seed, dev, s=1.5, cmax=100, r=8):
    """C4 keys (BASELINE.json configs[3]): a k-mer-count spectrum -- D
    distinct uniform 64-bit keys (counter_stream, TAG_BASES) whose
    multiplicities are bounded Zipf(s) on [1, cmax] drawn with the
    reference's own rejection-inversion sampler (fk/workloads.py:81-118), each
    key repeated that many times and the stream shuffled (the structure of
    the reference's ur_count, fk/workloads.py:66-71, with Zipfian instead of
    uniform counts).  D is sized so the canonical table fills alpha * 2^q
    slots (plain Zipf ranks leave the table nearly empty).
    The multiplicities are host numpy draws; keys, repetition and shuffle are
    generated on the device (setup, not timed)."""
    from paper_2212_09005_b200.workloads import TAG_BASES
    counts, mean_len = _kmer_counts(q, alpha, seed, s, cmax, r)
    d = len(counts)
    uniq = device_keys(torch, seed, TAG_BASES, d, dev)
    cnt = torch.from_numpy(counts).to(dev)
    occ = torch.repeat_interleave(uniq, cnt)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    occ = occ[torch.randperm(occ.numel(), device=dev, generator=g)]
    return {"occ": occ, "uniq": uniq, "counts": cnt, "n_occ": int(occ.numel()), "n_distinct": d,
            "s": s, "cmax": cmax, "mean_slots_per_key": mean_len}


def _workload_bytes(args, filt, ops, world):
    """Algorithmic bytes per item of each op of a secondary workload (the
    figure its `roofline.achieved` is computed from):
    * bulk TCF insert: the 8-B key read once plus the block table, fill and
      backing arrays read and written once per batch (2 x table bytes / n);
    * bulk TCF query: 8-B key + the 256-B b1 block (+ b2 on 14.4 %) + 1-B flag;
    * bulk TCF delete: as the query plus the block written back;
    * GQF bulk insert / delete (per occurrence / key): 8-B key read, one
      8-B partition scatter + gather, and the table read and written once per
      batch (2 x table bytes / items) -- SURVEY 8(d);
    * GQF count: 8-B key + occupieds, runends and slot sectors + 8-B count."""
    t = filt._local if world > 1 else filt
    if args.workload == "bulk_tcf":
        tab = sum(v.numel() for v in t._t.dev.values())
        n = ops[0][2]
        return {"insert": 8 + 2.0 * tab / n, "query_pos": 8 + 256 * 1.144 + 1, "query_neg": 8 + 512 + 1,
                "delete": 8 + 256 * 1.144 + 256 + 1}, tab
    tab = sum(v.numel() for v in t._cur.dev.values())
    b = {name: (8 + 16 + 2.0 * tab / n) for name, _, n in ops if name != "count"}
    b["count"] = 8 + 3 * 32 + 8
    return b, tab


def _workload_kernel(workload, op):
    if workload == "bulk_tcf":
        return {"insert": "fk_btcf_insert pipeline (CUB partition sort + k_btcf_merge + route + backing)",
                "query_pos": "k_btcf_query", "query_neg": "k_btcf_query",
                "delete": "fk_btcf_delete pipeline (sort + k_btcf_delete x2 + backing)"}[op]
    return {"bulk_insert": "fk_gqf_apply insert pipeline (hash + two MSD partition passes + shared-memory "
                           "aggregation + decode/merge + region-parallel placement)",
            "count": "k_gqf_count",
            "bulk_delete": "fk_gqf_apply delete pipeline (sort + reduce + found walk + decode/merge + "
                           "region-parallel placement)"}[op]


def _workload_traffic(workload, op, items):
    """DRAM bytes (read + write) of the op's kernels per launch of the op,
    from the newest committed ncu capture of that workload (profiles/
    r2*_<workload>_<op>_dram.json, written by scripts/prof_workloads.py)."""
    import glob
    for path in _newest_first(glob.glob(os.path.join(ROOT, "profiles", "*_%s_%s_dram.json" % (workload, op)))):
        d = json.load(open(path))
        return {"bytes_per_launch": d["dram_bytes"] * items / d["items"], "bytes_per_op": d["dram_bytes"] / d["items"],
                "source": os.path.relpath(path, ROOT)}
    return None


def run_workload(args, rank, world, local_rank):
    import torch
    local_rank %= torch.cuda.device_count()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
    filt, ops, x, desc, cpu_key = _workload_setup(args, rank, world, dev, torch)
    stream = torch.cuda.current_stream()

    def step(ev=None, inp=x):
        filt._reset()
        out = []
        for i, (_, fn, _) in enumerate(ops):
            if ev:
                ev[i].record(stream)
            out.append(fn(inp))
        if ev:
            ev[len(ops)].record(stream)
        return out

    clk = ClockSampler(local_rank).start()  # running before the timed region starts
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # at least ~1.5 s of timed steps, so the clock sampler sees the load
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    step()
    t1.record(stream)
    t1.synchronize()
    one = t0.elapsed_time(t1)
    steps = args.steps
    if not args.exact_steps:
        steps = max(steps, min(400, int(1500.0 / max(one, 1e-3)) + 1))
    if dist:
        t = torch.tensor([steps], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        steps = int(t.item())
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(len(ops) + 1)] for _ in range(steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with clk:
        t0.record(stream)
        for s in range(steps):
            step(evs[s])
        t1.record(stream)
        torch.cuda.synchronize()
    ms_total = t0.elapsed_time(t1)
    if dist:
        ms_total = max_over_ranks(torch, ms_total, dev)
    ms_step = ms_total / steps
    items = sum(n for _, _, n in ops)
    per_op = {}
    for i, (name, _, n) in enumerate(ops):
        ms = float(np.mean([evs[s][i].elapsed_time(evs[s][i + 1]) for s in range(steps)]))
        per_op[name] = {"ops_per_s": n / (ms / 1e3), "ms": ms, "items": n}
    e2e = None
    if not args.no_e2e:
        hx = {k: v.cpu().pin_memory() for k, v in x.items()}
        step(inp=hx)
        torch.cuda.synchronize()
        ne = max(1, min(steps, 3))
        tsum = time.perf_counter()
        for _ in range(ne):
            step(inp=hx)
        torch.cuda.synchronize()
        te = (time.perf_counter() - tsum) / ne
        if dist:
            te = max_over_ranks(torch, te, dev)
        e2e = {"value": items * world / te, "unit": UNIT, "ms_per_step": te * 1e3,
               "h2d_bytes_per_step": 8 * items,
               "d2h_bytes_per_step": sum(RESULT_BYTES.get(name, 0) * m for name, _, m in ops)}
    launches = count_launches(torch, step) if not args.no_launch_count else None
    peak, peak_kind = peaks()
    bpo, tab = _workload_bytes(args, filt, ops, world)
    dom = max(per_op, key=lambda k: per_op[k]["ms"])
    for name in per_op:
        gbs = bpo[name] * per_op[name]["ops_per_s"] / 1e9
        per_op[name].update({"bytes_per_op": bpo[name], "achieved_gbs": gbs, "frac_of_%s_hbm" % peak_kind: gbs / peak})
    traffic = _workload_traffic(args.workload, dom, per_op[dom]["items"])
    achieved = per_op[dom]["achieved_gbs"]
    res = {"metric": METRIC, "value": items * world / (ms_step / 1e3), "unit": UNIT, "n_gpus": world,
           "steps": steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "u16" if args.workload == "bulk_tcf" else "u8",
           "data": "synthetic",
           "config": {"workload": desc, "table_bytes": tab,
                      "l2": "no flush: inputs + tables rewritten per step (table %s the 126 MB L2)"
                            % ("inside" if tab < (126 << 20) else "larger than")},
           "per_op": per_op,
           "roofline": {"bound": "hbm", "kernel": _workload_kernel(args.workload, dom), "op": dom,
                        "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                        "peak_kind": peak_kind, "bytes_per_op": bpo[dom],
                        "traffic": traffic["bytes_per_launch"] if traffic else None,
                        "traffic_bytes_per_op": traffic["bytes_per_op"] if traffic else None,
                        "traffic_source": traffic["source"] if traffic else None},
           "e2e": e2e, "gpu_launches": launches * steps if launches is not None else None,
           "gpu_launches_per_step": launches, "clocks": clk.summary()}
    if rank == 0 and world == 1 and not args.no_cpu:
        res["cpu_baseline"] = cpu_baseline_workload(cpu_key)
    return res if rank == 0 else None


def cpu_baseline_workload(key):
    """The unmodified reference package (baseline/_ref) on all host cores on
    the same workload through its public bulk API with workers = cores
    (fk/bench.py:156-268); GQF C4 on a bounded q=22 sample of the same
    spectrum.  Median of 3 where one run takes under 5 s."""
    fk = ref_package()
    if fk is None:
        return _cpu_baseline_workload_kernels(key)
    threads = os.cpu_count() or 1
    kind, log_slots, load = key
    w = fk.workloads
    if kind == "bulk_tcf":
        nb = (1 << log_slots) // 128
        n = int(load * (1 << log_slots))
        keys = w.counter_stream(1, TAG_UNIFORM, n)
        negs = w.counter_stream(2, TAG_FPR, n)

        def run():
            f = fk.BulkTcf(fk.BulkTcfParams(num_blocks=nb))
            t = time.perf_counter()
            f.insert_batch(keys, workers=threads)
            f.query_batch(keys, workers=threads)
            f.query_batch(negs, workers=threads)
            f.delete_batch(keys, workers=threads)
            return 4 * n, time.perf_counter() - t
        what = "bulk TCF 2^%d slots, insert_batch + 2x query_batch + delete_batch" % log_slots
    else:
        if kind == "gqf_kmer":
            qs = min(log_slots, 22)
            occ, uniq = kmer_zipf_host(qs, load, 1)
            what = ("GQF q=%d (bounded sample of the q=%d run) k-mer Zipf spectrum at load %.2f, naive "
                    "bulk_insert + count_many + bulk_delete" % (qs, log_slots, load))
        else:
            qs = log_slots
            occ = w.gen_keys(w.WorkloadSpec("ur_count", n=int(load * (1 << qs)) // 4, seed=1))
            uniq = np.unique(occ)
            what = "GQF q=%d ur_count (full size), naive bulk_insert + count_many + bulk_delete" % qs

        def run():
            f = fk.Gqf(fk.GqfParams(q=qs))
            t = time.perf_counter()
            f.bulk_insert(occ, workers=threads)
            f.count_many(uniq, workers=threads)
            f.bulk_delete(uniq, workers=threads)
            return len(occ) + 2 * len(uniq), time.perf_counter() - t
    ops, dt = run()
    rates = [ops / dt]
    if dt < 5.0:
        rates += [o / d for o, d in (run(), run())]
    return {"value": float(np.median(rates)), "unit": UNIT, "cores": threads, "kind": "reference",
            "cpu_model": cpu_model(), "repeats": len(rates),
            "sample": "unmodified reference package (baseline/_ref) public API, workers=%d: %s (%d ops, %.1f s "
                      "per run, median of %d)" % (threads, what, ops, dt, len(rates))}


def _cpu_baseline_workload_kernels(key):
    """Fallback without baseline/_ref: the reference's compiled kernels +
    restated facade glue (oracle/ref_model.py)."""
    from oracle import ref_model
    if not ref_model.available():
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": "reference not built"}
    threads = os.cpu_count() or 1
    kind, log_slots, load = key
    if kind == "bulk_tcf":
        nb = (1 << log_slots) // 128
        n = int(load * (1 << log_slots))
        keys = counter_stream(1, TAG_UNIFORM, n)
        negs = counter_stream(2, TAG_FPR, n)
        f = ref_model.RefBulkTcf(nb, backing_slots=int(round(nb * 128 * 0.01)))
        t = time.perf_counter()
        f.insert_batch(keys, threads)
        f.query_batch(keys, threads)
        f.query_batch(negs, threads)
        f.delete_batch(keys, threads)
        dt = time.perf_counter() - t
        ops = 4 * n
    else:
        from paper_2212_09005_b200.workloads import WorkloadSpec, gen_keys
        qs = min(log_slots, 22)
        if kind == "gqf_kmer":
            occ, uniq = kmer_zipf_host(qs, load, 1)
        else:
            occ = gen_keys(WorkloadSpec("ur_count", n=int(load * (1 << qs)) // 4, seed=1))
            uniq = np.unique(occ)
        f = ref_model.RefGqf(qs)
        t = time.perf_counter()
        f.bulk_insert(occ, workers=threads)
        f.count_many(uniq, threads)
        f.bulk_delete(uniq, workers=threads)
        dt = time.perf_counter() - t
        ops = len(occ) + 2 * len(uniq)
    return {"value": ops / dt, "unit": UNIT, "cores": threads, "kind": "reference", "cpu_model": cpu_model(),
            "sample": "reference _ckernels (oracle/_ref) + restated facade glue: %s (%d ops, %.1f s)"
                      % (kind, ops, dt)}


def secondary_lines(args, rank, world, local_rank):
    """configs[0] (bulk TCF 2^20), configs[1] (C2: GQF q=22 ur_count) and
    configs[3] (C4: GQF q=28 k-mer Zipf at load 0.9), each a full line of its
    own (value, per-op, roofline, e2e, clocks, cpu_baseline), carried under
    the headline line's "secondary" key so the driver's single run records
    them."""
    import copy
    import torch
    out = {}
    for wl in ("bulk_tcf", "gqf", "gqf_kmer"):
        a = copy.copy(args)
        a.workload = wl
        a.log_slots_set = False
        a.load = 0.9
        a.steps = 3
        a.exact_steps = False
        out[wl] = run_workload(a, rank, world, local_rank)
        torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------------
# CPU baseline / reference arm: the UNMODIFIED reference package
# ---------------------------------------------------------------------------
#
# oracle/install_ref.sh pip-installs /root/reference/pkg (its Cython
# _ckernels built with the reference's own setup.py) into baseline/_ref,
# which travels to the GPU box.  The reference arm and the cpu_baseline legs
# drive that package through its public API and its own bench drivers
# (fk/bench.py:101-268: key-range slices on OS threads over the point API,
# workers= on the bulk API).  When baseline/_ref is absent, the compiled
# kernels in oracle/_ref with restated facade glue (oracle/ref_model.py)
# stand in.

REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def ref_package():
    """The reference `filterkit` from baseline/_ref with its compiled backend,
    or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "filterkit")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import filterkit
        import filterkit.bench  # noqa: F401
    except ImportError:
        return None
    if "c" not in filterkit.available_backends():
        return None
    return filterkit


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _ref_c3_driver(fk, log_slots, threads):
    cfg = fk.bench.BenchConfig(filter_id="tcf", op="insert", log_slots=log_slots, threads=threads)
    return fk.bench._PointTcfDriver(cfg)


def _ref_c3_step(fk, log_slots, keys, negs, threads):
    """One C3 step through the reference's own point-TCF driver
    (fk/bench.py:101-148; Tcf.insert_many/query_many/delete_many, fk/tcf.py:
    142-192, on key-range slices across OS threads): seconds per op."""
    d = _ref_c3_driver(fk, log_slots, threads)
    d.build()
    t = [time.perf_counter()]
    d.insert(keys, threads, 1)
    t.append(time.perf_counter())
    d.query(keys, threads)
    t.append(time.perf_counter())
    d.query(negs, threads)
    t.append(time.perf_counter())
    d.delete(keys, threads)
    t.append(time.perf_counter())
    return {op: t[i + 1] - t[i] for i, op in enumerate(("insert", "query_pos", "query_neg", "delete"))}


def _ref_c3_one_thread(fk, log_slots, keys, negs, threads, parts=8):
    """The single-thread figure on a bounded sample of the same
    step: the keys are cut into 8*parts pieces and every 8th piece is inserted
    (later deleted) by ONE thread, timed, the others by `threads` threads,
    untimed, in key order -- so the timed inserts see every load level; 1/8
    of the positives and of the negatives are queried by one thread.
    -> (ops, seconds)."""
    d = _ref_c3_driver(fk, log_slots, threads)
    d.build()
    f = d.filt
    pk = np.array_split(keys, 8 * parts)
    pn = np.array_split(negs, 8 * parts)
    ops, sec = 0, 0.0

    def phase(pieces, fn_one, fn_many, timed_every=8):
        nonlocal ops, sec
        for i, piece in enumerate(pieces):
            if i % timed_every == 0:
                t = time.perf_counter()
                fn_one(piece)
                sec += time.perf_counter() - t
                ops += len(piece)
            elif fn_many is not None:
                fn_many(piece)

    phase(pk, f.insert_many, lambda x: d.insert(x, threads, 1))
    phase(pk, f.query_many, None)
    phase(pn, f.query_many, None)
    phase(pk, f.delete_many, lambda x: d.delete(x, threads))
    return ops, sec


def _c3_keys_host(log_slots, load, fk=None):
    n = int(load * (1 << log_slots))
    gen = fk.workloads.counter_stream if fk is not None else counter_stream
    return gen(1, TAG_UNIFORM, n), gen(2, TAG_FPR, n)


def cpu_baseline(log_slots=28, load=0.9, repeats=3):
    """The reference package on all host cores, C3 at full size (2^28 slots,
    the same keys as the GPU run): median of `repeats` steps (fk/bench.py:
    77, :488)."""
    threads = os.cpu_count() or 1
    fk = ref_package()
    if fk is None:
        return _cpu_baseline_kernels(log_slots, load, threads)
    keys, negs = _c3_keys_host(log_slots, load, fk)
    rates = []
    for _ in range(repeats):
        tt = _ref_c3_step(fk, log_slots, keys, negs, threads)
        rates.append(4 * len(keys) / sum(tt.values()))
    return {"value": float(np.median(rates)), "unit": UNIT, "cores": threads, "kind": "reference",
            "cpu_model": cpu_model(), "repeats": repeats, "steps_ops_per_s": rates,
            "sample": "unmodified reference package (baseline/_ref, pip-installed from /root/reference/pkg, "
                      "compiled backend) through its own point-TCF bench driver (fk/bench.py:101-148): C3 at full "
                      "size, 2^%d slots at %.2f load, insert+pos+neg+delete of the same keys as the GPU run, "
                      "%d threads slicing the keys (fk/bench.py:86-97), median of %d steps"
                      % (log_slots, load, threads, repeats)}


def _cpu_baseline_kernels(log_slots, load, threads):
    """Fallback without baseline/_ref: the reference's compiled kernels
    (oracle/_ref) under restated facade glue (oracle/ref_model.py)."""
    from oracle import ref_model
    if not ref_model.available():
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                "sample": "unavailable: neither baseline/_ref nor oracle/_ref is built"}
    nb = (1 << log_slots) // 16
    keys, negs = _c3_keys_host(log_slots, load)
    f = ref_model.RefTcf(nb, backing_slots=int(round(nb * 16 * 0.01)))
    t = time.perf_counter()
    f.insert_many(keys, threads)
    f.query_many(keys, threads)
    f.query_many(negs, threads)
    f.delete_many(keys, threads)
    dt = time.perf_counter() - t
    return {"value": 4 * len(keys) / dt, "unit": UNIT, "cores": threads, "kind": "reference",
            "cpu_model": cpu_model(),
            "sample": "reference _ckernels (oracle/_ref) + restated facade glue, point TCF 2^%d slots at %.2f "
                      "load, insert+pos+neg+delete, %d threads" % (log_slots, load, threads)}


def run_reference(args, rank, world):
    """--impl reference: the unmodified reference package on the host cores,
    on our arm's config (C3: 2^28 slots, 0.9 load, the same keys), every
    step at full size."""
    if rank != 0:
        return None
    fk = ref_package()
    threads = os.cpu_count() or 1
    if fk is None:
        return {"impl": "reference", "unavailable": "baseline/_ref (reference package install) not present"}
    log_slots = args.log_slots
    keys, negs = _c3_keys_host(log_slots, args.load, fk)
    for _ in range(args.warmup):
        _ref_c3_step(fk, log_slots, keys, negs, threads)
    steps = [_ref_c3_step(fk, log_slots, keys, negs, threads) for _ in range(args.steps)]
    tot_t = sum(sum(st.values()) for st in steps)
    ops_step = 4 * len(keys)
    value = ops_step * args.steps / tot_t
    rates = [ops_step / sum(st.values()) for st in steps]
    per_op = {op: {"ops_per_s": len(keys) / float(np.mean([st[op] for st in steps])),
                   "ms": 1e3 * float(np.mean([st[op] for st in steps]))} for op in steps[0]}
    one_ops, one_s = _ref_c3_one_thread(fk, log_slots, keys, negs, threads)
    sample = ("unmodified reference package (baseline/_ref, pip-installed from /root/reference/pkg, compiled "
              "backend) through its own point-TCF bench driver (fk/bench.py:101-148): 2^%d slots at %.2f load, "
              "insert+pos+neg+delete of the GPU run's keys each step, %d threads slicing the keys "
              "(fk/bench.py:86-97)" % (log_slots, args.load, threads))
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u16",
            "data": "synthetic",
            "config": {"workload": "C3: point TCF, 2^%d slots/GPU (nb=2^%d x B=16, 16-bit tags, 1%% backing), "
                                   "uniform 64-bit keys, insert+pos query+neg query+delete at %.2f load"
                                   % (log_slots, log_slots - 4, args.load),
                       "keys_per_op_per_gpu": len(keys), "same_config_as_gpu_arm": True},
            "per_op": per_op, "median_step_ops_per_s": float(np.median(rates)),
            "one_thread": {"ops_per_s": one_ops / one_s, "ops": one_ops, "seconds": one_s,
                           "sample": "same table and keys; every 8th of 64 key pieces inserted/deleted by one "
                                     "thread (timed) between multi-thread pieces (untimed), 1/8 of the "
                                     "positive and negative queries by one thread"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                             "cpu_model": cpu_model(), "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["tcf", "bulk_tcf", "gqf", "gqf_kmer"], default="tcf")
    ap.add_argument("--log-slots", type=int, default=None)
    ap.add_argument("--load", type=float, default=0.9)
    ap.add_argument("--group-width", type=int, default=1)
    ap.add_argument("--mode", choices=["ordered", "concurrent"], default="ordered")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-concurrent", action="store_true")
    ap.add_argument("--no-launch-count", action="store_true")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the configs[0]/C2/C4 lines carried under 'secondary'")
    ap.add_argument("--exact-steps", action="store_true",
                    help="secondary workloads: time exactly --steps steps (default: at least ~1.5 s)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    args.log_slots_set = args.log_slots is not None
    if args.log_slots is None:
        args.log_slots = 28

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        res = run_reference(args, rank, world)
    else:
        if world > 1:
            import torch
            import torch.distributed as dist
            # FK_BENCH_BACKEND=gloo: test hook for several ranks on one GPU
            # (NCCL refuses that); the driver's runs use NCCL
            backend = os.environ.get("FK_BENCH_BACKEND", "nccl")
            dev_idx = local_rank % torch.cuda.device_count()
            torch.cuda.set_device(dev_idx)
            if backend == "nccl":
                # communicator init on stderr (comm / rank / nranks / transports) so the
                # scaling run's NCCL setup can be checked from the log
                os.environ.setdefault("NCCL_DEBUG", "INFO")
                os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
                dist.init_process_group("nccl", device_id=torch.device("cuda", dev_idx))
            else:
                dist.init_process_group(backend)
        res = (run_ours if args.workload == "tcf" else run_workload)(args, rank, world, local_rank)
        if args.workload == "tcf" and not args.no_secondary and not args.log_slots_set:
            sec = secondary_lines(args, rank, world, local_rank)
            if res is not None:
                res["secondary"] = sec
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
    if res is not None:
        print(json.dumps(res))


if __name__ == "__main__":
    main()
