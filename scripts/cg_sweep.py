#!/usr/bin/env python
"""C3 cooperative-group sweep (BASELINE.json configs[2]) and L2- vs
HBM-resident table sizes for the point TCF.

For every (log2 slots, B, G, mode): reset -> insert 0.9*2^s keys -> positive
query -> negative query -> delete, each op timed with CUDA events on the
launching stream (mean of `--steps` after `--warmup`).  G sweeps 1..16 at the
reference's default B=16 (TcfParams rejects G > B, fk/tcf.py:70-71) and G=32
at B=32 (the only way the reference API admits a 32-wide group).  Prints one
JSON line per point; keys are the bench's device counter_stream.

  python scripts/cg_sweep.py --log-slots 28 22 --modes ordered concurrent
"""

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def run_point(torch, log_slots, B, G, mode, steps, warmup, keys, negs):
    from paper_2212_09005_b200 import Tcf
    nb = (1 << log_slots) // B
    n = keys.numel()
    filt = Tcf(num_blocks=nb, block_slots=B, group_width=G, mode=mode)
    st = torch.cuda.current_stream()
    names = ("insert", "query_pos", "query_neg", "delete")
    ms = {k: [] for k in names}
    for s in range(warmup + steps):
        filt._reset()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record(st)
        codes = filt.insert_many(keys)
        ev[1].record(st)
        fpos = filt.query_many(keys)
        ev[2].record(st)
        fneg = filt.query_many(negs)
        ev[3].record(st)
        rem = filt.delete_many(keys)
        ev[4].record(st)
        torch.cuda.synchronize()
        if s >= warmup:
            for i, k in enumerate(names):
                ms[k].append(ev[i].elapsed_time(ev[i + 1]))
    per = {k: {"ms": float(np.mean(v)), "g_ops_per_s": n / (float(np.mean(v)) / 1e3) / 1e9} for k, v in ms.items()}
    step_ms = sum(p["ms"] for p in per.values())
    return {"log_slots": log_slots, "table_mib": (1 << log_slots) * 2 >> 20, "B": B, "G": G, "mode": mode,
            "keys": n, "per_op": per, "step_g_ops_per_s": 4 * n / (step_ms / 1e3) / 1e9,
            "checks": {"full": int((codes == 3).sum()), "false_neg": int((~fpos).sum()),
                       "fpr": float(fneg.float().mean()), "removed": int(rem.sum())}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log-slots", type=int, nargs="+", default=[28, 22])
    ap.add_argument("--modes", nargs="+", default=["ordered", "concurrent"])
    ap.add_argument("--groups", type=int, nargs="+", default=[1, 2, 4, 8, 16, 32])
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--load", type=float, default=0.9)
    a = ap.parse_args()
    import torch
    dev = torch.device("cuda", 0)
    for ls in a.log_slots:
        n = int(a.load * (1 << ls))
        keys = bench.device_keys(torch, 1, bench.TAG_UNIFORM, n, dev)
        negs = bench.device_keys(torch, 2, bench.TAG_FPR, n, dev)
        for mode in a.modes:
            for G in a.groups:
                B = 16 if G <= 16 else 32
                r = run_point(torch, ls, B, G, mode, a.steps, a.warmup, keys, negs)
                print(json.dumps(r), flush=True)
        del keys, negs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
