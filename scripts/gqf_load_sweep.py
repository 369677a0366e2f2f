#!/usr/bin/env python
"""C4 load-factor sweep (BASELINE.json configs[3]): GQF 2^q slots (q=28
default, r=8), k-mer-like Zipfian counting keys, alpha in 0.1..0.9.

The spectrum is bench.kmer_zipf_workload's (distinct uniform keys, bounded
Zipf(1.5) multiplicities on [1, 100], stream shuffled), generated once for
the largest alpha; a smaller alpha takes the prefix of distinct keys that
fills alpha * 2^q slots.  Per point: fresh filter -> naive bulk_insert of
every occurrence -> count_many(distinct) -> bulk_delete(distinct, all copies),
each timed with CUDA events (mean of --steps after --warmup), plus
size-independent checks: every count >= its multiplicity (a GQF never
undercounts), the fraction exactly equal, total items == occurrences, and an
empty table after the delete.  One JSON line per alpha.
"""

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--q", type=int, default=28)
    ap.add_argument("--alphas", type=float, nargs="+", default=[0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9])
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=1)
    a = ap.parse_args()
    import torch
    from paper_2212_09005_b200 import Gqf
    dev = torch.device("cuda", 0)
    amax = max(a.alphas)
    w = bench.kmer_zipf_workload(torch, a.q, amax, 1, dev)
    del w["occ"]
    uniq_all, cnt_all = w["uniq"], w["counts"]
    filt = Gqf(q=a.q)
    st = torch.cuda.current_stream()
    for alpha in a.alphas:
        d = int(round(w["n_distinct"] * alpha / amax))
        uniq, cnt = uniq_all[:d], cnt_all[:d]
        occ = torch.repeat_interleave(uniq, cnt)
        g = torch.Generator(device=dev)
        g.manual_seed(int(alpha * 1000))
        occ = occ[torch.randperm(occ.numel(), device=dev, generator=g)]
        names = ("bulk_insert", "count", "bulk_delete")
        ms = {k: [] for k in names}
        for s in range(a.warmup + a.steps):
            filt._reset()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
            ev[0].record(st)
            filt.bulk_insert(occ)
            ev[1].record(st)
            counts = filt.count_many(uniq)
            ev[2].record(st)
            torch.cuda.synchronize()
            lf = filt.load_factor()
            items = filt.total_items
            ev[3].record(st)
            found = filt.bulk_delete(uniq)
            ev[4].record(st)
            torch.cuda.synchronize()
            if s >= a.warmup:
                for k, (i, j) in zip(names, ((0, 1), (1, 2), (3, 4))):
                    ms[k].append(ev[i].elapsed_time(ev[j]))
        n_items = {"bulk_insert": occ.numel(), "count": d, "bulk_delete": d}
        per = {k: {"ms": float(np.mean(v)), "g_ops_per_s": n_items[k] / (float(np.mean(v)) / 1e3) / 1e9}
               for k, v in ms.items()}
        under = int((counts < cnt).sum())
        exact = float((counts == cnt).float().mean())
        print(json.dumps({
            "q": a.q, "r": 8, "alpha_target": alpha, "load_factor": lf, "distinct": d,
            "occurrences": int(occ.numel()), "per_op": per,
            "occurrences_per_s_insert": per["bulk_insert"]["g_ops_per_s"] * 1e9,
            "checks": {"undercounts": under, "exact_count_frac": exact, "total_items": int(items),
                       "items_match": int(items) == int(occ.numel()), "found_frac": float(found.float().mean()),
                       "empty_after_delete": filt.occupied_slots == 0}}), flush=True)
        del occ
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
