#!/usr/bin/env python
"""Ordered point-TCF tuning probe: per table size, time insert/delete at 0.9
load under the FK_ORD_* knobs given on the command line and read the
kernel's round statistics (ctl[5] main rounds, ctl[6] backing rounds,
ctl[7] keys carried) back from the workspace.

  python scripts/ord_tune.py --log-slots 20 22 28 --cfg "W=4096,RS=0,CTAS=0" ...
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def rup(x):
    return (x + 255) & ~255


def ctl_offset(nb, bs, n, rs):
    a = rup(((nb >> rs) + 1) * 4)
    a += rup(max(bs, 1) * 4)
    a += rup(n * 4)
    a += rup(n)
    return a


def default_rs(nb):
    rs = 0
    while (nb >> rs) > (1 << 22):
        rs += 1
    return rs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log-slots", type=int, nargs="+", default=[20, 22, 24, 28])
    ap.add_argument("--cfg", nargs="+", default=["default"])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--group-width", type=int, default=1)
    a = ap.parse_args()
    import torch
    from paper_2212_09005_b200 import Tcf, _lib
    dev = torch.device("cuda", 0)
    lib = _lib.load()
    for ls in a.log_slots:
        nb = (1 << ls) // 16
        n = int(0.9 * (1 << ls))
        keys = bench.device_keys(torch, 1, bench.TAG_UNIFORM, n, dev)
        filt = Tcf(num_blocks=nb, group_width=a.group_width, mode="ordered")
        for cfg in a.cfg:
            env = {}
            if cfg != "default":
                for kv in cfg.split(","):
                    k, v = kv.split("=")
                    env[{"W": "FK_ORD_WINDOW", "RS": "FK_ORD_RES_SHIFT", "CTAS": "FK_ORD_CTAS_PER_SM",
                         "H": "FK_ORD_HINTS", "OB": "FK_ORD_ONEBAR", "KB3": "FK_ORD_KB3",
                         "HO": "FK_ORD_HELD_ONLY"}[k]] = v
            for k in ("FK_ORD_WINDOW", "FK_ORD_RES_SHIFT", "FK_ORD_CTAS_PER_SM", "FK_ORD_HINTS", "FK_ORD_ONEBAR", "FK_ORD_KB3",
                      "FK_ORD_HELD_ONLY"):
                os.environ.pop(k, None)
            os.environ.update(env)
            rs = int(env.get("FK_ORD_RES_SHIFT", default_rs(nb)))
            nbytes = lib.fk_tcf_workspace_bytes(ctypes.byref(filt._geom), n, _lib.FK_ORDERED)
            ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
            off = ctl_offset(nb, filt.params.backing_slots, n, rs)
            codes = torch.empty(n, dtype=torch.uint8, device=dev)
            st = torch.cuda.current_stream()
            res = {}
            for op in ("insert", "delete"):
                res[op] = {"ms": []}
            for r in range(a.reps + 1):
                filt._reset()
                for op in ("insert", "delete"):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    fn = lib.fk_tcf_insert if op == "insert" else lib.fk_tcf_delete
                    if op == "insert":
                        rc = fn(ctypes.byref(filt._geom), filt._t.ptr("blocks"), filt._t.ptr("backing"),
                                _lib.dptr(keys), 0, None, n, _lib.dptr(codes), _lib.dptr(filt._counters_dev),
                                _lib.FK_ORDERED, _lib.dptr(ws), nbytes, _lib.stream_ptr(torch))
                    else:
                        rc = fn(ctypes.byref(filt._geom), filt._t.ptr("blocks"), filt._t.ptr("backing"),
                                _lib.dptr(keys), 0, n, _lib.dptr(codes), _lib.dptr(filt._counters_dev),
                                _lib.FK_ORDERED, _lib.dptr(ws), nbytes, _lib.stream_ptr(torch))
                    _lib.check(rc, op)
                    e1.record(st)
                    torch.cuda.synchronize()
                    if r:
                        res[op]["ms"].append(e0.elapsed_time(e1))
                    ctl = ws[off:off + 64].cpu().numpy().view(np.uint32)
                    res[op].update(rounds=int(ctl[5]), backing_rounds=int(ctl[6]), carried=int(ctl[7]),
                                   deferred=int(ctl[2]))
            for op in res:
                ms = float(np.mean(res[op].pop("ms")))
                res[op]["ms"] = ms
                res[op]["g_ops_per_s"] = n / ms / 1e6
                res[op]["us_per_round"] = 1e3 * ms / max(1, res[op]["rounds"] + res[op]["backing_rounds"])
            print(json.dumps({"log_slots": ls, "G": a.group_width, "cfg": cfg, "rs": rs, **res}), flush=True)
        del keys, filt
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
