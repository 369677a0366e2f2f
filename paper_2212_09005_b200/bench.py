"""``filterkit-bench`` for the B200 filters: the reference's benchmark and
validation CLI (/root/reference/pkg/src/filterkit/bench.py) with the same
flags, the same CSV schema and the same exit codes, driving the GPU facades.

    python -m paper_2212_09005_b200.bench --filter gqf --op insert \\
        --log-slots 22 --dist zipf --mode mapreduce --csv runs.csv

Contract kept from the reference (bench.py:1-12, :276-425):
  * one MetricsRecord / CSV row per repeat; header written only for a new
    file (bench.py:38-56, :399-411); `read_csv` parses rows back;
  * ops: insert, query, count (GQF), fpr (1 M fresh keys), delete (every
    other distinct key), fill-to-failure (4096-key chunks until the first
    failed placement / CapacityError);
  * every repeat ends with the filter's full `validate()`; a violation exits
    with code 2, a parameter error with code 1 (bench.py:478-485, :430-432);
  * key streams are the reference generators (workloads.gen_keys) with the
    same sizing (bench.py:239-262).

Deliberate differences (GPU execution model):
  * keys are uploaded to the device once before the timed region and the
    region ends with a device synchronisation; `wall_seconds` is host wall
    time around the device calls;
  * `--threads N` is recorded but spawns no host threads: the facades
    serialise batches per filter, and one batch already runs on every SM.
    The point TCF runs in its bit-exact ordered mode (one linearisation of
    the reference's threaded inserts); its free-threaded CAS mode
    (`Tcf(mode="concurrent")`) is a library option, not a CLI one, because
    with a whole batch in flight at once it loses placement quality on small
    tables (blocks fill past the shortcut before the less-full choice can
    spread them).
"""

from __future__ import annotations

import argparse
import csv
import statistics
import sys
import time
from dataclasses import dataclass, fields

import numpy as np

from .errors import CapacityError, FilterFullError, ValidationError
from .workloads import WorkloadSpec, gen_keys, measure_fpr

FPR_QUERIES = 1_000_000
FILL_CHUNK = 4096


class ParameterError(ValueError):
    """Bad flag combination or workload input (exit code 1)."""


@dataclass
class MetricsRecord:
    filter: str
    api: str
    op: str
    log_slots: int
    load_factor: float
    threads: int
    dist: str
    seed: int
    wall_seconds: float
    ops_per_sec: float
    fpr: float = None
    bits_per_item: float = None


CSV_FIELDS = [f.name for f in fields(MetricsRecord)]


@dataclass
class BenchConfig:
    filter_id: str
    op: str
    api: str = None
    log_slots: int = 16
    load: float = 0.9
    threads: int = 1
    dist: str = "uniform"
    zipf_s: float = 1.5
    kmer_file: str = None
    k: int = 28
    seed: int = 0
    batches: int = 1
    mode: str = "naive"
    no_backing: bool = False
    group_width: int = 1
    csv: str = None
    repeats: int = 3


def _sync():
    import torch
    torch.cuda.synchronize()


def _device(keys):
    import torch
    return torch.from_numpy(np.ascontiguousarray(keys, dtype=np.uint64).view(np.int64)).cuda()


# -- one adapter per filter: build / fill / probe / delete / accounting --------

class _Adapter:
    filter_id = api = None
    capacity = 0

    def live_items(self):
        c = self.filt.counters
        return c["inserts_ok"] - c["deletes_ok"]

    def load_factor(self):
        return self.filt.load_factor()


class _PointTcf(_Adapter):
    filter_id, api = "tcf", "point"
    B = 16

    def __init__(self, cfg):
        from .tcf import TcfParams
        if (1 << cfg.log_slots) % self.B:
            raise ParameterError("--log-slots must cover whole 16-slot blocks")
        self.params = TcfParams(num_blocks=(1 << cfg.log_slots) // self.B,
                                backing_fraction=0.0 if cfg.no_backing else 0.01,
                                group_width=cfg.group_width, seed=cfg.seed)
        self.capacity = self.params.main_slots

    def build(self):
        from .tcf import Tcf
        self.filt = Tcf(self.params, mode="ordered")

    def insert(self, keys, batches):
        full = 0
        for part in _split(keys, batches):
            full += int((self.filt.insert_many(part) == 3).sum())
        if full:
            raise FilterFullError("%d inserts found no slot" % full)

    def insert_until_full(self, keys):
        done = 0
        for lo in range(0, len(keys), FILL_CHUNK):
            codes = self.filt.insert_many(keys[lo:lo + FILL_CHUNK]).cpu().numpy()
            bad = np.flatnonzero(codes == 3)
            if len(bad):
                return done + int(bad[0])
            done += len(codes)
        return done

    def query(self, keys):
        self.filt.query_many(keys)

    def delete(self, keys):
        self.filt.delete_many(keys)


class _BulkTcf(_Adapter):
    filter_id, api = "tcf-bulk", "bulk"
    B = 128

    def __init__(self, cfg):
        from .tcf_bulk import BulkTcfParams
        if (1 << cfg.log_slots) % self.B:
            raise ParameterError("--log-slots must cover whole 128-slot blocks")
        self.params = BulkTcfParams(num_blocks=(1 << cfg.log_slots) // self.B,
                                    backing_fraction=0.0 if cfg.no_backing else 0.01, seed=cfg.seed)
        self.capacity = self.params.main_slots

    def build(self):
        from .tcf_bulk import BulkTcf
        self.filt = BulkTcf(self.params)

    def insert(self, keys, batches):
        for part in _split(keys, batches):
            failed = self.filt.insert_batch(part)
            if len(failed):
                raise FilterFullError("%d inserts found no slot" % len(failed))

    def insert_until_full(self, keys):
        done = 0
        for lo in range(0, len(keys), FILL_CHUNK):
            part = keys[lo:lo + FILL_CHUNK]
            nfail = len(self.filt.insert_batch(part))
            done += len(part) - nfail
            if nfail:
                return done
        return done

    def query(self, keys):
        self.filt.query_batch(keys)

    def delete(self, keys):
        self.filt.delete_batch(keys)


class _Gqf(_Adapter):
    filter_id = "gqf"

    def __init__(self, cfg, api):
        from .gqf import GqfParams
        self.api, self.mode = api, cfg.mode
        self.params = GqfParams(q=cfg.log_slots, r=8, seed=cfg.seed)
        self.capacity = self.params.logical_slots

    def build(self):
        from .gqf import Gqf
        self.filt = Gqf(self.params)

    def insert(self, keys, batches):
        if self.mode == "mapreduce":
            # aggregation is part of the measured algorithm (bench.py:219-222);
            # on the device: sort + run-length reduce of the key stream
            import torch
            uniq, counts = torch.unique(keys, sorted=True, return_counts=True)
            self.filt.bulk_insert(uniq, counts)
        elif self.api == "bulk":
            for part in _split(keys, batches):
                self.filt.bulk_insert(part)
        else:
            self.filt.insert_many(keys)

    def insert_until_full(self, keys):
        done = 0
        for lo in range(0, len(keys), FILL_CHUNK):
            part = keys[lo:lo + FILL_CHUNK]
            try:
                (self.filt.bulk_insert if self.api == "bulk" else self.filt.insert_many)(part)
            except CapacityError:
                return self.filt.distinct_items
            done += len(part)
        return done

    def query(self, keys):
        self.filt.count_many(keys)

    count = query

    def delete(self, keys):
        import torch
        ones = torch.ones(keys.numel(), dtype=torch.int64, device=keys.device)
        (self.filt.bulk_delete if self.api == "bulk" else self.filt.delete_many)(keys, ones)

    def live_items(self):
        return self.filt.distinct_items


def _split(keys, parts):
    n = keys.numel()
    cuts = np.linspace(0, n, parts + 1).astype(np.int64)
    return [keys[int(cuts[i]):int(cuts[i + 1])] for i in range(parts)]


def _adapter(cfg):
    if cfg.filter_id == "tcf":
        if cfg.api not in (None, "point"):
            raise ParameterError("--filter tcf is the point API; use --filter tcf-bulk for the bulk variant")
        return _PointTcf(cfg)
    if cfg.filter_id == "tcf-bulk":
        if cfg.api not in (None, "bulk"):
            raise ParameterError("--filter tcf-bulk only has a bulk API")
        return _BulkTcf(cfg)
    if cfg.filter_id == "gqf":
        return _Gqf(cfg, cfg.api or "point")
    raise ParameterError("unknown filter %r" % (cfg.filter_id,))


def _keys_for(cfg, capacity):
    """The reference's key stream for cfg.load of the capacity (bench.py:239-262)."""
    target = max(1, int(cfg.load * capacity))
    specs = {
        "uniform": lambda: WorkloadSpec("uniform", n=target, seed=cfg.seed),
        "ur_count": lambda: WorkloadSpec("ur_count", n=max(1, target // 4), seed=cfg.seed),
        "zipf": lambda: WorkloadSpec("zipf", n=target, seed=cfg.seed, zipf_s=cfg.zipf_s),
        "kmer": lambda: WorkloadSpec("kmer", kmer_file=cfg.kmer_file, kmer_k=cfg.k),
    }
    if cfg.dist not in specs:
        raise ParameterError("unknown distribution %r" % (cfg.dist,))
    try:
        keys = gen_keys(specs[cfg.dist]())
    except (OSError, ValueError) as err:
        raise ParameterError(str(err))
    return keys[:target] if cfg.dist == "kmer" else keys


def _timed(fn):
    _sync()
    t0 = time.perf_counter()
    fn()
    _sync()
    return time.perf_counter() - t0


def _one_run(cfg, ad, keys_host, keys):
    ad.build()
    op, fpr, achieved = cfg.op, None, None
    if op == "insert":
        wall = _timed(lambda: ad.insert(keys, cfg.batches))
        ops = keys.numel()
    elif op == "fill-to-failure":
        box = {}
        wall = _timed(lambda: box.setdefault("n", ad.insert_until_full(keys)))
        ops = box["n"]
        achieved = ops / ad.capacity
    elif op in ("query", "count", "fpr", "delete"):
        ad.insert(keys, cfg.batches)
        if op == "query":
            wall, ops = _timed(lambda: ad.query(keys)), keys.numel()
        elif op == "count":
            if not hasattr(ad, "count"):
                raise ParameterError("--op count requires --filter gqf")
            wall, ops = _timed(lambda: ad.count(keys)), keys.numel()
        elif op == "fpr":
            box = {}
            wall = _timed(lambda: box.setdefault("f", measure_fpr(ad.filt, FPR_QUERIES, cfg.seed + 1)))
            fpr, ops = box["f"], FPR_QUERIES
        else:
            half = _device(np.unique(keys_host)[::2])
            wall, ops = _timed(lambda: ad.delete(half)), half.numel()
    else:
        raise ParameterError("unknown op %r" % (op,))
    ad.filt.validate()
    items = ad.live_items()
    if achieved is None:
        achieved = ad.load_factor()
    return MetricsRecord(filter=ad.filter_id, api=ad.api, op=op, log_slots=cfg.log_slots,
                         load_factor=round(achieved, 6), threads=cfg.threads, dist=cfg.dist, seed=cfg.seed,
                         wall_seconds=round(wall, 6),
                         ops_per_sec=round(ops / wall, 3) if wall > 0 else float("inf"), fpr=fpr,
                         bits_per_item=round(ad.filt.size_bits() / items, 4) if items else None)


def run(cfg):
    """Execute a config; one MetricsRecord per repeat (bench.py:380-396)."""
    if not 0.0 < cfg.load <= 1.0:
        raise ParameterError("--load must be in (0, 1]")
    if cfg.threads < 1 or cfg.batches < 1 or cfg.repeats < 1:
        raise ParameterError("--threads, --batches, --repeats must be positive")
    if cfg.dist == "kmer" and not cfg.kmer_file:
        raise ParameterError("--dist kmer requires --kmer-file")
    if cfg.mode not in ("naive", "mapreduce"):
        raise ParameterError("--mode must be naive or mapreduce")
    if cfg.mode == "mapreduce" and cfg.filter_id != "gqf":
        raise ParameterError("--mode mapreduce applies to --filter gqf only")
    if cfg.no_backing and cfg.filter_id == "gqf":
        raise ParameterError("--no-backing applies to the two-choice filters")
    ad = _adapter(cfg)
    if cfg.op == "fill-to-failure":
        keys_host = gen_keys(WorkloadSpec("uniform", n=int(ad.capacity * 1.05) + FILL_CHUNK, seed=cfg.seed))
    else:
        keys_host = _keys_for(cfg, ad.capacity)
    keys = _device(keys_host)
    return [_one_run(cfg, ad, keys_host, keys) for _ in range(cfg.repeats)]


def write_csv(path, records):
    """Append rows; header only when the file is new or empty."""
    try:
        with open(path, "r", encoding="utf-8") as fh:
            fresh = not fh.readline()
    except FileNotFoundError:
        fresh = True
    with open(path, "a", newline="", encoding="utf-8") as fh:
        w = csv.DictWriter(fh, fieldnames=CSV_FIELDS)
        if fresh:
            w.writeheader()
        for rec in records:
            w.writerow({k: ("" if v is None else v) for k, v in vars(rec).items()})


_PARSE = {"log_slots": int, "threads": int, "seed": int, "load_factor": float, "wall_seconds": float,
          "ops_per_sec": float, "fpr": float, "bits_per_item": float}


def read_csv(path):
    with open(path, newline="", encoding="utf-8") as fh:
        return [MetricsRecord(**{k: (_PARSE[k](v) if v != "" else None) if k in _PARSE else v
                                 for k, v in row.items()}) for row in csv.DictReader(fh)]


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # usage errors are parameter errors: exit 1
        self.exit(1, "%s: error: %s\n" % (self.prog, message))


def build_parser():
    p = _Parser(prog="filterkit-bench", description="B200 filter benchmark and validation CLI")
    p.add_argument("--filter", required=True, choices=["tcf", "tcf-bulk", "gqf"])
    p.add_argument("--api", choices=["point", "bulk"])
    p.add_argument("--op", required=True, choices=["insert", "query", "fpr", "delete", "count", "fill-to-failure"])
    p.add_argument("--log-slots", type=int, default=16)
    p.add_argument("--load", type=float, default=0.9)
    p.add_argument("--threads", type=int, default=1)
    p.add_argument("--dist", default="uniform", choices=["uniform", "ur-count", "zipf", "kmer"])
    p.add_argument("--zipf-s", type=float, default=1.5)
    p.add_argument("--kmer-file")
    p.add_argument("--k", type=int, default=28)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--batches", type=int, default=1)
    p.add_argument("--mode", default="naive", choices=["naive", "mapreduce"])
    p.add_argument("--no-backing", action="store_true")
    p.add_argument("--group-width", type=int, default=1)
    p.add_argument("--csv")
    p.add_argument("--repeats", type=int, default=3)
    return p


def main(argv=None):
    a = build_parser().parse_args(argv)
    cfg = BenchConfig(filter_id=a.filter, api=a.api, op=a.op, log_slots=a.log_slots, load=a.load,
                      threads=a.threads, dist=a.dist.replace("-", "_"), zipf_s=a.zipf_s, kmer_file=a.kmer_file,
                      k=a.k, seed=a.seed, batches=a.batches, mode=a.mode, no_backing=a.no_backing,
                      group_width=a.group_width, csv=a.csv, repeats=a.repeats)
    try:
        records = run(cfg)
    except ParameterError as err:
        print("parameter error: %s" % err, file=sys.stderr)
        return 1
    except ValidationError as err:
        print("INVARIANT VIOLATION: %s" % err, file=sys.stderr)
        return 2
    if cfg.csv:
        write_csv(cfg.csv, records)
    r0 = records[0]
    print("%s/%s %s: median %.0f ops/s over %d runs, load %.3f%s%s"
          % (r0.filter, r0.api, r0.op, statistics.median(r.ops_per_sec for r in records), len(records),
             r0.load_factor, ", fpr %.6f" % r0.fpr if r0.fpr is not None else "",
             ", %.2f bits/item" % r0.bits_per_item if r0.bits_per_item is not None else ""))
    return 0


def console_main():
    sys.exit(main())


if __name__ == "__main__":
    sys.exit(main())
