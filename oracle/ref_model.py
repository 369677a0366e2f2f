"""oracle.ref_model -- the reference's OWN compiled kernels as a CPU baseline.

TEST / BASELINE INFRASTRUCTURE ONLY (bench.py's cpu_baseline and
``--impl reference`` legs, tests/test_oracle_vs_ref.py).  The product never
imports this.

``oracle/_ref/_ckernels*.so`` is /root/reference/pkg/src/filterkit/_ckernels.pyx
compiled by oracle/build_ref.sh.  The host glue below restates the reference
facades' few lines around each kernel call (fk/tcf.py:142-192) and its bench
harness's thread slicing (fk/bench.py:86-97): the compiled loops release the
GIL, so T Python threads run T cores.
"""

from __future__ import annotations

import glob
import os
import sys
import threading

import numpy as np

from .model import fingerprint_many

_REF_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref")


def available():
    return bool(glob.glob(os.path.join(_REF_DIR, "_ckernels*.so")))


_ck = None


def kernels():
    global _ck
    if _ck is None:
        if not available():
            raise RuntimeError("oracle/_ref not built (oracle/build_ref.sh)")
        if _REF_DIR not in sys.path:
            sys.path.insert(0, _REF_DIR)
        import _ckernels  # noqa: E402
        _ck = _ckernels
    return _ck


def run_threads(fn, arrays, threads):
    """fk/bench.py:86-97: slice the key array(s) across OS threads."""
    n = len(arrays[0])
    if threads <= 1:
        fn(*arrays)
        return
    cuts = np.linspace(0, n, threads + 1).astype(np.int64)
    ts = [threading.Thread(target=fn, args=tuple(a[cuts[i]:cuts[i + 1]] for a in arrays))
          for i in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()


class RefTcf:
    """Point TCF on the reference's compiled kernels (real CAS, GIL released)."""

    def __init__(self, num_blocks, block_slots=16, tag_bits=16, slot_dtype=np.uint16, backing_slots=0,
                 cut_slots=12, probe_limit=20, seed=0, group_width=1):
        self.ck = kernels()
        self.B, self.f, self.cut, self.pl, self.g = block_slots, tag_bits, cut_slots, probe_limit, group_width
        self.seed = seed
        self.blocks = np.zeros(num_blocks * block_slots, dtype=slot_dtype)
        self.backing = np.zeros(backing_slots, dtype=slot_dtype)

    def insert_many(self, keys, threads=1):
        codes = np.empty(len(keys), dtype=np.uint8)
        zeros = np.zeros(len(keys), dtype=np.uint64)

        def work(k, c, v):
            fps = fingerprint_many(k, self.seed)
            self.ck.tcf_insert_batch(self.blocks, self.backing, self.B, self.f, self.cut, self.pl, self.g,
                                     None, fps, v, c)
        run_threads(work, (keys, codes, zeros), threads)
        return codes

    def query_many(self, keys, threads=1):
        found = np.empty(len(keys), dtype=np.uint8)
        vals = np.empty(len(keys), dtype=np.uint64)

        def work(k, fo, va):
            fps = fingerprint_many(k, self.seed)
            self.ck.tcf_query_batch(self.blocks, self.backing, self.B, self.f, self.pl, self.g, None,
                                    fps, fo, va)
        run_threads(work, (keys, found, vals), threads)
        return found

    def delete_many(self, keys, threads=1):
        removed = np.empty(len(keys), dtype=np.uint8)

        def work(k, r):
            fps = fingerprint_many(k, self.seed)
            self.ck.tcf_delete_batch(self.blocks, self.backing, self.B, self.f, self.pl, self.g, None, fps, r)
        run_threads(work, (keys, removed), threads)
        return removed


def _split_ranges(nb, workers):
    step = (nb + workers - 1) // workers
    return [(lo, min(lo + step, nb)) for lo in range(0, nb, step)]


def _run_ranged(fn, nb, workers):
    """fk/tcf_bulk.py:164-175: disjoint block ranges on OS threads."""
    if workers <= 1 or nb == 1:
        fn(0, nb)
        return
    ts = [threading.Thread(target=fn, args=r) for r in _split_ranges(nb, workers)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()


class RefBulkTcf:
    """Bulk TCF: the reference facade's numpy glue (fk/tcf_bulk.py:133-325,
    restated) around the reference's compiled kernels, `workers` threads."""

    def __init__(self, num_blocks, block_slots=128, tag_bits=16, backing_slots=0, cut_slots=96, probe_limit=20,
                 seed=0):
        from .model import potc_pair_many, remap_tags
        self._pp, self._rt = potc_pair_many, remap_tags
        self.ck = kernels()
        self.nb, self.B, self.f, self.cut, self.pl, self.seed = num_blocks, block_slots, tag_bits, cut_slots, \
            probe_limit, seed
        self.blocks = np.zeros(num_blocks * block_slots, dtype=np.uint16)
        self.fill = np.zeros(num_blocks, dtype=np.uint32)
        self.backing = np.zeros(backing_slots, dtype=np.uint16)

    def _sorted(self, blk, words):
        comb = (blk.astype(np.uint64) << np.uint64(32)) | words.astype(np.uint64)
        order = np.argsort(comb, kind="stable")
        comb = comb[order]
        bounds = np.searchsorted(comb, np.arange(self.nb + 1, dtype=np.uint64) << np.uint64(32)).astype(np.int64)
        return order, (comb & np.uint64(0xFFFFFFFF)).astype(np.uint16), bounds

    def insert_batch(self, keys, workers=1):
        fps = fingerprint_many(keys, self.seed)
        words = self._rt(fps, self.f)
        b1, _ = self._pp(fps, self.nb)
        order, ws, bounds = self._sorted(b1, words)
        fps_s = fps[order]
        seg = bounds[1:] - bounds[:-1]
        take = np.minimum(seg, np.maximum(0, self.cut - self.fill.astype(np.int64)))
        starts = bounds[:-1].copy()
        ends = starts + take
        _run_ranged(lambda lo, hi: self.ck.btcf_merge_lists(self.blocks, self.fill, self.B, ws, starts, ends,
                                                            lo, hi), self.nb, workers)
        pos = np.arange(len(ws), dtype=np.int64)
        seg_id = np.searchsorted(bounds, pos, side="right") - 1
        left = pos[pos >= ends[seg_id]]
        if len(left):
            fl, wl = fps_s[left], ws[left]
            x, y = self._pp(fl, self.nb)
            dest = np.empty(len(left), dtype=np.int64)
            self.ck.btcf_route(self.fill, self.B, x.astype(np.int64), y.astype(np.int64), dest)
            order2, w2, b2d = self._sorted(dest + 1, wl)
            b2d = np.searchsorted(((dest + 1).astype(np.uint64) << np.uint64(32) | wl.astype(np.uint64))[order2],
                                  np.arange(self.nb + 2, dtype=np.uint64) << np.uint64(32)).astype(np.int64)
            st2, en2 = b2d[1:-1].copy(), b2d[2:].copy()
            _run_ranged(lambda lo, hi: self.ck.btcf_merge_lists(self.blocks, self.fill, self.B, w2, st2, en2,
                                                                lo, hi), self.nb, workers)
            nback = int(b2d[1])
            if nback:
                codes = np.empty(nback, dtype=np.uint8)
                self.ck.backing_insert_batch(self.backing, self.pl, self.f, fl[order2[:nback]].copy(), codes)

    def query_batch(self, keys, workers=1):
        found = np.empty(len(keys), dtype=np.uint8)

        def work(k, fo):
            self.ck.btcf_query_batch(self.blocks, self.fill, self.backing, self.B, self.f, self.pl,
                                     fingerprint_many(k, self.seed), fo)
        run_threads(work, (keys, found), workers)
        return found

    def delete_batch(self, keys, workers=1):
        fps = fingerprint_many(keys, self.seed)
        words = self._rt(fps, self.f)
        removed = np.zeros(len(keys), dtype=np.uint8)
        pending = np.arange(len(keys), dtype=np.int64)
        for choice in self._pp(fps, self.nb):
            if not len(pending):
                break
            order, ws, bounds = self._sorted(choice[pending], words[pending])
            hit = np.zeros(len(pending), dtype=np.uint8)
            _run_ranged(lambda lo, hi: self.ck.btcf_delete_blocklocal(
                self.blocks, self.fill, self.B, ws, bounds[:-1].copy(), bounds[1:].copy(), lo, hi, hit),
                self.nb, workers)
            hb = hit.astype(bool)
            removed[pending[order[hb]]] = 1
            pending = pending[order[~hb]]
        if len(pending) and len(self.backing):
            flags = np.empty(len(pending), dtype=np.uint8)
            self.ck.backing_delete_batch(self.backing, self.pl, self.f, fps[pending].copy(), flags)
            removed[pending[flags.astype(bool)]] = 1
        return removed


class RefGqf:
    """GQF: the reference facade's bulk glue (fk/gqf.py:286-371, restated:
    stable sort, region split, even regions then odd on `workers` threads,
    descending deletes) and its chunked count_many (gqf.py:182-193) around
    the reference's compiled kernels."""

    def __init__(self, q, r=8, seed=0, max_load=0.95):
        self.ck = kernels()
        self.q, self.r, self.seed = q, r, seed
        logical = 1 << q
        phys = logical + min(8192, logical)
        self.nregions = (phys + 8191) >> 13
        self.qregions = (logical + 8191) >> 13
        self.max_occ = int(max_load * logical)
        dt = {8: np.uint8, 16: np.uint16, 32: np.uint32, 64: np.uint64}[r]
        self.slots = np.zeros(phys, dtype=dt)
        self.occ = np.zeros(phys >> 6, dtype=np.uint64)
        self.run = np.zeros(phys >> 6, dtype=np.uint64)
        self.offs = np.zeros(self.nregions, dtype=np.int32)
        self.stats = np.zeros(3, dtype=np.int64)
        self.locks = self.ck.make_region_locks(self.nregions)

    def _fps(self, keys):
        return fingerprint_many(keys, self.seed, self.q + self.r)

    def _bulk(self, keys, counts, workers, op):
        fps = self._fps(keys)
        dflt = np.uint64(1) if op == "insert" else np.uint64(2 ** 63)
        deltas = np.full(len(fps), dflt, dtype=np.uint64) if counts is None else np.ascontiguousarray(
            counts, dtype=np.uint64)
        order = np.argsort(fps, kind="stable")
        fps, deltas = fps[order], deltas[order]
        marks = np.arange(self.qregions + 1, dtype=np.uint64) << np.uint64(self.r + 13)
        bounds = np.searchsorted(fps, marks)
        found = np.ones(len(fps), dtype=np.uint8)
        fails = []

        def region(g):
            lo, hi = int(bounds[g]), int(bounds[g + 1])
            if lo >= hi:
                return
            sh = np.zeros(1, dtype=np.int64)
            if op == "insert":
                code, _ = self.ck.gqf_insert_batch(self.slots, self.occ, self.run, self.offs, self.stats, self.locks,
                                                   self.q, self.r, self.max_occ, False, fps[lo:hi], deltas[lo:hi], sh)
                if code:
                    fails.append(code)
            else:
                fl = np.empty(hi - lo, dtype=np.uint8)
                self.ck.gqf_delete_batch(self.slots, self.occ, self.run, self.offs, self.stats, self.locks, self.q,
                                         self.r, False, fps[lo:hi][::-1].copy(), deltas[lo:hi][::-1].copy(), fl, sh)
                found[lo:hi] = fl[::-1]

        for parity in (0, 1):
            regs = [g for g in range(parity, self.qregions, 2) if bounds[g] < bounds[g + 1]]
            if workers <= 1 or len(regs) <= 1:
                for g in regs:
                    region(g)
            else:
                buckets = [regs[w::workers] for w in range(workers)]
                ts = [threading.Thread(target=lambda b=b: [region(g) for g in b]) for b in buckets if b]
                for t in ts:
                    t.start()
                for t in ts:
                    t.join()
        if fails:
            raise RuntimeError("reference GQF capacity error %d" % fails[0])
        inv = np.empty_like(order)
        inv[order] = np.arange(len(order))
        return found[inv]

    def bulk_insert(self, keys, counts=None, workers=4):
        self._bulk(keys, counts, workers, "insert")

    def bulk_delete(self, keys, counts=None, workers=4):
        return self._bulk(keys, counts, workers, "delete")

    def count_many(self, keys, workers=1):
        counts = np.empty(len(keys), dtype=np.uint64)

        def work(k, c):
            self.ck.gqf_count_batch(self.slots, self.occ, self.run, self.offs, self.locks, self.q, self.r, True,
                                    self._fps(k), c)
        run_threads(work, (keys, counts), workers)
        return counts
