"""oracle.model -- CPU restatement of the reference filter facades.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs as the *checker*.  The product
package (paper_2212_09005_b200) never imports this module.

The kernels run in oracle/fk_oracle.c (loaded with ctypes); the host-side
orchestration here restates, in order and with the same tie-breaks, the
reference facades:

* OracleTcf      -- fk/tcf.py:95-192 (point insert/query/delete)
* OracleBulkTcf  -- fk/tcf_bulk.py:93-325 (partition, shortcut, route, merge,
                    backing; 3-pass delete; query)
* OracleGqf      -- fk/gqf.py:98-371 (point insert/count/delete in input
                    order; bulk even/odd region phases, workers=1)

Geometry is passed in as plain integers (main/backing slot counts, cut line,
...), so the derivation rules live in exactly one place (the product's
*Params classes), which tests/golden pins against the reference's own values.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libfk_oracle.so")

MASK64 = (1 << 64) - 1
C_BLOCK1 = 0x9E3779B97F4A7C15
C_BLOCK2 = 0xC2B2AE3D27D4EB4F
C_BACK_START = 0x165667B19E3779F9
C_BACK_STEP = 0x27D4EB2F165667C5
REGION_BITS = 13
LOAD_CAPACITY, SHIFT_BOUND = 1, 2


def build(force=False):
    """Compile fk_oracle.c with gcc (the checker, not the product)."""
    src = os.path.join(_HERE, "fk_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        import subprocess
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o", _LIB_PATH, src])
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = ctypes.CDLL(_LIB_PATH)
        i64, i32, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        _lib.orc_mix64.restype = ctypes.c_uint64
        _lib.orc_mix64.argtypes = [ctypes.c_uint64]
        for name in ("orc_tcf_insert_batch", "orc_tcf_query_batch", "orc_tcf_delete_batch",
                     "orc_btcf_merge_lists", "orc_backing_insert_batch",
                     "orc_btcf_delete_blocklocal", "orc_backing_delete_batch",
                     "orc_btcf_query_batch", "orc_encoded_length"):
            getattr(_lib, name).restype = i64
        for name in ("orc_btcf_route", "orc_gqf_insert_batch", "orc_gqf_count_batch",
                     "orc_gqf_delete_batch", "orc_gqf_find_run"):
            getattr(_lib, name).restype = i32
        _lib.orc_encoded_length.argtypes = [ctypes.c_uint64, ctypes.c_uint64, i32]
        del i64, vp
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None and a.size else ctypes.c_void_p(0)


def _u64(keys):
    return np.ascontiguousarray(keys, dtype=np.uint64)


# -- hashing (fk/hashing.py:28-117), numpy-vectorised ------------------------

def mix64_many(x):
    x = _u64(x).copy()
    with np.errstate(over="ignore"):
        x ^= x >> np.uint64(30)
        x *= np.uint64(0xBF58476D1CE4E5B9)
        x ^= x >> np.uint64(27)
        x *= np.uint64(0x94D049BB133111EB)
        x ^= x >> np.uint64(31)
    return x


def fingerprint_many(keys, seed, bits=64):
    fp = mix64_many(_u64(keys) ^ np.uint64(seed & MASK64))
    if bits < 64:
        fp &= np.uint64((1 << bits) - 1)
    return fp


def potc_pair_many(fps, nb):
    fps = _u64(fps)
    return (mix64_many(fps ^ np.uint64(C_BLOCK1)) % np.uint64(nb),
            mix64_many(fps ^ np.uint64(C_BLOCK2)) % np.uint64(nb))


def remap_tags(fps, f):
    t = _u64(fps) & np.uint64((1 << f) - 1 if f < 64 else MASK64)
    return np.where(t < 2, t | np.uint64(2), t).astype(np.uint64)


def encoded_length(rem, count, r):
    return int(lib().orc_encoded_length(int(rem), int(count), int(r)))


def _wb(dtype):
    return np.dtype(dtype).itemsize


# -- point TCF ------------------------------------------------------------------

class OracleTcf:
    """fk/tcf.py:95-192 with sequential (single caller thread) semantics."""

    def __init__(self, num_blocks, block_slots, tag_bits, slot_dtype, backing_slots,
                 cut_slots, probe_limit, seed):
        self.nb, self.B, self.f = int(num_blocks), int(block_slots), int(tag_bits)
        self.cut, self.probe_limit, self.seed = int(cut_slots), int(probe_limit), int(seed)
        self.blocks = np.zeros(self.nb * self.B, dtype=slot_dtype)
        self.backing = np.zeros(int(backing_slots), dtype=slot_dtype)
        self.wb = _wb(slot_dtype)
        self.counters = {"inserts_ok": 0, "inserts_backing": 0, "deletes_ok": 0}

    def fps(self, keys):
        return fingerprint_many(keys, self.seed)

    def insert_fps(self, fps, values=None):
        fps = _u64(fps)
        vals = None if values is None else _u64(values)
        codes = np.empty(len(fps), dtype=np.uint8)
        nback = ctypes.c_int64(0)
        nok = lib().orc_tcf_insert_batch(
            _p(self.blocks), self.wb, ctypes.c_int64(self.nb), _p(self.backing),
            ctypes.c_int64(len(self.backing)), self.B, self.f, self.cut, self.probe_limit,
            _p(fps), _p(vals), ctypes.c_int64(len(fps)), _p(codes), ctypes.byref(nback))
        self.counters["inserts_ok"] += int(nok)
        self.counters["inserts_backing"] += int(nback.value)
        return codes

    def insert_many(self, keys, values=None):
        return self.insert_fps(self.fps(keys), values)

    def query_fps(self, fps):
        fps = _u64(fps)
        found = np.empty(len(fps), dtype=np.uint8)
        vals = np.empty(len(fps), dtype=np.uint64)
        lib().orc_tcf_query_batch(
            _p(self.blocks), self.wb, ctypes.c_int64(self.nb), _p(self.backing),
            ctypes.c_int64(len(self.backing)), self.B, self.f, self.probe_limit,
            _p(fps), ctypes.c_int64(len(fps)), _p(found), _p(vals))
        return found.astype(bool), vals

    def query_values_many(self, keys):
        return self.query_fps(self.fps(keys))

    def query_many(self, keys):
        return self.query_values_many(keys)[0]

    def delete_fps(self, fps):
        fps = _u64(fps)
        removed = np.empty(len(fps), dtype=np.uint8)
        n = lib().orc_tcf_delete_batch(
            _p(self.blocks), self.wb, ctypes.c_int64(self.nb), _p(self.backing),
            ctypes.c_int64(len(self.backing)), self.B, self.f, self.probe_limit,
            _p(fps), ctypes.c_int64(len(fps)), _p(removed))
        self.counters["deletes_ok"] += int(n)
        return removed.astype(bool)

    def delete_many(self, keys):
        return self.delete_fps(self.fps(keys))


# -- bulk TCF ---------------------------------------------------------------------

class OracleBulkTcf:
    """fk/tcf_bulk.py:93-325 (workers=1; the reference result is worker-invariant)."""

    def __init__(self, num_blocks, block_slots, tag_bits, slot_dtype, backing_slots,
                 cut_slots, probe_limit, seed):
        self.nb, self.B, self.f = int(num_blocks), int(block_slots), int(tag_bits)
        self.cut, self.probe_limit, self.seed = int(cut_slots), int(probe_limit), int(seed)
        self.dtype = np.dtype(slot_dtype)
        self.wb = self.dtype.itemsize
        self.blocks = np.zeros(self.nb * self.B, dtype=slot_dtype)
        self.fill = np.zeros(self.nb, dtype=np.uint32)
        self.backing = np.zeros(int(backing_slots), dtype=slot_dtype)
        self.counters = {"inserts_ok": 0, "inserts_backing": 0, "deletes_ok": 0}

    def fps(self, keys):
        return fingerprint_many(keys, self.seed)

    def _merge(self, words, starts, ends):
        rc = lib().orc_btcf_merge_lists(
            _p(self.blocks), self.wb, _p(self.fill), self.B, _p(words), _p(starts), _p(ends),
            ctypes.c_int64(0), ctypes.c_int64(self.nb))
        if rc:
            raise AssertionError("merge overfilled block %d" % (rc - 1))

    def _sorted_by_block(self, blocks_of, words):
        """Stable order by (block, word) and per-block [start, end) bounds."""
        combined = (_u64(blocks_of) << np.uint64(32)) | _u64(words)
        order = np.argsort(combined, kind="stable")
        combined = combined[order]
        bounds = np.searchsorted(
            combined, np.arange(self.nb + 1, dtype=np.uint64) << np.uint64(32)).astype(np.int64)
        return order, (combined & np.uint64(0xFFFFFFFF)).astype(self.dtype), bounds

    def insert_batch(self, keys):
        keys = _u64(keys)
        if len(keys) == 0:
            return keys
        fps = self.fps(keys)
        words = remap_tags(fps, self.f)
        b1, _ = potc_pair_many(fps, self.nb)
        order, wsorted, bounds = self._sorted_by_block(b1, words)
        fps_s, keys_s = fps[order], keys[order]
        # phase 1 (fk/tcf_bulk.py:191-208): shortcut up to the cut line
        seg = bounds[1:] - bounds[:-1]
        room = np.maximum(0, self.cut - self.fill.astype(np.int64))
        starts = bounds[:-1].copy()
        ends = starts + np.minimum(seg, room)
        self._merge(wsorted, starts, ends)
        # phase 2 (fk/tcf_bulk.py:210-245): sequential routing of the leftovers
        pos = np.arange(len(wsorted), dtype=np.int64)
        seg_id = np.searchsorted(bounds, pos, side="right") - 1
        left = pos[pos >= ends[seg_id]]
        n_fail = 0
        failed = keys[:0]
        if len(left):
            fl, wl, kl = fps_s[left], wsorted[left], keys_s[left]
            x, y = potc_pair_many(fl, self.nb)
            x, y = x.astype(np.int64), y.astype(np.int64)
            dest = np.empty(len(left), dtype=np.int64)
            rc = lib().orc_btcf_route(_p(self.fill), ctypes.c_int64(self.nb), self.B, _p(x), _p(y),
                                      ctypes.c_int64(len(left)), _p(dest))
            if rc:
                raise MemoryError()
            combined = ((dest + 1).astype(np.uint64) << np.uint64(32)) | wl.astype(np.uint64)
            order2 = np.argsort(combined, kind="stable")
            combined = combined[order2]
            w2 = (combined & np.uint64(0xFFFFFFFF)).astype(self.dtype)
            b2d = np.searchsorted(
                combined, np.arange(self.nb + 2, dtype=np.uint64) << np.uint64(32)).astype(np.int64)
            st2, en2 = b2d[1:-1].copy(), b2d[2:].copy()
            self._merge(w2, st2, en2)
            n_back = int(b2d[1])
            if n_back:
                fb = _u64(fl[order2[:n_back]])
                codes = np.empty(n_back, dtype=np.uint8)
                n_fail = int(lib().orc_backing_insert_batch(
                    _p(self.backing), self.wb, ctypes.c_int64(len(self.backing)), self.probe_limit,
                    self.f, _p(fb), ctypes.c_int64(n_back), _p(codes)))
                self.counters["inserts_backing"] += n_back - n_fail
                if n_fail:
                    failed = kl[order2[:n_back]][codes == 3]
        self.counters["inserts_ok"] += len(keys) - n_fail
        return failed

    def query_batch(self, keys):
        fps = self.fps(keys)
        found = np.empty(len(fps), dtype=np.uint8)
        lib().orc_btcf_query_batch(
            _p(self.blocks), self.wb, _p(self.fill), ctypes.c_int64(self.nb), _p(self.backing),
            ctypes.c_int64(len(self.backing)), self.B, self.f, self.probe_limit, _p(fps),
            ctypes.c_int64(len(fps)), _p(found))
        return found.astype(bool)

    def delete_batch(self, keys):
        keys = _u64(keys)
        fps = self.fps(keys)
        words = remap_tags(fps, self.f)
        removed = np.zeros(len(keys), dtype=np.uint8)
        pending = np.arange(len(keys), dtype=np.int64)
        for choice in potc_pair_many(fps, self.nb):
            if not len(pending):
                break
            order, ws, bounds = self._sorted_by_block(choice[pending], words[pending])
            hit = np.zeros(len(pending), dtype=np.uint8)
            st, en = bounds[:-1].copy(), bounds[1:].copy()
            lib().orc_btcf_delete_blocklocal(
                _p(self.blocks), self.wb, _p(self.fill), self.B, _p(ws), _p(st), _p(en),
                ctypes.c_int64(0), ctypes.c_int64(self.nb), _p(hit))
            hb = hit.astype(bool)
            removed[pending[order[hb]]] = 1
            pending = pending[order[~hb]]
        if len(pending) and len(self.backing):
            flags = np.empty(len(pending), dtype=np.uint8)
            fp_p = _u64(fps[pending])
            lib().orc_backing_delete_batch(
                _p(self.backing), self.wb, ctypes.c_int64(len(self.backing)), self.probe_limit,
                self.f, _p(fp_p), ctypes.c_int64(len(pending)), _p(flags))
            removed[pending[flags.astype(bool)]] = 1
        self.counters["deletes_ok"] += int(removed.sum())
        return removed.astype(bool)


# -- GQF --------------------------------------------------------------------------

class OracleGqf:
    """fk/gqf.py:98-371.  Bulk ops run the even/odd region phases with one worker."""

    def __init__(self, q, r, seed, max_occupied):
        self.q, self.r, self.seed, self.max_occupied = int(q), int(r), int(seed), int(max_occupied)
        logical = 1 << self.q
        self.phys = logical + min(1 << REGION_BITS, logical)
        self.num_regions = (self.phys + (1 << REGION_BITS) - 1) >> REGION_BITS
        self.quotient_regions = (logical + (1 << REGION_BITS) - 1) >> REGION_BITS
        self.dtype = {8: np.uint8, 16: np.uint16, 32: np.uint32, 64: np.uint64}[self.r]
        self.slots = np.zeros(self.phys, dtype=self.dtype)
        self.occ = np.zeros(self.phys >> 6, dtype=np.uint64)
        self.run = np.zeros(self.phys >> 6, dtype=np.uint64)
        self.offsets = np.zeros(self.num_regions, dtype=np.int32)
        self.stats = np.zeros(3, dtype=np.int64)
        self.shifted = 0

    def fps(self, keys):
        return fingerprint_many(keys, self.seed, self.q + self.r)

    def _args(self):
        return (_p(self.slots), self.slots.itemsize, _p(self.occ), _p(self.run), _p(self.offsets))

    def insert_fps(self, fps, deltas):
        """Returns (code, fail_index) like gqf_insert_batch (pk:772-801)."""
        fps, deltas = _u64(fps), _u64(deltas)
        sh = ctypes.c_int64(0)
        fail = ctypes.c_int64(-1)
        code = lib().orc_gqf_insert_batch(
            *self._args(), _p(self.stats), ctypes.c_int64(self.phys), self.q, self.r,
            ctypes.c_int64(self.max_occupied), _p(fps), _p(deltas), ctypes.c_int64(len(fps)),
            ctypes.byref(sh), ctypes.byref(fail))
        if code < 0:
            raise RuntimeError("oracle invariant violation (%d)" % code)
        self.shifted += sh.value
        return code, fail.value

    def insert_many(self, keys, counts=None):
        """fk/gqf.py:174-178 (workers=1): input order, raise at the first failure."""
        fps = self.fps(keys)
        deltas = np.ones(len(fps), np.uint64) if counts is None else _u64(counts)
        return self.insert_fps(fps, deltas)

    def count_fps(self, fps):
        fps = _u64(fps)
        out = np.empty(len(fps), dtype=np.uint64)
        rc = lib().orc_gqf_count_batch(*self._args(), ctypes.c_int64(self.phys), self.q, self.r,
                                       _p(fps), ctypes.c_int64(len(fps)), _p(out))
        if rc:
            raise RuntimeError("oracle invariant violation")
        return out

    def count_many(self, keys):
        return self.count_fps(self.fps(keys))

    def delete_fps(self, fps, deltas):
        fps, deltas = _u64(fps), _u64(deltas)
        found = np.zeros(len(fps), dtype=np.uint8)
        sh = ctypes.c_int64(0)
        rc = lib().orc_gqf_delete_batch(
            *self._args(), _p(self.stats), ctypes.c_int64(self.phys), self.q, self.r, _p(fps),
            _p(deltas), ctypes.c_int64(len(fps)), _p(found), ctypes.byref(sh))
        if rc:
            raise RuntimeError("oracle invariant violation")
        self.shifted += sh.value
        return found.astype(bool)

    def delete_many(self, keys, counts=None):
        fps = self.fps(keys)
        deltas = np.full(len(fps), 2 ** 63, np.uint64) if counts is None else _u64(counts)
        return self.delete_fps(fps, deltas)

    def find_run(self, quotient):
        s, e = ctypes.c_int64(), ctypes.c_int64()
        rc = lib().orc_gqf_find_run(_p(self.occ), _p(self.run), _p(self.offsets),
                                    ctypes.c_int64(self.phys), ctypes.c_int64(quotient),
                                    ctypes.byref(s), ctypes.byref(e))
        if rc:
            raise RuntimeError("oracle invariant violation")
        return s.value, e.value

    def _region_op(self, fps, deltas, op, stats):
        """One region's slice through the batch kernel (pk:772-801 /
        pk:827-847) against the given stats array; -> (code, found, shifted)."""
        sh = ctypes.c_int64(0)
        if op == "insert":
            fail = ctypes.c_int64(-1)
            code = lib().orc_gqf_insert_batch(
                *self._args(), _p(stats), ctypes.c_int64(self.phys), self.q, self.r,
                ctypes.c_int64(self.max_occupied), _p(fps), _p(deltas), ctypes.c_int64(len(fps)),
                ctypes.byref(sh), ctypes.byref(fail))
            found = None
        else:
            found = np.zeros(len(fps), dtype=np.uint8)
            code = lib().orc_gqf_delete_batch(
                *self._args(), _p(stats), ctypes.c_int64(self.phys), self.q, self.r, _p(fps),
                _p(deltas), ctypes.c_int64(len(fps)), _p(found), ctypes.byref(sh))
        if code < 0 or (op != "insert" and code):
            raise RuntimeError("oracle invariant violation (%d)" % code)
        return code, found, sh.value

    def _bulk(self, fps, deltas, op, workers=1):
        """fk/gqf.py:293-353: stable sort, even regions, then odd.

        workers > 1 runs the regions of one parity on threads, as the
        reference's own worker pool does (fk/gqf.py:326-345; regions of one
        parity never touch each other's slots, pk:758-769).  Each thread gets
        a private copy of _stats (the reference adds to one array atomically,
        pk:579-581) and the deltas are summed after the phase.  The load check
        then sees a stale occupancy, so a parallel insert phase that reports
        any capacity failure is an error here: it is only for batches that
        stay below max_occupied (the full-size parity tests)."""
        order = np.argsort(fps, kind="stable")
        fps, deltas = fps[order], deltas[order]
        marks = np.arange(self.quotient_regions + 1, dtype=np.uint64) << np.uint64(self.r + REGION_BITS)
        bounds = np.searchsorted(fps, marks)
        found = np.ones(len(fps), dtype=np.uint8)
        failures = []
        for parity in (0, 1):
            jobs = []
            for g in range(parity, self.quotient_regions, 2):
                lo, hi = int(bounds[g]), int(bounds[g + 1])
                if lo < hi:
                    jobs.append((g, lo, hi))
            if workers <= 1:
                for g, lo, hi in jobs:
                    if op == "insert":
                        code, _, sh = self._region_op(fps[lo:hi], deltas[lo:hi], op, self.stats)
                        if code:
                            failures.append((code, g))
                    else:
                        _, fl, sh = self._region_op(fps[lo:hi][::-1].copy(), deltas[lo:hi][::-1].copy(), op,
                                                    self.stats)
                        found[lo:hi] = fl[::-1]
                    self.shifted += sh
                continue
            from concurrent.futures import ThreadPoolExecutor
            base = self.stats.copy()

            def run(job):
                g, lo, hi = job
                st = base.copy()
                if op == "insert":
                    res = self._region_op(fps[lo:hi], deltas[lo:hi], op, st)
                else:
                    res = self._region_op(fps[lo:hi][::-1].copy(), deltas[lo:hi][::-1].copy(), op, st)
                return job, res, st - base

            with ThreadPoolExecutor(workers) as ex:
                for (g, lo, hi), (code, fl, sh), dst in ex.map(run, jobs):
                    if code:
                        raise RuntimeError("capacity failure in a parallel oracle phase (region %d)" % g)
                    if fl is not None:
                        found[lo:hi] = fl[::-1]
                    self.stats += dst
                    self.shifted += sh
        inv = np.empty_like(order)
        inv[order] = np.arange(len(order))
        return failures, found[inv].astype(bool)

    def bulk_insert(self, keys, counts=None, workers=1):
        """Returns the failure list [(code, region)] (empty on success)."""
        fps = self.fps(keys)
        if not len(fps):
            return []
        deltas = np.ones(len(fps), np.uint64) if counts is None else _u64(counts)
        return self._bulk(fps, deltas, "insert", workers)[0]

    def bulk_delete(self, keys, counts=None, workers=1):
        fps = self.fps(keys)
        if not len(fps):
            return np.zeros(0, dtype=bool)
        deltas = np.full(len(fps), 2 ** 63, np.uint64) if counts is None else _u64(counts)
        return self._bulk(fps, deltas, "delete", workers)[1]

    def image(self):
        return dict(slots=self.slots, occupieds=self.occ, runends=self.run,
                    offsets=self.offsets, stats=self.stats)
