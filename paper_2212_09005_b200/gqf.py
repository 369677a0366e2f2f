"""Counting quotient filter (GQF) on the B200.

Drop-in for filterkit.gqf (/root/reference/pkg/src/filterkit/gqf.py:52-492):
same ``GqfParams`` (fields, validation, derived geometry) and ``Gqf`` methods
(point insert/count/delete, phased bulk insert/delete, enumeration,
find_run, cluster_stats, validate) with the same table image
(``_slots``, ``_occupieds``, ``_runends``, ``_offsets``, ``_stats``).

Every count query is one kernel (csrc/gqf_impl.cuh: k_gqf_count, O(1) run
lookup through a derived spill index).  Every insert/delete batch -- point
or bulk -- is one call of fk_gqf_apply: the final image is the canonical
layout of the resulting (fingerprint -> count) multiset, which is exactly
what the reference produces whenever it raises no CapacityError; batches
that could raise run the reference's sequential algorithm on the device and
reproduce its partial application.  ``workers`` arguments are accepted and
ignored (the device is the parallelism).
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._device import DeviceTables, check_backend, keys_in, ret
from .countgroups import decode_run
from .errors import CapacityError, ValidationError
from .hashing import fingerprint_many, join_fingerprint

__all__ = ["GqfParams", "Gqf"]

REGION_BITS = 13
REGION_SLOTS = 1 << REGION_BITS
GQF_LOAD_CAPACITY = 1
GQF_SHIFT_BOUND = 2


def _slot_dtype(bits):
    return {8: np.uint8, 16: np.uint16, 32: np.uint32, 64: np.uint64}[bits]


@dataclass(frozen=True)
class GqfParams:
    """Geometry for a counting quotient filter (gqf.py:52-95)."""

    q: int
    r: int = 8
    seed: int = 0
    max_load: float = 0.95

    def __post_init__(self):
        if not 6 <= self.q <= 40:
            raise ValueError("q must be in [6, 40]")
        if self.r not in (8, 16, 32, 64):
            raise ValueError("r must be one of 8, 16, 32, 64")
        if self.q + self.r > 64:
            raise ValueError("q + r must be at most 64")
        if not 0.0 < self.max_load <= 1.0:
            raise ValueError("max_load must be in (0, 1]")

    @property
    def logical_slots(self):
        return 1 << self.q

    @property
    def padding_slots(self):
        return min(REGION_SLOTS, self.logical_slots)

    @property
    def physical_slots(self):
        return self.logical_slots + self.padding_slots

    @property
    def num_regions(self):
        return (self.physical_slots + REGION_SLOTS - 1) >> REGION_BITS

    @property
    def quotient_regions(self):
        return (self.logical_slots + REGION_SLOTS - 1) >> REGION_BITS

    @property
    def max_occupied(self):
        return int(self.max_load * self.logical_slots)


def _capacity_msg(code):
    if code == GQF_LOAD_CAPACITY:
        return "insert rejected: used slots reached the load ceiling"
    if code == GQF_SHIFT_BOUND:
        return "insert rejected: shift would cross the region hard bound"
    return "insert rejected (code %d)" % code


class Gqf:
    """Counting quotient filter on the B200 (one device, exclusive batches)."""

    _OCCUPIED, _ITEMS, _DISTINCT = 0, 1, 2

    def __init__(self, params=None, *, backend="auto", device=None, **kwargs):
        if params is None:
            params = GqfParams(**kwargs)
        elif kwargs:
            raise TypeError("pass either params or keyword fields, not both")
        check_backend(backend)
        self.params = p = params
        torch = _lib.require_cuda(device)
        self._torch = torch
        self._device = torch.device(device) if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        self._lib = _lib.load()
        phys = p.physical_slots
        dt = _slot_dtype(p.r)
        self._dtype = np.dtype(dt)
        spec = {"slots": (dt, phys), "occupieds": (np.uint64, phys >> 6), "runends": (np.uint64, phys >> 6),
                "offsets": (np.int32, p.num_regions), "stats": (np.int64, 3),
                "spill": (np.uint32, max(1, p.logical_slots >> 6))}
        self._cur = DeviceTables(torch, self._device, spec)
        self._nxt = None  # second image, allocated on the first rebuild
        self._spec = spec
        self._geom = _lib.GqfGeom(p.q, p.r, phys, p.num_regions, p.quotient_regions, p.max_occupied,
                                  p.seed & ((1 << 64) - 1))
        self._shift_lock = threading.Lock()
        self._op_lock = threading.Lock()
        self._shifted_slots = 0

    @property
    def backend(self):
        return "cuda"

    # -- table image (host mirrors of the device tables) -----------------------
    @property
    def _slots(self):
        return self._cur.host("slots")

    @property
    def _occupieds(self):
        return self._cur.host("occupieds")

    @property
    def _runends(self):
        return self._cur.host("runends")

    @property
    def _offsets(self):
        return self._cur.host("offsets")

    @property
    def _stats(self):
        return self._cur.host("stats")

    def _tables(self, t):
        return _lib.GqfTables(t.ptr("slots"), t.ptr("occupieds"), t.ptr("runends"), t.ptr("offsets"),
                              t.ptr("stats"), t.ptr("spill"))

    def _sync_in(self):
        """Push host edits of the image back and re-derive the run index."""
        if self._cur.before_device_op() & {"occupieds", "runends"}:
            _lib.check(self._lib.fk_gqf_rebuild_index(ctypes.byref(self._geom), ctypes.byref(self._tables(self._cur)),
                                                      _lib.stream_ptr(self._torch)), "gqf index")

    # -- derived views -----------------------------------------------------------
    def _stat(self, i):
        return int(self._cur.peek("stats")[i])

    @property
    def occupied_slots(self):
        return self._stat(self._OCCUPIED)

    @property
    def total_items(self):
        return self._stat(self._ITEMS)

    @property
    def distinct_items(self):
        return self._stat(self._DISTINCT)

    @property
    def shifted_slots(self):
        return self._shifted_slots

    def load_factor(self):
        return self.occupied_slots / self.params.logical_slots

    def size_bits(self):
        """Same accounting as the reference (gqf.py:147-151): slots, both bit
        vectors, offsets, plus 512 bits per region (its lock line)."""
        p = self.params
        phys = p.physical_slots
        return (phys * self._dtype.itemsize + 2 * (phys >> 6) * 8 + p.num_regions * 4) * 8 + p.num_regions * 512

    # -- hashing -----------------------------------------------------------------
    def _fps(self, keys):
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        return fingerprint_many(keys, self.params.seed, self.params.q + self.params.r)

    def fingerprint_of(self, key):
        return int(self._fps([key])[0])

    # -- device calls ---------------------------------------------------------------
    def _deltas(self, counts, n, kind):
        torch = self._torch
        if counts is None:
            return None
        if isinstance(counts, torch.Tensor):
            c = _lib.to_device_u64(torch, counts, self._device)
        else:
            c = np.ascontiguousarray(counts, dtype=np.uint64).reshape(-1)
            c = _lib.to_device_u64(torch, c, self._device)
        if c.numel() != n:
            raise ValueError("counts length does not match keys length")
        return c

    def _apply(self, keys, counts, op, order):
        torch = self._torch
        k, kind = keys_in(torch, keys, self._device)
        n = k.numel()
        d = self._deltas(counts, n, kind)
        # (0/1 bytes written by the kernels)
        found = torch.zeros(n, dtype=torch.bool, device=self._device) if op == _lib.FK_GQF_DELETE else None
        res = _lib.GqfResult()
        if n:
            with self._op_lock:
                self._sync_in()
                if self._nxt is None:
                    self._nxt = DeviceTables(torch, self._device, self._spec)
                rc = self._lib.fk_gqf_apply(
                    ctypes.byref(self._geom), ctypes.byref(self._tables(self._cur)),
                    ctypes.byref(self._tables(self._nxt)), _lib.dptr(k), 0, _lib.dptr(d), n, op, order,
                    _lib.dptr(found), ctypes.byref(res), _lib.stream_ptr(torch))
                _lib.check(rc, "gqf apply")
                if res.swapped:
                    self._cur, self._nxt = self._nxt, self._cur
                self._cur.after_device_write()
                self._nxt.after_device_write()
            with self._shift_lock:
                self._shifted_slots += int(res.shifted)
        return res, found, kind

    # -- point API ----------------------------------------------------------------------
    def insert(self, key, count=1):
        self.insert_many([key], [count])

    def insert_many(self, keys, counts=None, workers=1):
        """Insert in input order; raises CapacityError at the first failing key
        (the keys before it stay inserted, like gqf_insert_batch)."""
        res, _, _ = self._apply(keys, counts, _lib.FK_GQF_INSERT, _lib.FK_ORDER_POINT)
        if res.code:
            raise CapacityError(_capacity_msg(res.code))

    def count(self, key):
        return int(self.count_many([key])[0])

    def query(self, key):
        return self.count(key) > 0

    def count_many(self, keys, workers=1):
        torch = self._torch
        k, kind = keys_in(torch, keys, self._device)
        n = k.numel()
        out = torch.empty(n, dtype=torch.int64, device=self._device)
        if n:
            with self._op_lock:
                self._sync_in()
                rc = self._lib.fk_gqf_count(ctypes.byref(self._geom), ctypes.byref(self._tables(self._cur)),
                                            _lib.dptr(k), 0, n, _lib.dptr(out), _lib.stream_ptr(torch))
                _lib.check(rc, "gqf count")
        if kind == "numpy":
            return out.cpu().numpy().view(np.uint64)
        return ret(torch, out, kind)

    def delete(self, key, count=1):
        if count is None:
            count = 2 ** 63
        return bool(self.delete_many([key], [count])[0])

    def delete_many(self, keys, counts=None, workers=1):
        """Remove up to `counts` copies (all by default) in input order; per-key
        found flags."""
        res, found, kind = self._apply(keys, counts, _lib.FK_GQF_DELETE, _lib.FK_ORDER_POINT)
        return self._flags(found, kind)

    def _flags(self, found, kind):
        if kind == "numpy":
            return found.cpu().numpy()
        return ret(self._torch, found, kind)

    # -- bulk API ---------------------------------------------------------------------------
    def bulk_insert(self, keys, counts=None, workers=4):
        """Batch insert of (key, count) pairs (gqf.py:355-360 semantics)."""
        res, _, _ = self._apply(keys, counts, _lib.FK_GQF_INSERT, _lib.FK_ORDER_BULK)
        if res.code:
            raise CapacityError(_capacity_msg(res.code) + " (bulk batch partially applied)")

    def bulk_delete(self, keys, counts=None, workers=4):
        """Batch delete; counts=None removes all copies; per-key found flags
        with the reference's per-region descending application order."""
        torch = self._torch
        if (isinstance(keys, torch.Tensor) and keys.numel() == 0) or \
                (not isinstance(keys, torch.Tensor) and len(keys) == 0):
            return np.zeros(0, dtype=bool)
        res, found, kind = self._apply(keys, counts, _lib.FK_GQF_DELETE, _lib.FK_ORDER_BULK)
        return self._flags(found, kind)

    def _reset(self):
        """Zero the filter (benchmark helper; not in the reference API)."""
        with self._op_lock:
            self._cur.zero()
            self._shifted_slots = 0

    # -- enumeration and structure (host, over the mirrored image) ---------------------------
    def _derive_structure(self):
        """(quotients, run starts, run ends) by global rank/select over the
        bit vectors -- independent of the device's run index."""
        occ = np.unpackbits(self._cur.peek("occupieds").view(np.uint8), bitorder="little")
        run = np.unpackbits(self._cur.peek("runends").view(np.uint8), bitorder="little")
        quotients = np.flatnonzero(occ).astype(np.int64)
        ends = np.flatnonzero(run).astype(np.int64)
        if len(quotients) != len(ends):
            raise ValidationError("occupieds and runends set-bit counts differ")
        if not len(quotients):
            return quotients, quotients, ends
        prev_end = np.concatenate(([-1], ends[:-1]))
        return quotients, np.maximum(quotients, prev_end + 1), ends

    def items(self):
        return list(self.enumerate_items())

    def enumerate_items(self):
        """Stored (fingerprint, count) pairs in fingerprint order, decoded on
        the device (fk_gqf_enumerate) and yielded from host arrays."""
        fps, cnts = self.device_items()
        for f, c in zip(fps.tolist(), cnts.tolist()):
            yield f, c

    def device_items(self):
        """(fingerprints, counts) as numpy uint64 arrays, fingerprint order."""
        torch = self._torch
        n = ctypes.c_int64(0)
        with self._op_lock:
            self._sync_in()
            cap = max(1, self.distinct_items)
            for _ in range(2):
                fp = torch.empty(cap, dtype=torch.int64, device=self._device)
                cn = torch.empty(cap, dtype=torch.int64, device=self._device)
                rc = self._lib.fk_gqf_enumerate(ctypes.byref(self._geom), ctypes.byref(self._tables(self._cur)),
                                                _lib.dptr(fp), _lib.dptr(cn), cap, ctypes.byref(n),
                                                _lib.stream_ptr(torch))
                if rc == _lib.FK_E_INVARIANT:
                    raise ValidationError("table does not decode")
                _lib.check(rc, "gqf enumerate")
                if n.value <= cap:
                    break
                cap = n.value  # the distinct counter disagreed with the table
        k = n.value
        return (fp[:k].cpu().numpy().view(np.uint64), cn[:k].cpu().numpy().view(np.uint64))

    def _enumerate_host(self):
        r = self.params.r
        slots = self._cur.peek("slots")
        quotients, starts, ends = self._derive_structure()
        for qt, s, e in zip(quotients.tolist(), starts.tolist(), ends.tolist()):
            for rem, cnt in decode_run(slots, s, e, r):
                yield join_fingerprint(qt, rem, r), cnt

    def find_run(self, quotient):
        """[start, end] slot interval of a quotient's run; (-1, -1) if absent."""
        torch = self._torch
        qt = torch.tensor([int(quotient)], dtype=torch.int64, device=self._device)
        se = torch.empty(2, dtype=torch.int64, device=self._device)
        with self._op_lock:
            self._sync_in()
            rc = self._lib.fk_gqf_find_run(ctypes.byref(self._geom), ctypes.byref(self._tables(self._cur)),
                                           _lib.dptr(qt), 1, _lib.dptr(se), _lib.stream_ptr(torch))
            _lib.check(rc, "gqf find_run")
        s, e = se.cpu().tolist()
        return (int(s), int(e))

    def cluster_stats(self):
        """Max/mean/count of maximal contiguous used-slot spans (gqf.py:
        416-428), by a global rank/select over the bit vectors on the device
        (fk_gqf_cluster_stats)."""
        out = np.zeros(3, dtype=np.int64)
        with self._op_lock:
            self._sync_in()
            rc = self._lib.fk_gqf_cluster_stats(ctypes.byref(self._geom), ctypes.byref(self._tables(self._cur)),
                                                out.ctypes.data_as(ctypes.c_void_p), _lib.stream_ptr(self._torch))
        if rc == _lib.FK_E_INVARIANT:
            raise ValidationError("occupieds and runends set-bit counts differ")
        _lib.check(rc, "gqf cluster_stats")
        num, longest, total = (int(x) for x in out)
        if num == 0:
            return {"num_clusters": 0, "max_cluster": 0, "mean_cluster": 0.0}
        return {"num_clusters": num, "max_cluster": longest, "mean_cluster": total / num}

    def validate(self):
        """Structural invariants (gqf.py:430-492), checked on the device by
        fk_gqf_validate (global rank/select over the bit vectors, every run
        decoded in parallel).  On a violation, tables small enough to decode
        on the host re-run the reference's host checks so the message names
        the same first failure; larger ones report the device's first one."""
        first = self._device_validate()
        if first is None:
            return
        if self.params.physical_slots <= (1 << 22):
            self._validate_host()
        raise ValidationError(first)

    _VCHECKS = [(1, "occupieds and runends set-bit counts differ"),
                (2, "occupied quotient beyond logical table (quotient %d)"),
                (3, "run extends past physical table (quotient %d)"),
                (5, "run with negative length (quotient %d)"),
                (7, "run crossed its region hard bound (quotient %d)"),
                (8, "region %d offset != derived")]

    def _device_validate(self):
        """None if the table is valid, else the first failure's message."""
        out = np.zeros(24, dtype=np.int64)
        with self._op_lock:
            self._sync_in()
            rc = self._lib.fk_gqf_validate(ctypes.byref(self._geom), ctypes.byref(self._tables(self._cur)),
                                           out.ctypes.data_as(ctypes.c_void_p), _lib.stream_ptr(self._torch))
            _lib.check(rc, "gqf validate")
        mask = int(out[0])
        for code, msg in self._VCHECKS:
            if mask >> code & 1:
                return msg % int(out[8 + code]) if "%d" in msg else msg
        if int(out[1]) != self.occupied_slots:
            return "used slots %d != occupied counter %d" % (int(out[1]), self.occupied_slots)
        if int(out[5]) != int(out[4]):
            return "free slots hold residual data"
        for code, msg in ((11, "run of quotient %d does not decode"), (12, "run of quotient %d has unsorted groups")):
            if mask >> code & 1:
                return msg % int(out[8 + code])
        if int(out[2]) != self.total_items:
            return "decoded total %d != items counter %d" % (int(out[2]), self.total_items)
        if int(out[3]) != self.distinct_items:
            return "decoded distinct %d != distinct counter %d" % (int(out[3]), self.distinct_items)
        return None

    def _validate_host(self):
        """The reference's host-side checks over the mirrored image."""
        p = self.params
        phys = p.physical_slots
        quotients, starts, ends = self._derive_structure()
        if len(quotients):
            if quotients[-1] >= p.logical_slots:
                raise ValidationError("occupied quotient beyond logical table")
            if ends[-1] >= phys:
                raise ValidationError("run extends past physical table")
            if np.any(np.diff(ends) <= 0):
                raise ValidationError("runends not strictly increasing")
            if np.any(starts > ends):
                raise ValidationError("run with negative length")
            if np.any(starts[1:] <= ends[:-1]):
                raise ValidationError("runs overlap")
            if np.any((ends >> REGION_BITS) > (quotients >> REGION_BITS) + 1):
                raise ValidationError("run crossed its region hard bound")
        offsets = self._cur.peek("offsets")
        bounds = np.arange(p.num_regions, dtype=np.int64) << REGION_BITS
        idx = np.searchsorted(quotients, bounds)
        derived = np.where(idx > 0, np.maximum(0, ends[np.maximum(idx - 1, 0)] - bounds + 1) if len(ends) else 0, 0)
        bad = np.flatnonzero(derived != offsets)
        if len(bad):
            h = int(bad[0])
            raise ValidationError("region %d offset %d != derived %d" % (h, int(offsets[h]), int(derived[h])))
        used = np.zeros(phys + 1, dtype=np.int64)
        np.add.at(used, starts, 1)
        np.add.at(used, ends + 1, -1)
        used = np.cumsum(used[:phys]) > 0
        if int(used.sum()) != self.occupied_slots:
            raise ValidationError("used slots %d != occupied counter %d" % (int(used.sum()), self.occupied_slots))
        slots = self._cur.peek("slots")
        if np.any(slots[~used] != 0):
            raise ValidationError("free slots hold residual data")
        total = distinct = 0
        for qt, s, e in zip(quotients.tolist(), starts.tolist(), ends.tolist()):
            try:
                groups = decode_run(slots, s, e, p.r)
            except ValueError as err:
                raise ValidationError("run of quotient %d does not decode: %s" % (qt, err))
            rems = [g[0] for g in groups]
            if rems != sorted(set(rems)):
                raise ValidationError("run of quotient %d has unsorted groups" % qt)
            if any(c <= 0 for _, c in groups):
                raise ValidationError("run of quotient %d decoded count <= 0" % qt)
            total += sum(c for _, c in groups)
            distinct += len(groups)
        if total != self.total_items:
            raise ValidationError("decoded total %d != items counter %d" % (total, self.total_items))
        if distinct != self.distinct_items:
            raise ValidationError("decoded distinct %d != distinct counter %d" % (distinct, self.distinct_items))
