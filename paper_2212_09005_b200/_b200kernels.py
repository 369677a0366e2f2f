"""The reference's kernel contract, served by the B200 kernels.

This module has the exact surface of the module ``filterkit._backends.
get_backend()`` returns (/root/reference/pkg/src/filterkit/_backends.py:29-40,
implemented there by ``_ckernels.pyx`` and ``_pykernels.py``): the same
function names, arguments, return values, in-place mutation of the caller's
numpy arrays and error behaviour.  Registering it in the reference's
``_backends`` runs the reference's own facades --
Tcf, BulkTcf, Gqf -- on the sm_100a kernels through the C ABI in
include/filterkit_b200.h, one entry point per contract function.

Each call uploads the arrays it reads, runs the kernel, and writes back the
arrays it mutates, so the facades' numpy state stays authoritative.  That
round trip is the price of the raw-array contract; the package's own
facades (paper_2212_09005_b200.Tcf & co.) keep the tables resident in HBM
instead.  Calls are serialised by one lock: the reference lets several
threads call the point-TCF / GQF entries on one filter (real CAS / region
spinlocks, ck:99-106), and executing each batch atomically is one legal
linearisation of those calls.  Insert and delete batches run in the ordered
(sequential-semantics) mode, so every call is bit-identical to
``_ckernels`` processing the batch in input order.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _lib

# Registered in the compiled backend's slot: the reference's facades and
# tests key on this name (_backends.py:29-40, test_backends.py:44-47).
NAME = "c"
IMPL = "b200"

P_PRIMARY, P_SECONDARY, P_BACKING, P_FULL = 0, 1, 2, 3
GQF_OK, GQF_LOAD_CAPACITY, GQF_SHIFT_BOUND = 0, 1, 2
REGION_BITS = 13
REGION_SLOTS = 1 << REGION_BITS
_LOCK_STRIDE = 16

_call_lock = threading.Lock()
_BITVIEW = {1: np.uint8, 2: np.int16, 4: np.int32, 8: np.int64}


def make_region_locks(n):
    """Region lock words (unused: the device path needs no host locks; kept
    so the facades' arrays have the reference's shape, ck:99-101)."""
    return np.zeros(int(n) * _LOCK_STRIDE, dtype=np.int32)


def make_mutex():
    """No mutex: the kernels use hardware atomics (ck:104-106)."""
    return None


# -- plumbing -------------------------------------------------------------------

def _torch():
    return _lib.require_cuda()


def _dev(torch, a):
    """numpy array -> device tensor holding the same bytes."""
    a = np.ascontiguousarray(a)
    if a.size == 0:
        return torch.empty(0, dtype=torch.uint8, device="cuda")
    return torch.from_numpy(a.view(_BITVIEW[a.itemsize])).to("cuda")


def _back(t, a):
    """Copy a device tensor back into the caller's numpy array in place."""
    if a.size:
        a[...] = t.cpu().numpy().view(a.dtype).reshape(a.shape)


def _u64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


def _stream(torch):
    return _lib.stream_ptr(torch)


def _tile(g):
    t = 1
    while t * 2 <= min(int(g), 32):
        t *= 2
    return t


def _tcf_geom(blocks, backing, B, f, cut, probe_limit, group_width):
    return _lib.TcfGeom(len(blocks) // int(B), len(backing), int(B), int(f), blocks.itemsize, int(cut),
                        int(probe_limit), _tile(min(int(group_width), int(B))), 0)


def _btcf_geom(nb, B, f, itemsize, backing_slots=0, probe_limit=20):
    return _lib.BtcfGeom(int(nb), int(backing_slots), int(B), int(f), int(itemsize), int(B), int(probe_limit), 0, 0)


def _check(rc, what):
    if rc == _lib.FK_E_INVARIANT:
        raise RuntimeError("%s: invariant violation" % what)
    _lib.check(rc, what)


# -- point TCF (ck:193-355) ----------------------------------------------------------

def _tcf_mutate(fn_name, blocks, backing, geom, fps, extra, out, what):
    torch = _torch()
    lib = _lib.load()
    n = len(fps)
    with _call_lock:
        db, dk = _dev(torch, blocks), _dev(torch, backing)
        dfp = _dev(torch, _u64(fps))
        dout = torch.zeros(n, dtype=torch.uint8, device="cuda")
        cnt = torch.zeros(3, dtype=torch.int64, device="cuda")
        ws_n = lib.fk_tcf_workspace_bytes(ctypes.byref(geom), n, _lib.FK_ORDERED)
        ws = torch.empty(max(1, ws_n), dtype=torch.uint8, device="cuda")
        if fn_name == "insert":
            dv = _dev(torch, _u64(extra)) if extra is not None else None
            rc = lib.fk_tcf_insert(ctypes.byref(geom), _lib.dptr(db), _lib.dptr(dk), _lib.dptr(dfp), 1,
                                   _lib.dptr(dv), n, _lib.dptr(dout), _lib.dptr(cnt), _lib.FK_ORDERED,
                                   _lib.dptr(ws), ws_n, _stream(torch))
        else:
            rc = lib.fk_tcf_delete(ctypes.byref(geom), _lib.dptr(db), _lib.dptr(dk), _lib.dptr(dfp), 1, n,
                                   _lib.dptr(dout), _lib.dptr(cnt), _lib.FK_ORDERED, _lib.dptr(ws), ws_n,
                                   _stream(torch))
        _check(rc, what)
        torch.cuda.current_stream().synchronize()
        _back(db, blocks)
        _back(dk, backing)
        _back(dout, out)
        return [int(x) for x in cnt.cpu().tolist()]


def tcf_insert_batch(blocks, backing, B, f, cut_slots, probe_limit, group_width, mutex, fps, values, codes):
    """Insert packed (tag, value) words; returns (inserted, backing_placed)
    (ck:193-238)."""
    if len(fps) == 0:
        return 0, 0
    geom = _tcf_geom(blocks, backing, B, f, cut_slots, probe_limit, group_width)
    c = _tcf_mutate("insert", blocks, backing, geom, fps, values, codes, "tcf_insert_batch")
    return c[0], c[1]


def tcf_delete_batch(blocks, backing, B, f, probe_limit, group_width, mutex, fps, removed):
    """Tombstone the first slot matching each tag; returns the removal count
    (ck:303-355)."""
    if len(fps) == 0:
        return 0
    geom = _tcf_geom(blocks, backing, B, f, B, probe_limit, group_width)
    return _tcf_mutate("delete", blocks, backing, geom, fps, None, removed, "tcf_delete_batch")[2]


def tcf_query_batch(blocks, backing, B, f, probe_limit, group_width, mutex, fps, found, values_out):
    """Tag-membership queries; fills found / values_out, returns the hit count
    (ck:252-300)."""
    n = len(fps)
    if n == 0:
        return 0
    torch = _torch()
    lib = _lib.load()
    geom = _tcf_geom(blocks, backing, B, f, B, probe_limit, group_width)
    with _call_lock:
        db, dk, dfp = _dev(torch, blocks), _dev(torch, backing), _dev(torch, _u64(fps))
        dfound = torch.zeros(n, dtype=torch.uint8, device="cuda")
        dval = torch.zeros(n, dtype=torch.int64, device="cuda") if values_out is not None else None
        _check(lib.fk_tcf_query(ctypes.byref(geom), _lib.dptr(db), _lib.dptr(dk), _lib.dptr(dfp), 1, n,
                                _lib.dptr(dfound), _lib.dptr(dval), _stream(torch)), "tcf_query_batch")
        torch.cuda.current_stream().synchronize()
        _back(dfound, found)
        if values_out is not None:
            _back(dval, values_out)
        return int(np.count_nonzero(found))


# -- bulk TCF (ck:379-599) ----------------------------------------------------------

def btcf_merge_lists(blocks, fill, B, words, starts, ends, b_lo, b_hi):
    """Merge each block's sorted incoming words into its sorted prefix;
    returns 0, or 1 + the first block that would overflow (ck:379-405)."""
    torch = _torch()
    lib = _lib.load()
    nb = len(fill)
    geom = _btcf_geom(nb, B, 8 * blocks.itemsize, blocks.itemsize)
    words = np.ascontiguousarray(words, dtype=blocks.dtype)
    with _call_lock:
        db, dfill, dw = _dev(torch, blocks), _dev(torch, fill), _dev(torch, words)
        ds, de = _dev(torch, np.asarray(starts, np.int64)), _dev(torch, np.asarray(ends, np.int64))
        st = ctypes.c_int64(0)
        _check(lib.fk_btcf_merge_words(ctypes.byref(geom), _lib.dptr(db), _lib.dptr(dfill), _lib.dptr(dw),
                                       len(words), _lib.dptr(ds), _lib.dptr(de), int(b_lo), int(b_hi),
                                       ctypes.byref(st), _stream(torch)), "btcf_merge_lists")
        _back(db, blocks)
        _back(dfill, fill)
        return int(st.value)


def btcf_route(fill, B, b1s, b2s, dest):
    """Sequential two-choice routing of the leftovers (ck:408-444); dest gets
    the chosen block or -1.  Computed by the fixpoint router, which reaches
    the walk's exact decisions."""
    n = len(b1s)
    if n == 0:
        return
    torch = _torch()
    lib = _lib.load()
    with _call_lock:
        dfill = _dev(torch, np.ascontiguousarray(fill, dtype=np.uint32))
        da, db = _dev(torch, np.asarray(b1s, np.int64)), _dev(torch, np.asarray(b2s, np.int64))
        dd = torch.empty(n, dtype=torch.int64, device="cuda")
        _check(lib.fk_btcf_route(_lib.dptr(dfill), len(fill), int(B), _lib.dptr(da), _lib.dptr(db), n,
                                 _lib.dptr(dd), _stream(torch)), "btcf_route")
        _back(dd, dest)


def backing_insert_batch(backing, probe_limit, f, fps, codes):
    """Backing-table inserts for bulk overflow items, input order; returns
    the failure count (ck:447-466)."""
    n = len(fps)
    if n == 0:
        return 0
    torch = _torch()
    lib = _lib.load()
    geom = _btcf_geom(1, 2, f, backing.itemsize, len(backing), probe_limit)
    with _call_lock:
        dk, dfp = _dev(torch, backing), _dev(torch, _u64(fps))
        dc = torch.zeros(n, dtype=torch.uint8, device="cuda")
        fails = ctypes.c_int64(0)
        _check(lib.fk_backing_insert_batch(ctypes.byref(geom), _lib.dptr(dk), _lib.dptr(dfp), n, _lib.dptr(dc),
                                           ctypes.byref(fails), _stream(torch)), "backing_insert_batch")
        _back(dk, backing)
        _back(dc, codes)
        return int(fails.value)


def btcf_delete_blocklocal(blocks, fill, B, words, starts, ends, b_lo, b_hi, removed):
    """Remove one copy of each word from its assigned block; removed[k] per
    sorted item; returns the removal count (ck:482-512)."""
    torch = _torch()
    lib = _lib.load()
    nb = len(fill)
    geom = _btcf_geom(nb, B, 8 * blocks.itemsize, blocks.itemsize)
    words = np.ascontiguousarray(words, dtype=blocks.dtype)
    with _call_lock:
        db, dfill, dw = _dev(torch, blocks), _dev(torch, fill), _dev(torch, words)
        ds, de = _dev(torch, np.asarray(starts, np.int64)), _dev(torch, np.asarray(ends, np.int64))
        drem = _dev(torch, np.ascontiguousarray(removed, dtype=np.uint8))
        cnt = ctypes.c_int64(0)
        _check(lib.fk_btcf_delete_blocklocal(ctypes.byref(geom), _lib.dptr(db), _lib.dptr(dfill), _lib.dptr(dw),
                                             len(words), _lib.dptr(ds), _lib.dptr(de), int(b_lo), int(b_hi),
                                             _lib.dptr(drem), ctypes.byref(cnt), _stream(torch)),
               "btcf_delete_blocklocal")
        _back(db, blocks)
        _back(dfill, fill)
        _back(drem, removed)
        return int(cnt.value)


def backing_delete_batch(backing, probe_limit, f, fps, removed):
    """Backing-table deletes, input order; returns the removal count
    (ck:515-549)."""
    n = len(fps)
    if n == 0:
        return 0
    torch = _torch()
    lib = _lib.load()
    geom = _btcf_geom(1, 2, f, backing.itemsize, len(backing), probe_limit)
    with _call_lock:
        dk, dfp = _dev(torch, backing), _dev(torch, _u64(fps))
        dr = torch.zeros(n, dtype=torch.uint8, device="cuda")
        cnt = ctypes.c_int64(0)
        _check(lib.fk_backing_delete_batch(ctypes.byref(geom), _lib.dptr(dk), _lib.dptr(dfp), n, _lib.dptr(dr),
                                           ctypes.byref(cnt), _stream(torch)), "backing_delete_batch")
        _back(dk, backing)
        _back(dr, removed)
        return int(cnt.value)


def btcf_query_batch(blocks, fill, backing, B, f, probe_limit, fps, found):
    """Membership over sorted blocks; returns the hit count (ck:552-599)."""
    n = len(fps)
    if n == 0:
        return 0
    torch = _torch()
    lib = _lib.load()
    geom = _btcf_geom(len(fill), B, f, blocks.itemsize, len(backing), probe_limit)
    with _call_lock:
        db, dfill, dk, dfp = _dev(torch, blocks), _dev(torch, fill), _dev(torch, backing), _dev(torch, _u64(fps))
        dfound = torch.zeros(n, dtype=torch.uint8, device="cuda")
        _check(lib.fk_btcf_query(ctypes.byref(geom), _lib.dptr(db), _lib.dptr(dfill), _lib.dptr(dk),
                                 _lib.dptr(dfp), 1, n, _lib.dptr(dfound), _stream(torch)), "btcf_query_batch")
        torch.cuda.current_stream().synchronize()
        _back(dfound, found)
        return int(np.count_nonzero(found))


# -- GQF (ck:754-1296) ----------------------------------------------------------------

def _gqf_geom(q, r, phys, max_occupied=0):
    logical = 1 << int(q)
    nreg = (int(phys) + REGION_SLOTS - 1) // REGION_SLOTS
    qreg = (logical + REGION_SLOTS - 1) // REGION_SLOTS
    return _lib.GqfGeom(int(q), int(r), int(phys), nreg, qreg, int(max_occupied), 0)


class _GqfImage:
    """Device copies of the caller's GQF arrays (+ the derived run index)."""

    def __init__(self, torch, slots, occ, run, offsets, stats, q):
        self.host = (slots, occ, run, offsets, stats)
        self.dev = [_dev(torch, a) if a is not None else None for a in self.host]
        self.spill = torch.zeros(max(1, (1 << int(q)) >> 6), dtype=torch.int32, device="cuda")
        if stats is None:
            self.dev[4] = torch.zeros(3, dtype=torch.int64, device="cuda")
        if slots is None:
            self.dev[0] = torch.zeros(1, dtype=torch.int64, device="cuda")

    def tables(self):
        d = self.dev
        return _lib.GqfTables(_lib.dptr(d[0]), _lib.dptr(d[1]), _lib.dptr(d[2]), _lib.dptr(d[3]), _lib.dptr(d[4]),
                              _lib.dptr(self.spill))

    def write_back(self):
        for t, a in zip(self.dev, self.host):
            if a is not None:
                _back(t, a)


def gqf_find_run(occ, run, offsets, q, quotient):
    """Slot interval [start, end] of a quotient's run, (-1, -1) when absent
    (ck:780-787)."""
    torch = _torch()
    lib = _lib.load()
    phys = len(run) << 6
    geom = _gqf_geom(q, 8, phys)
    with _call_lock:
        img = _GqfImage(torch, None, occ, run, offsets, None, q)
        t = img.tables()
        _check(lib.fk_gqf_rebuild_index(ctypes.byref(geom), ctypes.byref(t), _stream(torch)), "gqf_find_run")
        dq = torch.tensor([int(quotient)], dtype=torch.int64, device="cuda")
        se = torch.empty(2, dtype=torch.int64, device="cuda")
        _check(lib.fk_gqf_find_run(ctypes.byref(geom), ctypes.byref(t), _lib.dptr(dq), 1, _lib.dptr(se),
                                   _stream(torch)), "gqf_find_run")
        s, e = se.cpu().tolist()
        return (int(s), int(e))


def gqf_insert_batch(slots, occ, run, offsets, stats, locks, q, r, max_occupied, use_locks, fps, deltas,
                     shift_out):
    """Insert a batch in input order; returns (code, fail_index), shift_out[0]
    accumulates moved slots (ck:1147-1202)."""
    n = len(fps)
    if n == 0:
        return GQF_OK, -1
    torch = _torch()
    lib = _lib.load()
    geom = _gqf_geom(q, r, len(slots), max_occupied)
    with _call_lock:
        img = _GqfImage(torch, slots, occ, run, offsets, stats, q)
        t = img.tables()
        dfp, dd = _dev(torch, _u64(fps)), _dev(torch, _u64(deltas))
        code, fail, sh = ctypes.c_int32(0), ctypes.c_int64(-1), ctypes.c_int64(0)
        _check(lib.fk_gqf_insert_batch(ctypes.byref(geom), ctypes.byref(t), _lib.dptr(dfp), _lib.dptr(dd), n,
                                       ctypes.byref(code), ctypes.byref(fail), ctypes.byref(sh), _stream(torch)),
               "gqf_insert_batch")
        img.write_back()
        shift_out[0] += sh.value
        return (int(code.value), int(fail.value)) if code.value else (GQF_OK, -1)


def gqf_count_batch(slots, occ, run, offsets, locks, q, r, use_locks, fps, counts):
    """Exact-or-over counts for a batch of fingerprints (ck:1205-1250)."""
    n = len(fps)
    if n == 0:
        return
    torch = _torch()
    lib = _lib.load()
    geom = _gqf_geom(q, r, len(slots))
    with _call_lock:
        img = _GqfImage(torch, slots, occ, run, offsets, None, q)
        t = img.tables()
        _check(lib.fk_gqf_rebuild_index(ctypes.byref(geom), ctypes.byref(t), _stream(torch)), "gqf_count_batch")
        dfp = _dev(torch, _u64(fps))
        dc = torch.empty(n, dtype=torch.int64, device="cuda")
        _check(lib.fk_gqf_count(ctypes.byref(geom), ctypes.byref(t), _lib.dptr(dfp), 1, n, _lib.dptr(dc),
                                _stream(torch)), "gqf_count_batch")
        _back(dc, counts)


def gqf_delete_batch(slots, occ, run, offsets, stats, locks, q, r, use_locks, fps, deltas, found, shift_out):
    """Delete a batch in input order; found flags per item, shift_out[0]
    accumulates moved slots; returns (0, -1) (ck:1253-1296)."""
    n = len(fps)
    if n == 0:
        return GQF_OK, -1
    torch = _torch()
    lib = _lib.load()
    geom = _gqf_geom(q, r, len(slots))
    with _call_lock:
        img = _GqfImage(torch, slots, occ, run, offsets, stats, q)
        t = img.tables()
        dfp, dd = _dev(torch, _u64(fps)), _dev(torch, _u64(deltas))
        dfound = torch.zeros(n, dtype=torch.uint8, device="cuda")
        sh = ctypes.c_int64(0)
        _check(lib.fk_gqf_delete_batch(ctypes.byref(geom), ctypes.byref(t), _lib.dptr(dfp), _lib.dptr(dd), n,
                                       _lib.dptr(dfound), ctypes.byref(sh), _stream(torch)), "gqf_delete_batch")
        img.write_back()
        _back(dfound, found)
        shift_out[0] += sh.value
        return GQF_OK, -1
