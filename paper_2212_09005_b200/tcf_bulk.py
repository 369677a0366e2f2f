"""Two-choice filter, bulk API, on the B200.

Drop-in for filterkit.tcf_bulk (/root/reference/pkg/src/filterkit/tcf_bulk.py:
43-374): same ``BulkTcfParams`` fields, validation and derivations, same
``BulkTcf`` methods (``insert_batch`` returns the failed keys, ``query_batch``
and ``delete_batch`` return per-key flags, ``partition``/``merge_block`` are
the public building blocks).  Blocks hold ``block_slots`` tag words sorted and
front-packed; the whole batch pipeline -- partition sort, shortcut merge,
two-choice routing, dest-grouped merge, backing overflow, 3-pass delete --
runs as sm_100a kernels behind the C ABI (csrc/tcf_bulk.cu).  Results are
bit-identical to the reference, whose routing is sequential and therefore
worker-invariant; ``workers=`` is accepted and ignored.

Inputs may be numpy arrays (results come back as numpy) or 64-bit CUDA
tensors (results stay on the device).
"""

from __future__ import annotations

import ctypes
import math
import threading
from dataclasses import dataclass

import numpy as np

from . import _device, _lib
from ._device import DeviceTables as _DeviceTables, check_backend as _check_backend, keys_in as _keys_in
from .errors import FilterFullError, ValidationError
from .hashing import EMPTY, TOMBSTONE

__all__ = ["BulkTcfParams", "BulkTcf"]

_NO_STATUS = 0xFFFFFFFF


@dataclass(frozen=True)
class BulkTcfParams:
    """Geometry for a bulk two-choice filter (tcf_bulk.py:43-77)."""

    num_blocks: int
    block_slots: int = 128
    tag_bits: int = 16
    seed: int = 0
    backing_fraction: float = 0.01
    probe_limit: int = 20
    shortcut_fraction: float = 0.75

    def __post_init__(self):
        if self.num_blocks < 1:
            raise ValueError("num_blocks must be positive")
        if self.block_slots < 2:
            raise ValueError("block_slots must be at least 2")
        if not 2 < self.tag_bits <= 32:
            raise ValueError("tag_bits must be in (2, 32]")
        if not 0.0 <= self.backing_fraction <= 1.0:
            raise ValueError("backing_fraction must be in [0, 1]")
        if not 0.0 < self.shortcut_fraction <= 1.0:
            raise ValueError("shortcut_fraction must be in (0, 1]")

    @property
    def main_slots(self):
        return self.num_blocks * self.block_slots

    @property
    def backing_slots(self):
        return int(round(self.main_slots * self.backing_fraction))  # tcf_bulk.py:71-72

    @property
    def cut_slots(self):
        return math.ceil(self.shortcut_fraction * self.block_slots)


def _dtype_for(bits):
    for dt in (np.uint8, np.uint16, np.uint32):
        if bits <= np.dtype(dt).itemsize * 8:
            return np.dtype(dt)
    raise ValueError("tag width over 32 bits")


class BulkTcf:
    """Two-choice filter driven by sorted batch operations (tcf_bulk.py:93)."""

    def __init__(self, params=None, *, backend="auto", device=None, **kwargs):
        if params is None:
            params = BulkTcfParams(**kwargs)
        elif kwargs:
            raise TypeError("pass either params or keyword fields, not both")
        _check_backend(backend)
        if params.block_slots > 8192:
            raise ValueError("block_slots > 8192 is not supported by the B200 build "
                             "(one block is staged in shared memory)")
        self.params = params
        torch = _lib.require_cuda(device)
        self._torch = torch
        self._device = torch.device(device) if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        self._lib = _lib.load()
        p = params
        dt = _dtype_for(p.tag_bits)
        self._dtype = dt
        self._t = _DeviceTables(torch, self._device, {
            "blocks": (dt, p.main_slots), "fill": (np.uint32, p.num_blocks),
            "backing": (dt, p.backing_slots)})
        self._counters_dev = torch.zeros(3, dtype=torch.int64, device=self._device)
        self._status = torch.empty(1, dtype=torch.int32, device=self._device)
        self._insert_res = torch.empty(2, dtype=torch.int64, device=self._device)
        self._geom = _lib.BtcfGeom(p.num_blocks, p.backing_slots, p.block_slots, p.tag_bits, dt.itemsize,
                                   p.cut_slots, p.probe_limit, 0, p.seed & ((1 << 64) - 1))
        self._op_lock = threading.Lock()

    @property
    def backend(self):
        return "cuda"

    # -- private host mirrors (reference tests read/mutate these) -----------
    @property
    def _blocks(self):
        return self._t.host("blocks")

    @property
    def _fill(self):
        return self._t.host("fill")

    @property
    def _backing(self):
        return self._t.host("backing")

    def _reset(self):
        """Zero every table and counter (benchmark helper; not in the reference API)."""
        with self._op_lock:
            self._t.zero()
            self._counters_dev.zero_()

    def _ptrs(self):
        return self._t.ptr("blocks"), self._t.ptr("fill"), self._t.ptr("backing")

    def _check_status(self, what):
        v = int(self._status.view(self._torch.int32).item()) & 0xFFFFFFFF
        if v != _NO_STATUS:
            raise AssertionError("%s overfilled block %d" % (what, v - 1))

    # -- batch building blocks ------------------------------------------------
    def _fps(self, keys):
        from .hashing import fingerprint_many
        return fingerprint_many(np.ascontiguousarray(keys, dtype=np.uint64), self.params.seed)

    def _words(self, fps):
        from .hashing import remap_tag_many
        return remap_tag_many(np.asarray(fps, dtype=np.uint64) & np.uint64((1 << self.params.tag_bits) - 1))

    def partition(self, keys):
        """Sort a batch by (primary block, tag word) on the device
        (tcf_bulk.py:123-143).  Returns numpy (block_ids, words, bounds,
        order) exactly as the reference."""
        torch = self._torch
        k, _ = _keys_in(torch, keys, self._device)
        n = k.numel()
        p = self.params
        sk = torch.empty(n, dtype=torch.int64, device=self._device)
        order = torch.empty(n, dtype=torch.int32, device=self._device)
        if n:
            _lib.check(self._lib.fk_btcf_partition(ctypes.byref(self._geom), _lib.dptr(k), 0, n, _lib.dptr(sk),
                                                   _lib.dptr(order), _lib.stream_ptr(torch)), "btcf partition")
        blk = sk >> p.tag_bits
        words = sk & ((1 << p.tag_bits) - 1)
        bounds = torch.searchsorted(blk.contiguous(), torch.arange(p.num_blocks + 1, device=self._device))
        return (blk.cpu().numpy(), words.cpu().numpy().astype(np.uint64), bounds.cpu().numpy().astype(np.int64),
                order.cpu().numpy().view(np.uint32).astype(np.int64))

    def merge_block(self, block_index, words):
        """Merge tag words into one block (public building block,
        tcf_bulk.py:145-162); raises FilterFullError when it cannot hold them."""
        torch = self._torch
        p = self.params
        w = np.sort(np.ascontiguousarray(words).astype(self._dtype))
        if int(self._t.peek("fill")[block_index]) + len(w) > p.block_slots:
            raise FilterFullError("block %d cannot take %d more words" % (block_index, len(w)))
        if not len(w):
            return
        wd = torch.from_numpy(w.astype(np.int64)).to(self._device)
        lo = torch.zeros(p.num_blocks, dtype=torch.int32, device=self._device)
        hi = torch.zeros(p.num_blocks, dtype=torch.int32, device=self._device)
        hi[block_index] = len(w)
        with self._op_lock:
            self._t.before_device_op()
            self._status.fill_(-1)
            b, f, _ = self._ptrs()
            _lib.check(self._lib.fk_btcf_merge_lists(ctypes.byref(self._geom), b, f, _lib.dptr(wd), _lib.dptr(lo),
                                                     _lib.dptr(hi), _lib.dptr(self._status),
                                                     _lib.stream_ptr(torch)), "btcf merge")
            self._t.after_device_write()
            v = int(self._status.item()) & 0xFFFFFFFF
        if v != _NO_STATUS:
            raise FilterFullError("block %d overflow" % (v - 1))

    # -- batch operations -------------------------------------------------------
    def insert_batch(self, keys, workers=1):
        """Insert a batch; returns the (possibly empty) array of failed keys
        (tcf_bulk.py:179-257), in the reference's order."""
        torch = self._torch
        k, kind = _keys_in(torch, keys, self._device)
        n = k.numel()
        if n == 0:
            return np.zeros(0, dtype=np.uint64) if kind == "numpy" else k[:0]
        failed = torch.empty(n, dtype=torch.int64, device=self._device)
        with self._op_lock:
            self._t.before_device_op()
            # [0] failure count (zeroed by the call), [1] status word (low half,
            # -1 = none): one fill before, one copy after
            res = self._insert_res
            res.fill_(-1)
            b, f, bk = self._ptrs()
            rc = self._lib.fk_btcf_insert(ctypes.byref(self._geom), b, f, bk, _lib.dptr(k), 0, n, _lib.dptr(failed),
                                          _lib.dptr(res), _lib.dptr(self._counters_dev), _lib.dptr(res[1:]),
                                          _lib.stream_ptr(torch))
            _lib.check(rc, "btcf insert")
            self._t.after_device_write()
            m, v = (int(x) for x in res.cpu())
            v &= 0xFFFFFFFF
            if v != _NO_STATUS:
                raise AssertionError("insert overfilled block %d" % (v - 1))
        out = failed[:m]
        if kind == "cuda":
            return out
        arr = out.cpu().numpy().view(np.uint64)
        return torch.from_numpy(arr.view(np.int64)) if kind == "host" else arr

    def query_batch(self, keys, workers=1):
        """Approximate membership per key (btcf_query_batch, ck:552-599)."""
        torch = self._torch
        k, kind = _keys_in(torch, keys, self._device)
        n = k.numel()
        found = torch.empty(n, dtype=torch.bool, device=self._device)  # the kernel writes 0/1 bytes
        if n:
            with self._op_lock:
                self._t.before_device_op()
                b, f, bk = self._ptrs()
                _lib.check(self._lib.fk_btcf_query(ctypes.byref(self._geom), b, f, bk, _lib.dptr(k), 0, n,
                                                   _lib.dptr(found), _lib.stream_ptr(torch)), "btcf query")
        if kind == "cuda":
            return found
        if kind == "host":
            return found.cpu()
        return found.cpu().numpy()

    def delete_batch(self, keys, workers=1):
        """Remove one stored copy per key; per-key success flags
        (tcf_bulk.py:283-325: primary blocks, secondary blocks, backing)."""
        torch = self._torch
        k, kind = _keys_in(torch, keys, self._device)
        n = k.numel()
        removed = torch.zeros(n, dtype=torch.bool, device=self._device)  # the kernels write 0/1 bytes
        if n:
            with self._op_lock:
                self._t.before_device_op()
                b, f, bk = self._ptrs()
                _lib.check(self._lib.fk_btcf_delete(ctypes.byref(self._geom), b, f, bk, _lib.dptr(k), 0, n,
                                                    _lib.dptr(removed), _lib.dptr(self._counters_dev),
                                                    _lib.stream_ptr(torch)), "btcf delete")
                self._t.after_device_write()
        if kind == "cuda":
            return removed
        if kind == "host":
            return removed.cpu()
        return removed.cpu().numpy()

    # -- inspection (quiescent; host mirrors) -----------------------------------
    def occupancy(self, block_index):
        return int(self._t.peek("fill")[block_index])

    def load_factor(self):
        return float(self._t.peek("fill").astype(np.int64).sum()) / self.params.main_slots

    def size_bits(self):
        p = self.params
        return (p.main_slots + p.backing_slots) * self._dtype.itemsize * 8 + p.num_blocks * 32

    @property
    def counters(self):
        c = self._counters_dev.cpu().tolist()
        return {"inserts_ok": int(c[0]), "inserts_backing": int(c[1]), "deletes_ok": int(c[2])}

    def items(self):
        """All stored (block_index, word) pairs; backing entries get -1
        (tcf_bulk.py:342-352).  Each block's filled prefix and the live
        backing slots are selected on the device (fk_live_slots)."""
        p = self.params
        with self._op_lock:
            self._t.before_device_op()
            bi, bw = _device.live_slots(self._torch, self._lib, self._t, "blocks", "fill", p.block_slots)
            ki, kw = _device.live_slots(self._torch, self._lib, self._t, "backing")
        out = list(zip((bi // p.block_slots).tolist(), [int(x) for x in bw.tolist()]))
        out.extend((-1, int(x)) for x in kw.tolist())
        return out

    _VMSG = ((1, "block %d fill over capacity"), (2, "block %d stores a reserved word"),
             (4, "block %d prefix not sorted"), (8, "block %d tail not empty"))

    def validate(self):
        """Sorted-block invariants (tcf_bulk.py:354-374), checked on the
        device (fk_btcf_validate); raises ValidationError.  On a violation,
        tables small enough for the host re-run the host checks so the
        message names the same first failure."""
        out = np.zeros(8, dtype=np.int64)
        with self._op_lock:
            self._t.before_device_op()
            b, f, bk = self._ptrs()
            _lib.check(self._lib.fk_btcf_validate(ctypes.byref(self._geom), b, f, bk,
                                                  out.ctypes.data_as(ctypes.c_void_p),
                                                  _lib.stream_ptr(self._torch)), "btcf validate")
        first = None
        for bit, msg in self._VMSG:
            if int(out[0]) & bit:
                first = msg % int(out[1 + bit.bit_length() - 1])
                break
        c = self.counters
        used = int(out[5]) + int(out[6])
        if first is None and used != c["inserts_ok"] - c["deletes_ok"]:
            first = "stored words (%d) do not match inserts-deletes (%d)" % (used, c["inserts_ok"] - c["deletes_ok"])
        if first is None:
            return
        if self.params.main_slots <= (1 << 22):
            self._validate_host()
        raise ValidationError(first)

    def _validate_host(self):
        """The reference's host checks over the mirrored image."""
        p = self.params
        B = p.block_slots
        blocks = self._t.peek("blocks").reshape(p.num_blocks, B)
        fill = self._t.peek("fill").astype(np.int64)
        if (fill > B).any():
            raise ValidationError("block %d fill over capacity" % int(np.flatnonzero(fill > B)[0]))
        idx = np.arange(B)[None, :]
        live = idx < fill[:, None]
        vals = blocks.astype(np.int64)
        bad = live & (vals < 2)
        if bad.any():
            raise ValidationError("block %d stores a reserved word" % int(np.flatnonzero(bad.any(1))[0]))
        unsorted = live[:, 1:] & (vals[:, 1:] < vals[:, :-1])
        if unsorted.any():
            raise ValidationError("block %d prefix not sorted" % int(np.flatnonzero(unsorted.any(1))[0]))
        tail = (~live) & (vals != EMPTY)
        if tail.any():
            raise ValidationError("block %d tail not empty" % int(np.flatnonzero(tail.any(1))[0]))
        bk = self._t.peek("backing")
        used = int(fill.sum()) + int(((bk != EMPTY) & (bk != TOMBSTONE)).sum())
        c = self.counters
        if used != c["inserts_ok"] - c["deletes_ok"]:
            raise ValidationError("stored words (%d) do not match inserts-deletes (%d)"
                                  % (used, c["inserts_ok"] - c["deletes_ok"]))
