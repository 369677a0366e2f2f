"""Two-choice filter, point API, on the B200.

Drop-in for filterkit.tcf (/root/reference/pkg/src/filterkit/tcf.py:31-249):
same ``Placement`` codes, ``TcfParams`` fields/validation/derivations, and
``Tcf`` methods.  Table state lives in HBM as torch CUDA tensors; every
insert/query/delete is one launch of the sm_100a kernels in
csrc/tcf_point*.cu through the C ABI (include/filterkit_b200.h).

Semantics of a batch call:

* ``mode="ordered"`` (default): the result -- codes, table bit image, query
  answers including false positives -- is bit-identical to the reference
  processing the batch from one caller thread (``tcf_insert_batch`` loop,
  _ckernels.pyx:210-237).
* ``mode="concurrent"``: the paper's free-threaded CAS insert (Alg. 1): the
  same placement policy applied by every key at once, i.e. the reference's
  behaviour under many concurrent caller threads.  Faster; the placement
  of keys that compete for a block is a race.

Inputs may be numpy arrays (synchronous, results come back as numpy) or
int64/uint64 CUDA tensors (asynchronous on the current stream, results stay
on the device).
"""

from __future__ import annotations

import math
import threading
from dataclasses import dataclass
from enum import IntEnum

import numpy as np

from . import _device, _lib
from ._device import DeviceTables as _DeviceTables, check_backend as _check_backend
from .errors import FilterFullError, ValidationError
from .hashing import EMPTY, TOMBSTONE

__all__ = ["Placement", "TcfParams", "Tcf"]


class Placement(IntEnum):
    """Where an insert landed (tcf.py:31-37)."""

    PRIMARY = 0
    SECONDARY = 1
    BACKING = 2
    FULL = 3


def _slot_dtype(bits):
    for dt in (np.uint8, np.uint16, np.uint32, np.uint64):
        if bits <= np.dtype(dt).itemsize * 8:
            return np.dtype(dt)
    raise ValueError("slot width over 64 bits")


@dataclass(frozen=True)
class TcfParams:
    """Geometry and hashing parameters (tcf.py:47-92, same defaults/checks)."""

    num_blocks: int
    block_slots: int = 16
    tag_bits: int = 16
    slot_bits: int = 16
    seed: int = 0
    backing_fraction: float = 0.01
    probe_limit: int = 20
    shortcut_fraction: float = 0.75
    group_width: int = 1

    def __post_init__(self):
        if self.num_blocks < 1:
            raise ValueError("num_blocks must be positive")
        if self.block_slots < 1:
            raise ValueError("block_slots must be positive")
        if not 2 < self.tag_bits <= self.slot_bits:
            raise ValueError("need 2 < tag_bits <= slot_bits")
        if self.block_slots * self.slot_bits > 1024:
            raise ValueError("block exceeds 1024 bits (block_slots * slot_bits)")
        if not 1 <= self.group_width <= self.block_slots:
            raise ValueError("group_width must be in [1, block_slots]")
        if not 0.0 <= self.backing_fraction <= 1.0:
            raise ValueError("backing_fraction must be in [0, 1]")
        if not 0.0 < self.shortcut_fraction <= 1.0:
            raise ValueError("shortcut_fraction must be in (0, 1]")

    @property
    def value_bits(self):
        return self.slot_bits - self.tag_bits

    @property
    def main_slots(self):
        return self.num_blocks * self.block_slots

    @property
    def backing_slots(self):
        # Python round() (half-to-even) on a float, exactly as tcf.py:86-87
        return int(round(self.main_slots * self.backing_fraction))

    @property
    def cut_slots(self):
        return math.ceil(self.shortcut_fraction * self.block_slots)

    @property
    def tile_width(self):
        """Cooperative-group tile the kernels use: group_width rounded down to
        a power of two (results never depend on it, _pykernels.py:86-91)."""
        g = 1
        while g * 2 <= min(self.group_width, 32):
            g *= 2
        return g


# ordered kernels index their input with 32 bits (fk_tcf_insert rejects
# n > 0xFFFFFFF0): longer ordered batches run as consecutive launches
_ORD_MAX_KEYS = 1 << 31

_MODES = {"ordered": _lib.FK_ORDERED, "concurrent": _lib.FK_CONCURRENT}


class Tcf:
    """Two-choice filter with point (per-key) operations on the B200."""

    def __init__(self, params=None, *, backend="auto", mode="ordered", device=None, **kwargs):
        if params is None:
            params = TcfParams(**kwargs)
        elif kwargs:
            raise TypeError("pass either params or keyword fields, not both")
        _check_backend(backend)
        if mode not in _MODES:
            raise ValueError("mode must be 'ordered' or 'concurrent'")
        self.params = params
        self.mode = mode
        p = params
        dt = _slot_dtype(p.slot_bits)
        if p.block_slots * dt.itemsize * 8 > 1024:
            # The reference bounds block_slots * slot_bits (tcf.py:61-75); the
            # kernels hold a block in at most 1024 bits of *storage* words
            # (slot_bits=12 is stored as uint16), so reject it here, not at
            # the first operation.
            raise ValueError(
                "block_slots * storage bits = %d * %d exceeds the 1024-bit block the B200 kernels hold "
                "(slot_bits=%d is stored as %s)" % (p.block_slots, dt.itemsize * 8, p.slot_bits, dt.name))
        torch = _lib.require_cuda(device)
        self._torch = torch
        self._device = torch.device(device) if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        self._lib = _lib.load()
        self._dtype = dt
        self._t = _DeviceTables(torch, self._device, {
            "blocks": (dt, p.main_slots), "backing": (dt, p.backing_slots)})
        self._counters_dev = torch.zeros(3, dtype=torch.int64, device=self._device)
        self._geom = _lib.TcfGeom(p.num_blocks, p.backing_slots, p.block_slots, p.tag_bits,
                                  dt.itemsize, p.cut_slots, p.probe_limit, p.tile_width,
                                  p.seed & ((1 << 64) - 1))
        self._op_lock = threading.Lock()
        self._pipe = None  # HostPipeline, created on the first large host-side batch

    def _pipe_wants(self, keys):
        from ._pipeline import PIPE_CHUNK
        if self._kind(keys) == "cuda":
            return False
        n = keys.numel() if isinstance(keys, self._torch.Tensor) else len(keys)
        return n >= 2 * (self._pipe.chunk if self._pipe is not None else PIPE_CHUNK)

    @property
    def backend(self):
        return "cuda"

    # -- private host mirrors (reference tests read/mutate these) -----------
    @property
    def _blocks(self):
        return self._t.host("blocks")

    @property
    def _backing(self):
        return self._t.host("backing")

    # -- plumbing -------------------------------------------------------------
    def _keys_in(self, keys):
        """-> (device int64 tensor, kind); kind is 'cuda' (results stay on the
        device, asynchronous), 'host' (a CPU torch tensor, e.g. pinned: results
        come back as CPU tensors) or 'numpy'."""
        torch = self._torch
        if isinstance(keys, torch.Tensor):
            kind = "cuda" if keys.is_cuda else "host"
        else:
            kind = "numpy"
        return _lib.to_device_u64(torch, keys, self._device), kind

    def _kind(self, keys):
        torch = self._torch
        if isinstance(keys, torch.Tensor):
            return "cuda" if keys.is_cuda else "host"
        return "numpy"

    def _pipelined(self, keys, op, out_dtype):
        """Host-resident batch through the chunked H2D / kernel / D2H pipeline
        (_pipeline.py); returns results in the caller's kind."""
        torch = self._torch
        from ._pipeline import HostPipeline
        if self._pipe is None:
            self._pipe = HostPipeline(torch, self._device)
        kind = self._kind(keys)
        if kind == "host":
            hk = keys.reshape(-1)
            hk = hk.view(torch.int64) if hk.dtype in (torch.int64, torch.uint64) else hk.to(torch.int64)
        else:
            hk = torch.from_numpy(np.ascontiguousarray(np.asarray(keys, dtype=np.uint64).reshape(-1))
                                  .view(np.int64))
        mode = _MODES[self.mode]
        geom, lib = ctypes_byref(self._geom), self._lib
        with self._op_lock:
            self._t.before_device_op()
            ws, wsb = self._workspace(min(hk.numel(), self._pipe.chunk), mode) if op != "query" else (None, 0)

            def launch(din, dout):
                k, o, m = din[0], dout[0], din[0].numel()
                sp = _lib.stream_ptr(torch)
                if op == "insert":
                    rc = lib.fk_tcf_insert(geom, self._t.ptr("blocks"), self._t.ptr("backing"), _lib.dptr(k), 0,
                                           None, m, _lib.dptr(o), _lib.dptr(self._counters_dev), mode,
                                           _lib.dptr(ws), wsb, sp)
                elif op == "delete":
                    rc = lib.fk_tcf_delete(geom, self._t.ptr("blocks"), self._t.ptr("backing"), _lib.dptr(k), 0,
                                           m, _lib.dptr(o), _lib.dptr(self._counters_dev), mode, _lib.dptr(ws),
                                           wsb, sp)
                else:
                    rc = lib.fk_tcf_query(geom, self._t.ptr("blocks"), self._t.ptr("backing"), _lib.dptr(k), 0,
                                          m, _lib.dptr(o), None, sp)
                _lib.check(rc, "tcf " + op)

            out, = self._pipe.run([hk], [out_dtype], launch)
            if op != "query":
                self._t.after_device_write()
        return out if kind == "host" else out.numpy()

    def _ret(self, t, kind):
        if kind == "cuda":
            return t
        if kind == "host":
            out = self._torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            out.copy_(t, non_blocking=True)
            self._torch.cuda.current_stream().synchronize()
            return out
        return t.cpu().numpy()

    def _reset(self):
        """Zero every table and counter (benchmark helper; not in the reference API)."""
        with self._op_lock:
            for t in self._t.dev.values():
                t.zero_()
            self._counters_dev.zero_()
            self._t.mirror.clear()
            self._t.lent.clear()

    def _check_values(self, values, n, on_dev):
        torch = self._torch
        if values is None:
            return None
        vb = self.params.value_bits
        if isinstance(values, torch.Tensor):
            v = _lib.to_device_u64(torch, values, self._device)
            if v.numel() != n:
                raise ValueError("values length does not match keys length")
            if vb < 64 and n:
                bad = (v.view(torch.int64) >> vb) != 0 if vb > 0 else v != 0
                if bool(bad.any()):
                    raise ValueError("value does not fit in %d bits" % vb)
            return v
        vals = np.ascontiguousarray(values, dtype=np.uint64).reshape(-1)
        if len(vals) != n:
            raise ValueError("values length does not match keys length")
        if vb < 64 and len(vals) and int(vals.max()) >> vb:
            raise ValueError("value does not fit in %d bits" % vb)
        return _lib.to_device_u64(torch, vals, self._device)

    def _workspace(self, n, mode):
        nbytes = self._lib.fk_tcf_workspace_bytes(ctypes_byref(self._geom), n, mode)
        if not nbytes:
            return None, 0
        return self._torch.empty(nbytes, dtype=self._torch.uint8, device=self._device), nbytes

    # -- point operations -------------------------------------------------------
    def insert(self, key, value=0):
        code = int(self.insert_many([key], [value])[0])
        if code == Placement.FULL:
            raise FilterFullError("no free slot in either block or backing table")
        return Placement(code)

    def insert_many(self, keys, values=None):
        """Insert a batch; returns a Placement code per key (no raise)."""
        torch = self._torch
        if values is None and self._pipe_wants(keys):
            return self._pipelined(keys, "insert", torch.uint8)
        k, on_dev = self._keys_in(keys)
        n = k.numel()
        v = self._check_values(values, n, on_dev)
        codes = torch.empty(n, dtype=torch.uint8, device=self._device)
        if n:
            mode = _MODES[self.mode]
            step = _ORD_MAX_KEYS if self.mode == "ordered" else n
            with self._op_lock:
                self._t.before_device_op()
                ws, wsb = self._workspace(min(n, step), mode)
                # ordered batches past the kernels' 32-bit input index run as
                # consecutive launches (in order: the same sequential result)
                for lo in range(0, n, step):
                    m = min(step, n - lo)
                    rc = self._lib.fk_tcf_insert(
                        ctypes_byref(self._geom), self._t.ptr("blocks"), self._t.ptr("backing"),
                        _lib.dptr(k[lo:lo + m]), 0, _lib.dptr(v[lo:lo + m] if v is not None else None), m,
                        _lib.dptr(codes[lo:lo + m]), _lib.dptr(self._counters_dev), mode, _lib.dptr(ws), wsb,
                        _lib.stream_ptr(torch))
                    _lib.check(rc, "tcf insert")
                self._t.after_device_write()
        return self._ret(codes, on_dev)

    def query(self, key):
        return bool(self.query_many([key])[0])

    def query_value(self, key):
        found, values = self.query_values_many([key])
        return bool(found[0]), int(values[0])

    def query_many(self, keys):
        if self._pipe_wants(keys):
            return self._pipelined(keys, "query", self._torch.bool)
        return self._query(keys, False)[0]

    def query_values_many(self, keys):
        return self._query(keys, True)

    def _query(self, keys, want_values):
        torch = self._torch
        k, on_dev = self._keys_in(keys)
        n = k.numel()
        found = torch.empty(n, dtype=torch.bool, device=self._device)  # the kernel writes 0/1 bytes
        vals = torch.empty(n if want_values else 0, dtype=torch.int64, device=self._device)
        if n:
            with self._op_lock:
                self._t.before_device_op()
                rc = self._lib.fk_tcf_query(
                    ctypes_byref(self._geom), self._t.ptr("blocks"), self._t.ptr("backing"),
                    _lib.dptr(k), 0, n, _lib.dptr(found), _lib.dptr(vals), _lib.stream_ptr(torch))
                _lib.check(rc, "tcf query")
        if on_dev == "cuda":
            return found, (vals if want_values else None)
        if on_dev == "host":
            return self._ret(found, "host"), (self._ret(vals, "host") if want_values else None)
        return found.cpu().numpy(), (vals.cpu().numpy().view(np.uint64) if want_values else None)

    def delete(self, key):
        return bool(self.delete_many([key])[0])

    def delete_many(self, keys):
        torch = self._torch
        if self._pipe_wants(keys):
            return self._pipelined(keys, "delete", torch.bool)
        k, on_dev = self._keys_in(keys)
        n = k.numel()
        removed = torch.empty(n, dtype=torch.bool, device=self._device)  # the kernels write 0/1 bytes
        if n:
            mode = _MODES[self.mode]
            step = _ORD_MAX_KEYS if self.mode == "ordered" else n
            with self._op_lock:
                self._t.before_device_op()
                ws, wsb = self._workspace(min(n, step), mode)
                for lo in range(0, n, step):
                    m = min(step, n - lo)
                    rc = self._lib.fk_tcf_delete(
                        ctypes_byref(self._geom), self._t.ptr("blocks"), self._t.ptr("backing"),
                        _lib.dptr(k[lo:lo + m]), 0, m, _lib.dptr(removed[lo:lo + m]),
                        _lib.dptr(self._counters_dev), mode, _lib.dptr(ws), wsb, _lib.stream_ptr(torch))
                    _lib.check(rc, "tcf delete")
                self._t.after_device_write()
        if on_dev == "cuda":
            return removed
        if on_dev == "host":
            return self._ret(removed, "host")
        return removed.cpu().numpy()

    # -- inspection (quiescent; host mirrors) ------------------------------------
    def items(self):
        """All stored (block_index, tag, value) triples, backing entries with
        block_index -1 (tcf.py:196-208); the live slots are selected on the
        device (fk_live_slots), only they cross to the host."""
        p = self.params
        fmask = (1 << p.tag_bits) - 1
        with self._op_lock:
            self._t.before_device_op()
            bi, bw = _device.live_slots(self._torch, self._lib, self._t, "blocks")
            ki, kw = _device.live_slots(self._torch, self._lib, self._t, "backing")
        out = []
        for idx, words, main in ((bi, bw, True), (ki, kw, False)):
            w = [int(x) for x in words.tolist()]
            blk = (idx // p.block_slots).tolist() if main else [-1] * len(w)
            out.extend((b, x & fmask, x >> p.tag_bits) for b, x in zip(blk, w))
        return out

    def occupancy(self, block_index):
        p = self.params
        blk = self._t.peek("blocks")[block_index * p.block_slots:(block_index + 1) * p.block_slots]
        return int((blk > TOMBSTONE).sum())

    def _census(self):
        """(live main, reserved-tag main, live backing, reserved-tag backing),
        counted on the device (fk_tcf_census)."""
        out = np.zeros(4, dtype=np.int64)
        with self._op_lock:
            self._t.before_device_op()
            _lib.check(self._lib.fk_tcf_census(ctypes_byref(self._geom), self._t.ptr("blocks"),
                                               self._t.ptr("backing"), out.ctypes.data_as(_ctypes_vp()),
                                               _lib.stream_ptr(self._torch)), "tcf census")
        return [int(x) for x in out]

    def load_factor(self):
        return self._census()[0] / self.params.main_slots

    def size_bits(self):
        p = self.params
        return (p.main_slots + p.backing_slots) * self._dtype.itemsize * 8

    @property
    def counters(self):
        c = self._counters_dev.cpu().tolist()
        return {"inserts_ok": int(c[0]), "inserts_backing": int(c[1]), "deletes_ok": int(c[2])}

    def validate(self):
        """Structural invariants (tcf.py:232-249) from a device census;
        raises ValidationError."""
        live_m, bad_m, live_b, bad_b = self._census()
        for name, bad in (("main", bad_m), ("backing", bad_b)):
            if bad:
                raise ValidationError("%s table holds a used slot with a reserved tag" % name)
        used_total = live_m + live_b
        c = self.counters
        expect = c["inserts_ok"] - c["deletes_ok"]
        if used_total != expect:
            raise ValidationError("stored slots (%d) do not match inserts-deletes (%d)"
                                  % (used_total, expect))


def ctypes_byref(x):
    import ctypes
    return ctypes.byref(x)


def _ctypes_vp():
    import ctypes
    return ctypes.c_void_p
