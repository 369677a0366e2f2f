"""Device-resident table buffers with host mirrors, shared by the facades."""

from __future__ import annotations

import numpy as np

from . import _lib


def check_backend(backend):
    if backend not in ("auto", "cuda", "c"):
        if backend == "py":
            raise RuntimeError("the pure-Python backend does not exist in the B200 build")
        raise ValueError("unknown backend %r (expected 'auto' or 'cuda')" % (backend,))


class DeviceTables:
    """Named device byte buffers with lazily synced host mirrors.

    Reading ``_blocks`` & co. returns a host numpy copy (D2H on first access
    after a device write).  Tests in the reference mutate those arrays in
    place; a handed-out mirror is therefore pushed back (H2D)
    before the next device operation.
    """

    def __init__(self, torch, device, spec):
        self.torch, self.device = torch, device
        self.spec = dict(spec)  # name -> (dtype, count)
        self.dev = {n: torch.zeros(max(1, c * np.dtype(dt).itemsize), dtype=torch.uint8, device=device)
                    for n, (dt, c) in self.spec.items()}
        self.mirror = {}
        self.lent = set()

    def ptr(self, name):
        dt, c = self.spec[name]
        return _lib.dptr(self.dev[name]) if c else _lib.c_vp(0)

    def _fetch(self, name):
        if name not in self.mirror:
            dt, c = self.spec[name]
            self.mirror[name] = _lib.host_view(self.torch, self.dev[name], dt)[:c] if c else \
                np.zeros(0, dtype=dt)
        return self.mirror[name]

    def host(self, name):
        """The mutable mirror handed to callers (the reference's private
        arrays); it is pushed back before every later device operation."""
        m = self._fetch(name)
        self.lent.add(name)
        return m

    def peek(self, name):
        """Read-only view of the mirror for the facades' own inspection
        methods: not lent, so it never triggers a push-back."""
        v = self._fetch(name).view()
        v.flags.writeable = False
        return v

    def before_device_op(self):
        """Push handed-out mirrors back (they stay lent -- the caller may still
        hold and edit them -- until a device write replaces them); returns
        the set of names pushed."""
        pushed = set()
        for name in self.lent:
            dt, c = self.spec[name]
            if c:
                src = self.torch.from_numpy(np.ascontiguousarray(self.mirror[name]).view(np.uint8).copy())
                self.dev[name][: src.numel()].copy_(src.to(self.device))
                pushed.add(name)
        return pushed

    def zero(self):
        for t in self.dev.values():
            t.zero_()
        self.mirror.clear()
        self.lent.clear()

    def after_device_write(self):
        self.mirror.clear()
        self.lent.clear()


def live_slots(torch, lib, tables, name, fill_name=None, block_slots=1):
    """(positions, words) of the live slots of table `name`, selected on the
    device (fk_live_slots) so only the live entries cross to the host."""
    dt, c = tables.spec[name]
    if not c:
        return np.zeros(0, np.int64), np.zeros(0, dt)
    dev = tables.dev[name]
    idx = torch.empty(c, dtype=torch.int64, device=dev.device)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev.device)
    fill = _lib.dptr(tables.dev[fill_name]) if fill_name else None
    _lib.check(lib.fk_live_slots(_lib.dptr(dev), np.dtype(dt).itemsize, c, fill, block_slots, _lib.dptr(idx),
                                 _lib.dptr(cnt), _lib.stream_ptr(torch)), "live slots")
    m = int(cnt.item())
    idx = idx[:m]
    itemsize = np.dtype(dt).itemsize
    tdt = {1: torch.uint8, 2: torch.int16, 4: torch.int32, 8: torch.int64}[itemsize]
    words = dev[: c * itemsize].view(tdt)[idx]
    return idx.cpu().numpy(), words.cpu().numpy().view(dt)


def keys_in(torch, keys, device):
    """-> (device int64 tensor, kind): kind 'cuda' (results stay on device,
    asynchronous), 'host' (CPU torch tensor; results come back as CPU
    tensors) or 'numpy'."""
    if isinstance(keys, torch.Tensor):
        kind = "cuda" if keys.is_cuda else "host"
    else:
        kind = "numpy"
    return _lib.to_device_u64(torch, keys, device), kind


def ret(torch, t, kind):
    """Return a device result in the caller's flavour."""
    if kind == "cuda":
        return t
    if kind == "host":
        out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        out.copy_(t, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return out
    return t.cpu().numpy()
