"""Hash-prefix sharding of the filters across GPUs (one process per GPU).

The reference is a single-process package; this is the new build's scale-out
path.  Each rank owns an independent sub-filter and every batch
call is: partition the rank's keys by owner (fk_shard_partition, a stable
device partition on a fingerprint prefix) -> an all-gather of the G per-owner
counts -> the keys move to their owners (by default the peer-memory dispatch
kernel, NVLink stores into the owners' buffers; FK_SHARD_PEER=0: one NCCL
all-to-all) -> the local sub-filter kernel on what arrived, in (source rank,
input index) order -> the per-key results move back (peer-memory combine or
the reverse all-to-all) -> fk_shard_unpermute back to input order.

* TCF: owner = top log2(G) bits of mix64(key ^ seed).  b1, b2, the tag and the
  backing schedule come from other hash streams, so shard s is exactly a
  ``Tcf(num_blocks / G)`` over the keys it owns.
* GQF: owner = top log2(G) bits of the q-bit quotient.  The shard's own
  ``Gqf(q - log2 G, r)`` sees the low q' + r fingerprint bits, so its counts
  (and every answer) equal a single global ``Gqf(q, r)``'s.

``world`` must be a power of two (1, 2, 4, 8).  ``_Router`` (the all-to-all
fallback) uses ``torch.distributed.all_to_all_single`` on the group's backend
(NCCL over NVLink on the B200 box).  ``_Router`` takes its partition / unpermute ops as
an object so that the exchange logic can be exercised with world_size-2
gloo on CPU (tests/test_sharding_cpu.py); the product ops are the CUDA
kernels and refuse non-CUDA tensors.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

__all__ = ["ShardedTcf", "ShardedBulkTcf", "ShardedGqf", "CudaShardOps"]


def _log2_exact(g):
    lg = int(g).bit_length() - 1
    if g < 1 or (1 << lg) != g:
        raise ValueError("the number of shards must be a power of two (got %d)" % g)
    return lg


class CudaShardOps:
    """Partition / unpermute through the C ABI (csrc/shard.cu)."""

    def __init__(self, torch):
        self.torch = torch
        self.lib = _lib.load()

    def partition(self, keys, vals, seed, shift, log2g):
        torch = self.torch
        if not keys.is_cuda:
            raise RuntimeError("sharded filters route CUDA tensors only (no CPU path)")
        n = keys.numel()
        dev = keys.device
        ko = torch.empty(n, dtype=torch.int64, device=dev)
        vo = torch.empty(n, dtype=torch.int64, device=dev) if vals is not None else None
        perm = torch.empty(n, dtype=torch.int32, device=dev)
        counts = torch.empty(1 << log2g, dtype=torch.int64, device=dev)
        _lib.check(self.lib.fk_shard_partition(_lib.dptr(keys), _lib.dptr(vals), n, seed & ((1 << 64) - 1), shift,
                                               log2g, _lib.dptr(ko), _lib.dptr(vo), _lib.dptr(perm),
                                               _lib.dptr(counts), _lib.stream_ptr(torch)), "shard partition")
        return ko, vo, perm, counts

    def partition_perm(self, keys, seed, shift, log2g):
        """Stable owner permutation and per-owner counts only (no gather)."""
        torch = self.torch
        n = keys.numel()
        perm = torch.empty(n, dtype=torch.int32, device=keys.device)
        counts = torch.empty(1 << log2g, dtype=torch.int64, device=keys.device)
        _lib.check(self.lib.fk_shard_partition(_lib.dptr(keys), None, n, seed & ((1 << 64) - 1), shift, log2g,
                                               None, None, _lib.dptr(perm), _lib.dptr(counts),
                                               _lib.stream_ptr(torch)), "shard partition")
        return perm, counts

    def unpermute(self, perm, src):
        torch = self.torch
        out = torch.empty_like(src)
        eb = src.element_size()
        _lib.check(self.lib.fk_shard_unpermute(_lib.dptr(perm), _lib.dptr(src), src.numel(), eb, _lib.dptr(out),
                                               _lib.stream_ptr(torch)), "shard unpermute")
        return out


class _Router:
    """Owner routing of one rank's batch and the way back (8(e) steps 1-5)."""

    def __init__(self, torch, group, world, seed, shift, ops):
        self.torch, self.group, self.world = torch, group, world
        self.log2g = _log2_exact(world)
        self.seed, self.shift, self.ops = seed, shift, ops
        self.stage = False  # gloo moves host tensors only: stage device buffers through the host
        if world > 1:
            import torch.distributed as dist
            self.stage = dist.get_backend(group) == "gloo"

    def _a2a(self, out, inp, out_splits=None, in_splits=None):
        import torch.distributed as dist
        if self.stage and inp.is_cuda:
            o = out.cpu()
            dist.all_to_all_single(o, inp.cpu(), out_splits, in_splits, group=self.group)
            out.copy_(o)
        else:
            dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)

    def route(self, keys, vals=None):
        """-> (keys that this rank owns, their values, plan for unroute)."""
        torch = self.torch
        if self.world == 1:
            return keys, vals, None
        import torch.distributed as dist
        ko, vo, perm, counts = self.ops.partition(keys, vals, self.seed, self.shift, self.log2g)
        rcounts = torch.empty_like(counts)
        self._a2a(rcounts, counts)
        send = counts.tolist()
        recv = rcounts.tolist()
        rk = torch.empty(sum(recv), dtype=keys.dtype, device=keys.device)
        self._a2a(rk, ko, recv, send)
        rv = None
        if vals is not None:
            rv = torch.empty(sum(recv), dtype=vals.dtype, device=vals.device)
            self._a2a(rv, vo, recv, send)
        return rk, rv, (perm, send, recv)

    def unroute(self, res, plan):
        """Per-key results for the keys this rank received -> results for this
        rank's own keys, in its input order."""
        if plan is None:
            return res
        perm, send, recv = plan
        back = self.torch.empty(sum(send), dtype=res.dtype, device=res.device)
        self._a2a(back, res.contiguous(), send, recv)
        return self.ops.unpermute(perm, back)

    def _coll_device(self):
        if self.stage or not self.torch.cuda.is_available():
            return "cpu"
        return "cuda"

    def any_flag(self, flag):
        """Max of a small int over ranks (error propagation after a batch)."""
        if self.world == 1:
            return int(flag)
        import torch.distributed as dist
        t = self.torch.tensor([int(flag)], dtype=self.torch.int64, device=self._coll_device())
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return int(t.item())

    def sum(self, values):
        if self.world == 1:
            return list(values)
        import torch.distributed as dist
        t = self.torch.tensor(list(values), dtype=self.torch.int64, device=self._coll_device())
        dist.all_reduce(t, group=self.group)
        return t.tolist()


class _PeerBuffers:
    """Device buffers every rank can store into: allocated whole (cudaMalloc)
    so a CUDA IPC handle covers them, the other ranks' buffers opened into
    this process (NVLink peer mappings).  Capacities grow by a decision every
    rank makes identically from the all-gathered count matrix, so sizing needs
    no extra collective; handles are exchanged only when they grow.  The flag
    words of the stream-ordered handoff (one u32 per source rank) are
    allocated once and never move."""

    NAMES = ("keys", "vals", "back")

    def __init__(self, torch, group, world, rank):
        self.torch, self.group, self.world, self.rank = torch, group, world, rank
        self.lib = _lib.load()
        self.cap = 0
        self.local = {}   # name -> own device pointer
        self.peers = {}   # name -> [pointer of rank r's buffer] (own included)
        self.tables = {}  # name -> int64 CUDA tensor of the pointers (kernel argument)

    def _close_peers(self, names):
        for name in names:
            for r, ptr in enumerate(self.peers.get(name, [])):
                if r != self.rank and ptr:
                    self.lib.fk_ipc_close(ctypes.c_void_p(ptr))
            self.peers.pop(name, None)
            self.tables.pop(name, None)

    def _free_local(self, names):
        for name in names:
            if self.local.get(name):
                self.lib.fk_ipc_free(ctypes.c_void_p(self.local.pop(name)))

    def _exchange(self, names, nbytes):
        """Allocate `names` (nbytes each), exchange handles, map the peers'."""
        import torch.distributed as dist
        torch = self.torch
        handles = {}
        for name in names:
            ptr = ctypes.c_void_p()
            _lib.check(self.lib.fk_ipc_alloc(nbytes, ctypes.byref(ptr)), "ipc alloc")
            self.local[name] = ptr.value
            h = ctypes.create_string_buffer(64)
            _lib.check(self.lib.fk_ipc_get_handle(ptr, h), "ipc handle")
            handles[name] = h.raw
        everyone = [None] * self.world
        dist.all_gather_object(everyone, handles, group=self.group)  # once per growth, not per batch
        ok = True
        for name in names:
            ptrs = []
            for r in range(self.world):
                if r == self.rank:
                    ptrs.append(self.local[name])
                    continue
                out = ctypes.c_void_p()
                h = ctypes.create_string_buffer(everyone[r][name], 64)
                if self.lib.fk_ipc_open(h, ctypes.byref(out)) != 0:
                    ok = False
                ptrs.append(out.value or 0)
            self.peers[name] = ptrs
            self.tables[name] = torch.tensor(ptrs, dtype=torch.int64, device="cuda")
        oks = [None] * self.world  # every rank must reach every other one, or nobody uses it
        dist.all_gather_object(oks, ok, group=self.group)
        return all(oks)

    def ensure(self, want):
        """Every rank calls it with the same `want` (items)."""
        import torch.distributed as dist
        if want <= self.cap:
            return
        cap = max(int(want), 2 * self.cap, 1 << 16)
        first = self.cap == 0
        if not first:
            # unmap the peers' old buffers everywhere before anyone frees its own
            self._close_peers(self.NAMES)
            dist.barrier(group=self.group)
            self._free_local(self.NAMES)
        ok = self._exchange(self.NAMES, cap * 8)
        if first and ok:
            ok = self._exchange(("flags",), 4 * self.world)
            if ok:
                self.view("flags", self.world, self.torch.int32).zero_()
                self.torch.cuda.current_stream().synchronize()
                dist.barrier(group=self.group)  # flags are zero before any peer signals
        if not ok:
            self.release()
            raise _NoPeerAccess()
        self.cap = cap

    def release(self):
        names = self.NAMES + ("flags",)
        self._close_peers(names)
        self._free_local(names)
        self.cap = 0

    def view(self, name, n, dtype):
        """This rank's own buffer `name` as a CUDA tensor of n items of dtype."""
        return _DevView.make(self.torch, self.local[name], n, dtype)

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


class _NoPeerAccess(RuntimeError):
    """Some rank could not map another rank's buffers (no CUDA IPC / P2P)."""


class _DevView:
    """A torch CUDA tensor over a raw device pointer (no ownership)."""

    @staticmethod
    def make(torch, ptr, n, dtype):
        itemsize = torch.empty(0, dtype=dtype).element_size()

        class _Iface:
            __cuda_array_interface__ = {"shape": (int(n),), "typestr": {1: "|u1", 4: "<i4", 8: "<i8"}[itemsize],
                                        "data": (int(ptr), False), "version": 3}
        t = torch.as_tensor(_Iface(), device="cuda")
        return t.view(dtype) if t.dtype != dtype else t


def exchange_plan(C, me):
    """Offsets of the peer exchange from the all-gathered count matrix
    C[source][owner] (int64 numpy), as rank `me` needs them: seg_start[o] (my
    owner-o group in my partitioned order), dst_off[o] (where it lands in
    owner o's receive buffer: after the earlier sources' groups), recv_off[s]
    (source s's run in my receive buffer, G+1 entries), back_off[s] (where my
    results for source s land in its partitioned order), and the buffer
    capacity every rank derives identically."""
    C = np.asarray(C, dtype=np.int64)
    G = C.shape[0]
    seg_start = np.concatenate(([0], np.cumsum(C[me])[:-1]))
    dst_off = (np.cumsum(C, axis=0) - C)[me]
    recv_off = np.concatenate(([0], np.cumsum(C[:, me])))
    back_off = (np.cumsum(C, axis=1) - C)[:, me]
    want = int(max(C.sum(axis=0).max(), C.sum(axis=1).max())) if G else 0
    return seg_start, dst_off, recv_off, back_off, want


class _PeerRouter(_Router):
    """Owner routing through peer memory instead of an all-to-all: the
    dispatch kernel stores every key (8 bytes) into its owner's receive
    buffer, the combine kernel stores every result into its source's return
    buffer in the source's owner-grouped order, and stream-ordered flag
    kernels hand the buffers over between GPUs.  Per batch: one all-gather of
    the G per-owner counts (a tensor collective) and one host synchronisation
    (to read them); no barriers."""

    WAIT_TIMEOUT_S = 120.0

    def __init__(self, torch, group, world, seed, shift, ops):
        super().__init__(torch, group, world, seed, shift, ops)
        import torch.distributed as dist
        self.rank = dist.get_rank(group)
        self.bufs = _PeerBuffers(torch, group, world, self.rank)
        self.fallback = False  # set collectively if peer mappings are unavailable
        self.epoch = 0

    def _handoff(self):
        """Stream-ordered: signal every peer that this rank's exchange stores
        are done, then wait until every peer signalled the same epoch."""
        self.epoch = (self.epoch + 1) & 0xFFFFFFFF
        lib, sp = self.ops.lib, _lib.stream_ptr(self.torch)
        _lib.check(lib.fk_shard_signal(_lib.dptr(self.bufs.tables["flags"]), self.log2g, self.rank, self.epoch, sp),
                   "shard signal")
        _lib.check(lib.fk_shard_wait(ctypes.c_void_p(self.bufs.local["flags"]), self.log2g, self.epoch,
                                     self.WAIT_TIMEOUT_S, sp), "shard wait")

    def route(self, keys, vals=None):
        torch = self.torch
        if self.world == 1:
            return keys, vals, None
        if self.fallback:
            return super().route(keys, vals)
        import torch.distributed as dist
        perm, counts = self.ops.partition_perm(keys, self.seed, self.shift, self.log2g)
        c = counts.to(self._coll_device())
        allc = [torch.empty_like(c) for _ in range(self.world)]
        dist.all_gather(allc, c, group=self.group)
        C = torch.stack(allc).cpu().numpy()  # the batch's one host synchronisation
        me = self.rank
        seg_start, dst_off, recv_off, back_off, want = exchange_plan(C, me)
        try:
            self.bufs.ensure(want)
        except _NoPeerAccess:  # collective decision: every rank falls back together
            self.fallback = True
            return super().route(keys, vals)
        recv_n = int(recv_off[-1])
        offs = torch.tensor(np.concatenate([seg_start, dst_off, recv_off, back_off]), dtype=torch.int64,
                            device=keys.device)
        G = self.world
        ss, do, ro, bo = offs[:G], offs[G:2 * G], offs[2 * G:3 * G + 1], offs[3 * G + 1:]
        t = self.bufs.tables
        _lib.check(self.ops.lib.fk_shard_dispatch(_lib.dptr(keys), _lib.dptr(vals), _lib.dptr(perm), keys.numel(),
                                                  self.seed & ((1 << 64) - 1), self.shift, self.log2g, _lib.dptr(ss),
                                                  _lib.dptr(do), _lib.dptr(t["keys"]),
                                                  _lib.dptr(t["vals"]) if vals is not None else None,
                                                  _lib.stream_ptr(torch)), "shard dispatch")
        self._handoff()  # every source's keys have landed in this rank's receive buffer
        rk = self.bufs.view("keys", recv_n, torch.int64)
        rv = self.bufs.view("vals", recv_n, torch.int64) if vals is not None else None
        return rk, rv, (perm, keys.numel(), recv_n, ro, bo)

    def unroute(self, res, plan):
        if plan is None:
            return res
        if self.fallback:
            return super().unroute(res, plan)
        torch = self.torch
        perm, n, recv_n, ro, bo = plan
        res = res.contiguous()
        _lib.check(self.ops.lib.fk_shard_combine(_lib.dptr(res), recv_n, res.element_size(), self.log2g,
                                                 _lib.dptr(ro), _lib.dptr(bo), _lib.dptr(self.bufs.tables["back"]),
                                                 _lib.stream_ptr(torch)), "shard combine")
        self._handoff()  # every owner has stored this rank's results
        return self.ops.unpermute(perm, self.bufs.view("back", n, res.dtype))


def failed_flags(torch, keys, failed):
    """Per-item failure flags (u8) for a batch whose failed keys came back as
    a multiset of values: a key that failed m times flags its LAST m copies
    (the local insert places the earlier copies of equal keys first), so
    duplicates where only some copies failed are not all reported."""
    flag = torch.zeros(keys.numel(), dtype=torch.uint8, device=keys.device)
    if failed.numel() == 0 or keys.numel() == 0:
        return flag
    uf, fcnt = torch.unique(failed, return_counts=True)
    order = torch.argsort(keys, stable=True)
    ks = keys[order]
    _, inv, gcnt = torch.unique_consecutive(ks, return_inverse=True, return_counts=True)
    gend = torch.cumsum(gcnt, 0)[inv]                      # one past each item's group end
    from_end = gend - 1 - torch.arange(ks.numel(), device=keys.device)
    pos = torch.searchsorted(uf, ks).clamp(max=uf.numel() - 1)
    m = torch.where(uf[pos] == ks, fcnt[pos], torch.zeros_like(fcnt[pos]))
    flag[order] = (from_end < m).to(torch.uint8)
    return flag


def _make_router(torch, group, world, seed, shift, ops):
    """The peer-memory router on CUDA groups of more than one rank (set
    FK_SHARD_PEER=0 for the all-to-all one); the all-to-all router otherwise
    (and for the host-side test doubles)."""
    import os
    if world > 1 and isinstance(ops, CudaShardOps) and os.environ.get("FK_SHARD_PEER", "1") != "0":
        return _PeerRouter(torch, group, world, seed, shift, ops)
    return _Router(torch, group, world, seed, shift, ops)


def _world(group):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def _as_device_keys(torch, keys, device):
    if isinstance(keys, torch.Tensor):
        return keys.reshape(-1).view(torch.int64).to(device), "cuda" if keys.is_cuda else "host"
    arr = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64).reshape(-1))
    return torch.from_numpy(arr.view(np.int64)).to(device), "numpy"


class _Sharded:
    def _init_common(self, group, ops):
        import torch
        self._torch = torch
        self.group = group
        self.world, self.rank = _world(group)
        self._ops = ops if ops is not None else CudaShardOps(torch)

    def _keys(self, keys):
        return _as_device_keys(self._torch, keys, self._local._device)


class ShardedTcf(_Sharded):
    """Point TCF over `world` GPUs: a global ``TcfParams`` (num_blocks divisible
    by the world size) split into per-rank ``Tcf(num_blocks / world)``."""

    def __init__(self, params=None, *, mode="ordered", group=None, ops=None, **kwargs):
        from .tcf import Tcf, TcfParams
        self._init_common(group, ops)
        if params is None:
            params = TcfParams(**kwargs)
        if params.num_blocks % self.world:
            raise ValueError("num_blocks must be divisible by the number of shards")
        self.params = params
        local = TcfParams(num_blocks=params.num_blocks // self.world, block_slots=params.block_slots,
                          tag_bits=params.tag_bits, slot_bits=params.slot_bits, seed=params.seed,
                          backing_fraction=params.backing_fraction, probe_limit=params.probe_limit,
                          shortcut_fraction=params.shortcut_fraction, group_width=params.group_width)
        self._local = Tcf(local, mode=mode)
        self.mode = mode
        lg = _log2_exact(self.world)
        self._router = _make_router(self._torch, group, self.world, params.seed, 64 - lg, self._ops)

    def _reset(self):
        self._local._reset()

    def _run(self, keys, fn, values=None):
        k, kind = self._keys(keys)
        v = None
        if values is not None:
            v, _ = _as_device_keys(self._torch, values, self._local._device)
        rk, rv, plan = self._router.route(k, v)
        res = fn(rk, rv)
        return self._router.unroute(res, plan), kind

    def insert_many(self, keys, values=None):
        out, kind = self._run(keys, lambda k, v: self._local.insert_many(k, v), values)
        return out if kind == "cuda" else out.cpu().numpy()

    def query_many(self, keys):
        out, kind = self._run(keys, lambda k, v: self._local.query_many(k).to(self._torch.uint8))
        return out.bool() if kind == "cuda" else out.cpu().numpy().astype(bool)

    def delete_many(self, keys):
        out, kind = self._run(keys, lambda k, v: self._local.delete_many(k).to(self._torch.uint8))
        return out.bool() if kind == "cuda" else out.cpu().numpy().astype(bool)

    @property
    def counters(self):
        c = self._local.counters
        tot = self._router.sum([c["inserts_ok"], c["inserts_backing"], c["deletes_ok"]])
        return {"inserts_ok": tot[0], "inserts_backing": tot[1], "deletes_ok": tot[2]}

    def load_factor(self):
        used = self._router.sum([int(round(self._local.load_factor() * self._local.params.main_slots))])[0]
        return used / self.params.main_slots


class ShardedBulkTcf(_Sharded):
    """Bulk TCF over `world` GPUs (per-rank ``BulkTcf(num_blocks / world)``).
    ``insert_batch`` returns this rank's keys that found no slot (in input
    order)."""

    def __init__(self, params=None, *, group=None, ops=None, **kwargs):
        from .tcf_bulk import BulkTcf, BulkTcfParams
        self._init_common(group, ops)
        if params is None:
            params = BulkTcfParams(**kwargs)
        if params.num_blocks % self.world:
            raise ValueError("num_blocks must be divisible by the number of shards")
        self.params = params
        local = BulkTcfParams(num_blocks=params.num_blocks // self.world, block_slots=params.block_slots,
                              tag_bits=params.tag_bits, seed=params.seed, backing_fraction=params.backing_fraction,
                              probe_limit=params.probe_limit, shortcut_fraction=params.shortcut_fraction)
        self._local = BulkTcf(local)
        lg = _log2_exact(self.world)
        self._router = _make_router(self._torch, group, self.world, params.seed, 64 - lg, self._ops)

    def _reset(self):
        self._local._reset()

    def insert_batch(self, keys, workers=1):
        torch = self._torch
        k, kind = self._keys(keys)
        rk, _, plan = self._router.route(k)
        failed = self._local.insert_batch(rk)
        flag = failed_flags(torch, rk, failed)
        mine = self._router.unroute(flag, plan).bool()
        out = k[mine]
        return out if kind == "cuda" else out.cpu().numpy().view(np.uint64)

    def query_batch(self, keys, workers=1):
        k, kind = self._keys(keys)
        rk, _, plan = self._router.route(k)
        out = self._router.unroute(self._local.query_batch(rk).to(self._torch.uint8), plan)
        return out.bool() if kind == "cuda" else out.cpu().numpy().astype(bool)

    def delete_batch(self, keys, workers=1):
        k, kind = self._keys(keys)
        rk, _, plan = self._router.route(k)
        out = self._router.unroute(self._local.delete_batch(rk).to(self._torch.uint8), plan)
        return out.bool() if kind == "cuda" else out.cpu().numpy().astype(bool)


class ShardedGqf(_Sharded):
    """GQF over `world` GPUs: a global ``GqfParams(q, r)`` split into per-rank
    ``Gqf(q - log2 world, r)`` by the top quotient bits; counts equal the
    global filter's.  A CapacityError on any shard is raised on every rank
    after the batch's reverse exchange."""

    def __init__(self, params=None, *, group=None, ops=None, **kwargs):
        from .gqf import Gqf, GqfParams
        self._init_common(group, ops)
        if params is None:
            params = GqfParams(**kwargs)
        lg = _log2_exact(self.world)
        if params.q - lg < 6:
            raise ValueError("q too small for %d shards" % self.world)
        self.params = params
        local = GqfParams(q=params.q - lg, r=params.r, seed=params.seed, max_load=params.max_load)
        self._local = Gqf(local)
        self._router = _make_router(self._torch, group, self.world, params.seed, local.q + params.r, self._ops)

    def _reset(self):
        self._local._reset()

    def _mutate(self, keys, counts, fn):
        from .errors import CapacityError
        torch = self._torch
        k, kind = self._keys(keys)
        c = None
        if counts is not None:
            c, _ = _as_device_keys(torch, counts, self._local._device)
        rk, rc, plan = self._router.route(k, c)
        err = None
        res = None
        try:
            res = fn(rk, rc)
        except CapacityError as e:
            err = e
        if res is None:
            res = torch.zeros(rk.numel(), dtype=torch.uint8, device=rk.device)
        out = self._router.unroute(res.to(torch.uint8), plan)
        if self._router.any_flag(err is not None):
            raise err if err is not None else CapacityError("capacity exceeded on another shard "
                                                            "(bulk batch partially applied)")
        return out, kind

    def bulk_insert(self, keys, counts=None, workers=4):
        self._mutate(keys, counts, lambda k, c: self._local.bulk_insert(k, c))

    def insert_many(self, keys, counts=None, workers=1):
        self._mutate(keys, counts, lambda k, c: self._local.insert_many(k, c))

    def bulk_delete(self, keys, counts=None, workers=4):
        out, kind = self._mutate(keys, counts, lambda k, c: self._local.bulk_delete(k, c))
        return out.bool() if kind == "cuda" else out.cpu().numpy().astype(bool)

    def delete_many(self, keys, counts=None, workers=1):
        out, kind = self._mutate(keys, counts, lambda k, c: self._local.delete_many(k, c))
        return out.bool() if kind == "cuda" else out.cpu().numpy().astype(bool)

    def count_many(self, keys, workers=1):
        k, kind = self._keys(keys)
        rk, _, plan = self._router.route(k)
        out = self._router.unroute(self._local.count_many(rk), plan)
        return out if kind == "cuda" else out.cpu().numpy().view(np.uint64)

    @property
    def total_items(self):
        return self._router.sum([self._local.total_items])[0]

    @property
    def distinct_items(self):
        return self._router.sum([self._local.distinct_items])[0]
