"""Hash-prefix sharding of the filters across GPUs (one process per GPU).

The reference is a single-process package; this is the new build's scale-out
path.  Each rank owns an independent sub-filter and every batch
call is: partition the rank's keys by owner (fk_shard_partition, a stable
device partition on a fingerprint prefix) -> one NCCL all-to-all of the keys
(after a G-int count exchange) -> the local sub-filter kernel on what arrived,
in (source rank, input index) order -> the reverse all-to-all of the per-key
results -> fk_shard_unpermute back to input order.  There is no other
data-path collective.

* TCF: owner = top log2(G) bits of mix64(key ^ seed).  b1, b2, the tag and the
  backing schedule come from other hash streams, so shard s is exactly a
  ``Tcf(num_blocks / G)`` over the keys it owns.
* GQF: owner = top log2(G) bits of the q-bit quotient.  The shard's own
  ``Gqf(q - log2 G, r)`` sees the low q' + r fingerprint bits, so its counts
  (and every answer) equal a single global ``Gqf(q, r)``'s.

``world`` must be a power of two (1, 2, 4, 8).  The exchange uses
``torch.distributed.all_to_all_single`` on the group's backend (NCCL over
NVLink on the B200 box).  ``_Router`` takes its partition / unpermute ops as
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
    so a CUDA IPC handle covers them, handles exchanged once per growth, the
    other ranks' buffers opened into this process (NVLink peer mappings)."""

    NAMES = ("keys", "vals", "src", "out")

    def __init__(self, torch, group, world, rank):
        self.torch, self.group, self.world, self.rank = torch, group, world, rank
        self.lib = _lib.load()
        self.cap = 0
        self.local = {}   # name -> own device pointer
        self.peers = {}   # name -> [pointer of rank r's buffer] (own included)
        self.tables = {}  # name -> int64 CUDA tensor of the pointers (kernel argument)

    def _free(self):
        for name in self.NAMES:
            for r, ptr in enumerate(self.peers.get(name, [])):
                if r != self.rank and ptr:
                    self.lib.fk_ipc_close(ctypes.c_void_p(ptr))
            if self.local.get(name):
                self.lib.fk_ipc_free(ctypes.c_void_p(self.local[name]))
        self.local, self.peers, self.tables = {}, {}, {}

    def ensure(self, need):
        """Collective: every rank calls it with its own need (items)."""
        import torch.distributed as dist
        torch = self.torch
        objs = [None] * self.world
        dist.all_gather_object(objs, int(need), group=self.group)
        want = max(objs)
        if want <= self.cap:
            return
        cap = max(want, 2 * self.cap, 1 << 16)
        self._free()
        handles = {}
        for name in self.NAMES:
            ptr = ctypes.c_void_p()
            _lib.check(self.lib.fk_ipc_alloc(cap * 8, ctypes.byref(ptr)), "ipc alloc")
            self.local[name] = ptr.value
            h = ctypes.create_string_buffer(64)
            _lib.check(self.lib.fk_ipc_get_handle(ptr, h), "ipc handle")
            handles[name] = h.raw
        everyone = [None] * self.world
        dist.all_gather_object(everyone, handles, group=self.group)
        ok = True
        for name in self.NAMES:
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
        # every rank must be able to reach every other one, or nobody uses it
        oks = [None] * self.world
        dist.all_gather_object(oks, ok, group=self.group)
        if not all(oks):
            self._free()
            raise _NoPeerAccess()
        self.cap = cap

    def view(self, name, n, dtype):
        """This rank's own buffer `name` as a CUDA tensor of n items of dtype."""
        return _DevView.make(self.torch, self.local[name], n, dtype)

    def __del__(self):
        try:
            self._free()
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
            __cuda_array_interface__ = {"shape": (int(n),), "typestr": {1: "|u1", 8: "<i8"}[itemsize],
                                        "data": (int(ptr), False), "version": 3}
        t = torch.as_tensor(_Iface(), device="cuda")
        return t.view(dtype) if t.dtype != dtype else t


class _PeerRouter(_Router):
    """Owner routing through peer memory instead of an all-to-all: the
    dispatch kernel stores every key into its owner's receive buffer, the
    combine kernel stores every result into its source rank's output buffer
    (fk_shard_dispatch / fk_shard_combine).  Only per-owner counts (G ints)
    and a barrier per direction go through torch.distributed."""

    def __init__(self, torch, group, world, seed, shift, ops):
        super().__init__(torch, group, world, seed, shift, ops)
        import torch.distributed as dist
        self.rank = dist.get_rank(group)
        self.bufs = _PeerBuffers(torch, group, world, self.rank)
        self.fallback = False  # set collectively if peer mappings are unavailable

    def _barrier(self):
        import torch.distributed as dist
        self.torch.cuda.current_stream().synchronize()
        dist.barrier(group=self.group)

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
        C = np.array([a.tolist() for a in allc], dtype=np.int64)  # C[source][owner]
        me = self.rank
        recv_n = int(C[:, me].sum())
        try:
            self.bufs.ensure(max(recv_n, keys.numel()))
        except _NoPeerAccess:  # collective decision: every rank falls back together
            self.fallback = True
            return super().route(keys, vals)
        seg_start = np.concatenate(([0], np.cumsum(C[me])[:-1]))
        dst_off = np.cumsum(C, axis=0) - C  # rows above: earlier source ranks
        dev = keys.device
        ss = torch.tensor(seg_start, dtype=torch.int64, device=dev)
        do = torch.tensor(dst_off[me], dtype=torch.int64, device=dev)
        t = self.bufs.tables
        lib = self.ops.lib
        _lib.check(lib.fk_shard_dispatch(_lib.dptr(keys), _lib.dptr(vals), _lib.dptr(perm), keys.numel(),
                                         self.seed & ((1 << 64) - 1), self.shift, self.log2g, me, _lib.dptr(ss),
                                         _lib.dptr(do), _lib.dptr(t["keys"]),
                                         _lib.dptr(t["vals"]) if vals is not None else None, _lib.dptr(t["src"]),
                                         _lib.stream_ptr(torch)), "shard dispatch")
        self._barrier()  # every rank's keys have landed in its owners' buffers
        rk = self.bufs.view("keys", recv_n, torch.int64)
        rv = self.bufs.view("vals", recv_n, torch.int64) if vals is not None else None
        return rk, rv, (keys.numel(), recv_n)

    def unroute(self, res, plan):
        if plan is None:
            return res
        if self.fallback:
            return super().unroute(res, plan)
        torch = self.torch
        n, recv_n = plan
        res = res.contiguous()
        eb = res.element_size()
        src = self.bufs.view("src", recv_n, torch.int64)
        _lib.check(self.ops.lib.fk_shard_combine(_lib.dptr(src), _lib.dptr(res), recv_n, eb,
                                                 _lib.dptr(self.bufs.tables["out"]), _lib.stream_ptr(torch)),
                   "shard combine")
        self._barrier()  # every owner has stored this rank's results
        return self.bufs.view("out", n, res.dtype).clone()


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
        flag = torch.isin(rk, failed).to(torch.uint8) if failed.numel() else \
            torch.zeros(rk.numel(), dtype=torch.uint8, device=rk.device)
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
