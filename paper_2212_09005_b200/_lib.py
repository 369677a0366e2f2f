"""ctypes binding of libfkb200.so (the C ABI in include/filterkit_b200.h).

The product path has exactly one backend: these sm_100a kernels.  If the
library or a CUDA device is missing, every filter constructor raises
immediately -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfkb200.so")

FK_ORDERED, FK_CONCURRENT = 0, 1
FK_E_INVARIANT = -9
FK_E_ARG = -1000

c_i64, c_i32, c_u64, c_vp, c_sz = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_size_t


class TcfGeom(ctypes.Structure):
    _fields_ = [("num_blocks", c_i64), ("backing_slots", c_i64), ("block_slots", c_i32),
                ("tag_bits", c_i32), ("slot_bytes", c_i32), ("cut_slots", c_i32),
                ("probe_limit", c_i32), ("group_width", c_i32), ("seed", c_u64)]


class BtcfGeom(ctypes.Structure):
    _fields_ = [("num_blocks", c_i64), ("backing_slots", c_i64), ("block_slots", c_i32),
                ("tag_bits", c_i32), ("slot_bytes", c_i32), ("cut_slots", c_i32),
                ("probe_limit", c_i32), ("reserved", c_i32), ("seed", c_u64)]


class GqfGeom(ctypes.Structure):
    _fields_ = [("q", c_i32), ("r", c_i32), ("phys", c_i64), ("num_regions", c_i64),
                ("quotient_regions", c_i64), ("max_occupied", c_i64), ("seed", c_u64)]


class GqfTables(ctypes.Structure):
    _fields_ = [("slots", c_vp), ("occupieds", c_vp), ("runends", c_vp), ("offsets", c_vp),
                ("stats", c_vp), ("spill", c_vp)]


class GqfResult(ctypes.Structure):
    _fields_ = [("code", c_i32), ("swapped", c_i32), ("fail_index", c_i64), ("fail_region", c_i64),
                ("shifted", c_i64)]


FK_GQF_INSERT, FK_GQF_DELETE = 0, 1
FK_ORDER_POINT, FK_ORDER_BULK = 0, 1

_SIGS = {
    "fk_version": (ctypes.c_char_p, []),
    "fk_abi_version": (c_i32, []),
    "fk_device_setup": (c_i32, [c_i32]),
    "fk_device_l2_fetch_bytes": (c_i32, []),
    "fk_hash_streams": (c_i32, [c_vp, c_i64, c_u64, c_i32, c_u64, c_u64, c_vp, c_vp]),
    "fk_sector_gather": (c_i32, [c_vp, c_i64, c_i64, c_u64, c_vp, c_vp]),
    "fk_sector_rmw": (c_i32, [c_vp, c_i64, c_i64, c_u64, c_vp]),
    "fk_fastmod_check": (c_i32, [c_vp, c_i64, c_u64, c_vp, c_vp]),
    "fk_counter_stream": (c_i32, [c_u64, c_u64, c_u64, c_i64, c_vp, c_vp]),
    "fk_tcf_workspace_bytes": (c_sz, [ctypes.POINTER(TcfGeom), c_i64, c_i32]),
    "fk_tcf_insert": (c_i32, [ctypes.POINTER(TcfGeom), c_vp, c_vp, c_vp, c_i32, c_vp, c_i64, c_vp,
                              c_vp, c_i32, c_vp, c_sz, c_vp]),
    "fk_tcf_census": (c_i32, [ctypes.POINTER(TcfGeom), c_vp, c_vp, c_vp, c_vp]),
    "fk_tcf_query": (c_i32, [ctypes.POINTER(TcfGeom), c_vp, c_vp, c_vp, c_i32, c_i64, c_vp, c_vp, c_vp]),
    "fk_tcf_delete": (c_i32, [ctypes.POINTER(TcfGeom), c_vp, c_vp, c_vp, c_i32, c_i64, c_vp, c_vp,
                              c_i32, c_vp, c_sz, c_vp]),
    "fk_btcf_insert": (c_i32, [ctypes.POINTER(BtcfGeom), c_vp, c_vp, c_vp, c_vp, c_i32, c_i64, c_vp, c_vp,
                               c_vp, c_vp, c_vp]),
    "fk_btcf_validate": (c_i32, [ctypes.POINTER(BtcfGeom), c_vp, c_vp, c_vp, c_vp, c_vp]),
    "fk_btcf_query": (c_i32, [ctypes.POINTER(BtcfGeom), c_vp, c_vp, c_vp, c_vp, c_i32, c_i64, c_vp, c_vp]),
    "fk_btcf_delete": (c_i32, [ctypes.POINTER(BtcfGeom), c_vp, c_vp, c_vp, c_vp, c_i32, c_i64, c_vp, c_vp,
                               c_vp]),
    "fk_btcf_partition": (c_i32, [ctypes.POINTER(BtcfGeom), c_vp, c_i32, c_i64, c_vp, c_vp, c_vp]),
    "fk_btcf_merge_lists": (c_i32, [ctypes.POINTER(BtcfGeom), c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "fk_btcf_route": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "fk_btcf_merge_words": (c_i32, [ctypes.POINTER(BtcfGeom), c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_i64,
                                    ctypes.POINTER(c_i64), c_vp]),
    "fk_btcf_delete_blocklocal": (c_i32, [ctypes.POINTER(BtcfGeom), c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_i64,
                                          c_i64, c_vp, ctypes.POINTER(c_i64), c_vp]),
    "fk_backing_insert_batch": (c_i32, [ctypes.POINTER(BtcfGeom), c_vp, c_vp, c_i64, c_vp, ctypes.POINTER(c_i64),
                                        c_vp]),
    "fk_backing_delete_batch": (c_i32, [ctypes.POINTER(BtcfGeom), c_vp, c_vp, c_i64, c_vp, ctypes.POINTER(c_i64),
                                        c_vp]),
    "fk_gqf_cluster_stats": (c_i32, [ctypes.POINTER(GqfGeom), ctypes.POINTER(GqfTables), c_vp, c_vp]),
    "fk_kmer_windows": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_vp, c_vp]),
    "fk_pcg64_raw": (c_i32, [c_u64, c_u64, c_u64, c_u64, c_u64, c_i64, c_vp, c_vp]),
    "fk_bounded_integers": (c_i32, [c_u64, c_u64, c_u64, c_u64, c_i64, c_i64, c_i64, c_vp, ctypes.POINTER(c_i64),
                                    c_vp]),
    "fk_zipf_bounded": (c_i32, [c_u64, c_u64, c_u64, c_u64, ctypes.c_double, c_i64, c_i64, ctypes.c_double,
                                ctypes.c_double, ctypes.c_double, c_vp, ctypes.POINTER(c_i64), c_vp]),
    "fk_mix_offsets": (c_i32, [c_u64, c_vp, c_i64, c_vp, c_vp]),
    "fk_shuffle_u64": (c_i32, [c_vp, c_i64, c_u64, c_vp, c_vp]),
    "fk_live_slots": (c_i32, [c_vp, c_i32, c_i64, c_vp, c_i32, c_vp, c_vp, c_vp]),
    "fk_shard_partition": (c_i32, [c_vp, c_vp, c_i64, c_u64, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "fk_shard_unpermute": (c_i32, [c_vp, c_vp, c_i64, c_i32, c_vp, c_vp]),
    "fk_shard_dispatch": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_u64, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "fk_shard_combine": (c_i32, [c_vp, c_i64, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "fk_shard_signal": (c_i32, [c_vp, c_i32, ctypes.c_uint32, ctypes.c_uint32, c_vp]),
    "fk_shard_wait": (c_i32, [c_vp, c_i32, ctypes.c_uint32, ctypes.c_double, c_vp]),
    "fk_ipc_alloc": (c_i32, [c_i64, ctypes.POINTER(c_vp)]),
    "fk_ipc_free": (c_i32, [c_vp]),
    "fk_ipc_get_handle": (c_i32, [c_vp, c_vp]),
    "fk_ipc_open": (c_i32, [c_vp, ctypes.POINTER(c_vp)]),
    "fk_ipc_close": (c_i32, [c_vp]),
    "fk_gqf_count": (c_i32, [ctypes.POINTER(GqfGeom), ctypes.POINTER(GqfTables), c_vp, c_i32, c_i64, c_vp, c_vp]),
    "fk_gqf_find_run": (c_i32, [ctypes.POINTER(GqfGeom), ctypes.POINTER(GqfTables), c_vp, c_i64, c_vp, c_vp]),
    "fk_gqf_rebuild_index": (c_i32, [ctypes.POINTER(GqfGeom), ctypes.POINTER(GqfTables), c_vp]),
    "fk_gqf_validate": (c_i32, [ctypes.POINTER(GqfGeom), ctypes.POINTER(GqfTables), c_vp, c_vp]),
    "fk_gqf_enumerate": (c_i32, [ctypes.POINTER(GqfGeom), ctypes.POINTER(GqfTables), c_vp, c_vp, c_i64,
                                 ctypes.POINTER(c_i64), c_vp]),
    "fk_gqf_insert_batch": (c_i32, [ctypes.POINTER(GqfGeom), ctypes.POINTER(GqfTables), c_vp, c_vp, c_i64,
                                    ctypes.POINTER(c_i32), ctypes.POINTER(c_i64), ctypes.POINTER(c_i64), c_vp]),
    "fk_gqf_delete_batch": (c_i32, [ctypes.POINTER(GqfGeom), ctypes.POINTER(GqfTables), c_vp, c_vp, c_i64, c_vp,
                                    ctypes.POINTER(c_i64), c_vp]),
    "fk_gqf_apply": (c_i32, [ctypes.POINTER(GqfGeom), ctypes.POINTER(GqfTables), ctypes.POINTER(GqfTables),
                             c_vp, c_i32, c_vp, c_i64, c_i32, c_i32, c_vp, ctypes.POINTER(GqfResult), c_vp]),
}

_lib = None
_lock = threading.Lock()


def exported_symbols():
    """Names the Python side binds (tests check the .so exports all of them)."""
    return sorted(_SIGS)


def load():
    """Load libfkb200.so and bind every entry point; raises if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    "libfkb200.so is not built (%s); run __graft_entry__.build() -- "
                    "there is no CPU fallback" % LIB_PATH)
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


class KernelError(RuntimeError):
    pass


def check(rc, what):
    """Map a C-ABI return code to an exception (never silently ignored)."""
    if rc == 0:
        return 0
    if rc == FK_E_INVARIANT:
        raise RuntimeError("%s: invariant violation" % what)
    if rc == FK_E_ARG:
        raise ValueError("%s: invalid arguments" % what)
    if rc < 0:
        raise KernelError("%s: CUDA error %d" % (what, -rc))
    return rc


_setup_done = set()


def require_cuda(device=None):
    """torch with a CUDA device, the library loaded and the device set up."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("the B200 filter kernels need a CUDA device; none is visible "
                           "(there is no CPU fallback)")
    lib = load()
    idx = torch.device(device).index if device is not None else None
    if idx is None:
        idx = torch.cuda.current_device()
    if idx not in _setup_done:
        with torch.cuda.device(idx):
            check(lib.fk_device_setup(int(os.environ.get("FK_L2_FETCH_BYTES", "32"))), "device setup")
        _setup_done.add(idx)
    return torch


def dptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None and t.numel() else ctypes.c_void_p(0)


def stream_ptr(torch):
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def to_device_u64(torch, keys, device):
    """numpy/torch/sequence of 64-bit keys -> contiguous int64 CUDA tensor (bit view)."""
    if isinstance(keys, torch.Tensor):
        t = keys.reshape(-1)
        if t.dtype in (torch.int64, torch.uint64):
            t = t.view(torch.int64)
        else:
            t = t.to(torch.int64)
        if not t.is_cuda:
            return t.to(device, non_blocking=t.is_pinned()).contiguous()
        return t.to(device).contiguous()
    arr = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64).reshape(-1))
    return torch.from_numpy(arr.view(np.int64)).to(device)


def host_view(torch, t, dtype):
    """Device byte tensor -> numpy array of `dtype` (synchronous D2H)."""
    return t.detach().cpu().numpy().view(dtype)


def to_device_bytes(torch, arr, device):
    a = np.ascontiguousarray(arr)
    return torch.from_numpy(a.view(np.uint8).reshape(-1).copy()).to(device)
