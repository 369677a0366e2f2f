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
