"""Multi-process sharding logic on CPU: world_size-2 gloo through the real
_Router exchange path (count all-to-all, key all-to-all, reverse all-to-all,
unpermute).  The partition/unpermute ops and the per-shard filters are the
CPU oracle here (tests only); on the GPU box they are the CUDA kernels.

Checks: every key reaches the shard its fingerprint prefix
names, shards see (source rank, input index) order, answers come back in
each rank's input order, TCF shard s equals an oracle Tcf(nb / G) fed exactly
its keys, and sharded GQF counts equal one global GQF's counts.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


class NumpyShardOps:
    """Test double of CudaShardOps (same contract as fk_shard_partition)."""

    def partition(self, keys, vals, seed, shift, log2g):
        from oracle import model
        k = keys.numpy().view(np.uint64)
        h = model.fingerprint_many(k, seed)
        owner = (h >> np.uint64(shift)) & np.uint64((1 << log2g) - 1) if log2g else np.zeros(len(k), np.uint64)
        perm = np.argsort(owner, kind="stable")
        counts = np.bincount(owner.astype(np.int64), minlength=1 << log2g).astype(np.int64)
        vo = torch.from_numpy(vals.numpy()[perm].copy()) if vals is not None else None
        return (torch.from_numpy(k[perm].view(np.int64).copy()), vo, torch.from_numpy(perm.astype(np.int32)),
                torch.from_numpy(counts))

    def unpermute(self, perm, src):
        out = torch.empty_like(src)
        out[perm.long()] = src
        return out


def _owner(keys, seed, shift, g):
    from oracle import model
    return ((model.fingerprint_many(keys, seed) >> np.uint64(shift)) & np.uint64(g - 1)).astype(np.int64)


def _keys_of(rank, n):
    import sys
    sys.path.insert(0, ROOT)
    from paper_2212_09005_b200.workloads import counter_stream
    return counter_stream(100 + rank, 0x5851F42D4C957F2D, n)


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import model
        from paper_2212_09005_b200.sharding import _Router
        ops = NumpyShardOps()
        out = {}
        # ---- point TCF: 2 shards of nb/2 blocks --------------------------------
        nb, seed = 512, 7
        keys = _keys_of(rank, 3000)
        r = _Router(torch, None, world, seed, 64 - 1, ops)
        rk, _, plan = r.route(torch.from_numpy(keys.view(np.int64)))
        tcf = model.OracleTcf(nb // world, 16, 16, np.uint16, int(round(nb // world * 16 * 0.01)), 12, 20, seed)
        rkn = rk.numpy().view(np.uint64)
        codes = tcf.insert_many(rkn)
        back = r.unroute(torch.from_numpy(codes), plan).numpy()
        found = r.unroute(torch.from_numpy(tcf.query_many(rkn).astype(np.uint8)), plan).numpy()
        out["tcf_recv"] = rkn
        out["tcf_codes"] = back
        out["tcf_found"] = found
        out["tcf_blocks"] = tcf.blocks.copy()
        # ---- GQF: global q=14 -> 2 shards of q=13; counts with values ------------
        gq, gr = 14, 8
        gk = np.concatenate([_keys_of(rank, 3000), _keys_of(rank, 500)])
        cnt = (np.arange(len(gk)) % 5 + 1).astype(np.uint64)
        rg = _Router(torch, None, world, seed, (gq - 1) + gr, ops)
        rkk, rcc, plan2 = rg.route(torch.from_numpy(gk.view(np.int64)), torch.from_numpy(cnt.view(np.int64)))
        g = model.OracleGqf(gq - 1, gr, seed, int(0.95 * (1 << (gq - 1))))
        code, _ = g.insert_many(rkk.numpy().view(np.uint64), rcc.numpy().view(np.uint64))
        assert code == 0
        c = g.count_many(rkk.numpy().view(np.uint64))
        out["gqf_counts"] = rg.unroute(torch.from_numpy(c.view(np.int64)), plan2).numpy().view(np.uint64)
        out["gqf_keys"] = gk
        out["gqf_cnt"] = cnt
        assert rg.any_flag(rank == 1) == 1
        assert r.sum([rank + 1, 10]) == [3, 20]
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def results():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    return res


def test_tcf_routing_and_shard_images(results, oracle):
    world, seed, nb = 2, 7, 512
    keys = [_keys_of(r, 3000) for r in range(world)]
    for s in range(world):
        # shard s received (rank 0's keys it owns, then rank 1's), input order
        exp = np.concatenate([k[_owner(k, seed, 63, world) == s] for k in keys])
        assert np.array_equal(results[s]["tcf_recv"], exp)
        t = oracle.OracleTcf(nb // world, 16, 16, np.uint16, int(round(nb // world * 16 * 0.01)), 12, 20, seed)
        t.insert_many(exp)
        assert np.array_equal(results[s]["tcf_blocks"], t.blocks)
    for r in range(world):
        assert results[r]["tcf_found"].all()  # no false negatives after the round trip
        own = _owner(keys[r], seed, 63, world)
        for s in range(world):
            exp = np.concatenate([k[_owner(k, seed, 63, world) == s] for k in keys])
            t = oracle.OracleTcf(nb // world, 16, 16, np.uint16, int(round(nb // world * 16 * 0.01)), 12, 20,
                                 seed)
            codes = t.insert_many(exp)
            mine = codes[:int((own == s).sum())] if r == 0 else codes[len(exp) - int((own == s).sum()):]
            assert np.array_equal(results[r]["tcf_codes"][own == s], mine)


def test_gqf_sharded_counts_equal_global(results, oracle):
    world, seed = 2, 7
    g = oracle.OracleGqf(14, 8, seed, int(0.95 * (1 << 14)))
    allk = np.concatenate([results[r]["gqf_keys"] for r in range(world)])
    allc = np.concatenate([results[r]["gqf_cnt"] for r in range(world)])
    code, _ = g.insert_many(allk, allc)
    assert code == 0
    for r in range(world):
        assert np.array_equal(results[r]["gqf_counts"], g.count_many(results[r]["gqf_keys"]))


@pytest.mark.parametrize("G", [2, 4, 8])
def test_peer_exchange_plan_round_trip(G):
    """The peer-memory exchange's offsets (exchange_plan), played through in
    numpy exactly as the kernels address memory: dispatch stores key i of
    owner o at dst_off[o] + i - seg_start[o] of o's receive buffer, combine
    stores received item j of source s at back_off[s] + j - recv_off[s] of
    s's return buffer, the source unpermutes.  Every owner receives each
    source's keys in (source rank, input order) with no tag, and every
    source gets each key's answer back at its input position."""
    from paper_2212_09005_b200.sharding import exchange_plan
    rng = np.random.default_rng(G)
    n = [int(rng.integers(0, 300)) for _ in range(G)]
    n[0] = 0  # an empty batch still takes part
    keys = [rng.integers(0, 1 << 62, n[r]).astype(np.int64) for r in range(G)]
    owner = [(k * 2654435761 >> 7) % G for k in keys]
    perm = [np.argsort(o, kind="stable") for o in owner]
    C = np.array([np.bincount(owner[r], minlength=G) for r in range(G)], dtype=np.int64)
    plans = [exchange_plan(C, r) for r in range(G)]
    assert len({p[4] for p in plans}) == 1  # every rank sizes the buffers the same way
    cap = plans[0][4]
    recv = [np.full(cap, -1, np.int64) for _ in range(G)]
    for r in range(G):  # dispatch
        ss, do = plans[r][0], plans[r][1]
        for i, p in enumerate(perm[r]):
            o = owner[r][p]
            recv[o][do[o] + i - ss[o]] = keys[r][p]
    for o in range(G):  # owners see (source rank, input order)
        ro = plans[o][2]
        expect = np.concatenate([keys[s][owner[s] == o] for s in range(G)]) if C[:, o].sum() else np.zeros(0)
        assert np.array_equal(recv[o][:ro[-1]], expect)
    back = [np.full(cap, -1, np.int64) for _ in range(G)]
    for o in range(G):  # combine: the answer is the key itself, doubled
        ro, bo = plans[o][2], plans[o][3]
        for j in range(ro[-1]):
            s = int(np.searchsorted(ro, j, side="right") - 1)
            back[s][bo[s] + j - ro[s]] = 2 * recv[o][j]
    for r in range(G):  # unpermute
        out = np.empty(n[r], np.int64)
        out[perm[r]] = back[r][:n[r]]
        assert np.array_equal(out, 2 * keys[r])


def test_failed_flags_counts_duplicates():
    """Sharded bulk insert: a key that failed m times flags its last m copies
    only (not every copy, as a membership test would)."""
    from paper_2212_09005_b200.sharding import failed_flags
    keys = torch.tensor([5, 7, 5, 9, 5, 7, 11], dtype=torch.int64)
    failed = torch.tensor([5, 7, 5], dtype=torch.int64)
    got = failed_flags(torch, keys, failed).tolist()
    assert got == [0, 0, 1, 0, 1, 1, 0]
    assert failed_flags(torch, keys, failed[:0]).tolist() == [0] * 7
