"""The sharded facades end to end on the B200 with two ranks.

The GPU box has one GPU, and NCCL refuses two ranks on one device, so the
two processes share cuda:0 over a gloo group (the router stages the
all-to-all buffers through the host for gloo).  Everything else is the
product path: CUDA partition / unpermute kernels, per-rank CUDA sub-filters,
reverse exchange.  Checks every rank's answers against oracles of the shards
and of one global GQF.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, q, peer="1"):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), FK_SHARD_PEER=peer)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from conftest import counter_keys
        from paper_2212_09005_b200.sharding import ShardedBulkTcf, ShardedGqf, ShardedTcf
        out = {}
        keys = counter_keys(60 + rank, 20_000)
        st = ShardedTcf(num_blocks=4096)
        out["router"] = type(st._router).__name__
        out["codes"] = st.insert_many(keys)
        out["found"] = st.query_many(keys)
        out["neg"] = st.query_many(counter_keys(80 + rank, 5000))
        out["blocks"] = st._local._blocks.copy()
        # uneven batches, one of them empty: the exchange is still collective
        out["uneven"] = st.query_many(keys[:0] if rank == 0 else keys[:100])
        out["removed"] = st.delete_many(keys[::2])
        out["counters"] = st.counters
        sb = ShardedBulkTcf(num_blocks=512)
        out["bfailed"] = sb.insert_batch(keys)
        out["bfound"] = sb.query_batch(keys)
        sg = ShardedGqf(q=15)
        gk = np.concatenate([keys[:8000], keys[:3000]])
        sg.bulk_insert(gk)
        out["gcount"] = sg.count_many(keys[:10_000])
        out["gkeys"] = gk
        out["total"] = sg.total_items
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("peer", ["1", "0"])
def test_two_rank_sharded_facades(oracle, peer):
    """peer = 1: the fused peer-memory exchange (fk_shard_dispatch /
    fk_shard_combine over CUDA IPC mappings, stream-ordered fk_shard_signal /
    fk_shard_wait handoffs); 0: the all-to-all router."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, peer)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=400) for _ in procs)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    from conftest import counter_keys
    keys = [counter_keys(60 + r, 20_000) for r in range(2)]
    own = [((oracle.fingerprint_many(k, 0) >> np.uint64(63)) & np.uint64(1)).astype(int) for k in keys]
    # shard s = oracle Tcf(4096 / 2) fed (rank 0's owned keys, then rank 1's)
    for s in range(2):
        recv = np.concatenate([keys[r][own[r] == s] for r in range(2)])
        o = oracle.OracleTcf(2048, 16, 16, np.uint16, int(round(2048 * 16 * 0.01)), 12, 20, 0)
        codes = o.insert_many(recv)
        assert np.array_equal(res[s]["blocks"], o.blocks)
        n0 = int((own[0] == s).sum())
        assert np.array_equal(res[0]["codes"][own[0] == s], codes[:n0])
        assert np.array_equal(res[1]["codes"][own[1] == s], codes[n0:])
    assert res[0]["router"] == ("_PeerRouter" if peer == "1" else "_Router")
    assert len(res[0]["uneven"]) == 0 and len(res[1]["uneven"]) == 100 and res[1]["uneven"].all()
    for r in range(2):
        assert res[r]["found"].all() and res[r]["removed"].all()
        assert res[r]["neg"].mean() < 0.01
        assert len(res[r]["bfailed"]) == 0 and res[r]["bfound"].all()
    assert res[0]["counters"]["inserts_ok"] == 40_000 and res[0]["counters"]["deletes_ok"] == 20_000
    g = oracle.OracleGqf(15, 8, 0, int(0.95 * (1 << 15)))
    assert g.bulk_insert(np.concatenate([res[r]["gkeys"] for r in range(2)])) == []
    for r in range(2):
        assert np.array_equal(res[r]["gcount"], g.count_many(keys[r][:10_000]))
    assert res[0]["total"] == 22_000
