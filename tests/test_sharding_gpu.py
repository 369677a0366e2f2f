"""Sharding kernels on the B200 (csrc/shard.cu) and per-shard parity.

One GPU, so the all-to-all itself is covered by the gloo tests; here the
CUDA partition/unpermute are checked bit-exact against a numpy restatement,
G virtual shards are built on one device from the kernel's partition, and
each shard's filter is compared with the oracle fed the same keys (TCF image
bit-exact; GQF counts equal one global filter's).
"""

import numpy as np
import pytest

from conftest import counter_keys

pytestmark = pytest.mark.gpu


def _np_partition(keys, seed, shift, log2g, oracle):
    h = oracle.fingerprint_many(keys, seed)
    owner = (h >> np.uint64(shift)) & np.uint64((1 << log2g) - 1) if log2g else np.zeros(len(keys), np.uint64)
    perm = np.argsort(owner, kind="stable")
    return keys[perm], perm, np.bincount(owner.astype(np.int64), minlength=1 << log2g)


@pytest.mark.parametrize("log2g,shift", [(0, 64), (1, 63), (3, 61), (3, 30), (2, 40)])
def test_partition_and_unpermute_bit_exact(oracle, log2g, shift):
    import torch
    from paper_2212_09005_b200.sharding import CudaShardOps
    ops = CudaShardOps(torch)
    keys = counter_keys(4, 300_001)
    vals = np.arange(len(keys), dtype=np.uint64) * np.uint64(3)
    kd = torch.from_numpy(keys.view(np.int64)).cuda()
    vd = torch.from_numpy(vals.view(np.int64)).cuda()
    ko, vo, perm, counts = ops.partition(kd, vd, 11, shift, log2g)
    ek, eperm, ecounts = _np_partition(keys, 11, shift, log2g, oracle)
    assert np.array_equal(ko.cpu().numpy().view(np.uint64), ek)
    assert np.array_equal(perm.cpu().numpy(), eperm.astype(np.int32))
    assert np.array_equal(counts.cpu().numpy(), ecounts)
    assert np.array_equal(vo.cpu().numpy().view(np.uint64), vals[eperm])
    back = ops.unpermute(perm, ko)
    assert np.array_equal(back.cpu().numpy().view(np.uint64), keys)
    flags = (ko & 1).to(torch.uint8)
    assert np.array_equal(ops.unpermute(perm, flags).cpu().numpy(), (keys & np.uint64(1)).astype(np.uint8))


def _virtual_exchange(torch, ops, batches, seed, shift, log2g):
    """G ranks' batches -> per-shard received keys (source rank, input order)."""
    G = 1 << log2g
    parts = []
    for b in batches:
        ko, _, perm, counts = ops.partition(torch.from_numpy(b.view(np.int64)).cuda(), None, seed, shift, log2g)
        c = counts.cpu().tolist()
        off = np.concatenate([[0], np.cumsum(c)])
        parts.append([ko[off[s]:off[s + 1]] for s in range(G)])
    return [torch.cat([parts[r][s] for r in range(len(batches))]) for s in range(G)]


def test_virtual_shards_tcf_parity(oracle):
    import torch
    from paper_2212_09005_b200 import Tcf
    from paper_2212_09005_b200.sharding import CudaShardOps
    ops = CudaShardOps(torch)
    G, nb = 4, 4096
    batches = [counter_keys(30 + r, 12_000) for r in range(G)]
    recv = _virtual_exchange(torch, ops, batches, 0, 62, 2)
    for s in range(G):
        f = Tcf(num_blocks=nb // G)
        o = oracle.OracleTcf(nb // G, 16, 16, np.uint16, f.params.backing_slots, 12, 20, 0)
        codes = f.insert_many(recv[s])
        assert np.array_equal(codes.cpu().numpy(), o.insert_many(recv[s].cpu().numpy().view(np.uint64)))
        assert np.array_equal(f._blocks, o.blocks) and np.array_equal(f._backing, o.backing)


def test_virtual_shards_gqf_counts_equal_global(oracle):
    import torch
    from paper_2212_09005_b200 import Gqf
    from paper_2212_09005_b200.sharding import CudaShardOps
    ops = CudaShardOps(torch)
    G, q, r = 4, 16, 8
    batches = [np.concatenate([counter_keys(40 + i, 9000), counter_keys(40 + i, 2000)]) for i in range(G)]
    recv = _virtual_exchange(torch, ops, batches, 5, (q - 2) + r, 2)
    shards = [Gqf(q=q - 2, r=r, seed=5) for _ in range(G)]
    for s in range(G):
        shards[s].bulk_insert(recv[s])
    glob = oracle.OracleGqf(q, r, 5, int(0.95 * (1 << q)))
    allk = np.concatenate(batches)
    assert glob.bulk_insert(allk) == []
    for s in range(G):
        got = shards[s].count_many(recv[s]).cpu().numpy().view(np.uint64)
        assert np.array_equal(got, glob.count_many(recv[s].cpu().numpy().view(np.uint64)))


def test_world1_sharded_facades_match_plain():
    """Without torch.distributed the sharded facades are the local filter."""
    from paper_2212_09005_b200 import Gqf, Tcf
    from paper_2212_09005_b200.sharding import ShardedBulkTcf, ShardedGqf, ShardedTcf
    keys = counter_keys(9, 20_000)
    st, t = ShardedTcf(num_blocks=2048), Tcf(num_blocks=2048)
    assert np.array_equal(st.insert_many(keys), t.insert_many(keys))
    assert np.array_equal(st.query_many(keys[:5000]), t.query_many(keys[:5000]))
    assert np.array_equal(st.delete_many(keys[::2]), t.delete_many(keys[::2]))
    assert st.counters == t.counters
    sb = ShardedBulkTcf(num_blocks=256)
    assert len(sb.insert_batch(keys)) == 0 and sb.query_batch(keys).all()
    sg, g = ShardedGqf(q=14), Gqf(q=14)
    sg.bulk_insert(keys[:5000])
    g.bulk_insert(keys[:5000])
    assert np.array_equal(sg.count_many(keys[:6000]), g.count_many(keys[:6000]))
    assert sg.total_items == 5000
