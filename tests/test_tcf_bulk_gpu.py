"""Bulk-TCF parity on the B200: the CUDA path (through the C ABI) vs the
reference's own goldens and the CPU oracle (oracle/model.py OracleBulkTcf).

Everything is bit-exact: the failed-key list and its order, the sorted block
image, fill, backing table, query answers (false positives included),
removed flags and counters -- the reference routes sequentially, so its
result is a pure function of (state, batch) and the device reproduces it.
Mirrors /root/reference/pkg/tests/test_tcf_bulk.py and test_backends.py:115-137.
"""

import numpy as np
import pytest

from conftest import counter_keys

pytestmark = pytest.mark.gpu


def _pair(oracle, **kw):
    from paper_2212_09005_b200 import BulkTcf
    f = BulkTcf(**kw)
    p = f.params
    o = oracle.OracleBulkTcf(p.num_blocks, p.block_slots, p.tag_bits, f._dtype, p.backing_slots, p.cut_slots,
                             p.probe_limit, p.seed)
    return f, o


def _same(f, o):
    assert np.array_equal(f._fill, o.fill)
    assert np.array_equal(f._blocks, o.blocks)
    assert np.array_equal(f._backing, o.backing)
    assert f.counters == o.counters


@pytest.mark.parametrize("name", ["a", "b", "c"])
def test_reference_goldens(golden, name):
    """Fixtures produced by the reference's compiled backend (make_golden.py)."""
    from paper_2212_09005_b200 import BulkTcf
    t = golden("tcf_bulk")
    f = BulkTcf(num_blocks=int(t[name + "_nb"][0]))
    failed = f.insert_batch(t[name + "_keys"])
    assert np.array_equal(failed, t[name + "_failed"])
    assert np.array_equal(f._blocks.astype(np.uint64), t[name + "_blocks_ins"])
    assert np.array_equal(f._fill, t[name + "_fill_ins"])
    assert np.array_equal(f._backing.astype(np.uint64), t[name + "_backing_ins"])
    assert np.array_equal(f.query_batch(t[name + "_probe"]).astype(np.uint8), t[name + "_found"])
    assert np.array_equal(f.delete_batch(t[name + "_dkeys"]).astype(np.uint8), t[name + "_removed"])
    assert np.array_equal(f._blocks.astype(np.uint64), t[name + "_blocks_del"])
    assert np.array_equal(f._fill, t[name + "_fill_del"])
    assert np.array_equal(f._backing.astype(np.uint64), t[name + "_backing_del"])
    c = f.counters
    assert [c["inserts_ok"], c["inserts_backing"], c["deletes_ok"]] == t[name + "_counters"].tolist()


@pytest.mark.parametrize("load", [0.85, 0.9])
def test_c1_scale_parity(oracle, load):
    """2^20 slots (8192 blocks x 128), one batch to the load, then queries and
    a delete of half the keys plus absent ones."""
    f, o = _pair(oracle, num_blocks=8192)
    n = int(load * 2 ** 20)
    keys = counter_keys(1, n)
    assert np.array_equal(f.insert_batch(keys), o.insert_batch(keys))
    _same(f, o)
    probe = np.concatenate([keys[::3], counter_keys(2, 300_000)])
    qa = f.query_batch(probe)
    assert np.array_equal(qa, o.query_batch(probe))
    assert qa[: len(keys[::3])].all()
    d = np.concatenate([keys[::2], counter_keys(3, 50_000)])
    assert np.array_equal(f.delete_batch(d), o.delete_batch(d))
    _same(f, o)
    f.validate()


def test_multi_batch_and_overfill(oracle):
    """Batches into a partly filled table, then past capacity: the backing
    table fills and failed keys come back in the reference's order."""
    f, o = _pair(oracle, num_blocks=300, backing_fraction=0.005)
    for s, n in enumerate([10_000, 15_000, 9_000, 8_000]):
        keys = counter_keys(10 + s, n)
        a, b = f.insert_batch(keys), o.insert_batch(keys)
        assert np.array_equal(a, b), s
        _same(f, o)
    assert len(a) > 0
    d = counter_keys(11, 15_000)
    assert np.array_equal(f.delete_batch(d), o.delete_batch(d))
    _same(f, o)


@pytest.mark.parametrize("kw", [dict(tag_bits=8), dict(tag_bits=20), dict(tag_bits=32, block_slots=40),
                                dict(block_slots=7, shortcut_fraction=0.5), dict(backing_fraction=0.0),
                                dict(block_slots=2), dict(block_slots=1000, tag_bits=12)])
def test_geometries(oracle, kw):
    nb = 97
    f, o = _pair(oracle, num_blocks=nb, **kw)
    cap = nb * f.params.block_slots
    for s in range(3):
        keys = counter_keys(20 + s, int(0.4 * cap))
        assert np.array_equal(f.insert_batch(keys), o.insert_batch(keys)), (kw, s)
        _same(f, o)
    probe = np.concatenate([counter_keys(20, 500), counter_keys(99, 2000)])
    assert np.array_equal(f.query_batch(probe), o.query_batch(probe))
    d = np.concatenate([counter_keys(21, int(0.4 * cap)), counter_keys(98, 300)])
    assert np.array_equal(f.delete_batch(d), o.delete_batch(d))
    _same(f, o)


def test_duplicates_and_repeated_deletes(oracle):
    """Duplicate keys in a batch share (block, word): merge keeps every copy,
    deletes remove one copy per request while copies remain."""
    f, o = _pair(oracle, num_blocks=64)
    base = counter_keys(5, 2000)
    keys = np.concatenate([base, base[:700], base[:50], base[:50]])
    assert np.array_equal(f.insert_batch(keys), o.insert_batch(keys))
    _same(f, o)
    d = np.concatenate([base[:100], base[:100], base[:100], base[:100], counter_keys(6, 100)])
    assert np.array_equal(f.delete_batch(d), o.delete_batch(d))
    _same(f, o)


def test_partition_and_merge_block(oracle):
    """Public building blocks (test_tcf_bulk.py:15-58)."""
    from paper_2212_09005_b200 import BulkTcf
    from paper_2212_09005_b200.hashing import potc_pair_many
    f = BulkTcf(num_blocks=50)
    keys = counter_keys(7, 3000)
    blocks, words, bounds, order = f.partition(keys)
    fps = f._fps(keys)
    w = f._words(fps)
    b1, _ = potc_pair_many(fps, 50)
    comb = (b1.astype(np.uint64) << np.uint64(32)) | w
    ref = np.argsort(comb, kind="stable")
    assert np.array_equal(order, ref)
    assert np.array_equal(blocks, (comb[ref] >> np.uint64(32)).astype(np.int64))
    assert np.array_equal(words, comb[ref] & np.uint64(0xFFFFFFFF))
    assert np.array_equal(bounds, np.searchsorted(comb[ref], np.arange(51, dtype=np.uint64) << np.uint64(32)))
    f.merge_block(3, np.array([9, 4, 300, 4], dtype=np.uint16))
    f.merge_block(3, np.array([5, 1000], dtype=np.uint16))
    assert f._blocks[3 * 128:3 * 128 + 7].tolist() == [4, 4, 5, 9, 300, 1000, 0]
    assert f.occupancy(3) == 6
    from paper_2212_09005_b200 import FilterFullError
    with pytest.raises(FilterFullError):
        f.merge_block(4, np.arange(2, 200, dtype=np.uint16))


def test_device_tensors_and_validate():
    import torch
    from paper_2212_09005_b200 import BulkTcf, ValidationError
    f = BulkTcf(num_blocks=512)
    keys = counter_keys(8, 50_000)
    kd = torch.from_numpy(keys.view(np.int64)).cuda()
    failed = f.insert_batch(kd)
    assert failed.is_cuda and failed.numel() == 0
    assert bool(f.query_batch(kd).all())
    assert f.counters["inserts_ok"] == 50_000
    f.validate()
    assert abs(f.load_factor() - 50_000 / (512 * 128)) < 1e-12
    rem = f.delete_batch(kd[:1000])
    assert rem.is_cuda and bool(rem.all())
    f.validate()
    blk = f._blocks
    b = int(np.flatnonzero(f._fill)[0])
    assert f._fill[b] >= 2
    blk[b * 128], blk[b * 128 + 1] = 0xFFFF, 2
    with pytest.raises(ValidationError):
        f.validate()


def test_device_validate_agrees_with_host_checks():
    """BulkTcf.validate runs on the device (fk_btcf_validate); every kind of
    corruption the reference's host checks reject is rejected, and a clean
    table passes."""
    from paper_2212_09005_b200 import BulkTcf, ValidationError
    f = BulkTcf(num_blocks=256)
    f.insert_batch(counter_keys(71, 25_000))
    f.validate()
    B = f.params.block_slots
    fill = f._fill
    blk = int(np.flatnonzero(fill > 3)[0])
    base = blk * B

    def corrupt(fn):
        blocks, fl = f._blocks, f._fill
        saved = (blocks.copy(), fl.copy())
        fn(blocks, fl)
        with pytest.raises(ValidationError):
            f.validate()
        blocks[:] = saved[0]
        fl[:] = saved[1]
        f.validate()

    corrupt(lambda b, fl: fl.__setitem__(blk, B + 1))                      # fill over capacity
    corrupt(lambda b, fl: b.__setitem__(base + 1, 1))                      # reserved word in the prefix
    corrupt(lambda b, fl: b.__setitem__(base, b[base + 2] + 1))            # unsorted prefix
    corrupt(lambda b, fl: b.__setitem__(base + int(fl[blk]), 77))          # tail not empty
    corrupt(lambda b, fl: fl.__setitem__(blk, fl[blk] - 1) or b.__setitem__(base + int(fl[blk]), 0))  # count mismatch


@pytest.mark.parametrize("mode", ["blocks", "jacobi", "seq", "prefix"])
def test_route_modes_bit_exact(oracle, monkeypatch, mode):
    """The four routers (per-block fixpoint sweeps -- the default --, the
    global-prefix fixpoint, the one-warp walk and the block-parallel prefix
    walk) give the reference's sequential
    decisions (ck:408-444): configs[0] at 0.9 load, then an overfilled small
    table where both blocks of some leftovers are full (dest = -1, backing)."""
    monkeypatch.setenv("FK_ROUTE", mode)
    f, o = _pair(oracle, num_blocks=8192)
    keys = counter_keys(41, int(0.9 * 2 ** 20))
    assert np.array_equal(f.insert_batch(keys), o.insert_batch(keys))
    _same(f, o)
    f, o = _pair(oracle, num_blocks=200, backing_fraction=0.02)
    for s, n in enumerate([20_000, 8_000, 4_000]):
        keys = counter_keys(50 + s, n)
        assert np.array_equal(f.insert_batch(keys), o.insert_batch(keys)), s
        _same(f, o)


def test_route_long_segments_fall_back(oracle, monkeypatch, capfd):
    """More than 1024 leftovers on one block: the per-block router hands the
    batch to the global-prefix fixpoint, same decisions as the reference's
    walk (ck:408-444)."""
    monkeypatch.setenv("FK_ROUTE_STATS", "1")
    f, o = _pair(oracle, num_blocks=8, backing_fraction=0.5)
    keys = counter_keys(61, 20_000)
    assert np.array_equal(f.insert_batch(keys), o.insert_batch(keys))
    _same(f, o)
    err = capfd.readouterr().err
    assert "fk route (blocks)" in err and "converged=2" in err, err[-500:]


def test_items_selected_on_device():
    """BulkTcf.items selects each block's filled prefix and the live backing
    slots on the device (fk_live_slots): the reference's (block, word) list
    (tcf_bulk.py:342-352), in its order."""
    from paper_2212_09005_b200 import BulkTcf
    f = BulkTcf(num_blocks=256)
    keys = counter_keys(93, int(256 * 128 * 1.03))  # overfill: backing entries
    f.insert_batch(keys)
    f.delete_batch(keys[::9])
    p = f.params
    blocks, fill, backing = f._blocks, f._fill, f._backing
    want = []
    for b in range(p.num_blocks):
        want.extend((b, int(w)) for w in blocks[b * p.block_slots:b * p.block_slots + int(fill[b])].tolist())
    want.extend((-1, int(w)) for w in backing[backing > 1].tolist())
    assert any(b == -1 for b, _ in want)
    assert f.items() == want
