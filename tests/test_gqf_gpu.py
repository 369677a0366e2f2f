"""GQF parity on the B200: the CUDA path vs the CPU oracle / reference goldens.

Bit-exact: table image (_slots/_occupieds/_runends/_offsets/_stats), counts,
delete found flags, capacity errors (code, failure point, partial image).
"""

import numpy as np
import pytest

from conftest import counter_keys

pytestmark = pytest.mark.gpu

IMG = ("slots", "occupieds", "runends", "offsets", "stats")
_INV1 = pow(0xBF58476D1CE4E5B9, -1, 2 ** 64)
_INV2 = pow(0x94D049BB133111EB, -1, 2 ** 64)
M64 = 2 ** 64 - 1


def _unshift(x, s):
    y = x
    for _ in range(64 // s + 1):
        y = x ^ (y >> s)
    return y


def unmix64(x):
    x = _unshift(x, 31)
    x = (x * _INV2) & M64
    x = _unshift(x, 27)
    x = (x * _INV1) & M64
    return _unshift(x, 30)


def craft(g, pairs):
    p = g.params
    return np.array([unmix64((qt << p.r) | rem) ^ p.seed for qt, rem in pairs], dtype=np.uint64)


def _oracle(g, oracle):
    p = g.params
    return oracle.OracleGqf(p.q, p.r, p.seed, p.max_occupied)


def same_image(g, o):
    img = o.image()
    for nm in IMG:
        assert np.array_equal(getattr(g, "_" + nm), img[nm]), nm


def golden_image(g, t, pre):
    for nm in IMG:
        assert np.array_equal(getattr(g, "_" + nm), t[pre + nm]), (pre, nm)


@pytest.mark.parametrize("r", [8, 16])
def test_golden_sequence(golden, r):
    from paper_2212_09005_b200 import Gqf
    t = golden("gqf")
    pre = "r%d_" % r
    g = Gqf(q=14, r=r)
    g.insert_many(t[pre + "k"], t[pre + "c"])
    golden_image(g, t, pre + "ins_")
    assert np.array_equal(g.count_many(t[pre + "k"]), t[pre + "count"])
    assert np.array_equal(g.delete_many(t[pre + "dk"], t[pre + "dc"]).astype(np.uint8), t[pre + "dfound"])
    golden_image(g, t, pre + "del_")
    g.bulk_insert(t[pre + "k2"])
    golden_image(g, t, pre + "bulk_")
    assert np.array_equal(g.bulk_delete(t[pre + "kk"]).astype(np.uint8), t[pre + "bfound"])
    golden_image(g, t, pre + "bdel_")
    g.validate()


def test_golden_duplicates_and_mapreduce(golden):
    from paper_2212_09005_b200 import Gqf
    t = golden("gqf")
    g = Gqf(q=16, r=8)
    g.bulk_insert(t["ur_keys"])
    golden_image(g, t, "ur_")
    uq, uc = np.unique(t["ur_keys"], return_counts=True)
    assert np.array_equal(g.count_many(uq), t["ur_count"])
    g2 = Gqf(q=16, r=8)
    g2.bulk_insert(uq, uc.astype(np.uint64))
    golden_image(g2, t, "ur_")


def test_golden_capacity_partial_image(golden):
    from paper_2212_09005_b200 import CapacityError, Gqf
    t = golden("gqf")
    g = Gqf(q=10, r=8)
    with pytest.raises(CapacityError):
        g.insert_many(t["cap_k"])
    golden_image(g, t, "cap_")
    g.validate()


def test_crafted_layouts():
    from paper_2212_09005_b200 import Gqf
    g = Gqf(q=8, r=8, seed=1)
    g.insert_many(craft(g, [(50, 9), (50, 3), (50, 200)]))
    assert g.find_run(50) == (50, 52)
    assert g._slots[50:53].tolist() == [3, 9, 200]
    g = Gqf(q=8, r=8, seed=2)
    g.insert_many(craft(g, [(5, 10), (5, 20), (6, 30), (7, 40)]))
    assert [g.find_run(x) for x in (5, 6, 7)] == [(5, 6), (7, 7), (8, 8)]
    assert g.find_run(99) == (-1, -1)
    g = Gqf(q=8, r=8, seed=6)
    key = int(craft(g, [(10, 7)])[0])
    for add in (1, 1, 298):
        g.insert(key, count=add)
    assert g.count(key) == 300
    assert g._slots[10:14].tolist() == [7, 4, 43, 7]
    assert g.delete(key, count=250) and g.count(key) == 50
    assert g.delete(key, count=50) and g.count(key) == 0 and not g.query(key)
    g.validate()


@pytest.mark.parametrize("q,r,n,seed", [(12, 8, 1200, 1), (16, 16, 20_000, 2), (18, 8, 78_000, 3)])
def test_point_ops_vs_oracle(oracle, q, r, n, seed):
    from paper_2212_09005_b200 import Gqf
    rng = np.random.default_rng(seed)
    g = Gqf(q=q, r=r, seed=seed)
    o = _oracle(g, oracle)
    keys = rng.integers(0, 2 ** 63, n, dtype=np.uint64)
    counts = rng.integers(1, 4, n, dtype=np.uint64)
    code, _ = o.insert_many(keys, counts)
    assert code == 0
    g.insert_many(keys, counts)
    same_image(g, o)
    probe = np.concatenate([keys[: n // 2], rng.integers(0, 2 ** 63, n // 2, dtype=np.uint64)])
    assert np.array_equal(g.count_many(probe), o.count_many(probe))
    for qt in rng.integers(0, 1 << q, 200).tolist():
        assert g.find_run(qt) == o.find_run(qt)
    d = np.concatenate([keys[::3], keys[:100], probe[-100:]])
    dc = rng.integers(1, 3, len(d), dtype=np.uint64)
    assert np.array_equal(g.delete_many(d, dc), o.delete_many(d, dc))
    same_image(g, o)
    g.validate()


@pytest.mark.parametrize("dist", ["uniform", "ur_count", "zipf"])
def test_bulk_ops_vs_oracle(oracle, dist):
    from paper_2212_09005_b200 import Gqf
    from paper_2212_09005_b200.workloads import WorkloadSpec, gen_keys
    q = 18
    spec = {"uniform": WorkloadSpec("uniform", n=int(0.85 * 2 ** q), seed=4),
            "ur_count": WorkloadSpec("ur_count", n=int(0.9 * 2 ** q) // 8, seed=4),
            "zipf": WorkloadSpec("zipf", n=200_000, seed=4, universe=100_000)}[dist]
    keys = gen_keys(spec)
    g = Gqf(q=q, r=8)
    o = _oracle(g, oracle)
    assert o.bulk_insert(keys) == []
    g.bulk_insert(keys)
    same_image(g, o)
    g.validate()
    dk = np.concatenate([keys[::4], keys[:1000]])
    assert np.array_equal(g.bulk_delete(dk), o.bulk_delete(dk))
    same_image(g, o)
    dc = np.full(5000, 3, np.uint64)
    assert np.array_equal(g.bulk_delete(keys[-5000:], dc), o.bulk_delete(keys[-5000:], dc))
    same_image(g, o)
    g.validate()


def test_bulk_equals_point_equals_mapreduce(oracle):
    from paper_2212_09005_b200 import Gqf
    rng = np.random.default_rng(9)
    keys = rng.integers(0, 2 ** 40, 40_000, dtype=np.uint64)
    keys = np.concatenate([keys, keys[:5000], keys[:100]])
    a, b, c = Gqf(q=16, r=8), Gqf(q=16, r=8), Gqf(q=16, r=8)
    a.bulk_insert(keys)
    b.insert_many(rng.permutation(keys))
    u, cnt = np.unique(keys, return_counts=True)
    c.bulk_insert(u, cnt.astype(np.uint64))
    for nm in IMG:
        assert np.array_equal(getattr(a, "_" + nm), getattr(b, "_" + nm))
        assert np.array_equal(getattr(a, "_" + nm), getattr(c, "_" + nm))


def test_load_capacity_point_and_bulk(oracle):
    from paper_2212_09005_b200 import CapacityError, Gqf
    rng = np.random.default_rng(11)
    for trial in range(3):
        keys = rng.integers(0, 2 ** 50, 1100 + 50 * trial, dtype=np.uint64)
        g = Gqf(q=10, r=8)
        o = _oracle(g, oracle)
        code, idx = o.insert_many(keys)
        assert code != 0
        with pytest.raises(CapacityError):
            g.insert_many(keys)
        same_image(g, o)
        g = Gqf(q=10, r=8)
        o = _oracle(g, oracle)
        assert o.bulk_insert(keys) != []
        with pytest.raises(CapacityError):
            g.bulk_insert(keys)
        same_image(g, o)


def test_shift_bound_rem0_unary(oracle):
    """A remainder-0 group spends one slot per copy (countgroups.py:14-16):
    a large count crosses the region hard bound -> SHIFT_BOUND, table intact."""
    from paper_2212_09005_b200 import CapacityError, Gqf
    g = Gqf(q=15, r=8, seed=3)
    o = _oracle(g, oracle)
    k = craft(g, [(100, 0), (8000, 5), (8100, 0)])
    cnt = np.array([20_000, 1, 9000], dtype=np.uint64)
    code, idx = o.insert_many(k, cnt)
    assert code == 2
    with pytest.raises(CapacityError, match="hard bound"):
        g.insert_many(k, cnt)
    same_image(g, o)
    g.validate()


def test_validate_detects_corruption():
    from paper_2212_09005_b200 import Gqf, ValidationError
    g = Gqf(q=14, r=8)
    g.insert_many(np.random.default_rng(3).integers(0, 2 ** 40, 8000, dtype=np.uint64))
    g.validate()
    s = g._slots
    i = int(np.flatnonzero(s == 0)[-1])
    s[i] = 7
    with pytest.raises(ValidationError):
        g.validate()
    s[i] = 0
    g.validate()
    g._offsets[1] += 1
    with pytest.raises(ValidationError):
        g.validate()


def test_mirror_edits_reach_device():
    from paper_2212_09005_b200 import Gqf
    g = Gqf(q=10, r=8, seed=2)
    key = int(craft(g, [(7, 9)])[0])
    g.insert(key, 5)
    assert g.count(key) == 5
    s = g._slots
    pos = g.find_run(7)[0]
    assert s[pos:pos + 3].tolist() == [9, 3, 9]  # count 5 = [rem, (5-2) % 9, rem]
    # rewrite the group by hand as [9, 9] (= count 2) and move the runend
    s[pos:pos + 3] = [9, 9, 0]
    rb = g._runends
    rb[(pos + 2) >> 6] &= ~np.uint64(1 << ((pos + 2) & 63))
    rb[(pos + 1) >> 6] |= np.uint64(1 << ((pos + 1) & 63))
    assert g.count(key) == 2  # the device saw the edited image and re-derived its index


def test_empty_and_stats():
    from paper_2212_09005_b200 import Gqf
    g = Gqf(q=8)
    g.bulk_insert(np.zeros(0, np.uint64))
    assert len(g.bulk_delete(np.zeros(0, np.uint64))) == 0
    assert g.occupied_slots == 0 and g.total_items == 0 and g.distinct_items == 0
    g.insert_many([1, 2, 3], [1, 1, 5])
    assert g.total_items == 7 and g.distinct_items == 3
    assert g.size_bits() == (g.params.physical_slots * 8 + 2 * (g.params.physical_slots // 64) * 64
                             + g.params.num_regions * 32) + g.params.num_regions * 512


def test_shift_instrumentation():
    from paper_2212_09005_b200 import Gqf
    g = Gqf(q=13, r=8, seed=28)
    keys = np.unique(np.random.default_rng(12).integers(0, 2 ** 50, 3000, dtype=np.uint64))
    g.bulk_insert(keys, workers=2)
    assert g.shifted_slots == 0
    g = Gqf(q=13, r=8, seed=28)
    g.insert_many(np.random.default_rng(12).integers(0, 2 ** 50, 3000, dtype=np.uint64))
    assert g.shifted_slots > 0


def _host_raises(g):
    from paper_2212_09005_b200 import ValidationError
    try:
        g._validate_host()
    except ValidationError:
        return True
    return False


@pytest.mark.parametrize("r", [8, 16])
def test_device_validate_agrees_with_host(r):
    """fk_gqf_validate flags exactly the tables the reference's host checks
    reject (gqf.py:430-492), over valid fills and a catalogue of corruptions."""
    from paper_2212_09005_b200 import Gqf
    rng = np.random.default_rng(11 + r)
    g = Gqf(q=14, r=r, seed=5)
    keys = rng.integers(0, 2 ** 40, 2500, dtype=np.uint64)
    g.bulk_insert(keys, rng.integers(1, 300, 2500).astype(np.uint64))
    assert g._device_validate() is None and not _host_raises(g)
    base = {n: getattr(g, n).copy() for n in ("_slots", "_occupieds", "_runends", "_offsets", "_stats")}

    def restore():
        for n, a in base.items():
            getattr(g, n)[:] = a

    used = np.flatnonzero(g._slots)
    corruptions = [
        ("_slots", lambda a: a.__setitem__(int(np.flatnonzero(a == 0)[-1]), 7)),      # residual data
        ("_slots", lambda a: a.__setitem__(int(used[len(used) // 2]), 0)),             # group damage
        ("_slots", lambda a: a.__setitem__(int(used[len(used) // 3]), a[used[len(used) // 3]] ^ 0x5)),
        ("_offsets", lambda a: a.__setitem__(1, a[1] + 1)),
        ("_stats", lambda a: a.__setitem__(0, a[0] + 1)),
        ("_stats", lambda a: a.__setitem__(1, a[1] - 1)),
        ("_stats", lambda a: a.__setitem__(2, a[2] + 3)),
        ("_runends", lambda a: a.__setitem__(3, a[3] ^ (1 << 17))),                    # count mismatch
        ("_occupieds", lambda a: a.__setitem__(5, a[5] ^ (1 << 40))),
    ]
    for name, fn in corruptions:
        fn(getattr(g, name))
        host = _host_raises(g)
        dev = g._device_validate()
        assert host == (dev is not None), (name, dev)
        restore()
    assert g._device_validate() is None


def test_device_validate_large_table():
    """q=24 (16.8 M slots): validation runs on the device in well under a
    second; the host decode loop would take minutes."""
    import time
    import torch
    from paper_2212_09005_b200 import Gqf
    g = Gqf(q=24, r=8)
    keys = torch.randint(-2 ** 62, 2 ** 62, (6_000_000,), dtype=torch.int64, device="cuda")
    g.bulk_insert(keys)
    t = time.perf_counter()
    g.validate()
    assert time.perf_counter() - t < 5.0
    assert g.total_items == 6_000_000


@pytest.mark.parametrize("with_counts", [False, True])
def test_capacity_large_point_batch_prefix_path(oracle, with_counts):
    """Point batches longer than the direct sequential threshold apply their
    longest safe prefix canonically and only the tail sequentially: the
    partial image (hence the failing index) still equals the reference's."""
    from paper_2212_09005_b200 import CapacityError, Gqf
    rng = np.random.default_rng(5 + with_counts)
    keys = rng.integers(0, 2 ** 52, 9000, dtype=np.uint64)
    cnt = rng.integers(1, 6, 9000).astype(np.uint64) if with_counts else None
    g = Gqf(q=13, r=8, seed=4)
    o = _oracle(g, oracle)
    code, idx = o.insert_many(keys, cnt)
    assert code == 1 and idx > 2048
    with pytest.raises(CapacityError):
        g.insert_many(keys, cnt)
    same_image(g, o)
    g.validate()


def test_shift_bound_inside_large_point_batch(oracle):
    from paper_2212_09005_b200 import CapacityError, Gqf
    g = Gqf(q=15, r=8, seed=3)
    o = _oracle(g, oracle)
    rng = np.random.default_rng(9)
    keys = rng.integers(0, 2 ** 52, 4000, dtype=np.uint64)
    keys[2600] = craft(g, [(100, 0)])[0]
    cnt = np.ones(4000, dtype=np.uint64)
    cnt[2600] = 20_000
    code, idx = o.insert_many(keys, cnt)
    assert code == 2 and idx == 2600
    with pytest.raises(CapacityError, match="hard bound"):
        g.insert_many(keys, cnt)
    same_image(g, o)


@pytest.mark.parametrize("r", [8, 16])
def test_small_batches_region_path_equals_oracle(oracle, monkeypatch, r):
    """Batches with few distinct fingerprints take the region-local insert
    path (k_gqf_insert_regions on a copy of the table); the image after every
    batch must equal the oracle's, with the full rebuild path as control."""
    from paper_2212_09005_b200 import Gqf
    rng = np.random.default_rng(20 + r)
    for limit in ("0", "100000"):
        monkeypatch.setenv("FK_GQF_SMALL", limit)
        g = Gqf(q=16, r=r, seed=7)
        o = _oracle(g, oracle)
        for step in range(12):
            keys = rng.integers(0, 2 ** 60, int(rng.integers(1, 3000)), dtype=np.uint64)
            if step % 3 == 1:
                keys = np.concatenate([keys, keys[: len(keys) // 2]])  # repeats in the batch
            cnt = rng.integers(1, 40, len(keys)).astype(np.uint64) if step % 2 else None
            if step % 4 == 3:
                g.insert_many(keys, cnt)
                o.insert_many(keys, cnt)
            else:
                g.bulk_insert(keys, cnt)
                o.bulk_insert(keys, cnt)
            same_image(g, o)
        g.validate()


@pytest.mark.parametrize("r", [8, 16])
def test_small_delete_batches_region_path_equals_oracle(oracle, monkeypatch, r):
    """Small delete batches run the reference's sequential delete per region
    (descending for bulk_delete, input order for delete_many): found flags
    and images equal the oracle's, with the rebuild path as control."""
    from paper_2212_09005_b200 import Gqf
    for limit in ("0", "100000"):
        rng = np.random.default_rng(40 + r)
        monkeypatch.setenv("FK_GQF_SMALL", limit)
        g = Gqf(q=16, r=r, seed=9)
        o = _oracle(g, oracle)
        pool = rng.integers(0, 2 ** 60, 10_000, dtype=np.uint64)
        cnt = rng.integers(1, 50, len(pool)).astype(np.uint64)
        monkeypatch.setenv("FK_GQF_SMALL", "0")  # build the table through the rebuild path
        g.bulk_insert(pool, cnt)
        o.bulk_insert(pool, cnt)
        monkeypatch.setenv("FK_GQF_SMALL", limit)
        same_image(g, o)
        for step in range(10):
            d = pool[rng.integers(0, len(pool), int(rng.integers(1, 2000)))]
            d = np.concatenate([d, d[: len(d) // 3], rng.integers(0, 2 ** 60, 50, dtype=np.uint64)])
            dc = rng.integers(1, 200, len(d)).astype(np.uint64) if step % 2 else None
            if step % 3 == 2:
                got, want = g.delete_many(d, dc), o.delete_many(d, dc)
            else:
                got, want = g.bulk_delete(d, dc), o.bulk_delete(d, dc)
            assert np.array_equal(np.asarray(got).astype(bool), np.asarray(want).astype(bool)), (limit, step)
            same_image(g, o)
        g.validate()


@pytest.mark.parametrize("order", ["point", "bulk"])
def test_small_batches_hitting_capacity_fall_back_exactly(oracle, monkeypatch, order):
    """A small batch that overflows (load ceiling) on the region-local path
    leaves the table untouched there and is replayed by the exact path: the
    partial image equals the reference's, batch after batch."""
    from paper_2212_09005_b200 import CapacityError, Gqf
    rng = np.random.default_rng(77)
    g = Gqf(q=12, r=8, seed=1)
    o = _oracle(g, oracle)
    base = rng.integers(0, 2 ** 60, 3700, dtype=np.uint64)
    g.bulk_insert(base)
    o.bulk_insert(base)
    monkeypatch.setenv("FK_GQF_SMALL", "100000")
    raised = 0
    for step in range(40):
        keys = rng.integers(0, 2 ** 60, 12, dtype=np.uint64)
        cnt = rng.integers(1, 4, 12).astype(np.uint64)
        try:
            if order == "point":
                g.insert_many(keys, cnt)
            else:
                g.bulk_insert(keys, cnt)
        except CapacityError:
            raised += 1
        if order == "point":
            o.insert_many(keys, cnt)
        else:
            o.bulk_insert(keys, cnt)
        same_image(g, o)
    assert raised > 0


@pytest.mark.parametrize("order", ["point", "bulk"])
def test_small_batch_at_load_ceiling_keeps_input_order(oracle, order):
    """Occupancy max_occupied - 1, batch [new key A, existing key B] with B's
    increment not growing its group and fp(B) < fp(A): the reference inserts A
    (occupancy reaches the ceiling) and raises on B (pk:592-593).  The
    region-local small path applies in sorted order and must not succeed
    where the reference raises.  q = 15: four quotient regions, so regions of
    one parity run in parallel."""
    from paper_2212_09005_b200 import CapacityError, Gqf
    g = Gqf(q=15, r=8, seed=4)
    o = _oracle(g, oracle)
    p = g.params
    rng = np.random.default_rng(123)
    pairs = rng.choice(1 << (p.q + p.r), size=p.max_occupied + 64, replace=False)
    pairs = [(int(x) >> p.r, int(x) & 0xFF) for x in pairs]
    # B: (quotient 5, remainder 10) with count 1000 (4 slots; 1001 is 4 slots too)
    pairs = [pr for pr in pairs if pr[0] not in (5, 20000)]
    kb = craft(g, [(5, 10)])
    g.bulk_insert(kb, np.array([1000], np.uint64))
    o.bulk_insert(kb, np.array([1000], np.uint64))
    fill = craft(g, pairs[: p.max_occupied - 1 - int(o.stats[0])])
    g.bulk_insert(fill)
    o.bulk_insert(fill)
    assert int(o.stats[0]) == p.max_occupied - 1
    same_image(g, o)
    ka = craft(g, [(20000, 7)])  # another region, fingerprint above B's
    batch = np.concatenate([ka, kb])
    if order == "point":
        with pytest.raises(CapacityError):
            g.insert_many(batch)
        assert o.insert_many(batch) == (1, 1)
    else:
        # bulk order is sorted (B, then A): the reference succeeds, and so must we
        assert o.bulk_insert(batch) == []
        g.bulk_insert(batch)
    same_image(g, o)
    assert int(g._stats[0]) <= p.max_occupied


@pytest.mark.parametrize("r", [8, 16])
def test_device_enumerate_equals_host_decode(r):
    """enumerate_items decodes on the device (fk_gqf_enumerate); it yields
    exactly the host decode of the mirrored image, in fingerprint order."""
    from paper_2212_09005_b200 import Gqf
    rng = np.random.default_rng(90 + r)
    g = Gqf(q=15, r=r, seed=3)
    pool = rng.integers(0, 2 ** 60, 6000, dtype=np.uint64)
    g.bulk_insert(pool[rng.integers(0, len(pool), 12000)], rng.integers(1, 400, 12000).astype(np.uint64))
    g.bulk_delete(pool[::5])
    dev = list(g.enumerate_items())
    host = list(g._enumerate_host())
    assert dev == host and len(dev) == g.distinct_items
    fps = [f for f, _ in dev]
    assert fps == sorted(fps)
    assert sum(c for _, c in dev) == g.total_items


@pytest.mark.parametrize("r", [8, 16])
def test_runs_spilling_into_padding(oracle, r):
    """Quotients packed against the end of the logical table push their runs
    into the padding region: the derived run index must still find them
    (counts, find_run, device enumeration) exactly like the reference."""
    from paper_2212_09005_b200 import Gqf
    rng = np.random.default_rng(5 + r)
    g = Gqf(q=12, r=r, seed=11)
    o = _oracle(g, oracle)
    qs = rng.integers(3900, 4096, 700)
    rems = rng.integers(1, 1 << r, 700)
    keys = np.unique(craft(g, list(zip(qs.tolist(), rems.tolist()))))
    cnt = rng.integers(1, 50, len(keys)).astype(np.uint64)
    g.bulk_insert(keys, cnt)
    o.bulk_insert(keys, cnt)
    same_image(g, o)
    _, _, ends = g._derive_structure()
    assert ends.max() >= 1 << 12  # runs end in the padding
    assert np.array_equal(g.count_many(keys), o.count_many(keys))
    for qt in (3900, 4000, 4095):
        assert g.find_run(qt) == o.find_run(qt)
    assert list(g.enumerate_items()) == list(g._enumerate_host())
    g.validate()


@pytest.mark.parametrize("seed,q", [(0, 11), (1, 11), (2, 11), (3, 6), (4, 7)])
def test_churn_fuzz_vs_oracle(oracle, monkeypatch, seed, q):
    """Random churn at high load (the reference's dict-oracle fuzz, here
    against the oracle image): point and bulk inserts/deletes with counts,
    small batches (region-local paths) and large ones (rebuild), capacity
    errors included; image, counts and found flags after every step."""
    from paper_2212_09005_b200 import CapacityError, Gqf
    rng = np.random.default_rng(500 + seed)
    g = Gqf(q=q, r=8, seed=seed)
    o = _oracle(g, oracle)
    pool = rng.integers(0, 2 ** 62, 3 << (q - 2), dtype=np.uint64)
    # a quarter of the pool packed against the end of the table (runs into the padding)
    m = 1 << (q - 2)
    tail = craft(g, [(int(x), int(y)) for x, y in zip(rng.integers((1 << q) - max(8, m // 2), 1 << q, m),
                                                       rng.integers(0, 256, m))])
    pool = np.concatenate([pool, tail])
    raised = 0
    for step in range(80):
        size = int(rng.choice([1, 5, 40, 400])) if q > 8 else int(rng.choice([1, 3, 12, 40]))
        keys = pool[rng.integers(0, len(pool), size)]
        cnt = rng.integers(1, 20, size).astype(np.uint64) if rng.random() < 0.5 else None
        small = rng.random() < 0.5
        monkeypatch.setenv("FK_GQF_SMALL", "100000" if small else "0")
        op = rng.integers(0, 4)
        if op == 0:
            try:
                g.insert_many(keys, cnt)
            except CapacityError:
                raised += 1
            o.insert_many(keys, cnt)
        elif op == 1:
            try:
                g.bulk_insert(keys, cnt)
            except CapacityError:
                pass
            try:
                o.bulk_insert(keys, cnt)
            except Exception:
                pass
        elif op == 2:
            assert np.array_equal(np.asarray(g.delete_many(keys, cnt)), o.delete_many(keys, cnt).astype(bool))
        else:
            assert np.array_equal(np.asarray(g.bulk_delete(keys, cnt)),
                                  np.asarray(o.bulk_delete(keys, cnt)).astype(bool))
        same_image(g, o)
        assert np.array_equal(g.count_many(pool), o.count_many(pool))
    assert raised > 0  # the capacity paths ran
    g.validate()
    assert list(g.enumerate_items()) == list(g._enumerate_host())


@pytest.mark.parametrize("q,r,n,dup", [(20, 8, 600_000, 0), (18, 16, 150_000, 7), (22, 16, 2_000_000, 3)])
def test_partition_counting_equals_full_sort(oracle, monkeypatch, q, r, n, dup):
    """Plain counted bulk inserts of large batches are counted by two MSD
    partition passes and shared-memory hash aggregation (k_part_*); the
    image equals the sort + run-length path's (FK_GQF_PART=0) and, where the
    C oracle is quick, the oracle's.  (22, 16): 38-bit fingerprints."""
    from paper_2212_09005_b200 import Gqf
    rng = np.random.default_rng(q + r)
    base = rng.integers(0, 2 ** 63, n, dtype=np.uint64)
    keys = np.concatenate([base] + [base[: n // (4 * dup)]] * dup) if dup else base
    keys = rng.permutation(keys)
    monkeypatch.setenv("FK_GQF_PART_MIN", "1000")
    a = Gqf(q=q, r=r)
    a.bulk_insert(keys)
    monkeypatch.setenv("FK_GQF_PART", "0")
    b = Gqf(q=q, r=r)
    b.bulk_insert(keys)
    for name in ("_slots", "_occupieds", "_runends", "_offsets", "_stats"):
        assert np.array_equal(getattr(a, name), getattr(b, name)), name
    a.validate()
    if n <= 600_000:
        o = _oracle(a, oracle)
        assert o.bulk_insert(keys) == []
        same_image(a, o)


def test_partition_counting_overflow_falls_back(oracle, monkeypatch):
    """A partition with more distinct fingerprints than its shared-memory
    table holds (table capped at 8 entries here) makes the batch recount on
    the sort + run-length path: same image and counts as the oracle."""
    from paper_2212_09005_b200 import Gqf
    rng = np.random.default_rng(11)
    base = rng.integers(0, 2 ** 63, 60_000, dtype=np.uint64)
    keys = rng.permutation(np.concatenate([base, np.full(20_000, base[7], np.uint64)]))
    monkeypatch.setenv("FK_GQF_PART_MIN", "1000")
    monkeypatch.setenv("FK_GQF_PART_SLOTS", "8")
    g = Gqf(q=17, r=16)
    o = _oracle(g, oracle)
    g.bulk_insert(keys)
    assert o.bulk_insert(keys) == []
    same_image(g, o)
    assert g.count_many(base[7:8])[0] == o.count_many(base[7:8])[0]


def _unmix64(h):
    """Inverse of the SplitMix64 finalizer (hashing.mix64): keys whose
    fingerprints are chosen."""
    M = (1 << 64) - 1

    def unshift(x, s):
        y = x
        for _ in range(64 // s + 1):
            y = x ^ (y >> s)
        return y & M

    x = unshift(h & M, 31)
    x = (x * pow(0x94D049BB133111EB, -1, 1 << 64)) & M
    x = unshift(x, 27)
    x = (x * pow(0xBF58476D1CE4E5B9, -1, 1 << 64)) & M
    return unshift(x, 30)


def test_partition_counting_long_clusters_sort(oracle, monkeypatch):
    """The aggregation's order-preserving hash puts fingerprints that share
    their top bits in one probe cluster; 3000 consecutive fingerprints in one
    partition make a cluster too long for the odd-even rounds, so the
    partition is ordered by the bitonic fallback: same image as the sort +
    run-length path and the oracle."""
    from paper_2212_09005_b200 import Gqf
    from paper_2212_09005_b200.hashing import fingerprint_many
    q, r = 18, 16
    g = Gqf(q=q, r=r)
    seed = g.params.seed
    top = 0x2A5 << (q + r - 10)
    want = [top | j for j in range(3000)]
    structured = np.array([_unmix64(h) ^ seed for h in want], dtype=np.uint64)
    assert np.array_equal(fingerprint_many(structured, seed, q + r), np.array(want, dtype=np.uint64))
    rng = np.random.default_rng(5)
    keys = rng.permutation(np.concatenate([np.repeat(structured, 3),
                                           rng.integers(0, 2 ** 63, 40_000, dtype=np.uint64)]))
    monkeypatch.setenv("FK_GQF_PART_MIN", "1000")
    g.bulk_insert(keys)
    monkeypatch.setenv("FK_GQF_PART", "0")
    b = Gqf(q=q, r=r)
    b.bulk_insert(keys)
    for name in ("_slots", "_occupieds", "_runends", "_offsets", "_stats"):
        assert np.array_equal(getattr(g, name), getattr(b, name)), name
    o = _oracle(g, oracle)
    assert o.bulk_insert(keys) == []
    same_image(g, o)
    assert (g.count_many(structured) == 3).all()


def _host_cluster_stats(g):
    """The reference's cluster_stats (gqf.py:416-428) on the host mirrors."""
    occ = np.unpackbits(g._occupieds.view(np.uint8), bitorder="little")
    run = np.unpackbits(g._runends.view(np.uint8), bitorder="little")
    quotients, ends = np.flatnonzero(occ), np.flatnonzero(run)
    if not len(quotients):
        return {"num_clusters": 0, "max_cluster": 0, "mean_cluster": 0.0}
    starts = np.maximum(quotients, np.concatenate(([-1], ends[:-1])) + 1)
    breaks = np.flatnonzero(starts[1:] > ends[:-1] + 1)
    c_starts = np.concatenate(([0], breaks + 1))
    c_ends = np.concatenate((breaks, [len(starts) - 1]))
    lengths = ends[c_ends] - starts[c_starts] + 1
    return {"num_clusters": int(len(lengths)), "max_cluster": int(lengths.max()),
            "mean_cluster": float(lengths.mean())}


@pytest.mark.parametrize("q,r,load", [(12, 8, 0.0), (14, 8, 0.5), (16, 16, 0.9), (20, 8, 0.93)])
def test_cluster_stats_on_device_equal_reference_formula(q, r, load):
    """Gqf.cluster_stats runs on the device (fk_gqf_cluster_stats): equal to
    the reference's host derivation over the same image, empty table and
    runs spilling into the padding included."""
    from paper_2212_09005_b200 import Gqf
    g = Gqf(q=q, r=r)
    n = int(load * (1 << q) * 0.8)
    if n:
        rng = np.random.default_rng(q)
        keys = rng.integers(0, 2 ** 63, n, dtype=np.uint64)
        g.bulk_insert(np.concatenate([keys, keys[: n // 5]]))
    assert g.cluster_stats() == _host_cluster_stats(g)


@pytest.mark.parametrize("q", [10, 16])
def test_r32_point_bulk_and_counts_vs_oracle(oracle, q):
    """32-bit remainders (GqfParams admits r = 32, gqf.py:52-95; u32 slots):
    point and bulk counted inserts, counts, bulk and point deletes and the
    image equal the oracle's."""
    from paper_2212_09005_b200 import Gqf
    rng = np.random.default_rng(q + 32)
    n = int(0.4 * (1 << q))
    keys = rng.integers(0, 2 ** 63, n, dtype=np.uint64)
    g = Gqf(q=q, r=32)
    o = _oracle(g, oracle)
    assert g._slots.dtype == np.uint32
    g.bulk_insert(np.concatenate([keys, keys[: n // 3]]))
    assert o.bulk_insert(np.concatenate([keys, keys[: n // 3]])) == []
    same_image(g, o)
    extra = rng.integers(0, 2 ** 63, n // 20, dtype=np.uint64)
    cnt = rng.integers(1, 40, n // 20).astype(np.uint64)
    g.insert_many(extra, cnt)
    o.insert_many(extra, cnt)
    same_image(g, o)
    probe = np.concatenate([keys[::3], extra, rng.integers(0, 2 ** 63, 2000, dtype=np.uint64)])
    assert np.array_equal(g.count_many(probe), o.count_many(probe))
    d = np.concatenate([keys[::2], keys[:50]])
    assert np.array_equal(g.bulk_delete(d), o.bulk_delete(d))
    same_image(g, o)
    assert np.array_equal(g.delete_many(extra[:20], cnt[:20]), o.delete_many(extra[:20], cnt[:20]))
    same_image(g, o)
    g.validate()


@pytest.mark.parametrize("r", [8, 16])
def test_local_apply_in_place_equals_oracle(oracle, monkeypatch, r):
    """Batches that touch at most a quarter of the regions are applied in
    place, region by region (apply_local_t: only the regions holding new
    items and their successors are decoded, merged, placed and rewritten);
    images equal the oracle's after every batch -- inserts with and without
    counts, point and bulk order, deletes with absent keys -- and the shift
    metric equals the whole-table path's (FK_GQF_LOCAL=0)."""
    from paper_2212_09005_b200 import Gqf
    monkeypatch.setenv("FK_GQF_SMALL", "0")  # the small-batch path would take these batches
    rng = np.random.default_rng(40 + r)
    q = 22
    base = rng.integers(0, 2 ** 62, int(0.6 * (1 << q)), dtype=np.uint64)
    g, h = Gqf(q=q, r=r, seed=3), Gqf(q=q, r=r, seed=3)
    o = _oracle(g, oracle)
    for f in (g, h, o):
        f.bulk_insert(base)
    cur, local_runs = g._cur, 0
    for step in range(10):
        keys = rng.integers(0, 2 ** 62, int(rng.integers(5, 40)), dtype=np.uint64)
        keys = np.concatenate([keys, base[rng.integers(0, len(base), 10)]])  # <= 50 regions + successors
        cnt = rng.integers(1, 30, len(keys)).astype(np.uint64) if step % 2 else None
        kind = step % 4
        outs = []
        for f, local in ((g, "1"), (h, "0"), (o, None)):
            if local is not None:
                monkeypatch.setenv("FK_GQF_LOCAL", local)
            if kind == 0:
                outs.append(f.bulk_insert(keys, cnt))
            elif kind == 1:
                outs.append(f.insert_many(keys, cnt))
            elif kind == 2:
                outs.append(np.asarray(f.bulk_delete(keys, cnt)).astype(bool))
            else:
                outs.append(np.asarray(f.delete_many(keys, cnt)).astype(bool))
        if kind >= 2:
            assert np.array_equal(outs[0], outs[2]) and np.array_equal(outs[1], outs[2]), step
        same_image(g, o)
        assert g.shifted_slots == h.shifted_slots, step
        local_runs += g._cur is cur  # applied in place: the image was not swapped for a rebuilt one
        cur = g._cur
    assert local_runs == 10
    g.validate()


def test_local_apply_capacity_falls_back_exactly(oracle, monkeypatch):
    """A mid-size point batch that crosses the load ceiling: the local path's
    plan pass sees the ceiling and the exact sequential path reproduces the
    reference's partial application and CapacityError."""
    from paper_2212_09005_b200 import CapacityError, Gqf
    monkeypatch.setenv("FK_GQF_SMALL", "0")
    rng = np.random.default_rng(77)
    q = 22
    g = Gqf(q=q, r=8, max_load=0.5)
    o = _oracle(g, oracle)
    # every occurrence of the fill takes one slot: 50 slots left under the ceiling
    fill = rng.integers(0, 2 ** 62, g.params.max_occupied - 50, dtype=np.uint64)
    g.bulk_insert(fill)
    o.bulk_insert(fill)
    keys = rng.integers(0, 2 ** 62, 25, dtype=np.uint64)  # ~4 slots each
    cnt = np.full(25, 400, np.uint64)
    with pytest.raises(CapacityError):
        g.insert_many(keys, cnt)
    code, _ = o.insert_many(keys, cnt)
    assert code != 0
    same_image(g, o)
