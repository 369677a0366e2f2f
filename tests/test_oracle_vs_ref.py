"""The C restatement (oracle/) against the reference's OWN compiled kernels
(oracle/_ref, built from /root/reference/pkg/src/filterkit/_ckernels.pyx by
oracle/build_ref.sh) on fresh random workloads -- the second pin of the
oracle next to the golden fixtures.  CPU only; skipped when the reference
build is absent (it is built here by __graft_entry__.build())."""

import numpy as np
import pytest

from conftest import counter_keys

ref_model = pytest.importorskip("oracle.ref_model")
pytestmark = pytest.mark.skipif(not ref_model.available(), reason="oracle/_ref not built")


@pytest.mark.parametrize("nb,load,seed", [(256, 0.9, 0), (4096, 0.95, 3), (100, 1.1, 7)])
def test_point_tcf_oracle_equals_reference(oracle, nb, load, seed):
    from paper_2212_09005_b200 import TcfParams
    p = TcfParams(num_blocks=nb, seed=seed)
    o = oracle.OracleTcf(nb, 16, 16, np.uint16, p.backing_slots, p.cut_slots, p.probe_limit, seed)
    r = ref_model.RefTcf(nb, backing_slots=p.backing_slots, cut_slots=p.cut_slots, probe_limit=p.probe_limit,
                         seed=seed)
    keys = counter_keys(100 + seed, int(load * nb * 16))
    dup = np.concatenate([keys, keys[: len(keys) // 7]])
    assert np.array_equal(o.insert_many(dup), r.insert_many(dup, threads=1))
    assert np.array_equal(o.blocks, r.blocks) and np.array_equal(o.backing, r.backing)
    probe = np.concatenate([keys[::3], counter_keys(900 + seed, 5000)])
    assert np.array_equal(o.query_many(probe).astype(np.uint8), r.query_many(probe, threads=1))
    d = np.concatenate([keys[::2], counter_keys(901 + seed, 500)])
    assert np.array_equal(o.delete_many(d), r.delete_many(d, threads=1))
    assert np.array_equal(o.blocks, r.blocks) and np.array_equal(o.backing, r.backing)


@pytest.mark.parametrize("nb,load", [(64, 0.85), (512, 0.9), (512, 1.02)])
def test_bulk_tcf_oracle_equals_reference(oracle, nb, load):
    from paper_2212_09005_b200 import BulkTcfParams
    p = BulkTcfParams(num_blocks=nb)
    o = oracle.OracleBulkTcf(nb, 128, 16, np.uint16, p.backing_slots, p.cut_slots, p.probe_limit, 0)
    r = ref_model.RefBulkTcf(nb, backing_slots=p.backing_slots, cut_slots=p.cut_slots, probe_limit=p.probe_limit)
    keys = counter_keys(33 + nb, int(load * nb * 128))
    for part in np.array_split(keys, 3):  # (the baseline glue returns no failed-key list)
        o.insert_batch(part)
        r.insert_batch(part, workers=1)
    assert np.array_equal(o.blocks, r.blocks) and np.array_equal(o.fill, r.fill)
    assert np.array_equal(o.backing, r.backing)
    probe = np.concatenate([keys[::5], counter_keys(77, 4000)])
    assert np.array_equal(np.asarray(o.query_batch(probe)).astype(bool),
                          np.asarray(r.query_batch(probe, workers=1)).astype(bool))
    d = keys[::4]
    assert np.array_equal(np.asarray(o.delete_batch(d)).astype(bool),
                          np.asarray(r.delete_batch(d, workers=1)).astype(bool))
    assert np.array_equal(o.blocks, r.blocks) and np.array_equal(o.fill, r.fill)


@pytest.mark.parametrize("q,r_bits", [(12, 8), (14, 16)])
def test_gqf_oracle_equals_reference(oracle, q, r_bits):
    rng = np.random.default_rng(q * 10 + r_bits)
    o = oracle.OracleGqf(q, r_bits, 0, int(0.95 * (1 << q)))
    r = ref_model.RefGqf(q, r_bits)
    pool = rng.integers(0, 2 ** 62, int(0.25 * (1 << q)), dtype=np.uint64)
    keys = pool[rng.integers(0, len(pool), int(0.4 * (1 << q)))]
    cnt = rng.integers(1, 40, len(keys)).astype(np.uint64)
    o.bulk_insert(keys, cnt)
    r.bulk_insert(keys, cnt, workers=1)
    img = o.image()
    assert np.array_equal(img["slots"], r.slots) and np.array_equal(img["occupieds"], r.occ)
    assert np.array_equal(img["runends"], r.run) and np.array_equal(img["offsets"], r.offs)
    assert np.array_equal(img["stats"], r.stats)
    assert np.array_equal(o.count_many(pool), r.count_many(pool))
    d = pool[rng.integers(0, len(pool), len(pool) // 2)]
    dc = rng.integers(1, 30, len(d)).astype(np.uint64)
    assert np.array_equal(np.asarray(o.bulk_delete(d, dc)).astype(bool),
                          np.asarray(r.bulk_delete(d, dc, workers=1)).astype(bool))
    img = o.image()
    assert np.array_equal(img["slots"], r.slots) and np.array_equal(img["stats"], r.stats)
