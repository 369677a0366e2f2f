"""Full-size checks on the B200 (BASELINE.json configs at their real sizes):
bit-exact against the oracle where the oracle finishes in seconds (2^24
slots, the one-barrier ordered kernel at 0.9 load), and size-independent
properties at 2^28 slots / q = 26 where it would not."""

import numpy as np
import pytest

from conftest import counter_keys

pytestmark = pytest.mark.gpu


def test_ordered_2p24_at_0p9_load_bit_exact(oracle):
    """15.1 M keys into 2^24 slots (the one-barrier kernel's regime, with
    backing deferrals at 0.9 load): codes, image, counters, deletes."""
    from paper_2212_09005_b200 import Tcf
    f = Tcf(num_blocks=1 << 20)
    p = f.params
    o = oracle.OracleTcf(p.num_blocks, 16, 16, np.uint16, p.backing_slots, p.cut_slots, p.probe_limit, 0)
    keys = counter_keys(2024, int(0.9 * (1 << 24)))
    codes = f.insert_many(keys)
    assert np.array_equal(codes, o.insert_many(keys))
    assert int((codes == 2).sum()) > 0  # the backing phase ran
    assert np.array_equal(f._blocks, o.blocks) and np.array_equal(f._backing, o.backing)
    d = keys[::3]
    assert np.array_equal(f.delete_many(d), o.delete_many(d).astype(bool))
    assert np.array_equal(f._blocks, o.blocks) and np.array_equal(f._backing, o.backing)
    assert f.counters == o.counters


@pytest.mark.parametrize("mode", ["ordered", "concurrent"])
def test_c3_2p28_properties(mode):
    """C3 at full size: nothing FULL, no false negatives, FPR under the
    two-block bound; deleting every inserted key succeeds except where an
    earlier delete took an aliased slot (16-bit tags: a few per million, the
    reference's own sequential semantics), and exactly those slots stay."""
    import torch
    from paper_2212_09005_b200 import Tcf
    from paper_2212_09005_b200.workloads import TAG_FPR, TAG_UNIFORM, counter_stream_device
    n = int(0.9 * (1 << 28))
    keys = counter_stream_device(1, TAG_UNIFORM, n)
    negs = counter_stream_device(2, TAG_FPR, 1 << 24)
    f = Tcf(num_blocks=1 << 24, mode=mode)
    codes = f.insert_many(keys)
    assert int((codes == 3).sum()) == 0
    assert bool(f.query_many(keys).all())
    fpr = float(f.query_many(negs).float().mean())
    assert fpr <= 2 * 16 / 2 ** 16
    c = f.counters
    assert c["inserts_ok"] == n
    removed = f.delete_many(keys)
    c = f.counters
    assert c["deletes_ok"] == int(removed.sum()) >= n - n // 100_000
    main = int(((f._t.dev["blocks"].view(torch.int16).to(torch.int32) & 0xFFFF) > 1).sum())
    back = int(((f._t.dev["backing"].view(torch.int16).to(torch.int32) & 0xFFFF) > 1).sum())
    assert main + back == n - c["deletes_ok"]


def test_c4_q26_counting_properties():
    """C4-style counting at q = 26, load 0.9: no undercounts, >= 99.8 % exact,
    items = occurrences, device validation clean, empty after delete."""
    import sys
    import torch
    sys.path.insert(0, __import__("conftest").ROOT)
    import bench
    from paper_2212_09005_b200 import Gqf
    w = bench.kmer_zipf_workload(torch, 26, 0.9, 1, torch.device("cuda", 0))
    g = Gqf(q=26, r=8)
    g.bulk_insert(w["occ"])
    assert g.total_items == w["n_occ"]
    counts = g.count_many(w["uniq"])
    assert int((counts < w["counts"]).sum()) == 0
    assert float((counts == w["counts"]).float().mean()) >= 0.998
    assert 0.85 <= g.load_factor() <= 0.95
    g.validate()
    g.bulk_delete(w["uniq"])
    assert g.occupied_slots == 0 and g.total_items == 0
    g.validate()


def test_bulk_tcf_2p23_block_parallel_route_bit_exact(oracle):
    """2^23 slots (2^16 blocks: the block-parallel routing path) at 0.9 load
    in two batches: failed keys, image, fill, backing and deletes equal the
    oracle's."""
    from paper_2212_09005_b200 import BulkTcf
    f = BulkTcf(num_blocks=1 << 16)
    p = f.params
    o = oracle.OracleBulkTcf(p.num_blocks, 128, 16, np.uint16, p.backing_slots, p.cut_slots, p.probe_limit, 0)
    keys = counter_keys(2323, int(0.9 * (1 << 23)))
    for part in np.array_split(keys, 2):
        assert np.array_equal(np.asarray(f.insert_batch(part)), np.asarray(o.insert_batch(part)))
    assert np.array_equal(f._blocks, o.blocks) and np.array_equal(f._fill, o.fill)
    assert np.array_equal(f._backing, o.backing)
    d = keys[::3]
    assert np.array_equal(np.asarray(f.delete_batch(d)), np.asarray(o.delete_batch(d)).astype(bool))
    assert np.array_equal(f._blocks, o.blocks) and np.array_equal(f._fill, o.fill)
