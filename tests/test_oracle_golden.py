"""The CPU oracle (oracle/) against golden vectors produced by the reference
itself (tests/golden/make_golden.py).  This pins the checker every GPU parity
test relies on."""

import numpy as np
import pytest

from oracle import model as M


def _dt(bits):
    return {8: np.uint8, 16: np.uint16, 32: np.uint32, 64: np.uint64}[bits]


def test_hashing_vectors(golden):
    h = golden("hashing")
    ks = h["keys"]
    assert np.array_equal(M.mix64_many(ks), h["mix"])
    assert np.array_equal(M.fingerprint_many(ks, 9), h["fp_s9"])
    assert np.array_equal(M.fingerprint_many(ks, 0), h["fp_s0"])
    fp = h["fp_s9"]
    for nb in (1, 100, 8192, 65536, 2 ** 24, 1000003):
        b1, b2 = M.potc_pair_many(fp, nb)
        assert np.array_equal(b1, h["b1_%d" % nb]) and np.array_equal(b2, h["b2_%d" % nb])
    for bits in (30, 36, 40):
        assert np.array_equal(M.fingerprint_many(ks, 0, bits), h["fpbits_%d" % bits])
    # SURVEY 8(c) fixed vectors generated from the reference
    assert int(M.mix64_many([1])[0]) == 0x5692161D100B05E5
    assert int(M.fingerprint_many([12345], 9)[0]) == 0xD3A4DBED91799966


def test_encoded_length_matches_reference_codec(golden):
    g = golden("countgroups")
    for r, rem, count, length in g["meta"].tolist():
        assert M.encoded_length(rem, count, r) == length


@pytest.mark.parametrize("name", ["w8", "w16", "w32", "w64", "nob", "b7", "b32"])
def test_point_tcf_matches_reference(golden, name):
    t = golden("tcf_point")
    nb, B, f, w, bs, cut, pl, _ = t[name + "_geom"].tolist()
    o = M.OracleTcf(nb, B, f, _dt(w), bs, cut, pl, 0)
    vb = w - f
    codes = o.insert_many(t[name + "_keys"], t[name + "_vals"] if vb else None)
    assert np.array_equal(codes, t[name + "_codes"])
    assert np.array_equal(o.blocks.astype(np.uint64), t[name + "_blocks_ins"])
    assert np.array_equal(o.backing.astype(np.uint64), t[name + "_backing_ins"])
    found, vals = o.query_values_many(t[name + "_probe"])
    assert np.array_equal(found.astype(np.uint8), t[name + "_found"])
    assert np.array_equal(vals, t[name + "_qvals"])
    rem = o.delete_many(t[name + "_dkeys"])
    assert np.array_equal(rem.astype(np.uint8), t[name + "_removed"])
    assert np.array_equal(o.blocks.astype(np.uint64), t[name + "_blocks_del"])
    assert np.array_equal(o.backing.astype(np.uint64), t[name + "_backing_del"])
    c = o.counters
    assert [c["inserts_ok"], c["inserts_backing"], c["deletes_ok"]] == t[name + "_counters"].tolist()


@pytest.mark.parametrize("name", ["a", "b", "c"])
def test_bulk_tcf_matches_reference(golden, name):
    t = golden("tcf_bulk")
    nb = int(t[name + "_nb"][0])
    o = M.OracleBulkTcf(nb, 128, 16, np.uint16, int(round(nb * 128 * 0.01)), 96, 20, 0)
    failed = o.insert_batch(t[name + "_keys"])
    assert np.array_equal(failed, t[name + "_failed"])
    assert np.array_equal(o.blocks.astype(np.uint64), t[name + "_blocks_ins"])
    assert np.array_equal(o.fill, t[name + "_fill_ins"])
    assert np.array_equal(o.backing.astype(np.uint64), t[name + "_backing_ins"])
    assert np.array_equal(o.query_batch(t[name + "_probe"]).astype(np.uint8), t[name + "_found"])
    assert np.array_equal(o.delete_batch(t[name + "_dkeys"]).astype(np.uint8), t[name + "_removed"])
    assert np.array_equal(o.blocks.astype(np.uint64), t[name + "_blocks_del"])
    assert np.array_equal(o.fill, t[name + "_fill_del"])
    assert np.array_equal(o.backing.astype(np.uint64), t[name + "_backing_del"])
    c = o.counters
    assert [c["inserts_ok"], c["inserts_backing"], c["deletes_ok"]] == t[name + "_counters"].tolist()


def _same_image(o, t, pre):
    img = o.image()
    for nm in ("slots", "occupieds", "runends", "offsets", "stats"):
        assert np.array_equal(img[nm], t[pre + nm]), (pre, nm)


@pytest.mark.parametrize("r", [8, 16])
def test_gqf_matches_reference(golden, r):
    t = golden("gqf")
    pre = "r%d_" % r
    o = M.OracleGqf(14, r, 0, int(0.95 * (1 << 14)))
    code, _ = o.insert_many(t[pre + "k"], t[pre + "c"])
    assert code == 0
    _same_image(o, t, pre + "ins_")
    assert np.array_equal(o.count_many(t[pre + "k"]), t[pre + "count"])
    assert np.array_equal(o.delete_many(t[pre + "dk"], t[pre + "dc"]).astype(np.uint8), t[pre + "dfound"])
    _same_image(o, t, pre + "del_")
    assert o.bulk_insert(t[pre + "k2"]) == []
    _same_image(o, t, pre + "bulk_")
    assert np.array_equal(o.bulk_delete(t[pre + "kk"]).astype(np.uint8), t[pre + "bfound"])
    _same_image(o, t, pre + "bdel_")


def test_gqf_duplicates_and_capacity(golden):
    t = golden("gqf")
    o = M.OracleGqf(16, 8, 0, int(0.95 * (1 << 16)))
    assert o.bulk_insert(t["ur_keys"]) == []
    _same_image(o, t, "ur_")
    uq = np.unique(t["ur_keys"])
    assert np.array_equal(o.count_many(uq), t["ur_count"])
    o = M.OracleGqf(10, 8, 0, int(0.95 * (1 << 10)))
    code, idx = o.insert_many(t["cap_k"])
    assert (code != 0) == bool(t["cap_err"][0])
    _same_image(o, t, "cap_")


def test_kmer_windows_host_match_reference_golden(golden, tmp_path):
    """The host k-mer extractor (and the read parser the device path shares)
    equals the reference's on its own fixture (tests/golden/kmer.npz)."""
    from paper_2212_09005_b200.workloads import kmer_windows
    g = golden("kmer")
    p = tmp_path / "reads.fq"
    p.write_bytes(g["text"].tobytes())
    for k in (1, 4, 11, 21, 31, 32):
        assert np.array_equal(kmer_windows(str(p), k), g["k%d" % k]), k
