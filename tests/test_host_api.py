"""Host-side API parity: parameter derivations, hashing helpers and the
count-group codec against golden vectors from the reference."""

import numpy as np
import pytest

from paper_2212_09005_b200 import countgroups, hashing
from paper_2212_09005_b200.tcf import TcfParams


def test_tcf_param_derivations(golden):
    for nb, B, frac, sf, bs, cut in golden("params")["tcf"].tolist():
        p = TcfParams(num_blocks=nb, block_slots=B, backing_fraction=frac / 1000, shortcut_fraction=sf / 100)
        assert (p.backing_slots, p.cut_slots) == (bs, cut), (nb, B, frac, sf)


@pytest.mark.parametrize("kw", [dict(num_blocks=0), dict(num_blocks=4, tag_bits=2),
                                dict(num_blocks=4, tag_bits=17), dict(num_blocks=4, block_slots=65),
                                dict(num_blocks=4, group_width=17), dict(num_blocks=4, backing_fraction=1.5),
                                dict(num_blocks=4, shortcut_fraction=0.0)])
def test_tcf_param_validation(kw):
    with pytest.raises(ValueError):
        TcfParams(**kw)


def test_tile_width():
    assert TcfParams(num_blocks=1, group_width=1).tile_width == 1
    assert TcfParams(num_blocks=1, group_width=3).tile_width == 2
    assert TcfParams(num_blocks=1, group_width=16).tile_width == 16
    assert TcfParams(num_blocks=1, block_slots=32, group_width=32).tile_width == 32


def test_host_hashing_matches_reference(golden):
    h = golden("hashing")
    ks = h["keys"]
    assert np.array_equal(hashing.mix64_many(ks), h["mix"])
    assert np.array_equal(hashing.fingerprint_many(ks, 9), h["fp_s9"])
    fp = h["fp_s9"]
    for nb in (100, 65536, 2 ** 24):
        b1, b2 = hashing.potc_pair_many(fp, nb)
        assert np.array_equal(b1, h["b1_%d" % nb]) and np.array_equal(b2, h["b2_%d" % nb])
    for size in (10486, 2684355):
        st = np.array([hashing.backing_schedule(int(x), size) for x in fp[:300].tolist()], dtype=np.uint64)
        assert np.array_equal(st[:, 0], h["bstart_%d" % size][:300])
        assert np.array_equal(st[:, 1], h["bstep_%d" % size][:300])
    assert np.array_equal(hashing.remap_tag_many(fp & np.uint64(0xFFFF)), h["remap16"])
    assert hashing.mix64(1) == 0x5692161D100B05E5


def test_countgroup_codec_matches_reference(golden):
    g = golden("countgroups")
    words = g["words"].tolist()
    pos = 0
    for r, rem, count, length in g["meta"].tolist():
        ref = words[pos:pos + length]
        pos += length
        assert countgroups.encode_group(rem, count, r) == ref
        assert countgroups.encoded_length(rem, count, r) == length
        assert countgroups.parse_group(ref, 0, length - 1, r) == (rem, count, length)
    assert countgroups.encode_group(7, 300, 8) == [7, 4, 43, 7]  # test_countgroups.py:39-43


def test_tcf_storage_width_limit_raises_at_construction():
    """slot_bits=12 with 80 slots passes the reference's bit check (960 bits)
    but its uint16 storage needs 1280 bits per block: the B200 facade says so
    in Tcf.__init__ (before touching the device), not at the first op."""
    from paper_2212_09005_b200 import Tcf
    TcfParams(num_blocks=4, block_slots=80, tag_bits=12, slot_bits=12)  # reference-valid
    with pytest.raises(ValueError, match="1024-bit block"):
        Tcf(num_blocks=4, block_slots=80, tag_bits=12, slot_bits=12)
