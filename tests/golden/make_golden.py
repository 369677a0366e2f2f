"""Generate golden fixtures from the REFERENCE implementation itself.

Run in the build container (where /root/reference exists), against a built
copy of the reference package (its compiled `_ckernels` backend):

    cp -r /root/reference/pkg /tmp/refbuild && (cd /tmp/refbuild && python setup.py build_ext --inplace)
    python tests/golden/make_golden.py --ref /tmp/refbuild/src

Writes tests/golden/*.npz.  The fixtures pin (a) the oracle restatement in
oracle/ (tests/test_oracle_golden.py) and (b) the product's host-side
parameter derivations; the GPU tests then compare the CUDA path against the
pinned oracle on the same seeded inputs.
"""

import argparse
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/tmp/refbuild/src")
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    import filterkit as fk
    from filterkit import countgroups, hashing
    from filterkit.workloads import counter_stream, gen_keys, WorkloadSpec

    assert "c" in fk.available_backends(), "build the reference's compiled backend first"

    def keys(seed, n):
        return counter_stream(seed, 0x5851F42D4C957F2D, n)

    # ---- hashing -----------------------------------------------------------
    ks = np.concatenate([np.array([0, 1, 2, 12345, 0x0123456789ABCDEF, 2 ** 64 - 1, 2 ** 63],
                                  dtype=np.uint64), keys(7, 2000)])
    out = {"keys": ks, "mix": hashing.mix64_many(ks)}
    for seed in (0, 9, 2 ** 64 - 1):
        out["fp_s%d" % (seed % 1000)] = hashing.fingerprint_many(ks, seed & (2 ** 64 - 1))
    fp = hashing.fingerprint_many(ks, 9)
    for nb in (1, 100, 8192, 65536, 2 ** 24, 1000003):
        b1, b2 = hashing.potc_pair_many(fp, nb)
        out["b1_%d" % nb], out["b2_%d" % nb] = b1, b2
    for size in (10486, 2684355, 7):
        st = [hashing.backing_schedule(int(x), size) for x in fp.tolist()]
        out["bstart_%d" % size] = np.array([a for a, _ in st], dtype=np.uint64)
        out["bstep_%d" % size] = np.array([b for _, b in st], dtype=np.uint64)
    for bits in (30, 36, 40):
        out["fpbits_%d" % bits] = hashing.fingerprint_many(ks, 0, bits)
    out["remap16"] = hashing.remap_tag_many(fp & np.uint64(0xFFFF))
    np.savez_compressed(os.path.join(HERE, "hashing.npz"), **out)

    # ---- count groups --------------------------------------------------------
    rows = []
    for r in (8, 16):
        for rem in (0, 1, 2, 5, 7, 200, (1 << r) - 1):
            for count in (1, 2, 3, 4, 12, 255, 256, 257, 300, 1000, 70000, 2 ** 16 + 5, 2 ** 20 + 3):
                if rem == 0 and count > 3000:
                    continue
                words = countgroups.encode_group(rem, count, r)
                rows.append((r, rem, count, len(words), words))
    flat = np.array([w for row in rows for w in row[4]], dtype=np.uint64)
    np.savez_compressed(os.path.join(HERE, "countgroups.npz"),
                        meta=np.array([row[:4] for row in rows], dtype=np.int64), words=flat)

    # ---- params ------------------------------------------------------------
    tp = []
    for nb in (1, 3, 7, 100, 512, 65536, 2 ** 24):
        for frac in (0.0, 0.01, 0.015, 0.05, 1.0):
            for B in (1, 7, 16, 32):
                for sf in (0.75, 0.5, 1.0, 0.33):
                    p = fk.TcfParams(num_blocks=nb, block_slots=B, backing_fraction=frac, shortcut_fraction=sf)
                    tp.append((nb, B, int(frac * 1000), int(sf * 100), p.backing_slots, p.cut_slots))
    gp = []
    for q in range(6, 31):
        for ml in (0.95, 0.9, 1.0, 0.5):
            p = fk.GqfParams(q=q, max_load=ml)
            gp.append((q, int(ml * 100), p.physical_slots, p.num_regions, p.quotient_regions, p.max_occupied))
    bp = []
    for nb in (1, 16, 128, 8192):
        p = fk.BulkTcfParams(num_blocks=nb)
        bp.append((nb, p.main_slots, p.backing_slots, p.cut_slots))
    np.savez_compressed(os.path.join(HERE, "params.npz"), tcf=np.array(tp, np.int64),
                        gqf=np.array(gp, np.int64), btcf=np.array(bp, np.int64))

    # ---- point TCF -----------------------------------------------------------
    out = {}
    cases = [("w8", dict(tag_bits=8, slot_bits=8), 512, 8500, 0.01),
             ("w16", dict(tag_bits=16, slot_bits=16), 512, 8500, 0.01),
             ("w32", dict(tag_bits=16, slot_bits=32), 512, 8500, 0.01),
             ("w64", dict(tag_bits=16, slot_bits=64), 512, 8500, 0.01),
             ("nob", dict(), 256, 4600, 0.0),
             ("b7", dict(block_slots=7, tag_bits=12), 300, 2000, 0.02),
             ("b32", dict(block_slots=32), 128, 3900, 0.01)]
    for name, geom, nb, n, bf in cases:
        f = fk.Tcf(num_blocks=nb, backend="c", backing_fraction=bf, **geom)
        p = f.params
        k = keys(11, n)
        vb = p.slot_bits - p.tag_bits
        vals = (keys(12, n) & np.uint64((1 << vb) - 1)) if vb else np.zeros(n, np.uint64)
        out[name + "_keys"] = k
        out[name + "_vals"] = vals
        out[name + "_codes"] = f.insert_many(k, vals if vb else None)
        out[name + "_blocks_ins"] = f._blocks.astype(np.uint64)
        out[name + "_backing_ins"] = f._backing.astype(np.uint64)
        probe = np.concatenate([k[: n // 2], keys(13, n // 2)])
        out[name + "_probe"] = probe
        fo, vo = f.query_values_many(probe)
        out[name + "_found"], out[name + "_qvals"] = fo.astype(np.uint8), vo
        dk = np.concatenate([k[::3], k[:50]])
        out[name + "_dkeys"] = dk
        out[name + "_removed"] = f.delete_many(dk).astype(np.uint8)
        out[name + "_blocks_del"] = f._blocks.astype(np.uint64)
        out[name + "_backing_del"] = f._backing.astype(np.uint64)
        c = f.counters
        out[name + "_counters"] = np.array([c["inserts_ok"], c["inserts_backing"], c["deletes_ok"]], np.int64)
        out[name + "_geom"] = np.array([nb, p.block_slots, p.tag_bits, p.slot_bits, p.backing_slots,
                                        p.cut_slots, p.probe_limit, int(bf * 1000)], np.int64)
    np.savez_compressed(os.path.join(HERE, "tcf_point.npz"), **out)

    # ---- bulk TCF --------------------------------------------------------------
    out = {}
    for name, nb, n in (("a", 128, 13000), ("b", 128, 17500), ("c", 64, 9000)):
        f = fk.BulkTcf(num_blocks=nb, backend="c")
        k = keys(41, n)
        out[name + "_keys"] = k
        out[name + "_failed"] = f.insert_batch(k)
        out[name + "_blocks_ins"] = f._blocks.astype(np.uint64)
        out[name + "_fill_ins"] = f._fill.copy()
        out[name + "_backing_ins"] = f._backing.astype(np.uint64)
        probe = np.concatenate([k[:4000], keys(42, 4000)])
        out[name + "_probe"] = probe
        out[name + "_found"] = f.query_batch(probe).astype(np.uint8)
        dk = np.concatenate([k[::2], k[:30]])
        out[name + "_dkeys"] = dk
        out[name + "_removed"] = f.delete_batch(dk).astype(np.uint8)
        out[name + "_blocks_del"] = f._blocks.astype(np.uint64)
        out[name + "_fill_del"] = f._fill.copy()
        out[name + "_backing_del"] = f._backing.astype(np.uint64)
        c = f.counters
        out[name + "_counters"] = np.array([c["inserts_ok"], c["inserts_backing"], c["deletes_ok"]], np.int64)
        out[name + "_nb"] = np.array([nb], np.int64)
    np.savez_compressed(os.path.join(HERE, "tcf_bulk.npz"), **out)

    # ---- GQF -------------------------------------------------------------------
    out = {}
    rng = np.random.default_rng(5)

    def img(g, pre):
        for nm in ("slots", "occupieds", "runends", "offsets", "stats"):
            out[pre + nm] = getattr(g, "_" + nm).copy()

    for r in (8, 16):
        g = fk.Gqf(q=14, r=r, backend="c")
        k = rng.integers(0, 2 ** 40, 600, dtype=np.uint64)
        c = rng.integers(1, 300, 600, dtype=np.uint64)
        pre = "r%d_" % r
        out[pre + "k"], out[pre + "c"] = k, c
        g.insert_many(k, c)
        img(g, pre + "ins_")
        out[pre + "count"] = g.count_many(k)
        dk, dc = k[::3].copy(), c[::3] // 2
        out[pre + "dk"], out[pre + "dc"] = dk, dc
        out[pre + "dfound"] = g.delete_many(dk, dc).astype(np.uint8)
        img(g, pre + "del_")
        k2 = rng.integers(0, 2 ** 40, 500, dtype=np.uint64)
        out[pre + "k2"] = k2
        g.bulk_insert(k2, workers=1)
        img(g, pre + "bulk_")
        kk = np.concatenate([k[:200], k2[:200], k2[:50]])
        out[pre + "kk"] = kk
        out[pre + "bfound"] = g.bulk_delete(kk, workers=1).astype(np.uint8)
        img(g, pre + "bdel_")
        g.validate()
    # duplicate-heavy (ur_count) bulk insert at q=16 + map-reduce form
    g = fk.Gqf(q=16, r=8, backend="c")
    uk = gen_keys(WorkloadSpec("ur_count", n=2000, seed=3))
    out["ur_keys"] = uk
    g.bulk_insert(uk, workers=1)
    img(g, "ur_")
    uq, uc = np.unique(uk, return_counts=True)
    out["ur_count"] = g.count_many(uq)
    g2 = fk.Gqf(q=16, r=8, backend="c")
    g2.bulk_insert(uq, uc.astype(np.uint64), workers=1)
    for nm in ("slots", "occupieds", "runends", "offsets", "stats"):
        assert np.array_equal(getattr(g, "_" + nm), getattr(g2, "_" + nm))
    # capacity failure in insert_many: index + partial image
    g = fk.Gqf(q=10, r=8, backend="c")
    ck = rng.integers(0, 2 ** 40, 1100, dtype=np.uint64)
    out["cap_k"] = ck
    try:
        g.insert_many(ck)
        out["cap_err"] = np.array([0])
    except fk.CapacityError:
        out["cap_err"] = np.array([1])
    img(g, "cap_")
    np.savez_compressed(os.path.join(HERE, "gqf.npz"), **out)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
