"""Device hashing is bit-identical to the reference's host hashing."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run_streams(keys, seed, bits, nb, bs):
    import torch
    from paper_2212_09005_b200 import _lib
    lib = _lib.load()
    k = torch.from_numpy(np.ascontiguousarray(keys, np.uint64).view(np.int64)).cuda()
    out = torch.empty(5 * len(keys), dtype=torch.int64, device="cuda")
    _lib.check(lib.fk_hash_streams(_lib.dptr(k), len(keys), seed, bits, nb, bs, _lib.dptr(out), None), "hash")
    torch.cuda.synchronize()
    return out.cpu().numpy().view(np.uint64).reshape(-1, 5)


def test_streams_match_golden(golden):
    h = golden("hashing")
    ks = h["keys"]
    for nb in (1, 100, 8192, 65536, 2 ** 24, 1000003):
        for bs in (10486, 2684355, 7):
            got = _run_streams(ks, 9, 64, nb, bs)
            assert np.array_equal(got[:, 0], h["fp_s9"])
            assert np.array_equal(got[:, 1], h["b1_%d" % nb])
            assert np.array_equal(got[:, 2], h["b2_%d" % nb])
            assert np.array_equal(got[:, 3], h["bstart_%d" % bs])
            assert np.array_equal(got[:, 4], h["bstep_%d" % bs])
    for bits in (30, 36, 40):
        assert np.array_equal(_run_streams(ks, 0, bits, 0, 0)[:, 0], h["fpbits_%d" % bits])


def test_streams_match_oracle_10m(oracle):
    from conftest import counter_keys
    ks = counter_keys(77, 10_000_000)
    got = _run_streams(ks, 12345, 64, 2 ** 24, 2684355)
    fp = oracle.fingerprint_many(ks, 12345)
    b1, b2 = oracle.potc_pair_many(fp, 2 ** 24)
    assert np.array_equal(got[:, 0], fp)
    assert np.array_equal(got[:, 1], b1) and np.array_equal(got[:, 2], b2)
    with np.errstate(over="ignore"):
        st = oracle.mix64_many(fp ^ np.uint64(oracle.C_BACK_START)) % np.uint64(2684355)
        sp = (oracle.mix64_many(fp ^ np.uint64(oracle.C_BACK_STEP)) | np.uint64(1)) % np.uint64(2684355)
    assert np.array_equal(got[:, 3], st) and np.array_equal(got[:, 4], sp)


@pytest.mark.parametrize("d", [1, 2, 3, 7, 100, 10486, 65536, 2684355, 1000003, 2 ** 32 - 1, 2 ** 32 + 1,
                               2 ** 63 + 12345, 2 ** 64 - 1, 0x9E3779B97F4A7C15])
def test_fastmod_exact(d):
    import torch
    from paper_2212_09005_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(d % 1000)
    x = np.concatenate([rng.integers(0, 2 ** 64, 1_000_000, dtype=np.uint64, endpoint=False),
                        np.array([v % 2 ** 64 for v in (0, 1, d - 1, d, d + 1, 2 ** 64 - 1, 2 ** 64 - 2,
                                                        (2 ** 64 - 1) // d * d)], dtype=np.uint64)])
    xt = torch.from_numpy(x.view(np.int64)).cuda()
    out = torch.empty_like(xt)
    _lib.check(lib.fk_fastmod_check(_lib.dptr(xt), len(x), d, _lib.dptr(out), None), "fastmod")
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().view(np.uint64), x % np.uint64(d))


def test_counter_stream_device_matches_host():
    """fk_counter_stream == workloads.counter_stream (fk/workloads.py:23-26),
    including odd lengths, a start offset and a wrap past 2^64."""
    import torch
    from paper_2212_09005_b200 import _lib
    from paper_2212_09005_b200.workloads import (TAG_FPR, TAG_UNIFORM, counter_stream,
                                                 counter_stream_device)
    for seed, tag, n in ((1, TAG_UNIFORM, 1), (2, TAG_FPR, 7), (0, TAG_UNIFORM, 1_000_003),
                         (12345, 0xFFFFFFFFFFFFFFFF, 4097)):
        got = counter_stream_device(seed, tag, n).cpu().numpy().view(np.uint64)
        assert np.array_equal(got, counter_stream(seed, tag, n))
    # start offset = a window of the full stream; odd (8-byte aligned) output
    full = counter_stream(5, TAG_UNIFORM, 5000)
    out = torch.zeros(4001, dtype=torch.int64, device="cuda")
    lib = _lib.load()
    _lib.check(lib.fk_counter_stream(5, TAG_UNIFORM, 999, 4000, ctypes.c_void_p(out.data_ptr() + 8), None), "cs")
    torch.cuda.synchronize()
    assert np.array_equal(out[1:].cpu().numpy().view(np.uint64), full[999:4999])
    assert int(out[0]) == 0


def test_kmer_windows_device_match_reference_golden(golden, tmp_path):
    """Device k-mer extraction (fk_kmer_windows) equals the reference's
    windows on its fixture, for every k, in order."""
    from paper_2212_09005_b200.workloads import kmer_windows_device
    g = golden("kmer")
    p = tmp_path / "reads.fq"
    p.write_bytes(g["text"].tobytes())
    for k in (1, 4, 11, 21, 31, 32):
        got = kmer_windows_device(str(p), k).cpu().numpy().view(np.uint64)
        assert np.array_equal(got, g["k%d" % k]), k


@pytest.mark.parametrize("seed,start", [(0, 0), (123, 12345), (2 ** 63 + 5, 1)])
def test_pcg64_device_matches_numpy(seed, start):
    """numpy's default_rng bit generator on the device (fk_pcg64_raw), with
    jump-ahead to any position: random_raw, bit for bit."""
    from paper_2212_09005_b200.workloads import pcg64_raw_device
    g = np.random.default_rng(seed)
    if start:
        g.bit_generator.random_raw(start)
    want = g.bit_generator.random_raw(100_003)
    got = pcg64_raw_device(seed, 100_003, start=start).cpu().numpy().view(np.uint64)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("low,high", [(1, 101), (0, 7), (5, 6), (0, 2 ** 32), (-3, 1000003)])
def test_bounded_integers_device_match_numpy(low, high):
    """Generator.integers(low, high, n) on the device (fk_bounded_integers):
    Lemire's method on the buffered 32-bit draws, rejections included."""
    from paper_2212_09005_b200.workloads import integers_device
    for seed in (3, 99):
        want = np.random.default_rng(seed).integers(low, high, 300_001)
        got = integers_device(seed, low, high, 300_001).cpu().numpy()
        assert np.array_equal(got, want), (seed, low, high)


@pytest.mark.parametrize("s,universe", [(1.5, 1_000_000), (1.5, 100), (1.0, 5000), (2.5, 10 ** 9)])
def test_zipf_device_matches_host(s, universe):
    """The bounded-Zipf rejection-inversion sampler on the device
    (fk_zipf_bounded) draws the same ranks as the host restatement of the
    reference's sampler (fk/workloads.py:81-118) on the same generator."""
    from paper_2212_09005_b200.workloads import zipf_bounded, zipf_bounded_device
    seed = 1234 + int(universe)
    want = zipf_bounded(np.random.default_rng(seed), s, universe, 500_000)
    got = zipf_bounded_device(seed, s, universe, 500_000).cpu().numpy()
    assert np.array_equal(got, want)


def test_gen_keys_device_match_reference_streams():
    """gen_keys on the device: uniform and zipf streams equal the host
    generator's (the reference's, restated), ur_count has exactly its
    multiset."""
    from paper_2212_09005_b200.workloads import WorkloadSpec, gen_keys, gen_keys_device
    for spec in (WorkloadSpec("uniform", n=100_000, seed=3), WorkloadSpec("zipf", n=200_000, seed=5),
                 WorkloadSpec("zipf", n=50_000, seed=6, universe=1000, zipf_s=1.2)):
        assert np.array_equal(gen_keys_device(spec).cpu().numpy().view(np.uint64), gen_keys(spec)), spec
    spec = WorkloadSpec("ur_count", n=20_000, seed=7)
    got = np.sort(gen_keys_device(spec).cpu().numpy().view(np.uint64))
    assert np.array_equal(got, np.sort(gen_keys(spec)))
