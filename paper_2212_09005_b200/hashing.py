"""Host-side hashing helpers, API-compatible with filterkit.hashing
(/root/reference/pkg/src/filterkit/hashing.py:17-154).

The hot path never uses these: every kernel hashes on the device
(csrc/fk_common.cuh).  They exist so callers (and tests) that craft keys,
inspect fingerprints or unpack slot words keep working, and so the host can
compute derived values bit-identically to the device.
"""

from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
EMPTY = 0
TOMBSTONE = 1

_C_BLOCK1 = 0x9E3779B97F4A7C15
_C_BLOCK2 = 0xC2B2AE3D27D4EB4F
_C_BACK_START = 0x165667B19E3779F9
_C_BACK_STEP = 0x27D4EB2F165667C5

_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB


def mix64(x: int) -> int:
    """SplitMix64 finalizer on a Python int (hashing.py:28-36)."""
    x &= MASK64
    for shift, mul in ((30, _M1), (27, _M2)):
        x = ((x ^ (x >> shift)) * mul) & MASK64
    return x ^ (x >> 31)


def mix64_many(arr) -> np.ndarray:
    """Vectorised mix64 over uint64 (wrapping multiply)."""
    x = np.array(arr, dtype=np.uint64, copy=True)
    with np.errstate(over="ignore"):
        for shift, mul in ((30, _M1), (27, _M2)):
            x ^= x >> np.uint64(shift)
            x *= np.uint64(mul)
        x ^= x >> np.uint64(31)
    return x


def _width_mask(bits):
    if not 1 <= bits <= 64:
        raise ValueError(f"fingerprint width must be 1..64, got {bits}")
    return MASK64 if bits == 64 else (1 << bits) - 1


def fingerprint(key: int, seed: int = 0, bits: int = 64) -> int:
    return mix64((int(key) ^ int(seed)) & MASK64) & _width_mask(bits)


def fingerprint_many(keys, seed: int = 0, bits: int = 64) -> np.ndarray:
    m = _width_mask(bits)
    fp = mix64_many(np.asarray(keys, dtype=np.uint64) ^ np.uint64(seed & MASK64))
    if m != MASK64:
        fp &= np.uint64(m)
    return fp


def split_fingerprint(fp: int, q: int, r: int):
    if q + r > 64:
        raise ValueError(f"q + r must be <= 64, got {q}+{r}")
    return (fp >> r) & ((1 << q) - 1), fp & ((1 << r) - 1)


def join_fingerprint(quotient: int, remainder: int, r: int) -> int:
    return (quotient << r) | remainder


def potc_pair(fp: int, num_blocks: int):
    return mix64(fp ^ _C_BLOCK1) % num_blocks, mix64(fp ^ _C_BLOCK2) % num_blocks


def potc_pair_many(fps, num_blocks: int):
    fps = np.asarray(fps, dtype=np.uint64)
    nb = np.uint64(num_blocks)
    return mix64_many(fps ^ np.uint64(_C_BLOCK1)) % nb, mix64_many(fps ^ np.uint64(_C_BLOCK2)) % nb


def backing_schedule(fp: int, size: int):
    return mix64(fp ^ _C_BACK_START) % size, (mix64(fp ^ _C_BACK_STEP) | 1) % size


def remap_tag(tag: int) -> int:
    return tag | 2 if tag < 2 else tag


def remap_tag_many(tags) -> np.ndarray:
    tags = np.asarray(tags, dtype=np.uint64)
    return np.where(tags < 2, tags | np.uint64(2), tags).astype(np.uint64)


def pack_slot(tag: int, value: int, f: int, w: int) -> int:
    if tag >> f:
        raise ValueError(f"tag {tag:#x} wider than {f} bits")
    if value >> (w - f):
        raise ValueError(f"value {value:#x} wider than {w - f} bits")
    return (value << f) | remap_tag(tag)


def unpack_slot(word: int, f: int):
    return word & ((1 << f) - 1), word >> f
