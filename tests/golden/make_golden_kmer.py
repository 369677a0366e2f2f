"""Golden k-mer windows from the REFERENCE's own extractor
(filterkit.workloads.kmer_windows, workloads.py:147-191).

    python tests/golden/make_golden_kmer.py --ref /root/reference/pkg/src

Writes tests/golden/kmer.npz: a FASTQ/FASTA text (uint8) mixing read layouts
the parser must handle (multi-line reads, lowercase, N and other non-ACGT
bytes, reads shorter than k, a quality line starting with '@', blank lines,
CRLF) and the reference's windows for several k.
"""

import argparse
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def text(seed=5):
    rng = np.random.default_rng(seed)

    def pick(alphabet, n):
        return np.frombuffer(alphabet, dtype=np.uint8)[rng.integers(0, len(alphabet), int(n))].tobytes()
    out = [b">r0 multi-line\n"]
    for _ in range(4):
        out.append(pick(b"ACGTacgt", 61) + b"\n")
    out.append(b"\n@r1\n" + pick(b"ACGTN", 300) + b"\n+\n@IIIIIIII\n")
    out.append(b">short\nACG\n>crlf\r\n" + pick(b"ACGT", 90) + b"\r\n")
    out.append(b">r3\n" + pick(b"ACGTRY", 500) + b"\n")
    for i in range(20):
        out.append(b"@q%d\n" % i + pick(b"ACGT", rng.integers(5, 150)) + b"\n+\nIIII\n")
    return b"".join(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    a = ap.parse_args()
    sys.path.insert(0, a.ref)
    from filterkit.workloads import kmer_windows
    t = text()
    path = os.path.join(HERE, "_kmer_tmp.fq")
    open(path, "wb").write(t)
    out = {"text": np.frombuffer(t, dtype=np.uint8)}
    for k in (1, 4, 11, 21, 31, 32):
        out["k%d" % k] = kmer_windows(path, k)
    os.remove(path)
    np.savez_compressed(os.path.join(HERE, "kmer.npz"), **out)
    print("wrote", os.path.join(HERE, "kmer.npz"))


if __name__ == "__main__":
    main()
