"""Count-group codec (host side), API-compatible with filterkit.countgroups
(/root/reference/pkg/src/filterkit/countgroups.py:28-112).

A group stores `count` copies of remainder `rem` in r-bit slot words:
count 1 -> [rem]; 2 -> [rem, rem]; rem 0 -> [0]*count (unary); otherwise
[rem, (count-2) % rem, base-(2^r-1) digits of (count-2)//rem with digits
>= rem bumped by one, rem].  The device encoder/decoder (csrc/gqf*.cu) is
the same arithmetic; this module serves enumeration, validation and tests.
"""

from __future__ import annotations

__all__ = ["encode_group", "encoded_length", "parse_group", "decode_run"]


def _check(rem, count, r):
    if count <= 0:
        raise ValueError("count must be positive")
    if not 0 <= rem < (1 << r):
        raise ValueError("remainder out of range for r=%d" % r)


def encode_group(rem, count, r):
    _check(rem, count, r)
    if rem == 0 or count <= 2:
        return [rem] * count
    base = (1 << r) - 1
    v, low = divmod(count - 2, rem)
    out = [rem, low]
    while v:
        v, d = divmod(v, base)
        out.append(d + (d >= rem))
    out.append(rem)
    return out


def encoded_length(rem, count, r):
    if count <= 0:
        raise ValueError("count must be positive")
    if rem == 0 or count <= 2:
        return count
    base = (1 << r) - 1
    v, n = (count - 2) // rem, 3
    while v:
        v //= base
        n += 1
    return n


def parse_group(slots, i, end, r):
    head = int(slots[i])
    if head == 0:
        j = i
        while j <= end and int(slots[j]) == 0:
            j += 1
        return 0, j - i, j
    if i == end:
        return head, 1, i + 1
    nxt = int(slots[i + 1])
    if nxt > head:
        return head, 1, i + 1
    if nxt == head:
        return head, 2, i + 2
    base = (1 << r) - 1
    value, scale, j = 0, 1, i + 2
    while True:
        if j > end:
            raise ValueError("unterminated count group at slot %d" % i)
        d = int(slots[j])
        if d == head:
            break
        value += scale * (d - (d > head))
        scale *= base
        j += 1
    return head, nxt + head * value + 2, j + 1


def decode_run(slots, start, end, r):
    groups, i = [], start
    while i <= end:
        rem, count, i = parse_group(slots, i, end, r)
        groups.append((rem, count))
    return groups
