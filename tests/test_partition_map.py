"""Host restatement of the partitioned grouping's key map (part_group.cuh:
PartMap, part_digit) — no GPU. For every run constant c the map
T(v) = swap_{0,t}(v ^ (v_t ? c ^ e_t : 0)), t = lowest set bit of c, is an
involution-built bijection with T(c) = e_0, so a key v and its partner
v ^ c map to w and w ^ 1: they share the dense partition digit (top bits)
and the hashed digit (a hash of w >> 1), and the block's x side is the
bucket whose original key is the smaller one."""
import numpy as np


def fwd(v, c):
    if c == 0:
        return v
    t = (c & -c).bit_length() - 1
    cm = c ^ (1 << t)
    x = v ^ (cm if (v >> t) & 1 else 0)
    d = (x ^ (x >> t)) & 1
    return x ^ (d | (d << t))


def inv(w, c):
    if c == 0:
        return w
    t = (c & -c).bit_length() - 1
    cm = c ^ (1 << t)
    d = (w ^ (w >> t)) & 1
    x = w ^ (d | (d << t))
    return x ^ (cm if (x >> t) & 1 else 0)


def hashed_digit(w, k):
    return (((w >> 1) * 0x9E3779B1) & 0xFFFFFFFF) >> (32 - k) if k else 0


def test_partition_map_pairs_partners_as_neighbours():
    rng = np.random.default_rng(5)
    for M in (2, 5, 12, 16, 20, 24, 31):
        for _ in range(40):
            c = int(rng.integers(0, 1 << M))
            vs = [int(v) for v in rng.integers(0, 1 << M, 200)]
            ws = [fwd(v, c) for v in vs]
            assert all(0 <= w < (1 << M) for w in ws)
            assert all(inv(w, c) == v for v, w in zip(vs, ws))  # bijection
            if c:
                assert fwd(c, c) == 1  # T(c) = e_0
            for v, w in zip(vs, ws):
                w2 = fwd(v ^ c, c)
                assert w2 == (w ^ 1 if c else w)  # partner = neighbour bucket (or itself when c = 0)
                k = min(10, M - 1)
                assert (w >> (M - k)) == (w2 >> (M - k))  # same dense partition
                assert hashed_digit(w, k) == hashed_digit(w2, k)  # same hashed partition
                if c:
                    ve = inv(w & ~1, c)  # the even bucket's original key
                    assert ve in (v, v ^ c)


def test_partition_map_is_linear():
    rng = np.random.default_rng(6)
    for _ in range(200):
        M = int(rng.integers(2, 32))
        c, a, b = (int(x) for x in rng.integers(0, 1 << M, 3))
        assert fwd(a ^ b, c) == fwd(a, c) ^ fwd(b, c)
