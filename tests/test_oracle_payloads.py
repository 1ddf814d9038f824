"""Oracle pins for the payloads (P:92-99, P:115-117 name the problems; their
definitions are reading E15, fp32 order reading E17), the packed layout
(reading E16) and the checksums (reading E21).  Pins are independent fp64
evaluations with numpy, textbook forms, closed-form special cases and known
reference values.  CPU only."""
import math

import numpy as np
import pytest

import workloads
from conftest import golden


def test_packed_rank_closed_forms_equal_enumeration(orc):
    n = 96
    o = orc.index_write(2, False, n)
    pos = 0
    for i in range(n):
        for j in range(i):
            assert o[pos] == pos == orc.rank2_strict(i, j)
            pos += 1
    o = orc.index_write(2, True, n)
    pos = 0
    for i in range(n):
        for j in range(i + 1):
            assert o[pos] == pos == orc.rank2_incl(i, j)
            pos += 1
    n = 40
    o = orc.index_write(3, False, n, elem_bytes=8)
    pos = 0
    for k in range(n):
        for j in range(k):
            for i in range(j):
                assert o[pos] == pos == orc.rank3(i, j, k)
                pos += 1
    assert pos == math.comb(n, 3)


def test_rank3_large_is_exact(orc):
    # 64-bit ranks near the C4/C5 extremes (Python ints are exact)
    for (i, j, k) in [(0, 1, 2047), (2045, 2046, 2047), (5, 70000, 131071)]:
        assert orc.rank3(i, j, k) == math.comb(k, 3) + math.comb(j, 2) + i
    n = 1 << 17
    assert orc.rank2_strict(n - 1, n - 2) == n * (n - 1) // 2 - 1


def test_edm_against_fp64(orc):
    p = workloads.points(300, 7)
    d = orc.edm(p)
    ref = []
    P = p.astype(np.float64)
    for i in range(300):
        for j in range(i):
            ref.append(np.sqrt(((P[i] - P[j]) ** 2).sum()))
    ref = np.array(ref)
    # fp32: three rounded squares/sums and a correctly-rounded sqrt -> a few ulp
    assert np.max(np.abs(d - ref) / np.maximum(ref, 1e-30)) < 4e-7
    assert d.dtype == np.float32 and len(d) == 300 * 299 // 2


def test_edm_symmetric_and_zero_for_duplicates(orc):
    p = workloads.clustered_points(64, 3, copies=2)
    assert orc.edm_dist(p, 1, 0) == 0.0
    for (i, j) in [(5, 2), (63, 0), (40, 39)]:
        assert orc.edm_dist(p, i, j) == orc.edm_dist(p, j, i)


def _at_textbook(P, i, j, k):
    """Axilrod-Teller (1 + 3 cos g1 cos g2 cos g3) / (r_ij r_jk r_ik)^3 with the
    angles taken from dot products (fp64)."""
    a, b, c = P[i], P[j], P[k]
    def cosang(o, u, v):
        x, y = u - o, v - o
        return np.dot(x, y) / (np.linalg.norm(x) * np.linalg.norm(y))
    rij, rjk, rik = np.linalg.norm(a - b), np.linalg.norm(b - c), np.linalg.norm(a - c)
    return (1 + 3 * cosang(a, b, c) * cosang(b, a, c) * cosang(c, a, b)) / (rij * rjk * rik) ** 3


def test_atm_term_against_textbook(orc):
    p = workloads.points(40, 11)
    P = p.astype(np.float64)
    worst = 0.0
    for (i, j, k) in [(0, 1, 2), (3, 17, 39), (5, 6, 30), (10, 20, 21), (1, 2, 38)]:
        t = orc.atm_term(p, i, j, k, 0.0)
        ref = _at_textbook(P, i, j, k)
        worst = max(worst, abs(t - ref) / abs(ref))
    assert worst < 1e-4


def test_atm_equilateral_closed_form(orc):
    # side^2 = s  ->  E = (11/8) s^-4.5 (E15)
    s3 = math.sqrt(3.0)
    tri = np.array([[0, 0, 0], [1, 0, 0], [0.5, s3 / 2, 0]], np.float32)
    for eps2 in (0.0, 1e-2):
        s = 1.0 + eps2
        t = orc.atm_term(tri, 0, 1, 2, eps2)
        assert abs(t - 11 / 8 * s ** -4.5) / (11 / 8 * s ** -4.5) < 5e-6


def test_atm_sum_permutation_and_fp64(orc):
    p = workloads.points(48, 5)
    eps2 = np.float32(1e-2)
    s = orc.atm_sum(p, eps2)
    perm = np.random.default_rng(1).permutation(48)
    s2 = orc.atm_sum(p[perm], eps2)
    assert abs(s - s2) / abs(s) < 1e-6
    # independent fp64 evaluation of the softened sum
    P = p.astype(np.float64)
    e = float(eps2)
    tot = 0.0
    for k in range(48):
        for j in range(k):
            for i in range(j):
                a = ((P[i] - P[j]) ** 2).sum() + e
                b = ((P[j] - P[k]) ** 2).sum() + e
                c = ((P[i] - P[k]) ** 2).sum() + e
                tot += (8 * a * b * c + 3 * (a + c - b) * (a + b - c) * (b + c - a)) / (8 * (a * b * c) ** 2 * math.sqrt(a * b * c))
    assert abs(s - tot) / abs(tot) < 1e-5
    # the row split does not change the result (deterministic combination)
    assert orc.atm_sum(p, eps2, 0, 20) + orc.atm_sum(p, eps2, 20, 48) == pytest.approx(s, rel=1e-12)
    assert orc.atm_sum(p, eps2, nthreads=1) == orc.atm_sum(p, eps2, nthreads=4)


def test_tc_count(orc):
    p = workloads.points(60, 9)
    n = 60
    assert orc.tc_count(p, 1e9) == math.comb(n, 3)
    assert orc.tc_count(p, 0.0) == 0
    P = p.astype(np.float64)
    D = ((P[:, None, :] - P[None, :, :]) ** 2).sum(-1) < 0.5 ** 2
    ref = sum(1 for k in range(n) for j in range(k) for i in range(j) if D[i, j] and D[j, k] and D[i, k])
    assert orc.tc_count(p, 0.5) == ref
    assert orc.tc_count(p, 0.5, nthreads=1) == orc.tc_count(p, 0.5, 0, 30) + orc.tc_count(p, 0.5, 30, 60)


def test_mix64_reference_values(orc):
    # mix64(p ^ bits*K) with p=0, bits=k equals the k-th splitmix64(seed 0) output
    for k, ref in golden("splitmix64.txt"):
        cs = orc.cs_array(np.array([int(k)], np.uint64))
        assert cs["mix"] == int(ref, 16)


def test_linear_checksums_definition(orc):
    a = np.array([5, 7, 11], np.uint32)
    cs = orc.cs_array(a, p0=10)
    assert cs["count"] == 3
    assert cs["s0"] == 23
    assert cs["s1"] == 11 * 5 + 12 * 7 + 13 * 11


@pytest.mark.parametrize("m,inc,n", [(2, False, 700), (2, True, 513), (3, False, 120)])
def test_streaming_index_checksum_equals_array(orc, m, inc, n):
    arr = orc.index_write(m, inc, n)
    assert orc.cs_index(m, inc, n) == orc.cs_array(arr)
    # closed forms: S0 = V(V-1)/2, S1 = sum (p+1) p
    V = len(arr)
    cs = orc.cs_index(m, inc, n)
    M = 1 << 64
    assert cs["s0"] == (V * (V - 1) // 2) % M
    assert cs["s1"] == ((V - 1) * V * (V + 1) // 3) % M


def test_streaming_edm_checksum_equals_array(orc):
    p = workloads.points(600, 2)
    assert orc.cs_edm(p) == orc.cs_array(orc.edm(p))
    # row ranges combine additively (sharded evaluation)
    a, b = orc.cs_edm(p, 0, 333), orc.cs_edm(p, 333, 600)
    tot = orc.cs_edm(p)
    assert all((a[k] + b[k]) % (1 << 64) == tot[k] for k in tot if k != "xr")
    assert a["xr"] ^ b["xr"] == tot["xr"]
