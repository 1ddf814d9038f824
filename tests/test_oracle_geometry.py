"""Oracle pins: simplex geometry and recursive-set volumes (P:131-163, P:303-337,
P:425-470).  CPU only."""
import math

import pytest

from conftest import golden


def test_volume_golden(orc):
    for m, n, v in golden("volumes.txt"):
        assert orc.simplex_volume(int(m), int(n)) == int(v)


@pytest.mark.parametrize("m", [1, 2, 3, 4])
def test_volume_equals_brute_force_enumeration(orc, m):
    # Eq.(2) vs counting the Eq.(1) set (cell convention, reading E1) by brute force
    nmax = {1: 40, 2: 40, 3: 30, 4: 14}[m]
    for n in range(0, nmax):
        assert orc.enumerate_count(m, n) == orc.simplex_volume(m, n), (m, n)


def test_volume_textbook_binomial(orc):
    for m in range(1, 7):
        for n in range(1, 60):
            assert orc.simplex_volume(m, n) == math.comb(n + m - 1, m)
    # the paper's printed special cases
    for n in range(1, 200):
        assert orc.simplex_volume(2, n) == n * (n + 1) // 2
        assert orc.simplex_volume(3, n) == n * (n + 1) * (n + 2) // 6


def test_stacked_identity_eq3(orc):
    for m in range(2, 8):
        for n in range(1, 64):
            assert orc.stacked_volume(m, n) == orc.simplex_volume(m, n)


def test_membership_examples(orc):
    # S:68-70
    assert orc.simplex_contains(2, 4, (0, 0))
    assert orc.simplex_contains(2, 4, (3, 0))
    assert not orc.simplex_contains(2, 4, (3, 1))
    assert not orc.simplex_contains(3, 2, (1, 1, 1))
    assert not orc.simplex_contains(2, 4, (-1, 0))


def test_bb_alpha_limit_eq4(orc):
    # Eq.(4): alpha -> m! - 1 ; finite form n^m / C(n+m-1, m) - 1
    for m in (2, 3, 4):
        a = orc.bb_alpha(m, 1 << 16)
        assert abs(a - (math.factorial(m) - 1)) < math.factorial(m) * 1e-3
    assert abs(orc.bb_alpha(2, 4) - 0.6) < 1e-12          # 16/10 - 1


def test_dispatch_golden(orc):
    for m, n, launched, useful in golden("dispatch.txt"):
        m, n = int(m), int(n)
        assert n ** m == int(launched)
        assert orc.simplex_volume(m, n) == int(useful)


def test_recursive_set_closed_forms(orc):
    rows = golden("paper_closed_forms.txt")
    for n, v2, v3, v3a in rows:
        n = int(n)
        assert orc.vs2(n) == int(v2)
        assert orc.vs3(n) == int(v3)
        assert orc.vs3_arity3(n) == int(v3a)
    for k in range(1, 25):
        n = 1 << k
        assert orc.vs2(n) == n * (n - 1) // 2
        assert orc.vs2(n) + n == orc.simplex_volume(2, n)
    for k in range(1, 21):                                        # n^3 < 2^64
        n = 1 << k
        assert orc.vs3(n) == (n ** 3 - n) // 6
        assert orc.vs3(n) == orc.simplex_volume(3, n - 1)        # P:559 "= V(Delta_{n-1})"
        assert orc.vs3_arity3(n) == (n ** 3 - 3 ** k) // 5       # P:460 (reading E8)


def test_arity3_and_two_branch_waste(orc):
    n = 1 << 10
    # arity-3 extra volume -> 1/5
    assert abs(orc.vs3_arity3(n) / orc.simplex_volume(3, n) - 1.2) < 0.012
    # grid (n/2)(n/2)(3n/4) vs V(S_n^3) -> 9/8 (12.5 %)
    grid = (n // 2) * (n // 2) * (3 * n // 4)
    assert abs(grid / orc.vs3(n) - 1.125) < 0.005 * 1.125


def test_floor_log2_plain(orc):
    # reading E3: floor(log2 y) = 31 - clz(y); checked against Python's bit_length
    for y in list(range(1, 5000)) + [2 ** 20, 2 ** 31 - 1, 2 ** 40 + 5]:
        assert orc.floor_log2(y) == y.bit_length() - 1
    # the paper's printed forms are wrong for every y (E3, E4): b - clz(y) is one too big
    for y in range(1, 1000):
        clz = 32 - y.bit_length()
        assert 32 - clz != orc.floor_log2(y)
        assert (2 << (32 - clz)) != (1 << orc.floor_log2(y))
