"""The general-m volume analysis (second half; P:425-470,
P:645-695; readings E8, E20, E30, E31): the library's host functions
(include/smap.h, smap_analysis.cu) against the oracle's top-down recurrence
and the values the paper prints.  CPU only (host-only C ABI functions)."""
import math

import pytest


@pytest.fixture(scope="module")
def sm():
    import paper_1610_07394_b200 as s
    return s


def test_oracle_recurrence_pins(orc):
    # the two maps' sets and the arity-3 set (reading E8) as special cases
    for k in range(1, 16):
        n = 1 << k
        assert orc.vsm(2, n) == n * (n - 1) // 2
        assert orc.vsm(3, n) == (n ** 3 - n) // 6
        assert orc.vsm(3, n, beta=3) == (n ** 3 - 3 ** k) // 5 == orc.vs3_arity3(n)
    # V(S_n^4) = (n^4 - n)/14 > V(Delta^4_{n-1}) = (n-1)n(n+1)(n+2)/24 for n >= 2
    assert [orc.vsm(4, n) for n in (4, 8, 16)] == [18, 292, 4680]
    for k in range(1, 14):
        n = 1 << k
        assert orc.vsm(4, n) == (n ** 4 - n) // 14
        # (equality at n = 2: 1 = 1; strict from n = 4 on -- the printed "> ... n >= 2" is off at n = 2)
        assert 24 * orc.vsm(4, n) >= (n - 1) * n * (n + 1) * (n + 2)
        assert n == 2 or 24 * orc.vsm(4, n) > (n - 1) * n * (n + 1) * (n + 2)
    assert orc.vsm(4, 12) == 2 ** 64 - 1                      # not a power of 1/r
    # alpha -> m!/(2^m - 2) - 1 = 5/7 (m=4, "approaches to 5/7"), 3 (m=5), 39 (m=7),
    # the printed "3x and 39x" being these alpha values (reading E20); Richardson on the O(1/n) tail
    for m, lim, k in ((4, 5 / 7, 14), (5, 3.0, 12), (7, 39.0, 9)):
        a1, a2 = orc.vsm_alpha(m, 1 << (k - 1)), orc.vsm_alpha(m, 1 << k)
        assert a1 < a2 < lim
        assert abs((2 * a2 - a1) - lim) <= 0.01 * lim
    # arity 3: alpha -> 1/5
    a1, a2 = orc.vsm_alpha(3, 1 << 19, beta=3), orc.vsm_alpha(3, 1 << 20, beta=3)
    assert abs((2 * a2 - a1) - 0.2) < 1e-3


@pytest.mark.parametrize("m", range(2, 9))
@pytest.mark.parametrize("beta", range(1, 7))
def test_library_volume_matches_oracle(sm, orc, m, beta):
    for rden in (2, 3):
        for k in range(0, 14):
            n = rden ** k
            want = orc.vsm(m, n, beta, rden)
            if want == 2 ** 64 - 1:
                with pytest.raises(sm.SmapError):
                    sm.smap_recursive_volume(m, n, beta, rden)
                continue
            assert sm.smap_recursive_volume(m, n, beta, rden) == want
            assert sm.smap_recursive_volume(m, n, beta, rden, closed=True) == want   # Eq. generic-m
    with pytest.raises(sm.SmapError):
        sm.smap_recursive_volume(m, 12, beta, 2)


def test_alpha_limit(sm, orc):
    for m in range(2, 9):
        assert sm.smap_alpha_limit(m) == pytest.approx(math.factorial(m) / (2 ** m - 2) - 1, rel=1e-15)
    assert sm.smap_alpha_limit(4) == pytest.approx(5 / 7)
    assert sm.smap_alpha_limit(5) == pytest.approx(3.0)
    assert sm.smap_alpha_limit(7) == pytest.approx(39.0)
    assert sm.smap_alpha_limit(3, 0.5, 3) == pytest.approx(0.2)           # arity 3
    assert sm.smap_alpha_limit(2) == 0.0 and sm.smap_alpha_limit(3) == 0.0   # lambda2, two-branch lambda3
    assert math.isinf(sm.smap_alpha_limit(3, 0.5, 8))                     # beta = 1/r^m: grows like n^m log n
    # the library's limit agrees with the oracle's finite-n extra volume
    for m, beta in ((4, 2), (5, 2), (3, 3), (4, 3)):
        a1, a2 = orc.vsm_alpha(m, 1 << 11, beta), orc.vsm_alpha(m, 1 << 12, beta)
        assert abs((2 * a2 - a1) - sm.smap_alpha_limit(m, 0.5, beta)) < 2e-3 * (1 + sm.smap_alpha_limit(m, 0.5, beta))


def test_r_star(sm):
    # 1/r^m - beta = m!; reading E30: the printed r = 1/(m^{-1/m}) = m^{1/m} is > 1
    assert sm.smap_r_star(2, 2) == pytest.approx(0.5, abs=1e-15)         # lambda2's r
    assert sm.smap_r_star(3, 2) == pytest.approx(0.5, abs=1e-15)         # lambda3's r
    assert sm.smap_r_star(4, 2) == pytest.approx(0.44285, abs=1e-5)
    assert sm.smap_r_star(5, 2) == pytest.approx(0.38259, abs=1e-5)
    for m in range(2, 9):
        for beta in (2, 3, 5):
            r = sm.smap_r_star(m, beta)
            assert (1 / r) ** m - beta == pytest.approx(math.factorial(m), rel=1e-12)
            assert sm.smap_alpha_limit(m, r, beta) == pytest.approx(0.0, abs=1e-9)
        assert m ** (1 / m) > 1.0                                          # the printed value cannot be a scale


def test_n0(sm):
    # r = 1/2, beta = 2 covers from n0 = 2 (m = 2, 3: equality V(S_n) = V(Delta_{n-1}); m = 4: "n >= 2")
    for m in (2, 3, 4, 5, 6):
        n0, ratio = sm.smap_find_n0(m, 0.5, 2, 4096)
        assert n0 == 2
        assert ratio == pytest.approx(1.0, rel=1e-12) if m <= 3 else ratio > 1.0
    # reading E31: under the exact constraint (r = r*) the continuous set never covers for m >= 4 --
    # V(S_n)/V(Delta_{n-1}) tends to 1 from below ("approach it from below" is required)
    for m in (4, 5, 6):
        n0, ratio = sm.smap_find_n0(m, sm.smap_r_star(m, 2), 2, 4096)
        assert n0 is None and 0.99 < ratio < 1.0
        _, r2 = sm.smap_find_n0(m, sm.smap_r_star(m, 2), 2, 1 << 16)
        assert ratio < r2 < 1.0
    with pytest.raises(sm.SmapError):
        sm.smap_find_n0(4, 1.5, 2, 100)


def test_r_cover(sm):
    # the least-extra-volume scaling that covers Delta^m_{n-1} from n0 on (the paper's open
    # optimisation): r in (r*, (beta+1)^{-1/m}); covers at that r, not just below it;
    # a larger n0 allows less extra volume; a larger beta moves the covering r
    for m in (4, 5):
        prev = None
        for n0 in (8, 64, 512):
            r = sm.smap_r_cover(m, 2, n0, 4096)
            assert sm.smap_r_star(m, 2) < r < (3.0) ** (-1 / m)
            assert sm.smap_find_n0(m, r, 2, 4096)[0] <= n0
            got = sm.smap_find_n0(m, r * (1 - 1e-6), 2, 4096)[0]
            assert got is None or got > n0
            a = sm.smap_alpha_limit(m, r, 2)
            assert a > 0.0
            if prev is not None:
                assert a < prev
            prev = a
