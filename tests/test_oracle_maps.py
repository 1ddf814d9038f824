"""Oracle pins for the block-space maps lambda2 and lambda3 (P:565-597,
reading R3).  Every map is pinned by exhaustive bijection against the plain
target set, by the independent recursive constructions, by SPEC's worked
examples and by the printed branch formulas.  CPU only."""
import pytest

from conftest import golden


def test_lambda2_golden(orc):
    for wx, wy, x, y in golden("lambda2_examples.txt"):
        assert orc.lambda2(int(wx), int(wy)) == (int(x), int(y))


def test_lambda2_n4_image(orc):
    img = {orc.lambda2(wx, wy) for wx in range(2) for wy in range(1, 4)}
    assert img == {(int(a), int(b)) for a, b in golden("lambda2_n4_image.txt")}


def test_grid_sizes_golden(orc):
    for kind, N, blocks, useful in golden("grid_sizes.txt"):
        N = int(N)
        if kind == "grid2":
            r = orc.check_cover2_blocks(N)
            assert (N // 2) * (N - 1) == int(blocks)
            assert r["mapped"] == int(useful)
        else:
            r = orc.check_cover3_blocks(N)
            assert (N // 2) * (N // 2) * (3 * N // 4) == int(blocks)
            assert r["mapped"] == int(useful)


@pytest.mark.parametrize("k", range(1, 13))
def test_lambda2_exhaustive_bijection(orc, k):
    N = 1 << k
    r = orc.check_cover2_blocks(N)
    assert r == {"mapped": N * (N - 1) // 2, "missing": 0, "duplicates": 0, "outside": 0}


@pytest.mark.parametrize("k", range(1, 12))
def test_lambda2_equals_recursive_set(orc, k):
    assert orc.check_rec2(1 << k) == 0


def test_lambda2_self_similarity(orc):
    # a block of the q-th copy at level l is displaced from its grid
    # position by (q 2^l, q 2^(l+1)); equivalently the q-th copy's image is the
    # q=0 copy's image translated by (2 q 2^l, 2 q 2^l) along the diagonal.
    N = 256
    for wy in range(1, N):
        b = 1 << (wy.bit_length() - 1)
        for wx in range(N // 2):
            q, u = divmod(wx, b)
            x, y = orc.lambda2(wx, wy)
            assert (x - wx, y - wy) == (q * b, 2 * q * b)
            x0, y0 = orc.lambda2(u, wy)
            assert (x, y) == (x0 + 2 * q * b, y0 + 2 * q * b)


def test_checker_not_vacuous(orc):
    # a unit translation must be flagged
    r = orc.check_cover2_blocks(64, corrupt=True)
    assert r["missing"] > 0 and (r["duplicates"] + r["outside"]) > 0
    r = orc.check_cover3_blocks(32, corrupt=True)
    assert r["missing"] > 0 and (r["duplicates"] + r["outside"]) > 0


def test_h_map_golden(orc):
    for N, wx, wy, wz, X, Y, Z in golden("h_map.txt"):
        c, xyz, _ = orc.lambda3(int(N), int(wx), int(wy), int(wz))
        assert c == orc.L3_INSIDE
        assert xyz == (int(X), int(Y), int(Z))


@pytest.mark.parametrize("k", range(3, 9))
def test_lambda3_exhaustive_bijection(orc, k):
    N = 1 << k
    r = orc.check_cover3_blocks(N)
    assert r["mapped"] == (N ** 3 - N) // 6
    assert r["missing"] == r["duplicates"] == r["outside"] == 0
    assert r["body_missing"] == r["body_duplicates"] == 0       # reading E14
    assert r["spare"] == N * N // 8
    assert r["spare"] + r["filler"] == 3 * N ** 3 // 16 - (N ** 3 - N) // 6


def test_lambda3_n4(orc):
    r = orc.check_cover3_blocks(4)
    assert r["mapped"] == 10 and r["missing"] == r["duplicates"] == r["outside"] == 0


@pytest.mark.parametrize("k", range(2, 8))
def test_lambda3_equals_recursive_fold(orc, k):
    assert orc.check_rec3(1 << k) == 0


def test_lambda3_main_cube_is_h(orc):
    # every main-orthotope block that lands inside is h(w) = w + (0, N/2, 0)
    N = 32
    for wz in range(N // 2):
        for wy in range(N // 2):
            for wx in range(N // 2):
                c, xyz, _ = orc.lambda3(N, wx, wy, wz)
                if c == orc.L3_INSIDE:
                    assert xyz == (wx, wy + N // 2, wz)


def test_lambda3_printed_branches(orc):
    """Slab blocks: the inside branch is the printed (w_x+qb, w_y+2qb, w_z-n/2)
     verbatim; the reflected branch is the printed
    (b(1+2q)-w_x, 2b(1+q)-w_y, 2b-w_z+n/2) with w_x, w_y read in
    copy-local coordinates, w_z in slab coordinates, minus the lattice
    correction 1 per axis (reading E11)."""
    N = 64
    h = N // 2
    seen_in = seen_out = 0
    for wz in range(h, 3 * N // 4):
        for wy in range(1, N // 2):
            b = 1 << (wy.bit_length() - 1)
            for wx in range(N // 2):
                q = wx // b
                c, xyz, _ = orc.lambda3(N, wx, wy, wz)
                if c == orc.L3_INSIDE:
                    assert xyz == (wx + q * b, wy + 2 * q * b, wz - h)
                    seen_in += 1
                elif c == orc.L3_REFLECTED:
                    u, v, w = wx - q * b, wy - b, wz - h
                    # printed constants with local coordinates and slab-local w_z - n/2 ... :
                    X = b * (1 + 2 * q) - u - 1
                    Y = 2 * b * (1 + q) - v - 1
                    Z = 2 * b - w - 1
                    assert xyz == (X, Y, Z)
                    seen_out += 1
    assert seen_in > 0 and seen_out > 0


def test_lambda3_tie_rule_diagonal_reflects(orc):
    # blocks whose h-image lies ON the diagonal plane x+z = y take the
    # reflected branch ("diagonal or outside")
    N = 32
    for wz in range(N // 2):
        for wy in range(N // 2):
            for wx in range(N // 2):
                if wx + wz == wy + N // 2:
                    assert orc.lambda3(N, wx, wy, wz)[0] == orc.L3_REFLECTED
