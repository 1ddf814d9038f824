"""Oracle pins for the lambda2 "level-square" launch order (reading E22,
include/smap.h launch-order note).  The launch order is an implementation
choice (the paper fixes none), so it is pinned by what must hold for
ANY launch order -- every grid block visited exactly once, hence an exact
element cover, also across omega_x shards -- and by an independent nested-loop
enumeration of the square walk (level b = 1, 2, 4, ...; one b x b copy square
at a time, rows b .. 2b-1 in order) compared with the oracle's O(1) per-block
decode (or_block_coords, order=1).  CPU only."""
import numpy as np
import pytest

SQ_CASES = [(256, 4, 1), (256, 4, 4), (64, 1, 2), (1024, 16, 1), (512, 8, 8), (128, 2, 16)]


@pytest.mark.parametrize("n,rho,G", SQ_CASES)
@pytest.mark.parametrize("inclusive", [False, True])
def test_square_order_exact_cover(orc, n, rho, G, inclusive):
    hits = None
    launched = 0
    for r in range(G):
        hits, res = orc.element_hits(2, inclusive, False, n, rho, rank=r, G=G, hits=hits, order="squares")
        launched += res["launched"]
        assert res["outside"] == 0
    V = n * (n + 1) // 2 if inclusive else n * (n - 1) // 2
    assert len(hits) == V and bool((hits == 1).all())
    assert launched == (n * (n + rho) // 2 if inclusive else n * n // 2)


def square_walk(N, W, wx0, inclusive):
    """Grid blocks omega = (wx, wy) of one shard in the level-square order,
    by plain nested loops: row 0 first, then for each level b the copy
    squares s (columns wx0 + s b .. wx0 + s b + b - 1) one at a time, row by
    row; a shard narrower than one copy walks its rows [b, 2b) whole; finally
    row N (inclusive)."""
    out = [(wx0 + x, 0) for x in range(W)]
    b = 1
    while b < N:
        if b <= W:
            for s in range(W // b):
                for wy in range(b, 2 * b):
                    for c in range(b):
                        out.append((wx0 + s * b + c, wy))
        else:
            for wy in range(b, 2 * b):
                for x in range(W):
                    out.append((wx0 + x, wy))
        b *= 2
    if inclusive:
        out += [(wx0 + x, N) for x in range(W)]
    return out


@pytest.mark.parametrize("N,G", [(2, 1), (8, 1), (16, 2), (64, 4), (128, 1), (128, 16), (256, 8)])
@pytest.mark.parametrize("inclusive", [False, True])
def test_square_order_is_the_nested_square_walk(orc, N, G, inclusive):
    W = N // 2 // G
    for r in range(G):
        rows = orc.map_dump(2, inclusive, False, N, rank=r, G=G, order="rows")
        sq = orc.map_dump(2, inclusive, False, N, rank=r, G=G, order="squares")
        walk = square_walk(N, W, r * W, inclusive)
        assert len(walk) == len(sq) == len(rows)
        assert len(set(walk)) == len(walk)                      # a walk visits each block once
        # the record of the k-th square-order block = the row-order record of its omega
        idx = np.array([wy * W + (wx - r * W) for wx, wy in walk], np.int64)
        assert np.array_equal(sq, rows[idx])


@pytest.mark.parametrize("N", [16, 64, 256])
def test_square_order_rows_stay_in_one_band(orc, N):
    # the point of the order: consecutive blocks of one square land in the same
    # 2b-row band of the triangle (the copy q = s sits at rows I in [2qb+b, 2qb+2b))
    sq = orc.map_dump(2, False, False, N, order="squares")
    W = N // 2
    b = 1
    k = W                                                       # after row 0
    while b < N:
        if b <= W:
            for s in range(W // b):
                blk = sq[k:k + b * b]
                I = blk[:, 1]
                assert I.min() >= 2 * s * b + b and I.max() < 2 * s * b + 2 * b
                k += b * b
        else:
            k += b * W
        b *= 2
