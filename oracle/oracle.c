/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for arXiv 1610.07394
 * ("Possibilities of Recursive GPU Mapping for Discrete Orthogonal Simplices").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / `--impl reference` legs may load this library.
 * It shares NO code, header, table or constant generator with the CUDA path
 * (paper_1610_07394_b200/csrc); neither side includes or links the other.
 *
 * Citations: "P:a-b" = /root/reference/PAPER.md lines a-b (LaTeX source),
 * "S:a-b" = SPEC.md lines a-b.  "Reading Ek" = the numbered reading in
 * DESIGN.md section 3 (where the paper is silent, garbled or inconsistent).
 *
 * Conventions (readings E1, E13, E16):
 *   - m=2 strict pairs     {(i,j): 0 <= j < i < n}        ~ Delta^2_{n-1}
 *   - m=2 inclusive pairs  {(i,j): 0 <= j <= i < n}       ~ Delta^2_n
 *   - m=3 strict triples   {(i,j,k): 0 <= i < j < k < n}  ~ Delta^3_{n-2}
 *   - packed layout = position in the plain nested-loop enumeration
 *     (m=2: i outer, j inner; m=3: k outer, j middle, i inner).
 *
 * Pins (tests/test_oracle_*.py, tests/golden/): closed forms of Eq.(2)/(3),
 * brute-force enumeration of Eq.(1), the recursive-set volume recurrences,
 * SPEC's worked examples, exhaustive bijection of both maps, agreement with
 * the independent recursive constructions, fp64 numpy evaluation of the
 * payloads, and closed-form payload special cases.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC
 * (no FMA contraction: every fp32 operation below rounds exactly as written).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

/* ======================================================================
 * L0 -- simplex geometry
 * ====================================================================== */

/* Eq.(2): V(Delta_n^m) = C(n+m-1, m) = n(n+1)...(n+m-1)/m!.
 * Multiplicative form: after step i the running value is C(n+i-1, i). */
uint64_t or_simplex_volume(int m, uint64_t n)
{
    if (m < 1 || n == 0) return 0;
    u128 r = 1;
    for (int i = 1; i <= m; i++) r = r * (u128)(n + (uint64_t)i - 1) / (u128)i;
    return (uint64_t)r;
}

/* Eq.(1), with the cell convention of reading E1:
 * x in Delta_n^m  <=>  x_i >= 0 for all i  and  sum_i x_i <= n-1. */
int or_simplex_contains(int m, uint64_t n, const int64_t *x)
{
    if (n == 0) return 0;
    int64_t s = 0;
    for (int i = 0; i < m; i++) {
        if (x[i] < 0) return 0;
        s += x[i];
    }
    return s <= (int64_t)n - 1;
}

/* Brute force: count the points of the box [0,n)^m that satisfy Eq.(1). */
uint64_t or_enumerate_count(int m, uint64_t n)
{
    if (m < 1 || m > 6 || n == 0) return 0;
    int64_t x[6] = {0, 0, 0, 0, 0, 0};
    uint64_t count = 0;
    for (;;) {
        count += (uint64_t)or_simplex_contains(m, n, x);
        int d = 0;                                  /* odometer increment */
        while (d < m && ++x[d] == (int64_t)n) { x[d] = 0; d++; }
        if (d == m) break;
    }
    return count;
}

/* Eq.(3): V(Delta_n^{m}) = sum_{i=1..n} V(Delta_i^{m-1}). */
uint64_t or_stacked_volume(int m, uint64_t n)
{
    uint64_t s = 0;
    for (uint64_t i = 1; i <= n; i++) s += or_simplex_volume(m - 1, i);
    return s;
}

/* Eq.(4), P:157-161 at finite n: alpha = V(Pi_n^m)/V(Delta_n^m) - 1 with the
 * bounding box Pi_n^m = [0,n)^m. */
double or_bb_alpha(int m, uint64_t n)
{
    double box = 1.0;
    for (int i = 0; i < m; i++) box *= (double)n;
    return box / (double)or_simplex_volume(m, n) - 1.0;
}

/* V(S_n^2) = (n/2)^2 + 2 V(S_{n/2}^2), V(S_2^2) = 1 (so V(S_1)=0). */
uint64_t or_vs2_recurrence(uint64_t n)
{
    if (n <= 1) return 0;
    return (n / 2) * (n / 2) + 2 * or_vs2_recurrence(n / 2);
}

/* two-branch V(S_n^3) = (n/2)^3 + 2 V(S_{n/2}^3). */
uint64_t or_vs3_recurrence(uint64_t n)
{
    if (n <= 1) return 0;
    return (n / 2) * (n / 2) * (n / 2) + 2 * or_vs3_recurrence(n / 2);
}

/* arity-3 V(S_n^3) = (n/2)^3 + 3 V(S_{n/2}^3) (analysis only). */
uint64_t or_vs3_arity3_recurrence(uint64_t n)
{
    if (n <= 1) return 0;
    return (n / 2) * (n / 2) * (n / 2) + 3 * or_vs3_arity3_recurrence(n / 2);
}

/* the general recursive set V(S_n^m) = (r n)^m + beta V(S_{r n}^m), r = 1/rden,
 * written top-down exactly as printed (V(S_1) = 0); UINT64_MAX when n is not a power of
 * rden or a value overflows 64 bits.  r = 1/2, beta = 2 is lambda2's set (m = 2) and the
 * two-branch tetrahedral set (m = 3); beta = 3, m = 3 the arity-3 set. */
uint64_t or_vsm_recurrence(int m, uint64_t n, uint64_t beta, uint64_t rden)
{
    if (n <= 1) return n == 1 ? 0 : UINT64_MAX;
    if (n % rden != 0) return UINT64_MAX;
    uint64_t sub = or_vsm_recurrence(m, n / rden, beta, rden);
    if (sub == UINT64_MAX) return UINT64_MAX;
    u128 cube = 1;
    for (int i = 0; i < m; i++) {
        cube *= (u128)(n / rden);
        if (cube >> 64) return UINT64_MAX;
    }
    u128 v = cube + (u128)beta * sub;
    return (v >> 64) ? UINT64_MAX : (uint64_t)v;
}

/* the extra volume at a finite n, V(S_n^m) / V(Delta_n^m) - 1, with V(Delta_n^m)
 * = C(n+m-1, m) by counting in long double (pins the limit numerically at large n) */
double or_vsm_alpha(int m, uint64_t n, uint64_t beta, uint64_t rden)
{
    uint64_t vs = or_vsm_recurrence(m, n, beta, rden);
    if (vs == UINT64_MAX) return NAN;
    long double vd = 1.0L;
    for (int i = 0; i < m; i++) vd = vd * (long double)(n + i) / (long double)(i + 1);
    return (double)((long double)vs / vd - 1.0L);
}

/* ======================================================================
 * L2 -- block-space maps
 * ====================================================================== */

/* floor(log2 y) by repeated halving -- the plain definition (the paper's
 * clz identities at P:373 and P:379 are errata; readings E3/E4). */
int or_floor_log2(uint64_t y)
{
    if (y == 0) return -1;
    int l = 0;
    while (y >= 2) { y /= 2; l++; }
    return l;
}

static uint64_t or_pow2(int l)
{
    uint64_t r = 1;
    for (int i = 0; i < l; i++) r *= 2;
    return r;
}

/* lambda2, P:346-359 (Eq. map2d):  b = 2^floor(log2 w_y),  q = floor(w_x/b),
 *   lambda(w) = (w_x + q b, w_y + 2 q b).
 * Image (x, y) with x < y: x is the block column J, y the block row I
 * (reading E13).  Defined for w_y >= 1 only (reading E5); returns -1 else. */
int or_lambda2(uint64_t wx, uint64_t wy, uint64_t *x, uint64_t *y)
{
    if (wy == 0) return -1;
    uint64_t b = or_pow2(or_floor_log2(wy));
    uint64_t q = wx / b;
    *x = wx + q * b;
    *y = wy + 2 * q * b;
    return 0;
}

/* Independent pin for lambda2: the recursive set S_N^2 of P:307-312 read as
 * a construction.  Rows w_y >= N/2 are the main (N/2)x(N/2) orthotope at the
 * identity; the remaining rows hold two copies of S_{N/2}^2, the left one at
 * offset (0,0) and the right one shifted by (N/2, N/2). */
int or_rec2(uint64_t wx, uint64_t wy, uint64_t N, uint64_t *x, uint64_t *y)
{
    if (wy == 0 || N < 2) return -1;
    if (wy >= N / 2) { *x = wx; *y = wy; return 0; }
    if (wx < N / 4) return or_rec2(wx, wy, N / 2, x, y);
    if (or_rec2(wx - N / 4, wy, N / 2, x, y)) return -1;
    *x += N / 2;
    *y += N / 2;
    return 0;
}

/* lambda3, reading R3 (E11/E12) of P:565-597.  Grid (N/2, N/2, 3N/4).
 * Target frame T_N = {(X,Y,Z): X,Z >= 0, X+Z < Y <= N-1} (|T_N| = (N^3-N)/6,
 * P:559).  Steps in the paper's order:
 *   main orthotope w_z < N/2: h(w) = w + (0, N/2, 0), kept when inside;
 *   otherwise the slab w_z >= N/2: b = 2^floor(log2 w_y), q = floor(w_x/b) as
 *   in lambda2, copy-local (u,v,w) = (w_x - qb, w_y - b, w_z - N/2);
 *   inside branch (w_x + qb, w_y + 2qb, w_z - N/2) and the
 *   "diagonal or outside" branch, a point reflection through the
 *   centre of the copy's cube top face (lattice form: 2qb+b-1-u, 2qb+2b-1-v,
 *   2b-1-w).  The main cube uses the same two branches with b = N/2, q = 0.
 * out[0..2] = (X,Y,Z) in the paper frame; out[3..5] = sorted block triple
 * (I,J,K) = (X, X+Z, Y), I <= J < K (reading E13).
 * Returns OR_L3_INSIDE / OR_L3_REFLECTED, or OR_L3_SPARE (slab row w_y = 0;
 * out[0] = body-diagonal block d = w_x + (N/2) w for w <= 1, else -1;
 * reading E14), or OR_L3_FILLER (w >= b; unused). */
enum { OR_L3_INSIDE = 0, OR_L3_REFLECTED = 1, OR_L3_SPARE = 2, OR_L3_FILLER = 3 };

int or_lambda3(uint64_t N, uint64_t wx, uint64_t wy, uint64_t wz, int64_t *out)
{
    int64_t b, q, u, v, w;
    int64_t h = (int64_t)N / 2;
    for (int t = 0; t < 6; t++) out[t] = -1;
    if ((int64_t)wz < h) {                       /* main orthotope (n/2)^3 */
        b = h; q = 0;
        u = (int64_t)wx; v = (int64_t)wy; w = (int64_t)wz;
    } else {                                     /* recursion slab */
        w = (int64_t)wz - h;
        if (wy == 0) {
            if (w <= 1) out[0] = (int64_t)wx + h * w;
            return OR_L3_SPARE;
        }
        b = (int64_t)or_pow2(or_floor_log2(wy));
        if (w >= b) return OR_L3_FILLER;
        q = (int64_t)wx / b;
        u = (int64_t)wx - q * b;
        v = (int64_t)wy - b;
    }
    int inside = (u + w < v + b);                /* image satisfies X+Z < Y */
    int64_t X, Y, Z;
    if (inside) {
        X = 2 * q * b + u;                       /* = w_x + q b           */
        Y = 2 * q * b + b + v;                   /* = w_y + 2 q b         */
        Z = w;                                   /* = w_z - n/2 (slab)    */
    } else {
        X = 2 * q * b + b - 1 - u;
        Y = 2 * q * b + 2 * b - 1 - v;
        Z = 2 * b - 1 - w;
    }
    out[0] = X; out[1] = Y; out[2] = Z;
    out[3] = X; out[4] = X + Z; out[5] = Y;
    return inside ? OR_L3_INSIDE : OR_L3_REFLECTED;
}

/* Independent pin for lambda3: the two-branch recursive set of P:525-563 as
 * a recursive construction, with the main cube folded by MEMBERSHIP (keep
 * h(w) if it lies in T_N, else reflect) instead of by the closed predicate,
 * and no floor-log2: the slab recurses into two half-size sub-problems at
 * offsets (0,0,0) and (N/2,N/2,0).  Returns 1 and (X,Y,Z), or 0 (unused). */
static int or_in_T(int64_t X, int64_t Y, int64_t Z) { return X >= 0 && Z >= 0 && X + Z < Y; }

int or_rec3(uint64_t N, uint64_t x, uint64_t y, uint64_t z, int64_t *out)
{
    int64_t s = (int64_t)N / 2;
    if ((int64_t)z < s) {
        int64_t X = (int64_t)x, Y = s + (int64_t)y, Z = (int64_t)z;    /* h(w) */
        if (!or_in_T(X, Y, Z)) {
            X = s - 1 - (int64_t)x;
            Y = s + s - 1 - (int64_t)y;
            Z = 2 * s - 1 - (int64_t)z;
        }
        out[0] = X; out[1] = Y; out[2] = Z;
        return 1;
    }
    if (N <= 2) return 0;
    int64_t w = (int64_t)z - s;
    if (y == 0) return 0;
    int64_t c = (int64_t)N / 4;
    int64_t sx = (int64_t)x / c;                 /* which sub-problem */
    int64_t cx = (int64_t)x - sx * c, cy, cz;
    if ((int64_t)y >= c) { cy = (int64_t)y - c; cz = w; }
    else {
        if (w >= (int64_t)N / 8) return 0;
        cy = (int64_t)y; cz = w + c;
    }
    if (!or_rec3(N / 2, (uint64_t)cx, (uint64_t)cy, (uint64_t)cz, out)) return 0;
    out[0] += sx * s;
    out[1] += sx * s;
    return 1;
}

/* ======================================================================
 * Block-level exhaustive cover checks (S:386-398 CoverageReport)
 * res = {mapped, missing, duplicates, outside}.  corrupt != 0 injects a unit
 * translation (x+1) into the image of every block with odd w_x, so that the
 * checker can be shown not to be vacuously green.
 * ====================================================================== */
int or_check_cover2_blocks(uint64_t N, int corrupt, int64_t *res)
{
    uint32_t *hit = calloc(N * N, sizeof(uint32_t));
    if (!hit) return -1;
    int64_t mapped = 0, outside = 0, missing = 0, dup = 0;
    for (uint64_t wy = 1; wy < N; wy++)
        for (uint64_t wx = 0; wx < N / 2; wx++) {
            uint64_t x, y;
            or_lambda2(wx, wy, &x, &y);
            if (corrupt && (wx & 1)) x += 1;
            mapped++;
            if (x < y && y < N) hit[y * N + x]++; else outside++;
        }
    for (uint64_t y = 0; y < N; y++)
        for (uint64_t x = 0; x < y; x++) {
            if (hit[y * N + x] == 0) missing++;
            if (hit[y * N + x] > 1) dup += hit[y * N + x] - 1;
        }
    free(hit);
    res[0] = mapped; res[1] = missing; res[2] = dup; res[3] = outside;
    return 0;
}

/* lambda3 over the full grid, target {I <= J < K < N}; the spare row's body
 * blocks must be exactly d = 0..N-1.  res additionally holds
 * {.., n_inside, n_reflected, n_spare, n_filler, body_missing, body_dup}. */
int or_check_cover3_blocks(uint64_t N, int corrupt, int64_t *res)
{
    uint32_t *hit = calloc(N * N * N, sizeof(uint32_t));
    uint32_t *body = calloc(N, sizeof(uint32_t));
    if (!hit || !body) { free(hit); free(body); return -1; }
    int64_t mapped = 0, outside = 0, missing = 0, dup = 0;
    int64_t cls[4] = {0, 0, 0, 0}, bmiss = 0, bdup = 0;
    for (uint64_t wz = 0; wz < 3 * N / 4; wz++)
        for (uint64_t wy = 0; wy < N / 2; wy++)
            for (uint64_t wx = 0; wx < N / 2; wx++) {
                int64_t o[6];
                int c = or_lambda3(N, wx, wy, wz, o);
                cls[c]++;
                if (c == OR_L3_SPARE) {
                    if (o[0] >= 0) { if (o[0] < (int64_t)N) body[o[0]]++; else outside++; }
                    continue;
                }
                if (c == OR_L3_FILLER) continue;
                int64_t I = o[3], J = o[4], K = o[5];
                if (corrupt && (wx & 1)) I += 1;
                mapped++;
                if (I >= 0 && I <= J && J < K && K < (int64_t)N) hit[(K * N + J) * N + I]++;
                else outside++;
            }
    for (uint64_t K = 0; K < N; K++)
        for (uint64_t J = 0; J < K; J++)
            for (uint64_t I = 0; I <= J; I++) {
                uint32_t h = hit[(K * N + J) * N + I];
                if (h == 0) missing++;
                if (h > 1) dup += h - 1;
            }
    for (uint64_t d = 0; d < N; d++) {
        if (body[d] == 0) bmiss++;
        if (body[d] > 1) bdup += body[d] - 1;
    }
    free(hit); free(body);
    res[0] = mapped; res[1] = missing; res[2] = dup; res[3] = outside;
    res[4] = cls[0]; res[5] = cls[1]; res[6] = cls[2]; res[7] = cls[3];
    res[8] = bmiss; res[9] = bdup;
    return 0;
}

/* Number of grid blocks on which lambda2 and rec2 disagree. */
int64_t or_check_rec2(uint64_t N)
{
    int64_t bad = 0;
    for (uint64_t wy = 1; wy < N; wy++)
        for (uint64_t wx = 0; wx < N / 2; wx++) {
            uint64_t x1, y1, x2, y2;
            or_lambda2(wx, wy, &x1, &y1);
            if (or_rec2(wx, wy, N, &x2, &y2) || x1 != x2 || y1 != y2) bad++;
        }
    return bad;
}

/* Number of grid blocks on which lambda3 (R3) and rec3 disagree (image or
 * mapped/unused classification). */
int64_t or_check_rec3(uint64_t N)
{
    int64_t bad = 0;
    for (uint64_t wz = 0; wz < 3 * N / 4; wz++)
        for (uint64_t wy = 0; wy < N / 2; wy++)
            for (uint64_t wx = 0; wx < N / 2; wx++) {
                int64_t a[6], r[3];
                int c = or_lambda3(N, wx, wy, wz, a);
                int ok = or_rec3(N, wx, wy, wz, r);
                int mapped = (c == OR_L3_INSIDE || c == OR_L3_REFLECTED);
                if (mapped != ok) { bad++; continue; }
                if (mapped && (a[0] != r[0] || a[1] != r[1] || a[2] != r[2])) bad++;
            }
    return bad;
}

/* ======================================================================
 * a5 -- packed ranks (reading E16).  The packed layout is DEFINED as the
 * position in the nested-loop enumeration (or_index_write below); these
 * closed forms are pinned against it by tests/test_oracle_payloads.py.
 * ====================================================================== */
uint64_t or_rank2_strict(uint64_t i, uint64_t j) { return i * (i - 1) / 2 + j; }
uint64_t or_rank2_incl(uint64_t i, uint64_t j)   { return i * (i + 1) / 2 + j; }
uint64_t or_rank3(uint64_t i, uint64_t j, uint64_t k)
{
    u128 ck3 = (u128)k * (k - 1) * (k - 2) / 6;
    return (uint64_t)ck3 + j * (j - 1) / 2 + i;
}
/* inclusive triples i <= j <= k in nested-loop order (k outer, i inner):
 * C(k+2,3) + C(j+1,2) + i  (the paper's Delta_n^3 in the cell convention, E1) */
uint64_t or_rank3_incl(uint64_t i, uint64_t j, uint64_t k)
{
    u128 t = (u128)k * (k + 1) * (k + 2) / 6;
    return (uint64_t)t + j * (j + 1) / 2 + i;
}

/* Useful-element count V of each domain (closed forms of L0). */
uint64_t or_domain_volume(int m, int inclusive, uint64_t n)
{
    if (m == 2) return inclusive ? or_simplex_volume(2, n) : or_simplex_volume(2, n - 1);
    if (m == 3) return inclusive ? or_simplex_volume(3, n) : (n >= 2 ? or_simplex_volume(3, n - 2) : 0);
    return 0;
}

/* ======================================================================
 * a4 -- thread -> element for the one-element-per-thread launch
 * (blocks of rho^m threads; readings E6, E14).
 * map: 0 = bounding box (identity + filter),
 *      1 = lambda,
 *      2 = enumeration baseline: the block coordinates come from
 *          the linear block rank (or_block_coords), the threads filter like BB.
 * Block coordinates (wx, wy, wz) are the paper's omega (BB / ENUM: the block).
 * Returns 1 and e[] = (i, j[, k]) for a useful thread, 0 for an idle one.
 * ====================================================================== */
int or_thread_elem2(int inclusive, int map, uint64_t N, uint64_t rho,
                    uint64_t wx, uint64_t wy, uint64_t tx, uint64_t ty, int64_t *e)
{
    if (map == 0 || map == 2) {                   /* BB / ENUM: block (J, I) = (wx, wy) */
        uint64_t i = wy * rho + ty, j = wx * rho + tx;
        if (inclusive ? (j <= i) : (j < i)) { e[0] = (int64_t)i; e[1] = (int64_t)j; return 1; }
        return 0;
    }
    if (inclusive && (wy == 0 || wy == N)) {      /* one diagonal block per row-0/row-N block */
        uint64_t D = (wy == 0) ? wx : wx + N / 2;
        if (tx > ty) return 0;
        e[0] = (int64_t)(D * rho + ty); e[1] = (int64_t)(D * rho + tx);
        return 1;
    }
    if (!inclusive && wy == 0) {                  /* diagonal pair D1 = wx, D2 = N-1-wx */
        uint64_t D1 = wx, D2 = N - 1 - wx;
        if (tx < ty) { e[0] = (int64_t)(D1 * rho + ty); e[1] = (int64_t)(D1 * rho + tx); return 1; }
        if (tx > ty) {                            /* D2 point-reflected inside the block */
            e[0] = (int64_t)(D2 * rho + rho - 1 - ty);
            e[1] = (int64_t)(D2 * rho + rho - 1 - tx);
            return 1;
        }
        return 0;
    }
    uint64_t J, I;
    or_lambda2(wx, wy, &J, &I);
    e[0] = (int64_t)(I * rho + ty); e[1] = (int64_t)(J * rho + tx);
    return 1;
}

int or_thread_elem3(int map, uint64_t N, uint64_t rho, uint64_t wx, uint64_t wy, uint64_t wz,
                    uint64_t a, uint64_t b, uint64_t c, int64_t *e)
{
    if (map == 0 || map == 2) {                   /* BB / ENUM: block (I, J, K) = (wx, wy, wz) */
        uint64_t i = wx * rho + a, j = wy * rho + b, k = wz * rho + c;
        if (i < j && j < k) { e[0] = (int64_t)i; e[1] = (int64_t)j; e[2] = (int64_t)k; return 1; }
        return 0;
    }
    int64_t o[6];
    int cls = or_lambda3(N, wx, wy, wz, o);
    if (cls == OR_L3_FILLER) return 0;
    if (cls == OR_L3_SPARE) {                     /* body-diagonal block d: a < b < c */
        if (o[0] < 0 || !(a < b && b < c)) return 0;
        uint64_t d = (uint64_t)o[0];
        e[0] = (int64_t)(d * rho + a); e[1] = (int64_t)(d * rho + b); e[2] = (int64_t)(d * rho + c);
        return 1;
    }
    uint64_t I = (uint64_t)o[3], J = (uint64_t)o[4], K = (uint64_t)o[5];
    if (I < J) {                                  /* interior block I < J < K */
        e[0] = (int64_t)(I * rho + a); e[1] = (int64_t)(J * rho + b); e[2] = (int64_t)(K * rho + c);
        return 1;
    }
    /* face block I == J < K: folds {I=J<K} (a<b) and {I<J=K} (a>b) */
    if (a < b) { e[0] = (int64_t)(I * rho + a); e[1] = (int64_t)(I * rho + b); e[2] = (int64_t)(K * rho + c); return 1; }
    if (a > b) { e[0] = (int64_t)(I * rho + c); e[1] = (int64_t)(K * rho + b); e[2] = (int64_t)(K * rho + a); return 1; }
    return 0;
}

/* Launch geometry of the one-element-per-thread grid (same definition as
 * include/smap.h, restated here): the block-linear id enumerates
 *   lambda2:  bid = wy*W + (wx - wx0),            wy in [0,H), H = N or N+1
 *   lambda3:  bid = (wz*(N/2) + wy)*W + (wx - wx0), wz in [0, 3N/4)
 *   BB2:      bid = I*N + J      (wx = J, wy = I)
 *   BB3:      bid = (K*N + J)*N + I
 *   ENUM2:    bid = row-major rank of the block (J, I) among J <= I
 *   ENUM3:    bid = colex rank of the block (I, J, K) among I <= J <= K
 * with W = N/(2G) columns per shard and wx0 = rank*W; threads within a block
 * are t = ty*rho + tx (m=2) and t = (c*rho + b)*rho + a (m=3). */
static uint64_t or_ipow(uint64_t b, int e) { uint64_t r = 1; while (e-- > 0) r *= b; return r; }

/* "Approach n from above": for any n the grid is the one of
 * n' = 2^ceil(log2 n), and threads whose element has an index >= n (the
 * largest index: i for pairs j < i, k for triples i < j < k) are idle. */
uint64_t or_padded_n(uint64_t n) { uint64_t p = 1; while (p < n) p *= 2; return p; }

uint64_t or_grid_blocks(int m, int inclusive, int map, uint64_t N, uint64_t G)
{
    if (map == 0) return or_ipow(N, m);
    if (map == 2) return m == 2 ? N * (N + 1) / 2 : N * (N + 1) * (N + 2) / 6;
    if (m == 2) return (N / 2 / G) * (inclusive ? N + 1 : N);
    return (N / 2 / G) * (N / 2) * (3 * N / 4);
}

/* The lambda2 "square" launch order (order = 1): rows 0 and N as in row
 * order; the rows [b, 2b) of level b are enumerated one b x b copy square at
 * a time (found here by plain search over the levels), row by row. */
static int or_block_coords(int m, int inclusive, int map, uint64_t N, uint64_t rank, uint64_t G,
                           int order, uint64_t bid, uint64_t *w)
{
    (void)inclusive;
    if (map == 0) {
        for (int d = 0; d < m; d++) { w[d] = bid % N; bid /= N; }
        return 0;
    }
    if (map == 2) {                  /* enumeration order, found by walking the rows (no roots) */
        if (m == 2) {
            uint64_t I = 0;
            while (bid >= I + 1) { bid -= I + 1; I++; }           /* row I holds I + 1 blocks */
            w[0] = bid; w[1] = I;
            return 0;
        }
        uint64_t K = 0, J = 0;
        while (bid >= (K + 1) * (K + 2) / 2) { bid -= (K + 1) * (K + 2) / 2; K++; }   /* layer K */
        while (bid >= J + 1) { bid -= J + 1; J++; }
        w[0] = bid; w[1] = J; w[2] = K;
        return 0;
    }
    uint64_t W = N / 2 / G, wx0 = rank * W;
    if (m == 2 && order == 1 && bid / W >= 1 && bid / W < N) {
        uint64_t b = 1;
        while (!(bid / W >= b && bid / W < 2 * b)) b *= 2;      /* level containing this row */
        uint64_t t = bid - b * W;
        if (b <= W) {
            uint64_t s = t / (b * b), r = t % (b * b);
            w[1] = b + r / b; w[0] = wx0 + s * b + r % b;
        } else {
            w[1] = b + t / W; w[0] = wx0 + t % W;
        }
        return 0;
    }
    w[0] = wx0 + bid % W; bid /= W;
    if (m == 2) { w[1] = bid; return 0; }
    w[1] = bid % (N / 2); w[2] = bid / (N / 2);
    return 0;
}

/* Writes, per launched thread in launch order, the packed rank of its element
 * or UINT64_MAX when idle.  len must equal grid_blocks * rho^m. */
int or_thread_dump(int m, int inclusive, int map, uint64_t n, uint64_t rho, uint64_t rank,
                   uint64_t G, int order, uint64_t *out, uint64_t len)
{
    /* m=3 inclusive (reading E24): the strict map of n + 2, element (i, j, k) = (i', j'-1, k'-2) */
    uint64_t nint = (m == 3 && inclusive) ? n + 2 : n;
    uint64_t N = or_padded_n(nint) / rho, T = or_ipow(rho, m);
    uint64_t nb = or_grid_blocks(m, inclusive, map, N, G);
    if (nb * T != len) return -1;
    for (uint64_t bid = 0; bid < nb; bid++) {
        uint64_t w[3] = {0, 0, 0};
        or_block_coords(m, inclusive, map, N, rank, G, order, bid, w);
        for (uint64_t t = 0; t < T; t++) {
            int64_t e[3];
            int ok;
            if (m == 2) ok = or_thread_elem2(inclusive, map, N, rho, w[0], w[1], t % rho, t / rho, e);
            else ok = or_thread_elem3(map, N, rho, w[0], w[1], w[2], t % rho, (t / rho) % rho, t / (rho * rho), e);
            uint64_t p = UINT64_MAX;
            if (ok && e[m == 2 ? 0 : 2] >= (int64_t)nint) ok = 0;  /* padded grid: beyond n */
            if (ok) {
                if (m == 2) p = inclusive ? or_rank2_incl((uint64_t)e[0], (uint64_t)e[1])
                                          : or_rank2_strict((uint64_t)e[0], (uint64_t)e[1]);
                else if (inclusive) p = or_rank3_incl((uint64_t)e[0], (uint64_t)e[1] - 1, (uint64_t)e[2] - 2);
                else p = or_rank3((uint64_t)e[0], (uint64_t)e[1], (uint64_t)e[2]);
            }
            out[bid * T + t] = p;
        }
    }
    return 0;
}

/* Element-level cover: adds one hit per useful thread of shard (rank, G)
 * into hits[p] (caller zeroes; length V).  res = {launched, useful, outside}
 * where outside counts elements that are not in the target domain. */
int or_element_hits(int m, int inclusive, int map, uint64_t n, uint64_t rho, uint64_t rank,
                    uint64_t G, int order, uint32_t *hits, uint64_t V, int64_t *res)
{
    uint64_t nint = (m == 3 && inclusive) ? n + 2 : n;     /* E24 */
    uint64_t N = or_padded_n(nint) / rho, T = or_ipow(rho, m);
    uint64_t nb = or_grid_blocks(m, inclusive, map, N, G);
    int64_t useful = 0, outside = 0;
    for (uint64_t bid = 0; bid < nb; bid++) {
        uint64_t w[3] = {0, 0, 0};
        or_block_coords(m, inclusive, map, N, rank, G, order, bid, w);
        for (uint64_t t = 0; t < T; t++) {
            int64_t e[3];
            int ok;
            if (m == 2) ok = or_thread_elem2(inclusive, map, N, rho, w[0], w[1], t % rho, t / rho, e);
            else ok = or_thread_elem3(map, N, rho, w[0], w[1], w[2], t % rho, (t / rho) % rho, t / (rho * rho), e);
            if (!ok) continue;
            if (e[m == 2 ? 0 : 2] >= (int64_t)nint && e[m == 2 ? 0 : 2] < (int64_t)(N * rho)) continue;  /* padded: idle */
            if (m == 3 && inclusive) { e[1] -= 1; e[2] -= 2; }  /* E24: back to i <= j <= k */
            int in;
            uint64_t p;
            if (m == 2) {
                in = e[1] >= 0 && e[0] < (int64_t)n && (inclusive ? e[1] <= e[0] : e[1] < e[0]);
                p = in ? (inclusive ? or_rank2_incl(e[0], e[1]) : or_rank2_strict(e[0], e[1])) : 0;
            } else {
                if (inclusive) {
                    in = e[0] >= 0 && e[0] <= e[1] && e[1] <= e[2] && e[2] < (int64_t)n;
                    p = in ? or_rank3_incl(e[0], e[1], e[2]) : 0;
                } else {
                    in = e[0] >= 0 && e[0] < e[1] && e[1] < e[2] && e[2] < (int64_t)n;
                    p = in ? or_rank3(e[0], e[1], e[2]) : 0;
                }
            }
            if (!in || p >= V) { outside++; continue; }
            hits[p]++;
            useful++;
        }
    }
    res[0] = (int64_t)(nb * T); res[1] = useful; res[2] = outside;
    return 0;
}

/* Useful elements carried by grid column wx (lambda maps; section 8e claim). */
int64_t or_column_work(int m, int inclusive, uint64_t n, uint64_t rho, uint64_t wx)
{
    uint64_t N = n / rho, T = or_ipow(rho, m);
    int64_t c = 0;
    if (m == 2) {
        uint64_t H = inclusive ? N + 1 : N;
        for (uint64_t wy = 0; wy < H; wy++)
            for (uint64_t t = 0; t < T; t++) {
                int64_t e[3];
                c += or_thread_elem2(inclusive, 1, N, rho, wx, wy, t % rho, t / rho, e);
            }
    } else {
        for (uint64_t wz = 0; wz < 3 * N / 4; wz++)
            for (uint64_t wy = 0; wy < N / 2; wy++)
                for (uint64_t t = 0; t < T; t++) {
                    int64_t e[3];
                    c += or_thread_elem3(1, N, rho, wx, wy, wz, t % rho, (t / rho) % rho, t / (rho * rho), e);
                }
    }
    return c;
}

/* ======================================================================
 * a6 -- payloads (the paper only names the problems, P:92-99, P:115-117;
 * definitions are reading E15, fp32 arithmetic order reading E17).
 * ====================================================================== */

/* Packed index write: out[p] = p in nested-loop order (defines the layout).
 * elem_bytes = 4 (uint32) or 8 (uint64). */
int or_index_write(int m, int inclusive, uint64_t n, void *out, int elem_bytes)
{
    uint64_t pos = 0;
    uint32_t *o4 = out; uint64_t *o8 = out;
    if (m == 2) {
        for (uint64_t i = 0; i < n; i++)
            for (uint64_t j = 0; inclusive ? j <= i : j < i; j++) {
                if (elem_bytes == 4) o4[pos] = (uint32_t)pos; else o8[pos] = pos;
                pos++;
            }
    } else {
        for (uint64_t k = 0; k < n; k++)
            for (uint64_t j = 0; inclusive ? j <= k : j < k; j++)
                for (uint64_t i = 0; inclusive ? i <= j : i < j; i++) {
                    if (elem_bytes == 4) o4[pos] = (uint32_t)pos; else o8[pos] = pos;
                    pos++;
                }
    }
    return 0;
}

/* Squared distance in fp32 (reading E17): d = p_b - p_a (three rounded
 * subtractions), r^2 = fma(dz, dz, fma(dy, dy, dx*dx)) with IEEE fused
 * multiply-adds (C99 fmaf, correctly rounded). */
static float or_r2(const float *pts, uint64_t a, uint64_t b)
{
    float dx = pts[3 * b + 0] - pts[3 * a + 0];
    float dy = pts[3 * b + 1] - pts[3 * a + 1];
    float dz = pts[3 * b + 2] - pts[3 * a + 2];
    float sx = dx * dx;
    float sxy = fmaf(dy, dy, sx);
    return fmaf(dz, dz, sxy);
}

/* EDM element: Euclidean distance ||x_i - x_j||_2 in fp32,
 * correctly-rounded sqrt. */
float or_edm_dist(const float *pts, uint64_t i, uint64_t j)
{
    return sqrtf(or_r2(pts, i, j));
}

/* Full strict-lower EDM in packed nested-loop order (i outer, j < i inner). */
int or_edm(uint64_t n, const float *pts, float *out)
{
    uint64_t pos = 0;
    for (uint64_t i = 0; i < n; i++)
        for (uint64_t j = 0; j < i; j++) out[pos++] = or_edm_dist(pts, i, j);
    return 0;
}

/* Softened Axilrod-Teller triple term (triple-interaction n-body, P:115-116;
 * reading E15, formula DESIGN.md section 3):
 *   a = r_ij^2 + eps2, b = r_jk^2 + eps2, c = r_ik^2 + eps2
 *   E = (8abc + 3(a+c-b)(a+b-c)(b+c-a)) / (8 (abc)^2 sqrt(abc))
 * which is (1 + 3 cos g1 cos g2 cos g3) / (r_ij r_jk r_ik)^3 via the law of
 * cosines.  Every fp32 operation is rounded in the order written. */
float or_atm_term(const float *pts, uint64_t i, uint64_t j, uint64_t k, float eps2)
{
    float a = or_r2(pts, i, j) + eps2;
    float b = or_r2(pts, j, k) + eps2;
    float c = or_r2(pts, i, k) + eps2;
    float ab = a * b;
    float abc = ab * c;
    float p1 = (a + c) - b;
    float p2 = (a + b) - c;
    float p3 = (b + c) - a;
    float p12 = p1 * p2;
    float P = p12 * p3;
    float num = (8.0f * abc) + (3.0f * P);
    float abc2 = abc * abc;
    float den = (8.0f * abc2) * sqrtf(abc);
    return num / den;
}

/* Neumaier compensated summation in fp64. */
typedef struct { double s, c; } or_nsum;
static void or_nadd(or_nsum *a, double x)
{
    double t = a->s + x;
    if (fabs(a->s) >= fabs(x)) a->c += (a->s - t) + x; else a->c += (x - t) + a->s;
    a->s = t;
}

static int or_threads(int nthreads)
{
#ifdef _OPENMP
    return nthreads > 0 ? nthreads : omp_get_max_threads();
#else
    (void)nthreads; return 1;
#endif
}

int or_max_threads(void) { return or_threads(0); }

/* Sum of ATM terms over i < j < k with k in [k_lo, k_hi), each k-row summed
 * in fp64 (Neumaier) and the rows combined in k order (thread-count
 * independent result). */
double or_atm_sum(uint64_t n, const float *pts, float eps2, uint64_t k_lo, uint64_t k_hi, int nthreads)
{
    if (k_hi > n) k_hi = n;
    if (k_lo >= k_hi) return 0.0;
    uint64_t R = k_hi - k_lo;
    double *row = calloc(R, sizeof(double));
    int nt = or_threads(nthreads);
    #pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
    for (uint64_t r = 0; r < R; r++) {
        uint64_t k = k_lo + r;
        or_nsum acc = {0.0, 0.0};
        for (uint64_t j = 0; j < k; j++)
            for (uint64_t i = 0; i < j; i++) or_nadd(&acc, (double)or_atm_term(pts, i, j, k, eps2));
        row[r] = acc.s + acc.c;
    }
    or_nsum tot = {0.0, 0.0};
    for (uint64_t r = 0; r < R; r++) or_nadd(&tot, row[r]);
    free(row);
    return tot.s + tot.c;
}

/* Triple correlation: 1 if all three pair distances are < R, compared
 * as r^2 < R*R in fp32. */
int or_tc_pred(const float *pts, uint64_t i, uint64_t j, uint64_t k, float R)
{
    float R2 = R * R;
    return or_r2(pts, i, j) < R2 && or_r2(pts, j, k) < R2 && or_r2(pts, i, k) < R2;
}

uint64_t or_tc_count(uint64_t n, const float *pts, float R, uint64_t k_lo, uint64_t k_hi, int nthreads)
{
    if (k_hi > n) k_hi = n;
    uint64_t total = 0;
    int nt = or_threads(nthreads);
    #pragma omp parallel for schedule(dynamic, 1) reduction(+:total) num_threads(nt)
    for (uint64_t k = k_lo; k < k_hi; k++)
        for (uint64_t j = 0; j < k; j++)
            for (uint64_t i = 0; i < j; i++) total += (uint64_t)or_tc_pred(pts, i, j, k, R);
    return total;
}

/* ======================================================================
 * a7 -- checksums of a (position, value) stream, order independent
 * (reading E21):
 *   cs[0] = count
 *   cs[1] = S0  = sum bits(v)            mod 2^64
 *   cs[2] = S1  = sum (p+1) * bits(v)    mod 2^64
 *   cs[3] = MIX = sum mix64(p ^ (bits(v) * K)) mod 2^64
 *   cs[4] = XR  = xor of bits(v)
 * bits(v) = the value's bit pattern zero-extended to 64 bits;
 * K = 0x9E3779B97F4A7C15; mix64 = the splitmix64 finaliser.
 * ====================================================================== */
static uint64_t or_mix64(uint64_t z)
{
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27; z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}

static void or_cs_add(uint64_t *cs, uint64_t p, uint64_t bits)
{
    cs[0] += 1;
    cs[1] += bits;
    cs[2] += (p + 1) * bits;
    cs[3] += or_mix64(p ^ (bits * 0x9E3779B97F4A7C15ULL));
    cs[4] ^= bits;
}

static uint32_t or_fbits(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

/* Checksum of a materialised array: element e is at position p0 + e. */
int or_cs_array(const void *arr, int kind /*0=u32,1=u64,2=f32*/, uint64_t p0, uint64_t len, uint64_t *cs)
{
    memset(cs, 0, 5 * sizeof(uint64_t));
    for (uint64_t e = 0; e < len; e++) {
        uint64_t bits = kind == 0 ? ((const uint32_t *)arr)[e]
                      : kind == 1 ? ((const uint64_t *)arr)[e]
                      : or_fbits(((const float *)arr)[e]);
        or_cs_add(cs, p0 + e, bits);
    }
    return 0;
}

/* Streaming checksum of the packed index write over outer rows [lo, hi)
 * (i for m=2, k for m=3); value = p (bits(p) = p for u32 and u64 layouts). */
int or_cs_index(int m, int inclusive, uint64_t n, uint64_t lo, uint64_t hi, int nthreads, uint64_t *cs)
{
    if (hi > n) hi = n;
    uint64_t c0 = 0, c1 = 0, c2 = 0, c3 = 0, c4 = 0;
    int nt = or_threads(nthreads);
    #pragma omp parallel for schedule(dynamic, 64) reduction(+:c0,c1,c2,c3) reduction(^:c4) num_threads(nt)
    for (uint64_t r = lo; r < hi; r++) {
        uint64_t c[5] = {0, 0, 0, 0, 0};
        if (m == 2) {
            uint64_t pos = inclusive ? or_rank2_incl(r, 0) : or_rank2_strict(r, 0);
            for (uint64_t j = 0; inclusive ? j <= r : j < r; j++, pos++) or_cs_add(c, pos, pos);
        } else {
            for (uint64_t j = 0; inclusive ? j <= r : j < r; j++) {
                uint64_t pos = inclusive ? or_rank3_incl(0, j, r) : or_rank3(0, j, r);
                for (uint64_t i = 0; inclusive ? i <= j : i < j; i++, pos++) or_cs_add(c, pos, pos);
            }
        }
        c0 += c[0]; c1 += c[1]; c2 += c[2]; c3 += c[3]; c4 ^= c[4];
    }
    cs[0] = c0; cs[1] = c1; cs[2] = c2; cs[3] = c3; cs[4] = c4;
    return 0;
}

/* Streaming checksum of the strict EDM over rows i in [lo, hi). */
int or_cs_edm(uint64_t n, const float *pts, uint64_t lo, uint64_t hi, int nthreads, uint64_t *cs)
{
    if (hi > n) hi = n;
    uint64_t c0 = 0, c1 = 0, c2 = 0, c3 = 0, c4 = 0;
    int nt = or_threads(nthreads);
    #pragma omp parallel for schedule(dynamic, 16) reduction(+:c0,c1,c2,c3) reduction(^:c4) num_threads(nt)
    for (uint64_t i = lo; i < hi; i++) {
        uint64_t c[5] = {0, 0, 0, 0, 0};
        uint64_t pos = or_rank2_strict(i, 0);
        for (uint64_t j = 0; j < i; j++, pos++) or_cs_add(c, pos, or_fbits(or_edm_dist(pts, i, j)));
        c0 += c[0]; c1 += c[1]; c2 += c[2]; c3 += c[3]; c4 ^= c[4];
    }
    cs[0] = c0; cs[1] = c1; cs[2] = c2; cs[3] = c3; cs[4] = c4;
    return 0;
}

/* ======================================================================
 * The lambda-order tile-blocked layout of m=2 outputs (E23; the
 * "succinct blocked" storage the paper pairs with block-space maps),
 * defined by enumeration: walk the shard's tiles in ROW launch order
 * (bid = wy*W + wx - wx0; for BB all tiles (I,J), J <= I, row-major) and give
 * each tile's elements the next positions, row by row (r = i - I*T), columns
 * in order; the strict row-0 slot holds D1's rows then D2's rows.
 * pos_of_rank[p] = position in this shard's array (-1 if another shard owns p).
 * ====================================================================== */
int or_tile_layout2(uint64_t n, uint64_t T, int inclusive, int map, uint64_t rank, uint64_t G,
                    int64_t *pos_of_rank, uint64_t V)
{
    uint64_t N = n / T;
    for (uint64_t p = 0; p < V; p++) pos_of_rank[p] = -1;
    int64_t pos = 0;
    /* helper: emit the elements of diagonal block D (strict: c < r; inclusive: c <= r) */
#define OR_EMIT(II, JJ, DIAGONAL)                                                       \
    for (uint64_t r = 0; r < T; r++)                                                     \
        for (uint64_t c = 0; c < T; c++) {                                               \
            uint64_t i = (II) * T + r, j = (JJ) * T + c;                                 \
            if ((DIAGONAL) && (inclusive ? c > r : c >= r)) continue;                    \
            uint64_t p = inclusive ? or_rank2_incl(i, j) : or_rank2_strict(i, j);        \
            if (p >= V) return -1;                                                       \
            pos_of_rank[p] = pos++;                                                      \
        }
    if (map == 0) {
        for (uint64_t I = 0; I < N; I++)
            for (uint64_t J = 0; J <= I; J++) { OR_EMIT(I, J, J == I) }
        return 0;
    }
    uint64_t W = N / 2 / G, wx0 = rank * W, H = inclusive ? N + 1 : N;
    for (uint64_t wy = 0; wy < H; wy++)
        for (uint64_t wx = wx0; wx < wx0 + W; wx++) {
            if (wy == 0 && !inclusive) {
                uint64_t D1 = wx, D2 = N - 1 - wx;
                OR_EMIT(D1, D1, 1)
                OR_EMIT(D2, D2, 1)
            } else if (inclusive && (wy == 0 || wy == N)) {
                uint64_t D = wy == 0 ? wx : wx + N / 2;
                OR_EMIT(D, D, 1)
            } else {
                uint64_t J, I;
                or_lambda2(wx, wy, &J, &I);
                OR_EMIT(I, J, 0)
            }
        }
#undef OR_EMIT
    return 0;
}

/* Streaming checksum (E21) of an m=2 payload written in the tile-blocked
 * layout, without materialising it: the same walk as or_tile_layout2, with the
 * slot offsets of each grid row counted up front (plain sums of the slot
 * sizes) so that the rows can be walked in parallel.
 * payload 0 = index write (value = canonical rank), 1 = EDM (strict only). */
int or_cs_tiles2(int payload, uint64_t n, uint64_t T, int inclusive, int map, uint64_t rank, uint64_t G,
                 const float *pts, int nthreads, uint64_t *cs)
{
    uint64_t N = n / T;
    if (payload == 1 && inclusive) return -1;
    uint64_t rows = map == 0 ? N : (inclusive ? N + 1 : N);
    uint64_t W = map == 0 ? 0 : N / 2 / G, wx0 = rank * W;
    int64_t *row_off = malloc((rows + 1) * sizeof(int64_t));
    uint64_t full = T * T, dstrict = T * (T - 1) / 2, dincl = T * (T + 1) / 2;
    row_off[0] = 0;
    for (uint64_t r = 0; r < rows; r++) {                  /* elements in grid row r */
        uint64_t s;
        if (map == 0) s = r * full + (inclusive ? dincl : dstrict);                 /* BB row I: I full + 1 diag */
        else if (!inclusive && r == 0) s = W * 2 * dstrict;
        else if (inclusive && (r == 0 || r == N)) s = W * dincl;
        else s = W * full;
        row_off[r + 1] = row_off[r] + (int64_t)s;
    }
    uint64_t c0 = 0, c1 = 0, c2 = 0, c3 = 0, c4 = 0;
    int nt = or_threads(nthreads);
    #pragma omp parallel for schedule(dynamic, 1) reduction(+:c0,c1,c2,c3) reduction(^:c4) num_threads(nt)
    for (uint64_t r = 0; r < rows; r++) {
        uint64_t c[5] = {0, 0, 0, 0, 0};
        uint64_t pos = (uint64_t)row_off[r];
        uint64_t ncols = map == 0 ? r + 1 : W;
        for (uint64_t k = 0; k < ncols; k++) {
            /* blocks of this slot: up to two (strict row 0) */
            uint64_t bI[2], bJ[2], nb = 1;
            int dg[2] = {0, 0};
            if (map == 0) { bI[0] = r; bJ[0] = k; dg[0] = (k == r); }
            else {
                uint64_t wx = wx0 + k, wy = r;
                if (!inclusive && wy == 0) { bI[0] = bJ[0] = wx; bI[1] = bJ[1] = N - 1 - wx; nb = 2; dg[0] = dg[1] = 1; }
                else if (inclusive && (wy == 0 || wy == N)) { bI[0] = bJ[0] = (wy == 0 ? wx : wx + N / 2); dg[0] = 1; }
                else { uint64_t J, I; or_lambda2(wx, wy, &J, &I); bI[0] = I; bJ[0] = J; }
            }
            for (uint64_t t = 0; t < nb; t++)
                for (uint64_t rr = 0; rr < T; rr++)
                    for (uint64_t cc = 0; cc < T; cc++) {
                        if (dg[t] && (inclusive ? cc > rr : cc >= rr)) continue;
                        uint64_t i = bI[t] * T + rr, j = bJ[t] * T + cc;
                        uint64_t bits;
                        if (payload == 0) bits = inclusive ? or_rank2_incl(i, j) : or_rank2_strict(i, j);
                        else bits = or_fbits(or_edm_dist(pts, i, j));
                        or_cs_add(c, pos, bits);
                        pos++;
                    }
        }
        c0 += c[0]; c1 += c[1]; c2 += c[2]; c3 += c[3]; c4 ^= c[4];
    }
    free(row_off);
    cs[0] = c0; cs[1] = c1; cs[2] = c2; cs[3] = c3; cs[4] = c4;
    return 0;
}

/* ======================================================================
 * m=3 tile-blocked layout (reading E26, the 3-D analogue of E23): every
 * T^3 tile is one contiguous slot, slots in the launch order of the tile
 * grid (lambda3 row order bid = (wz*N/2 + wy)*W + wx - wx0 within a shard;
 * BB colex over the tiles I <= J <= K); idle tiles have no slot.  Inside a
 * slot the elements follow the kernel's rows (k_l outer, j_l, i_l inner):
 *   interior I<J<K:          all (i_l, j_l, k_l)
 *   {I=J<K} segment:         i_l < j_l            (block triple (I, I, K))
 *   {I<J=K} segment:         j_l < k_l            (block triple (I, K, K))
 *   body I=J=K:              i_l < j_l < k_l
 * A lambda face tile (I=J<K) holds the {I=J<K} segment followed by the
 * {I<J=K} segment of (I, K) (reading E14); a BB tile holds its own class.
 * Defined here by enumeration, in the plain order above.
 * ====================================================================== */
typedef struct { uint64_t I, J, K; int kind; } or_seg3;   /* kind 0 interior, 1 {I=J<K}, 2 {I<J=K}, 3 body */

/* segments of the tile at launch position bid (returns the count, 0 = idle) */
static int or_tile3_segments(int map, uint64_t N, uint64_t rank, uint64_t G, uint64_t bid, or_seg3 *sg)
{
    if (map == 0) {                               /* BB: bid = (K*N + J)*N + I */
        uint64_t I = bid % N, J = (bid / N) % N, K = bid / (N * N);
        if (!(I <= J && J <= K)) return 0;
        sg[0].I = I; sg[0].J = J; sg[0].K = K;
        sg[0].kind = (I < J && J < K) ? 0 : (I == J && J < K) ? 1 : (I < J) ? 2 : 3;
        return 1;
    }
    uint64_t W = N / 2 / G, wx = rank * W + bid % W, wy = (bid / W) % (N / 2), wz = bid / W / (N / 2);
    int64_t o[6];
    int c = or_lambda3(N, wx, wy, wz, o);
    if (c == OR_L3_FILLER || (c == OR_L3_SPARE && o[0] < 0)) return 0;
    if (c == OR_L3_SPARE) { sg[0].I = sg[0].J = sg[0].K = (uint64_t)o[0]; sg[0].kind = 3; return 1; }
    uint64_t I = (uint64_t)o[3], J = (uint64_t)o[4], K = (uint64_t)o[5];
    if (I < J) { sg[0].I = I; sg[0].J = J; sg[0].K = K; sg[0].kind = 0; return 1; }
    sg[0].I = I; sg[0].J = I; sg[0].K = K; sg[0].kind = 1;
    sg[1].I = I; sg[1].J = K; sg[1].K = K; sg[1].kind = 2;
    return 2;
}

static uint64_t or_seg3_size(int kind, uint64_t T)
{
    switch (kind) {
    case 0: return T * T * T;
    case 1: case 2: return T * T * (T - 1) / 2;
    default: return T * (T - 1) * (T - 2) / 6;
    }
}

/* calls f(pos, rank) for every element of segment s, positions from *pos on */
#define OR_SEG3_WALK(s, T, POS, BODY)                                                        \
    for (uint64_t kl = 0; kl < (T); kl++)                                                    \
        for (uint64_t jl = 0; jl < (T); jl++) {                                              \
            if (((s).kind == 2 || (s).kind == 3) && jl >= kl) continue;                      \
            for (uint64_t il = 0; il < (T); il++) {                                          \
                if (((s).kind == 1 || (s).kind == 3) && il >= jl) continue;                  \
                uint64_t i_ = (s).I * (T) + il, j_ = (s).J * (T) + jl, k_ = (s).K * (T) + kl; \
                uint64_t rank_ = or_rank3(i_, j_, k_);                                       \
                BODY;                                                                        \
                (POS)++;                                                                     \
            }                                                                                \
        }

static uint64_t or_tile3_grid(int map, uint64_t N, uint64_t G)
{
    return map == 0 ? N * N * N : (N / 2 / G) * (N / 2) * (3 * N / 4);
}

int or_tile_layout3(uint64_t n, uint64_t T, int map, uint64_t rank, uint64_t G, int64_t *pos_of_rank, uint64_t V)
{
    uint64_t N = n / T, nb = or_tile3_grid(map, N, G);
    for (uint64_t p = 0; p < V; p++) pos_of_rank[p] = -1;
    uint64_t pos = 0;
    for (uint64_t bid = 0; bid < nb; bid++) {
        or_seg3 sg[2];
        int ns = or_tile3_segments(map, N, rank, G, bid, sg);
        for (int t = 0; t < ns; t++) {
            OR_SEG3_WALK(sg[t], T, pos, {
                if (rank_ >= V) return -1;
                pos_of_rank[rank_] = (int64_t)pos;
            })
        }
    }
    return 0;
}

/* Streaming checksum (E21) of the m=3 index write (value = canonical rank) in
 * the E26 layout: the slot offsets are counted up front (plain sums of the
 * segment sizes), then the tiles are walked in parallel. */
int or_cs_tiles3(uint64_t n, uint64_t T, int map, uint64_t rank, uint64_t G, int nthreads, uint64_t *cs)
{
    uint64_t N = n / T, nb = or_tile3_grid(map, N, G);
    uint64_t *off = malloc((nb + 1) * sizeof(uint64_t));
    if (!off) return -1;
    off[0] = 0;
    for (uint64_t bid = 0; bid < nb; bid++) {
        or_seg3 sg[2];
        int ns = or_tile3_segments(map, N, rank, G, bid, sg);
        uint64_t s = 0;
        for (int t = 0; t < ns; t++) s += or_seg3_size(sg[t].kind, T);
        off[bid + 1] = off[bid] + s;
    }
    uint64_t c0 = 0, c1 = 0, c2 = 0, c3 = 0, c4 = 0;
    int nt = or_threads(nthreads);
    #pragma omp parallel for schedule(dynamic, 4) reduction(+:c0,c1,c2,c3) reduction(^:c4) num_threads(nt)
    for (uint64_t bid = 0; bid < nb; bid++) {
        uint64_t c[5] = {0, 0, 0, 0, 0};
        or_seg3 sg[2];
        int ns = or_tile3_segments(map, N, rank, G, bid, sg);
        uint64_t pos = off[bid];
        for (int t = 0; t < ns; t++) {
            OR_SEG3_WALK(sg[t], T, pos, { or_cs_add(c, pos, rank_); })
        }
        c0 += c[0]; c1 += c[1]; c2 += c[2]; c3 += c[3]; c4 ^= c[4];
    }
    free(off);
    cs[0] = c0; cs[1] = c1; cs[2] = c2; cs[3] = c3; cs[4] = c4;
    return 0;
}

/* ======================================================================
 * Expected MAP_DUMP records (format of include/smap.h, restated): per grid
 * block in launch order, int32 {x0, x1, x2, cls}.
 * ====================================================================== */
int or_map_dump(int m, int inclusive, int map, uint64_t N, uint64_t rank, uint64_t G, int order,
                int32_t *out, uint64_t len)
{
    uint64_t nb = or_grid_blocks(m, inclusive, map, N, G);
    if (nb != len) return -1;
    for (uint64_t bid = 0; bid < nb; bid++) {
        uint64_t w[3] = {0, 0, 0};
        or_block_coords(m, inclusive, map, N, rank, G, order, bid, w);
        int32_t *r = out + 4 * bid;
        r[0] = r[1] = r[2] = r[3] = 0;
        if (m == 2 && (map == 0 || map == 2)) {
            r[0] = (int32_t)w[0]; r[1] = (int32_t)w[1];
            r[3] = w[0] < w[1] ? 0 : (w[0] == w[1] ? 3 : 4);
        } else if (m == 2) {
            if (w[1] == 0 && !inclusive) { r[0] = (int32_t)w[0]; r[1] = (int32_t)(N - 1 - w[0]); r[3] = 1; }
            else if (w[1] == 0) { r[0] = r[1] = (int32_t)w[0]; r[3] = 2; }
            else if (inclusive && w[1] == N) { r[0] = r[1] = (int32_t)(w[0] + N / 2); r[3] = 2; }
            else { uint64_t x, y; or_lambda2(w[0], w[1], &x, &y); r[0] = (int32_t)x; r[1] = (int32_t)y; r[3] = 0; }
        } else if (map == 0 || map == 2) {
            uint64_t I = w[0], J = w[1], K = w[2];
            r[0] = (int32_t)I; r[1] = (int32_t)J; r[2] = (int32_t)K;
            r[3] = (I < J && J < K) ? 0 : (I == J && J < K) ? 5 : (I < J && J == K) ? 6 : (I == J && J == K) ? 2 : 4;
        } else {
            int64_t o[6];
            int c = or_lambda3(N, w[0], w[1], w[2], o);
            if (c == OR_L3_INSIDE || c == OR_L3_REFLECTED) {
                r[0] = (int32_t)o[3]; r[1] = (int32_t)o[4]; r[2] = (int32_t)o[5]; r[3] = c;
            } else if (c == OR_L3_SPARE && o[0] >= 0) {
                r[0] = r[1] = r[2] = (int32_t)o[0]; r[3] = 2;
            } else {
                r[3] = 3;
            }
        }
    }
    return 0;
}

/* ======================================================================
 * "Approach n from below" (reading E28 in DESIGN.md), at tile
 * level.  P:399-404 reads: apply orthotopes Pi_{n_1}, Pi_{n_2}, ... with
 * n_1 = floor(log2 n) and n_i = log2(n - sum_{k<i} n_k), "plus a set of more
 * simpler mappings for the sub-orthotopes that remain un-mapped at each
 * level".  The printed n_i are logarithms where sizes are meant (reading
 * E7): the sizes are 2^floor(log2(n - sum_{k<i} n_k)), i.e. the binary
 * digits of n in descending order.  Applied to the M = ceil(n'/T) tiles per
 * side (n' = n, or n + 2 for the m = 3 inclusive set of reading E24):
 *   segments   S_s = [O_s, O_s + N_s), N_0 > N_1 > ... the binary digits of M,
 *              O_s = N_0 + ... + N_{s-1};
 *   m = 2      for s = 0, 1, ...: the triangle of S_s by lambda2
 *              over the inclusive tile grid (N_s/2) x (N_s + 1) (grid rows 0
 *              and N_s hold one diagonal tile each, reading E6; N_s = 1: the
 *              single diagonal tile), then the "simpler mappings" of the
 *              rectangles S_a x S_s, a < s, at the identity (J fastest);
 *   m = 3      for every segment triple a <= b <= c (c outer, then b, then a):
 *              a = b = c  the tetrahedron of S_a by lambda3 (reading R3) over
 *                         its (N/2, N/2, 3N/4) tile grid for N_a >= 8; for
 *                         N_a < 8 the C(N_a + 2, 3) tiles I <= J <= K in colex
 *                         order (a "simpler mapping");
 *              a < b = c  S_a x (triangle J <= K of S_b by the lambda2 grid above);
 *              a = b < c  (triangle I <= J of S_a by the lambda2 grid) x S_c;
 *              a < b < c  the box S_a x S_b x S_c at the identity.
 * Inside a piece the lower-ranked coordinates vary fastest (the order of the
 * packed layout): rectangle J then I; a < b = c the line I, then the lambda2
 * grid id (row order); a = b < c the lambda2 grid id, then K; box I, J, K.  Records have the
 * MAP_DUMP format {x0, x1, x2, cls}: m = 2 {J, I, 0, cls} with cls 0
 * off-diagonal, 2 diagonal tile; m = 3 {I, J, K, cls} with cls 0/1 the lambda3
 * branch (I = J: a face tile carrying {I=J<K} and {I<J=K}), 2 body tile,
 * 3 idle lambda3 tile (zeros), and for the other pieces cls 0 interior
 * (I < J < K), 5 face I = J < K, 6 face I < J = K, 2 body (I = J = K).
 * ====================================================================== */
int or_below_segments(uint64_t M, uint64_t *Ns, uint64_t *Os)
{
    int p = 0;
    uint64_t rest = M, off = 0;
    while (rest > 0) {
        uint64_t b = or_pow2(or_floor_log2(rest));   /* 2^floor(log2(M - sum so far)) */
        Ns[p] = b; Os[p] = off;
        off += b; rest -= b; p++;
    }
    return p;
}

/* the (J, K) tile of grid id g of the lambda2 inclusive tile grid of side N
 * (J <= K; returns 1 for a diagonal tile) */
static int or_below_tri(uint64_t N, uint64_t g, uint64_t *J, uint64_t *K)
{
    if (N == 1) { *J = *K = 0; return 1; }
    uint64_t W = N / 2, wx = g % W, wy = g / W;
    if (wy == 0) { *J = *K = wx; return 1; }
    if (wy == N) { *J = *K = wx + N / 2; return 1; }
    or_lambda2(wx, wy, J, K);
    return 0;
}

static uint64_t or_below_tri_count(uint64_t N) { return N == 1 ? 1 : (N / 2) * (N + 1); }

static void or_rec4(int32_t *r, uint64_t a, uint64_t b, uint64_t c, int cls)
{
    r[0] = (int32_t)a; r[1] = (int32_t)b; r[2] = (int32_t)c; r[3] = cls;
}

/* Tile records of the below decomposition in launch order; returns the
 * number of tiles (out may be NULL to count only). */
uint64_t or_below_tiles(int m, uint64_t M, int32_t *out)
{
    uint64_t Ns[64], Os[64], cnt = 0;
    int p = or_below_segments(M, Ns, Os);
    if (m == 2) {
        for (int s = 0; s < p; s++) {
            for (uint64_t g = 0; g < or_below_tri_count(Ns[s]); g++, cnt++) {
                uint64_t J, I;
                int d = or_below_tri(Ns[s], g, &J, &I);
                if (out) or_rec4(out + 4 * cnt, Os[s] + J, Os[s] + I, 0, d ? 2 : 0);
            }
            for (int a = 0; a < s; a++)           /* rectangle S_a x S_s, J fastest */
                for (uint64_t g = 0; g < Ns[a] * Ns[s]; g++, cnt++)
                    if (out) or_rec4(out + 4 * cnt, Os[a] + g % Ns[a], Os[s] + g / Ns[a], 0, 0);
        }
        return cnt;
    }
    for (int c = 0; c < p; c++)
        for (int b = 0; b <= c; b++)
            for (int a = 0; a <= b; a++) {
                if (a == b && b == c) {
                    uint64_t N = Ns[a], O = Os[a];
                    if (N >= 8) {
                        uint64_t nb = (N / 2) * (N / 2) * (3 * N / 4);
                        for (uint64_t g = 0; g < nb; g++, cnt++) {
                            if (!out) continue;
                            uint64_t wx = g % (N / 2), wy = (g / (N / 2)) % (N / 2), wz = g / (N / 2) / (N / 2);
                            int64_t o[6];
                            int k = or_lambda3(N, wx, wy, wz, o);
                            if (k == OR_L3_INSIDE || k == OR_L3_REFLECTED) or_rec4(out + 4 * cnt, O + o[3], O + o[4], O + o[5], k);
                            else if (k == OR_L3_SPARE && o[0] >= 0) or_rec4(out + 4 * cnt, O + o[0], O + o[0], O + o[0], 2);
                            else or_rec4(out + 4 * cnt, 0, 0, 0, 3);
                        }
                    } else {
                        for (uint64_t K = 0; K < N; K++)
                            for (uint64_t J = 0; J <= K; J++)
                                for (uint64_t I = 0; I <= J; I++, cnt++) {
                                    int cls = (I < J && J < K) ? 0 : (I == J && J < K) ? 5 : (I < J) ? 6 : 2;
                                    if (out) or_rec4(out + 4 * cnt, O + I, O + J, O + K, cls);
                                }
                    }
                } else if (b == c) {          /* a < b = c */
                    for (uint64_t g = 0; g < Ns[a] * or_below_tri_count(Ns[b]); g++, cnt++) {
                        uint64_t J, K;
                        int d = or_below_tri(Ns[b], g / Ns[a], &J, &K);
                        if (out) or_rec4(out + 4 * cnt, Os[a] + g % Ns[a], Os[b] + J, Os[b] + K, d ? 6 : 0);
                    }
                } else if (a == b) {          /* a = b < c: the triangle fastest, then K */
                    uint64_t tc = or_below_tri_count(Ns[a]);
                    for (uint64_t g = 0; g < Ns[c] * tc; g++, cnt++) {
                        uint64_t I, J;
                        int d = or_below_tri(Ns[a], g % tc, &I, &J);
                        if (out) or_rec4(out + 4 * cnt, Os[a] + I, Os[a] + J, Os[c] + g / tc, d ? 5 : 0);
                    }
                } else {                      /* a < b < c */
                    for (uint64_t g = 0; g < Ns[a] * Ns[b] * Ns[c]; g++, cnt++)
                        if (out) or_rec4(out + 4 * cnt, Os[a] + g % Ns[a], Os[b] + (g / Ns[a]) % Ns[b],
                                         Os[c] + g / Ns[a] / Ns[b], 0);
                }
            }
    return cnt;
}

/* Element-level cover of the below decomposition: one hit per element the
 * tile records carry (tile (I,J,K) holds the elements i = I*T + il etc.;
 * diagonal tiles clip to the domain, elements with the largest index >= n'
 * are filtered).  res = {tiles, useful, outside}. */
int or_below_element_hits(int m, int inclusive, uint64_t n, uint64_t T, uint32_t *hits, uint64_t V, int64_t *res)
{
    uint64_t nint = (m == 3 && inclusive) ? n + 2 : n;      /* E24 */
    uint64_t M = (nint + T - 1) / T;
    uint64_t nt = or_below_tiles(m, M, NULL);
    int32_t *rec = malloc(nt * 4 * sizeof(int32_t));
    if (!rec) return -1;
    or_below_tiles(m, M, rec);
    int64_t useful = 0, outside = 0;
    for (uint64_t t = 0; t < nt; t++) {
        int32_t *r = rec + 4 * t;
        if (m == 2) {
            uint64_t J = (uint64_t)r[0], I = (uint64_t)r[1];
            for (uint64_t rr = 0; rr < T; rr++)
                for (uint64_t cc = 0; cc < T; cc++) {
                    uint64_t i = I * T + rr, j = J * T + cc;
                    if (i >= n) continue;
                    if (r[3] == 2 && (inclusive ? cc > rr : cc >= rr)) continue;
                    int in = inclusive ? j <= i : j < i;
                    if (!in) { outside++; continue; }
                    uint64_t p = inclusive ? or_rank2_incl(i, j) : or_rank2_strict(i, j);
                    if (p >= V) { outside++; continue; }
                    hits[p]++; useful++;
                }
            continue;
        }
        if (r[3] == 3) continue;
        uint64_t I = (uint64_t)r[0], J = (uint64_t)r[1], K = (uint64_t)r[2];
        or_seg3 sg[2];
        int ns = 1;
        if (r[3] == 2) { sg[0].I = sg[0].J = sg[0].K = I; sg[0].kind = 3; }
        else if (I < J && J < K) { sg[0].I = I; sg[0].J = J; sg[0].K = K; sg[0].kind = 0; }
        else if (r[3] == 5) { sg[0].I = I; sg[0].J = I; sg[0].K = K; sg[0].kind = 1; }
        else if (r[3] == 6) { sg[0].I = I; sg[0].J = K; sg[0].K = K; sg[0].kind = 2; }
        else {                                   /* lambda3 face tile I = J < K: both folded sets (E14) */
            sg[0].I = I; sg[0].J = I; sg[0].K = K; sg[0].kind = 1;
            sg[1].I = I; sg[1].J = K; sg[1].K = K; sg[1].kind = 2;
            ns = 2;
        }
        for (int q = 0; q < ns; q++) {
            uint64_t pos = 0;
            OR_SEG3_WALK(sg[q], T, pos, {
                if (k_ >= nint) continue;
                uint64_t pp = rank_;
                int in = i_ < j_ && j_ < k_;
                if (in && inclusive) pp = or_rank3_incl(i_, j_ - 1, k_ - 2);
                if (!in || pp >= V) { outside++; continue; }
                hits[pp]++; useful++;
            })
            (void)pos;
        }
    }
    free(rec);
    res[0] = (int64_t)nt; res[1] = useful; res[2] = outside;
    return 0;
}

/* ======================================================================
 * Tile-blocked layout of the below decomposition (reading E29): the tiles
 * in the launch order of or_below_tiles, each one contiguous slot holding its
 * elements in the kernel's row order -- m=2 rows r then columns c (diagonal
 * tiles clipped to c < r / c <= r); m=3 the segments of E26 (k_l, j_l, i_l).
 * Slot sizes ignore the cut by n: an element whose largest index is >= n'
 * keeps its position as a hole (never written), so every slot size depends on
 * the tile class only.  pos_of_rank[p] = position of packed rank p.
 * ====================================================================== */
static uint64_t or_below_slot_size(int m, int inclusive, const int32_t *r, uint64_t T)
{
    if (m == 2) return r[3] == 2 ? (inclusive ? T * (T + 1) / 2 : T * (T - 1) / 2) : T * T;
    if (r[3] == 3) return 0;
    if (r[3] == 2) return T * (T - 1) * (T - 2) / 6;
    if (r[3] == 5 || r[3] == 6) return T * T * (T - 1) / 2;
    if (r[0] == r[1]) return T * T * (T - 1);              /* lambda3 face tile: both segments */
    return T * T * T;
}

/* calls BODY with (pos, rank) for every element of record r, positions from pos */
#define OR_BELOW_WALK(m, inclusive, nint, r, T, POS, BODY)                                              \
    do {                                                                                                \
        if ((m) == 2) {                                                                                 \
            uint64_t J_ = (uint64_t)(r)[0], I_ = (uint64_t)(r)[1];                                      \
            for (uint64_t rr = 0; rr < (T); rr++)                                                       \
                for (uint64_t cc = 0; cc < (T); cc++) {                                                 \
                    if ((r)[3] == 2 && ((inclusive) ? cc > rr : cc >= rr)) continue;                    \
                    uint64_t i_ = I_ * (T) + rr, j_ = J_ * (T) + cc;                                    \
                    if (i_ < (nint)) {                                                                  \
                        uint64_t rank_ = (inclusive) ? or_rank2_incl(i_, j_) : or_rank2_strict(i_, j_); \
                        BODY;                                                                           \
                    }                                                                                   \
                    (POS)++;                                                                            \
                }                                                                                       \
        } else if ((r)[3] != 3) {                                                                       \
            uint64_t I_ = (uint64_t)(r)[0], J_ = (uint64_t)(r)[1], K_ = (uint64_t)(r)[2];              \
            or_seg3 sg_[2];                                                                             \
            int ns_ = 1;                                                                                \
            if ((r)[3] == 2) { sg_[0].I = sg_[0].J = sg_[0].K = I_; sg_[0].kind = 3; }                  \
            else if (I_ < J_ && J_ < K_) { sg_[0].I = I_; sg_[0].J = J_; sg_[0].K = K_; sg_[0].kind = 0; } \
            else if ((r)[3] == 5) { sg_[0].I = I_; sg_[0].J = I_; sg_[0].K = K_; sg_[0].kind = 1; }    \
            else if ((r)[3] == 6) { sg_[0].I = I_; sg_[0].J = K_; sg_[0].K = K_; sg_[0].kind = 2; }    \
            else {                                                                                      \
                sg_[0].I = I_; sg_[0].J = I_; sg_[0].K = K_; sg_[0].kind = 1;                           \
                sg_[1].I = I_; sg_[1].J = K_; sg_[1].K = K_; sg_[1].kind = 2; ns_ = 2;                  \
            }                                                                                           \
            for (int q_ = 0; q_ < ns_; q_++)                                                            \
                for (uint64_t kl = 0; kl < (T); kl++)                                                   \
                    for (uint64_t jl = 0; jl < (T); jl++) {                                             \
                        if ((sg_[q_].kind == 2 || sg_[q_].kind == 3) && jl >= kl) continue;             \
                        for (uint64_t il = 0; il < (T); il++) {                                         \
                            if ((sg_[q_].kind == 1 || sg_[q_].kind == 3) && il >= jl) continue;         \
                            uint64_t i_ = sg_[q_].I * (T) + il, j_ = sg_[q_].J * (T) + jl, k_ = sg_[q_].K * (T) + kl; \
                            if (k_ < (nint)) {                                                          \
                                uint64_t rank_ = (inclusive) ? or_rank3_incl(i_, j_ - 1, k_ - 2) : or_rank3(i_, j_, k_); \
                                BODY;                                                                   \
                            }                                                                           \
                            (POS)++;                                                                    \
                        }                                                                               \
                    }                                                                                   \
        }                                                                                               \
    } while (0)

/* returns the layout length (slots incl. holes), or -1 */
int64_t or_below_tile_layout(int m, int inclusive, uint64_t n, uint64_t T, int64_t *pos_of_rank, uint64_t V)
{
    uint64_t nint = (m == 3 && inclusive) ? n + 2 : n;
    uint64_t M = (nint + T - 1) / T, nt = or_below_tiles(m, M, NULL);
    int32_t *rec = malloc(nt * 4 * sizeof(int32_t));
    if (!rec) return -1;
    or_below_tiles(m, M, rec);
    for (uint64_t p = 0; p < V; p++) pos_of_rank[p] = -1;
    uint64_t pos = 0;
    int bad = 0;
    for (uint64_t t = 0; t < nt; t++) {
        const int32_t *r = rec + 4 * t;
        uint64_t p0 = pos;
        OR_BELOW_WALK(m, inclusive, nint, r, T, pos, {
            if (rank_ >= V) bad = 1; else pos_of_rank[rank_] = (int64_t)pos;
        });
        if (pos - p0 != or_below_slot_size(m, inclusive, r, T)) bad = 1;
    }
    free(rec);
    return bad ? -1 : (int64_t)pos;
}

/* Streaming checksum (E21) of a payload written in the E29 layout: index
 * write (payload 0, value = packed rank) or EDM (payload 1, m=2 strict). */
int or_cs_below_tiles(int payload, int m, int inclusive, uint64_t n, uint64_t T, const float *pts, int nthreads,
                      uint64_t *cs)
{
    uint64_t nint = (m == 3 && inclusive) ? n + 2 : n;
    uint64_t M = (nint + T - 1) / T, nt = or_below_tiles(m, M, NULL);
    int32_t *rec = malloc(nt * 4 * sizeof(int32_t));
    uint64_t *off = malloc((nt + 1) * sizeof(uint64_t));
    if (!rec || !off) { free(rec); free(off); return -1; }
    or_below_tiles(m, M, rec);
    off[0] = 0;
    for (uint64_t t = 0; t < nt; t++) off[t + 1] = off[t] + or_below_slot_size(m, inclusive, rec + 4 * t, T);
    uint64_t c0 = 0, c1 = 0, c2 = 0, c3 = 0, c4 = 0;
    int ntr = or_threads(nthreads);
    #pragma omp parallel for schedule(dynamic, 4) reduction(+:c0,c1,c2,c3) reduction(^:c4) num_threads(ntr)
    for (uint64_t t = 0; t < nt; t++) {
        uint64_t c[5] = {0, 0, 0, 0, 0};
        const int32_t *r = rec + 4 * t;
        uint64_t pos = off[t];
        if (payload == 1 && m == 2) {
            OR_BELOW_WALK(2, inclusive, nint, r, T, pos, {
                (void)rank_;
                or_cs_add(c, pos, or_fbits(or_edm_dist(pts, i_, j_)));
            });
        } else {
            OR_BELOW_WALK(m, inclusive, nint, r, T, pos, { or_cs_add(c, pos, rank_); });
        }
        c0 += c[0]; c1 += c[1]; c2 += c[2]; c3 += c[3]; c4 ^= c[4];
    }
    free(rec); free(off);
    cs[0] = c0; cs[1] = c1; cs[2] = c2; cs[3] = c3; cs[4] = c4;
    return 0;
}
