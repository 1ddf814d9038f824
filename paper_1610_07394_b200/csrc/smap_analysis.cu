// smap_analysis.cu -- the paper's volume analysis of recursive orthotope sets
// for general m (second half): the arity-beta recursive
// set S_n^m with scaling r (Eq. generic-m; P:431-470 for the
// arity-3 tetrahedral set), the extra-volume limits, the scaling
// r* that meets the constraint 1/r^m - beta = m! (reading E30) and
// the coverage threshold n0 (reading E31).  Host-only C ABI
// functions (include/smap.h); no map exists for m >= 4 in the paper, so there
// is no device code here.
#include <cmath>
#include <cstdint>

#include "smap.h"

typedef unsigned __int128 u128;

namespace {

int ilog(uint64_t n, uint64_t base, bool *exact)      // k with base^k = n
{
    int k = 0;
    uint64_t v = 1;
    while (v < n) {
        if (v > UINT64_MAX / base) break;
        v *= base;
        k++;
    }
    *exact = v == n;
    return k;
}

bool pow_u128(uint64_t b, int e, u128 *out)             // b^e, false on overflow of 2^127
{
    u128 v = 1;
    for (int i = 0; i < e; i++) {
        if (v > (((u128)1) << 126) / (b ? b : 1)) return false;
        v *= b;
    }
    *out = v;
    return true;
}

double factorial(int m)
{
    double f = 1.0;
    for (int i = 2; i <= m; i++) f *= i;
    return f;
}

// continuous model of Eq. generic-m at real n >= 1
double vs_continuous(int m, double n, double r, int beta)
{
    const double inv = std::pow(1.0 / r, m) - beta;
    const double k = std::log(n) / std::log(1.0 / r);         // log_{1/r} n
    if (std::fabs(inv) < 1e-300) return std::pow(n, m) * k * std::pow(r, m);   // beta = 1/r^m: the degenerate sum
    return (std::pow(n, m) - std::pow((double)beta, k)) / inv;
}

// V(Delta^m_{n-1}) = C(n - 1 + m - 1, m), in double
double simplex_prev(int m, double n)
{
    double v = 1.0;
    for (int i = 0; i < m; i++) v *= (n - 1.0 + i) / (double)(i + 1);
    return v;
}

}  // namespace

extern "C" {

smap_status smap_recursive_volume(int m, uint64_t n, int beta, int r_den, uint64_t *vol)
{
    if (!vol || m < 1 || m > 16 || beta < 1 || r_den < 2 || n < 1) return SMAP_E_INVALID;
    bool exact;
    const int k = ilog(n, (uint64_t)r_den, &exact);
    if (!exact) return SMAP_E_INVALID;
    // V(n) = (n / r_den)^m + beta V(n / r_den), V(1) = 0 -- evaluated bottom-up in 128 bits
    u128 v = 0, side = 1;
    for (int lvl = 1; lvl <= k; lvl++) {                    // level side n_l = r_den^lvl, its cube side r_den^(lvl-1)
        u128 cube;
        if (!pow_u128((uint64_t)side, m, &cube)) return SMAP_E_INVALID;
        v = cube + (u128)beta * v;
        if (v >> 64) return SMAP_E_INVALID;
        side *= (u128)r_den;
    }
    *vol = (uint64_t)v;
    return SMAP_OK;
}

smap_status smap_recursive_volume_closed(int m, uint64_t n, int beta, int r_den, uint64_t *vol)
{
    if (!vol || m < 1 || m > 16 || beta < 1 || r_den < 2 || n < 1) return SMAP_E_INVALID;
    bool exact;
    const int k = ilog(n, (uint64_t)r_den, &exact);
    if (!exact) return SMAP_E_INVALID;
    u128 nm, bk, rm;
    if (!pow_u128(n, m, &nm) || !pow_u128((uint64_t)beta, k, &bk) || !pow_u128((uint64_t)r_den, m, &rm))
        return SMAP_E_INVALID;
    u128 v;
    if (rm == (u128)beta) {                                 // beta = 1/r^m: k equal terms (n r)^m
        v = nm / rm * (u128)k;
    } else if (rm > (u128)beta) {                           // (n^m - beta^k) / (1/r^m - beta)
        v = (nm - bk) / (rm - (u128)beta);
    } else {                                                // (beta^k - n^m) / (beta - 1/r^m)
        v = (bk - nm) / ((u128)beta - rm);
    }
    if (v >> 64) return SMAP_E_INVALID;
    *vol = (uint64_t)v;
    return SMAP_OK;
}

double smap_alpha_limit(int m, double r, int beta)
{
    if (m < 1 || !(r > 0.0 && r < 1.0)) return NAN;
    const double d = std::pow(1.0 / r, m) - beta;
    if (!(d > 0.0)) return INFINITY;                        // the recursive volume grows faster than n^m
    return factorial(m) / d - 1.0;                          // lim V(S_n^m) / V(Delta_n^m) - 1
}

double smap_r_star(int m, int beta)
{
    if (m < 1 || beta < 0) return NAN;
    return std::pow(factorial(m) + beta, -1.0 / m);         // 1/r^m - beta = m! (reading E30)
}

smap_status smap_find_n0(int m, double r, int beta, uint64_t n_max, uint64_t *n0, double *ratio_at_nmax)
{
    if (!n0 || m < 1 || m > 16 || !(r > 0.0 && r < 1.0) || beta < 1 || n_max < 2 || n_max > ((uint64_t)1 << 24))
        return SMAP_E_INVALID;
    // scan down from n_max: n0 = the smallest n such that V_S(n') >= V(Delta_{n'-1}) for every n' in [n, n_max]
    uint64_t first = 0;
    for (uint64_t n = n_max; n >= 2; n--) {
        const double vs = vs_continuous(m, (double)n, r, beta), vd = simplex_prev(m, (double)n);
        if (!(vs >= vd * (1.0 - 1e-12))) break;
        first = n;
    }
    *n0 = first;
    if (ratio_at_nmax) *ratio_at_nmax = vs_continuous(m, (double)n_max, r, beta) / simplex_prev(m, (double)n_max);
    return SMAP_OK;
}

smap_status smap_r_cover(int m, int beta, uint64_t n0, uint64_t n_max, double *r)
{
    if (!r || m < 1 || m > 16 || beta < 1 || n0 < 2 || n0 > n_max || n_max > ((uint64_t)1 << 20)) return SMAP_E_INVALID;
    // covers(r): V_S(n) >= V(Delta^m_{n-1}) for every n in [n0, n_max] (continuous model).
    // D = 1/r^m - beta falls as r grows: more recursive volume, more extra volume (alpha = m!/D - 1).
    // The least extra volume that still covers from n0 is the smallest covering r: bisect between
    // r* (D = m!, never covers for m >= 4, reading E31) and the r of D = 1 (covers for n0 >= 2).
    auto covers = [&](double rr) {
        for (uint64_t n = n0; n <= n_max; n++)
            if (!(vs_continuous(m, (double)n, rr, beta) >= simplex_prev(m, (double)n))) return false;
        return true;
    };
    double a = smap_r_star(m, beta), b = std::pow(beta + 1.0, -1.0 / m);
    if (covers(a)) { *r = a; return SMAP_OK; }
    if (!covers(b)) return SMAP_E_UNSUPPORTED;
    for (int it = 0; it < 60; it++) {
        const double mid = 0.5 * (a + b);
        if (covers(mid)) b = mid; else a = mid;
    }
    *r = b;
    return SMAP_OK;
}

}  // extern "C"
