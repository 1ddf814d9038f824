// smap_api.cu -- implementation of the C ABI declared in include/smap.h:
// argument validation, plan construction (grid extents, shard ranges and the
// closed forms of DESIGN.md s.5), scratch ownership, kernel dispatch and the
// deterministic fp64 finalize (a7).  No CPU fallback: every payload runs in
// the sm_100a kernels of smap_thread{2,3}.cu / smap_tile{2,3}.cu.
#include <cstdio>
#include <cstdarg>
#include <cstring>
#include <string>
#include <vector>

#include "smap.h"
#include "smap_device.cuh"

using namespace smap;

struct smap_plan_s {
    smap_plan_desc d;
    Params P;                 // per-plan launch parameters (pts/out/param set per run)
    uint64_t V;               // volume of the whole domain
    uint64_t useful;          // elements owned by this shard
    uint64_t launched;        // grid_blocks * rho^m
    int elem64;               // index-write element is uint64
    int device;
    unsigned ctas;            // TILE: CTAs launched
    Result *d_res = nullptr;
    Result *h_res = nullptr;  // pinned
    double *d_partials = nullptr;
    uint64_t npartials = 0;
    double *d_scratch = nullptr;
    uint32_t *d_adj = nullptr;      // TC pair-predicate bitmap (TILE)
    uint32_t *d_tcpairs = nullptr;  // TC, sharded lambda plan: the bitmap block pairs this shard reads
    uint32_t ntcpairs = 0;
    int tcpairs_done = 0;           // (the shard analysis ran; d_tcpairs null = build every pair)
    Piece *d_pieces = nullptr;      // SMAP_MAP_BELOW decomposition
    std::vector<uint32_t> segN, segO;   // SMAP_MAP_BELOW: the binary-digit segments of M (sizes, offsets)
    uint64_t layout_len = 0;        // SMAP_MAP_BELOW tile-blocked layout: slots incl. holes (E29)
    std::vector<Piece> pieces;
    float *d_stage = nullptr;
    smap_result *d_rec = nullptr;   // smap_run_host: device record
    smap_result *h_rec = nullptr;   // smap_run_host: pinned host record
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaStream_t last_stream = nullptr;
    uint32_t last_launches = 0;
    int ran = 0;
    int res_dirty = 1;              // the result block may be nonzero (a fresh allocation, or an smap_run's results)
};

static thread_local std::string g_err;

static smap_status fail(smap_status s, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

static smap_status cuda_fail(cudaError_t e, const char *where)
{
    return fail(e == cudaErrorMemoryAllocation ? SMAP_E_NOMEM : SMAP_E_CUDA, "%s: %s (%s)", where,
                cudaGetErrorString(e), cudaGetErrorName(e));
}

#define CK(call)                                                  \
    do {                                                          \
        cudaError_t e_ = (call);                                  \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call);       \
    } while (0)

// Makes the plan's device current for the scope of one entry point and
// restores the caller's device on every exit path.
struct DevGuard {
    int prev = -1;
    bool switched = false;
    cudaError_t enter(int dev)
    {
        cudaError_t e = cudaGetDevice(&prev);
        if (e != cudaSuccess || prev == dev) return e;
        e = cudaSetDevice(dev);
        switched = e == cudaSuccess;
        return e;
    }
    ~DevGuard()
    {
        if (switched) cudaSetDevice(prev);
    }
};

static bool is_pow2(int64_t x) { return x > 0 && (x & (x - 1)) == 0; }
static int ilog2(int64_t x) { int l = 0; while ((int64_t)1 << (l + 1) <= x) l++; return l; }

// "Approach n from below" (reading E28): the pieces of the M-tile
// simplex in launch order (include/smap.h); returns the total tile count.
static uint64_t below_pieces(int m, int64_t M, int T, bool incl, std::vector<Piece> &out, uint64_t *slots,
                             std::vector<uint32_t> &Ns, std::vector<uint32_t> &Os)
{
    for (int64_t rest = M, off = 0; rest > 0;) {        // binary digits of M, largest first
        const int64_t b = (int64_t)1 << ilog2(rest);
        Ns.push_back((uint32_t)b); Os.push_back((uint32_t)off);
        off += b; rest -= b;
    }
    const int p = (int)Ns.size();
    uint64_t start = 0;
    uint64_t sbase = 0;
    auto add = [&](uint8_t kind, int a, int b, int c, uint64_t count, uint64_t slots) {
        Piece pc;
        pc.start = start; pc.kind = kind; pc.sbase = sbase;
        sbase += slots;
        pc.Oa = Os[a]; pc.Ob = Os[b]; pc.Oc = Os[c];
        pc.ea = (uint8_t)ilog2(Ns[a]); pc.eb = (uint8_t)ilog2(Ns[b]); pc.ec = (uint8_t)ilog2(Ns[c]);
        out.push_back(pc);
        start += count;
    };
    auto tri = [](uint64_t N) { return N == 1 ? (uint64_t)1 : (N / 2) * (N + 1); };   // lambda2 inclusive tile grid
    // E29 slot totals: a triangle piece holds N diagonal tiles (size sd) and (N/2)(N-1) full ones
    auto tri_slots = [](uint64_t N, uint64_t sd, uint64_t sf) { return N * sd + (N / 2) * (N - 1) * sf; };
    const uint64_t T2 = (uint64_t)T * T, T3 = T2 * T, Tf = T2 * (T - 1) / 2, Tb = (uint64_t)T * (T - 1) * (T - 2) / 6;
    if (m == 2) {
        const uint64_t sd = incl ? (uint64_t)T * (T + 1) / 2 : (uint64_t)T * (T - 1) / 2;
        for (int s = 0; s < p; s++) {
            add(PK_TRI2, s, s, s, tri(Ns[s]), tri_slots(Ns[s], sd, T2));
            for (int a = 0; a < s; a++) add(PK_RECT2, a, s, s, (uint64_t)Ns[a] * Ns[s], (uint64_t)Ns[a] * Ns[s] * T2);
        }
        *slots = sbase;
        return start;
    }
    for (int c = 0; c < p; c++)
        for (int b = 0; b <= c; b++)
            for (int a = 0; a <= b; a++) {
                const uint64_t Na = Ns[a], Nb = Ns[b], Nc = Ns[c];
                if (a == c) {                 // interior C(N,3) T^3 + faces C(N,2) T^2(T-1) + bodies N C(T,3)
                    const uint64_t sl = Na * (Na - 1) * (Na - 2) / 6 * T3 + Na * (Na - 1) / 2 * 2 * Tf + Na * Tb;
                    if (Na >= 8) add(PK_TET3, a, a, a, (Na / 2) * (Na / 2) * (3 * Na / 4), sl);
                    else add(PK_TETS, a, a, a, Na * (Na + 1) * (Na + 2) / 6, sl);
                } else if (b == c) {
                    add(PK_LT, a, b, c, Na * tri(Nb), Na * tri_slots(Nb, Tf, T3));
                } else if (a == b) {
                    add(PK_TL, a, b, c, Nc * tri(Na), Nc * tri_slots(Na, Tf, T3));
                } else {
                    add(PK_BOX, a, b, c, Na * Nb * Nc, Na * Nb * Nc * T3);
                }
            }
    *slots = sbase;
    return start;
}

namespace smap {
__global__ void k_result_combine(const smap_result *recs, int G, smap_result *dst);
}

extern "C" {

int smap_abi_version(void) { return SMAP_ABI_VERSION; }

const char *smap_last_error(void) { return g_err.c_str(); }

uint64_t smap_volume(int m, int64_t n, int diag)
{
    if (n <= 0) return 0;
    unsigned __int128 N = (unsigned __int128)n;
    if (m == 2) return (uint64_t)(diag == SMAP_DIAG_INCLUSIVE ? N * (N + 1) / 2 : N * (N - 1) / 2);
    if (m == 3 && diag == SMAP_DIAG_INCLUSIVE) return (uint64_t)(N * (N + 1) * (N + 2) / 6);
    if (m == 3) return n < 3 ? 0 : (uint64_t)(N * (N - 1) * (N - 2) / 6);
    return 0;
}

smap_status smap_plan(const smap_plan_desc *d, smap_plan_t *out)
{
    g_err.clear();
    if (!d || !out) return fail(SMAP_E_INVALID, "smap_plan: NULL argument");
    *out = nullptr;
    const int m = d->m;
    const int64_t n = d->n;
    const int rho = d->rho;
    const bool lam = d->map == SMAP_MAP_LAMBDA;
    const bool incl = d->diag == SMAP_DIAG_INCLUSIVE;
    const bool tile = d->granularity == SMAP_GRAN_TILE;
    const int G = d->shard_count;
    if (m != 2 && m != 3) return fail(SMAP_E_INVALID, "m must be 2 or 3 (got %d)", m);
    if (d->map != SMAP_MAP_BB && d->map != SMAP_MAP_LAMBDA && d->map != SMAP_MAP_ENUM && d->map != SMAP_MAP_BELOW)
        return fail(SMAP_E_INVALID, "bad map %d", d->map);
    const bool enm = d->map == SMAP_MAP_ENUM;
    const bool below = d->map == SMAP_MAP_BELOW;
    if (enm && tile) return fail(SMAP_E_INVALID, "the enumeration baseline map is THREAD granularity only");

    if (d->diag != SMAP_DIAG_STRICT && d->diag != SMAP_DIAG_INCLUSIVE) return fail(SMAP_E_INVALID, "bad diag %d", d->diag);
    if (d->granularity != SMAP_GRAN_THREAD && d->granularity != SMAP_GRAN_TILE)
        return fail(SMAP_E_INVALID, "bad granularity %d", d->granularity);
    if (n < (incl ? 1 : m) || n > ((int64_t)1 << 30)) return fail(SMAP_E_INVALID, "n must be in [m, 2^30] (got %lld)", (long long)n);
    // m=3 inclusive (the paper's Delta_n^3, i <= j <= k < n) runs as the strict set of
    // n + 2 through the bijection (i, j, k) -> (i, j + 1, k + 2), which preserves the
    // packed rank: C(k+2,3) + C(j+1,2) + i (reading E24)
    const int64_t nint = (m == 3 && incl) ? n + 2 : n;
    // "approach n from above": the grid is built for n' = 2^ceil(log2 n) and
    // the elements with an index >= n are filtered out in the kernels
    int64_t npad = 1;
    while (npad < nint) npad <<= 1;
    const bool padded = npad != nint;
    if (!is_pow2(rho) || (rho > npad && !below))
        return fail(SMAP_E_INVALID, "rho must be a power of two <= 2^ceil(log2 n) (got %d)", rho);
    if (!tile) {
        if ((m == 2 && rho > 32) || (m == 3 && rho > 8))
            return fail(SMAP_E_INVALID, "THREAD granularity needs rho^m <= 1024 (rho=%d, m=%d)", rho, m);
        if (d->persistent) return fail(SMAP_E_INVALID, "persistent CTAs need TILE granularity");
    } else {
        const bool ok = m == 2 ? (rho >= 32 && rho <= 512) : (rho >= 8 && rho <= 64);
        if (!ok) return fail(SMAP_E_INVALID, "TILE rho must be in %s (got %d)", m == 2 ? "{32,...,512}" : "{8,16,32,64}", rho);
        if (d->persistent < 0) return fail(SMAP_E_INVALID, "persistent must be >= 0");
    }
    const int64_t N = npad / rho;
    if (m == 2 && lam && N < 2) return fail(SMAP_E_INVALID, "lambda2 needs N = n/rho >= 2");
    if (m == 3 && lam && N < 8) return fail(SMAP_E_INVALID, "lambda3 needs N = n/rho >= 8 (body blocks, E14)");
    if (G < 1 || !is_pow2(G)) return fail(SMAP_E_INVALID, "shard_count must be a power of two >= 1");
    if (!lam && G != 1) return fail(SMAP_E_INVALID, "BB, ENUM and BELOW plans are unsharded");
    if (lam && (N / 2) % G != 0) return fail(SMAP_E_INVALID, "shard_count %d does not divide N/2 = %lld", G, (long long)(N / 2));
    if (d->shard_rank < 0 || d->shard_rank >= G) return fail(SMAP_E_INVALID, "shard_rank out of range");
    if (d->order != SMAP_ORDER_ROWS && d->order != SMAP_ORDER_SQUARES) return fail(SMAP_E_INVALID, "bad order %d", d->order);
    if (d->layout != SMAP_LAYOUT_ROWS && d->layout != SMAP_LAYOUT_TILES) return fail(SMAP_E_INVALID, "bad layout %d", d->layout);
    if (d->layout == SMAP_LAYOUT_TILES && !tile)
        return fail(SMAP_E_INVALID, "the tile-blocked layout is for TILE plans");
    if (d->layout == SMAP_LAYOUT_TILES && m == 3 && incl && !below)
        return fail(SMAP_E_UNSUPPORTED, "the m=3 tile-blocked layout is for the strict diagonal");
    if (padded && G != 1) return fail(SMAP_E_UNSUPPORTED, "sharding needs n to be a power of two (padded grids are not volume-balanced)");
    if (padded && !below && d->layout == SMAP_LAYOUT_TILES)
        return fail(SMAP_E_UNSUPPORTED, "the lambda/BB tile-blocked layout needs n to be a power of two (BELOW: any n)");

    smap_plan_s *p = new (std::nothrow) smap_plan_s();
    if (!p) return fail(SMAP_E_NOMEM, "host allocation failed");
    p->d = *d;
    Params &P = p->P;
    memset(&P, 0, sizeof P);
    P.n = (int)nint; P.N = (int)N; P.log2N = ilog2(N); P.rho = rho; P.log2rho = ilog2(rho);
    P.layout = d->layout;
    if (below) {                              // M = ceil(n'/rho) tiles per side, any M
        const int64_t M = (nint + rho - 1) / rho;
        P.N = (int)M; P.log2N = 0;
        P.W = (int)M; P.log2W = 0; P.wx0 = 0;
        P.nblocks = below_pieces(m, M, rho, incl, p->pieces, &p->layout_len, p->segN, p->segO);
        P.npieces = (int)p->pieces.size();
    } else if (lam) {
        P.W = (int)(N / 2 / G); P.log2W = ilog2(P.W); P.wx0 = d->shard_rank * P.W;
        P.order = m == 2 ? d->order : 0;
        P.nblocks = m == 2 ? (uint64_t)P.W * (uint64_t)(incl ? N + 1 : N)
                           : (uint64_t)P.W * (uint64_t)(N / 2) * (uint64_t)(3 * N / 4);
    } else if (enm) {                         // blocks J <= I (m=2) / I <= J <= K (m=3)
        P.W = (int)N; P.log2W = P.log2N; P.wx0 = 0;
        P.nblocks = m == 2 ? (uint64_t)N * (N + 1) / 2 : (uint64_t)N * (N + 1) * (N + 2) / 6;
    } else {
        P.W = (int)N; P.log2W = P.log2N; P.wx0 = 0;
        P.nblocks = m == 2 ? (uint64_t)N * N : (uint64_t)N * N * N;
    }
    uint64_t rm = 1;
    for (int k = 0; k < m; k++) rm *= (uint64_t)rho;
    {   // every count and byte size of the plan must fit in 64 bits (m = 3 near n = 2^21 would wrap)
        typedef unsigned __int128 u128;
        const u128 Nn = (u128)n, lim = (u128)1 << 64;
        const u128 V128 = m == 2 ? Nn * (Nn + 1) / 2 : (Nn + 2) * (Nn + 1) * Nn / 6;   // >= the domain volume
        const u128 L128 = (u128)P.nblocks * rm;
        if (V128 * 8 >= lim || L128 >= lim || (u128)P.nblocks * 16 >= lim) {
            delete p;
            return fail(SMAP_E_INVALID, "n = %lld is too large: the volume or the launched-thread count of "
                                        "the plan exceeds 64 bits", (long long)n);
        }
    }
    p->launched = P.nblocks * rm;
    p->V = smap_volume(m, n, d->diag);
    p->useful = lam ? p->V / (uint64_t)G : p->V;
    p->elem64 = p->V > ((uint64_t)1 << 32);

    if (!tile && P.nblocks > 0x7fffffffull) {
        delete p;
        return fail(SMAP_E_INVALID, "grid of %llu blocks exceeds one launch; use TILE granularity",
                    (unsigned long long)P.nblocks);
    }
    int dev = d->device;
    if (dev == SMAP_DEVICE_NONE) {            // host-only plan: validation + closed forms, no device work
        p->device = dev;
        p->ctas = 0;
        *out = p;
        return SMAP_OK;
    }
    if (dev < 0) {
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) { delete p; return cuda_fail(e, "cudaGetDevice"); }
    }
    p->device = dev;
    DevGuard guard;                           // allocate on d->device, leave the caller's device current
    cudaError_t e = guard.enter(dev);
    if (e != cudaSuccess) { delete p; return cuda_fail(e, "cudaSetDevice"); }
    int sms = 0;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) { delete p; return cuda_fail(e, "cudaDeviceGetAttribute"); }
    if (tile) {
        uint64_t want = d->persistent > 0 ? (uint64_t)d->persistent * (uint64_t)sms : P.nblocks;
        if (want > P.nblocks) want = P.nblocks;
        if (want > 0x7fffffffull) { delete p; return fail(SMAP_E_INVALID, "too many tiles for one launch"); }
        p->ctas = (unsigned)want;
    }
    if ((e = cudaMalloc(&p->d_res, sizeof(Result))) != cudaSuccess ||
        (e = cudaMallocHost(&p->h_res, sizeof(Result))) != cudaSuccess ||
        (e = cudaEventCreate(&p->ev0)) != cudaSuccess || (e = cudaEventCreate(&p->ev1)) != cudaSuccess) {
        smap_destroy(p);
        return cuda_fail(e, "smap_plan scratch");
    }
    P.res = p->d_res;
    if (below) {
        e = cudaMalloc(&p->d_pieces, p->pieces.size() * sizeof(Piece));
        if (e == cudaSuccess)
            e = cudaMemcpy(p->d_pieces, p->pieces.data(), p->pieces.size() * sizeof(Piece), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) { smap_destroy(p); return cuda_fail(e, "smap_plan pieces"); }
        P.pieces = p->d_pieces;
    }
    *out = p;
    return SMAP_OK;
}

smap_status smap_plan_query(smap_plan_t p, smap_stats *st)
{
    if (!p || !st) return fail(SMAP_E_INVALID, "smap_plan_query: NULL argument");
    memset(st, 0, sizeof *st);
    st->grid_blocks = p->P.nblocks;
    st->launched_threads = p->launched;
    st->useful_elems = p->useful;
    st->wasted_threads = p->launched - p->useful;
    return SMAP_OK;
}

static int internal_pl(smap_plan_t p, smap_payload pl)
{
    switch (pl) {
    case SMAP_PAYLOAD_INDEX_WRITE: return p->elem64 ? PL_IW64 : PL_IW32;
    case SMAP_PAYLOAD_EDM: return PL_EDM;
    case SMAP_PAYLOAD_ATM: return PL_ATM;
    case SMAP_PAYLOAD_TC: return PL_TC;
    case SMAP_PAYLOAD_MAP_DUMP: return PL_MAPD;
    case SMAP_PAYLOAD_HITCOUNT: return PL_HIT;
    case SMAP_PAYLOAD_THREAD_DUMP: return PL_TDUMP;
    case SMAP_PAYLOAD_EMPTY: return PL_EMPTY;
    case SMAP_PAYLOAD_INDEX_WRITE_ATM: return p->elem64 ? PL_IWA64 : PL_IWA32;
    }
    return -1;
}

smap_status smap_out_bytes(smap_plan_t p, smap_payload pl, size_t *bytes)
{
    if (!p || !bytes) return fail(SMAP_E_INVALID, "smap_out_bytes: NULL argument");
    // tile layout: shard-local; BELOW: the slots incl. the holes of tiles cut by n (E29)
    const uint64_t Vout = p->d.layout != SMAP_LAYOUT_TILES ? p->V
                        : p->d.map == SMAP_MAP_BELOW ? p->layout_len : p->useful;
    switch (pl) {
    case SMAP_PAYLOAD_INDEX_WRITE:
    case SMAP_PAYLOAD_INDEX_WRITE_ATM: *bytes = (size_t)Vout * (p->elem64 ? 8 : 4); break;
    case SMAP_PAYLOAD_EDM: *bytes = (size_t)Vout * 4; break;
    case SMAP_PAYLOAD_HITCOUNT: *bytes = (size_t)Vout * 4; break;
    case SMAP_PAYLOAD_MAP_DUMP: *bytes = (size_t)p->P.nblocks * 16; break;
    case SMAP_PAYLOAD_THREAD_DUMP: *bytes = (size_t)p->launched * 8; break;
    case SMAP_PAYLOAD_ATM: case SMAP_PAYLOAD_TC: case SMAP_PAYLOAD_EMPTY: *bytes = 0; break;
    default: return fail(SMAP_E_INVALID, "unknown payload %d", (int)pl);
    }
    return SMAP_OK;
}

}  // extern "C"

// One validated run: the launch arguments derived by run_prepare.
struct RunArgs {
    int ipl = 0, cs = 0;
    bool tile = false, incl = false, atm = false, tc_bits = false;
    int64_t npad = 0;
    Params P;
};

// TC shard analysis (once per sharded lambda3 TILE plan, T = 32 / 64): enumerate the
// shard's tiles with the kernels' own decode and list the 32 x 32 blocks of the pair
// bitmap they read -- tables (I,J) (I,K) and the transposed (K,J) of an interior tile,
// (I,I) (I,K) (K,I) (K,K) of a face tile, (I,I) of a body tile, as (row block, word
// block) -- folded to unordered pairs (the pre-pass writes both orientations).  At
// G = 8 a shard reads 27-46 % of the bitmap (n = 8192).  Unsharded plans, other T and
// grids of more than 2^22 tiles keep the full pre-pass.
static smap_status tc_shard_pairs(smap_plan_t p)
{
    p->tcpairs_done = 1;
    const smap_plan_desc &d = p->d;
    const uint64_t T = (uint64_t)d.rho;
    if (d.map != SMAP_MAP_LAMBDA || d.shard_count <= 1 || (T != 32 && T != 64) || p->P.nblocks > ((uint64_t)1 << 22))
        return SMAP_OK;
    const uint64_t W32 = (uint64_t)p->P.N * T / 32, s = T / 32;          // 32-blocks per side, per tile block
    std::vector<uint8_t> need(W32 * W32, 0);
    auto mark = [&](uint64_t Y, uint64_t X) {           // tile-block pair (row block Y, word block X)
        for (uint64_t a = 0; a < s; a++)
            for (uint64_t b = 0; b < s; b++) {
                const uint64_t r = Y * s + a, c = X * s + b;
                need[(r > c ? r : c) * W32 + (r > c ? c : r)] = 1;
            }
    };
    for (uint64_t bid = 0; bid < p->P.nblocks; bid++) {
        const Blk3 B = decode_lambda3(bid, p->P);
        if (B.cls == 3) continue;
        if (B.cls == 2) { mark(B.I, B.I); continue; }
        if (B.I < B.J) { mark(B.J, B.I); mark(B.K, B.I); mark(B.J, B.K); }
        else { mark(B.I, B.I); mark(B.K, B.I); mark(B.I, B.K); mark(B.K, B.K); }
    }
    std::vector<uint32_t> list;
    for (uint64_t r = 0; r < W32; r++)
        for (uint64_t c = 0; c <= r; c++)
            if (need[r * W32 + c]) list.push_back((uint32_t)(r << 16 | c));
    if (list.size() == W32 * (W32 + 1) / 2) return SMAP_OK;   // every pair: the plain pass
    if (!list.empty()) {
        CK(cudaMalloc(&p->d_tcpairs, list.size() * sizeof(uint32_t)));
        CK(cudaMemcpy(p->d_tcpairs, list.data(), list.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    }
    p->ntcpairs = (uint32_t)list.size();
    if (list.empty()) {                                  // (a shard with no tile: keep a valid non-null marker)
        CK(cudaMalloc(&p->d_tcpairs, sizeof(uint32_t)));
    }
    return SMAP_OK;
}

// Validation and the plan's lazily allocated scratch (TC bitmap, ATM partials); the
// plan's device must be current.  No device work is queued.
static smap_status run_prepare(smap_plan_t p, smap_payload pl, const float *points, size_t points_bytes, float param,
                               void *out, size_t out_bytes, uint32_t flags, RunArgs *a)
{
    if (!p) return fail(SMAP_E_INVALID, "smap_run: NULL plan");
    if (p->device == SMAP_DEVICE_NONE) return fail(SMAP_E_INVALID, "smap_run on a host-only plan");
    const int ipl = internal_pl(p, pl);
    if (ipl < 0) return fail(SMAP_E_INVALID, "unknown payload %d", (int)pl);
    const smap_plan_desc &d = p->d;
    const bool tile = d.granularity == SMAP_GRAN_TILE;
    const bool incl = d.diag == SMAP_DIAG_INCLUSIVE;
    if (flags & ~(SMAP_RUN_CHECKSUM | SMAP_RUN_CHECKSUM_MIX | SMAP_RUN_XOR | SMAP_RUN_FAST_SQRT))
        return fail(SMAP_E_INVALID, "unknown flags 0x%x", flags);
    if ((flags & SMAP_RUN_FAST_SQRT) && ipl != PL_EDM) return fail(SMAP_E_INVALID, "SMAP_RUN_FAST_SQRT is an EDM flag");
    if (ipl == PL_EDM && (d.m != 2 || incl)) return fail(SMAP_E_INVALID, "EDM is defined on the m=2 strict domain");
    const bool atm = pl_atm(ipl);
    if ((atm || ipl == PL_TC) && d.m != 3) return fail(SMAP_E_INVALID, "ATM/TC are m=3 payloads");
    if (ipl == PL_EDM || atm || ipl == PL_TC) {
        const size_t need_pts = (size_t)d.n * 3 * sizeof(float);
        if (!points) return fail(SMAP_E_INVALID, "payload needs points");
        if (points_bytes < need_pts)
            return fail(SMAP_E_INVALID, "points buffer too small: need %zu bytes (n x 3 fp32), got %zu", need_pts, points_bytes);
        if ((reinterpret_cast<uintptr_t>(points) & 3) != 0) return fail(SMAP_E_INVALID, "points not 4-byte aligned");
    }
    if (atm && tile && d.m == 3 && d.rho > 32)
        return fail(SMAP_E_UNSUPPORTED, "ATM tiles are rho <= 32 (three rho x rho r^2 tables in shared memory)");
    if ((atm || ipl == PL_TC) && d.diag == SMAP_DIAG_INCLUSIVE)
        return fail(SMAP_E_UNSUPPORTED, "ATM / TC are defined on distinct triples (strict diagonal)");
    if (ipl == PL_TDUMP && tile) return fail(SMAP_E_INVALID, "THREAD_DUMP needs THREAD granularity");
    size_t need = 0;
    smap_out_bytes(p, pl, &need);
    if (need > 0 && (!out || out_bytes < need))
        return fail(SMAP_E_INVALID, "out buffer too small: need %zu bytes, got %zu", need, out ? out_bytes : (size_t)0);
    if (need > 0) {
        // the tile-blocked layouts are written with 16-B vector stores; the rows layout with
        // element-sized stores (and 16-B records for MAP_DUMP)
        const bool vec = d.layout == SMAP_LAYOUT_TILES || ipl == PL_MAPD;
        const uintptr_t align = vec ? 16 : (ipl == PL_TDUMP || (pl_iw(ipl) && p->elem64)) ? 8 : 4;
        if ((reinterpret_cast<uintptr_t>(out) & (align - 1)) != 0)
            return fail(SMAP_E_INVALID, "out must be %u-byte aligned for this payload / layout", (unsigned)align);
    }
    const bool csum_pl = pl_iw(ipl) || ipl == PL_EDM;
    const int cs = !csum_pl ? 0 : (flags & SMAP_RUN_CHECKSUM_MIX) ? 2 : (flags & SMAP_RUN_CHECKSUM) ? 1
                                 : (flags & SMAP_RUN_XOR) ? 3 : 0;
    uint64_t rm = 1;
    for (int k = 0; k < d.m; k++) rm *= (uint64_t)d.rho;
    const bool reduces = cs > 0 || atm || ipl == PL_TC;
    if (!tile && reduces && (rm % 32) != 0)
        return fail(SMAP_E_INVALID, "reductions need rho^m to be a multiple of 32 (rho^m = %llu)", (unsigned long long)rm);

    const bool tc_bits = ipl == PL_TC && tile;
    const int64_t npad = (int64_t)p->P.N * d.rho;          // bitmap over the grid's index range
    if (tc_bits && !p->d_adj)      // 32-row x 64-column blocks (adj_word, smap_tile3.cu)
        CK(cudaMalloc(&p->d_adj, (size_t)((npad + 31) / 32) * (size_t)(((npad + 31) / 32 + 1) / 2) * 256));
    if (tc_bits && !p->tcpairs_done) {
        smap_status st = tc_shard_pairs(p);
        if (st != SMAP_OK) return st;
    }
    if (atm) {
        const uint64_t np = tile ? p->ctas : p->P.nblocks;
        if (np > p->npartials) {
            cudaFree(p->d_partials); cudaFree(p->d_scratch);
            p->d_partials = nullptr; p->d_scratch = nullptr; p->npartials = 0;
            CK(cudaMalloc(&p->d_partials, np * sizeof(double)));
            CK(cudaMalloc(&p->d_scratch, (finalize_scratch_elems(np) + 1) * sizeof(double)));
            p->npartials = np;
        }
    }
    a->ipl = ipl; a->cs = cs; a->tile = tile; a->incl = incl; a->atm = atm; a->tc_bits = tc_bits; a->npad = npad;
    a->P = p->P;
    a->P.pts = points;
    a->P.param = param;
    a->P.fsqrt = (flags & SMAP_RUN_FAST_SQRT) ? 1 : 0;
    a->P.tc64 = (ipl == PL_TC && tile && d.rho == 64 && d.persistent >= 32) ? 1 : 0;
    a->P.out = out;
    a->P.partials = p->d_partials;
    a->P.adj = p->d_adj;
    return SMAP_OK;
}

// Queue the run's kernels on s (plus the CUDA events of smap_stats' kernel_ms when timed).
// rec (device smap_result *, optional): the run's record, written by the ATM
// finalize (or, for the other payloads, left to the caller: *rec_done false).
// lean (graph capture with a record): no memset of the result block (the graph's
// last kernel clears it behind the record; smap_graph_launch clears it first when
// an smap_run left results in it) and the small tail kernels as programmatic
// dependents.
static smap_status run_launch(smap_plan_t p, const RunArgs &a, cudaStream_t s, bool timed, smap_result *rec = nullptr,
                              bool lean = false, bool *rec_done = nullptr)
{
    const smap_plan_desc &d = p->d;
    uint32_t launches = 0;
    if (rec_done) *rec_done = false;
    if (!a.tc_bits && !lean) CK(cudaMemsetAsync(p->d_res, 0, sizeof(Result), s));   // (the TC pre-pass zeroes it itself)
    if (timed) CK(cudaEventRecord(p->ev0, s));
    cudaError_t e;
    if (a.tc_bits) {
        cudaError_t ea = launch_tc_adjacency(a.P.pts, (int)d.n, (int)a.npad, a.P.param, p->d_adj, p->d_res,
                                             p->d_tcpairs, p->ntcpairs, s);
        if (ea != cudaSuccess) return cuda_fail(ea, "TC adjacency launch");
        launches++;
    }
    if (!a.tile) e = d.m == 2 ? launch_thread2(a.P, d.map, a.incl, a.ipl, a.cs, s) : launch_thread3(a.P, d.map, a.ipl, a.cs, s);
    else e = d.m == 2 ? launch_tile2(a.P, d.rho, d.map, a.incl, a.ipl, a.cs, p->ctas, s)
                      : launch_tile3(a.P, d.rho, d.map, a.ipl, a.cs, p->ctas, s);
    if (e == cudaErrorInvalidValue) return fail(SMAP_E_UNSUPPORTED, "no kernel for this plan/payload combination");
    if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
    launches++;
    if (a.atm) {
        const uint64_t np = a.tile ? p->ctas : p->P.nblocks;
        e = launch_finalize(p->d_partials, np, p->d_scratch, p->d_res, s, &launches, rec, lean, lean);
        if (e != cudaSuccess) return cuda_fail(e, "finalize launch");
        if (rec_done) *rec_done = rec != nullptr;
    }
    if (timed) CK(cudaEventRecord(p->ev1, s));
    p->last_stream = s;
    p->last_launches = launches;
    p->ran = timed ? 1 : p->ran;
    if (timed) p->res_dirty = 1;        // results stay in the block (smap_stats_fetch / smap_result_reduce)
    return SMAP_OK;
}

extern "C" {

smap_status smap_run(smap_plan_t p, smap_payload pl, const float *points, size_t points_bytes, float param,
                     void *out, size_t out_bytes, uint32_t flags, void *stream)
{
    g_err.clear();
    if (!p) return fail(SMAP_E_INVALID, "smap_run: NULL plan");
    if (p->device == SMAP_DEVICE_NONE) return fail(SMAP_E_INVALID, "smap_run on a host-only plan");
    DevGuard guard;                           // the plan's device for this call; restored on every return
    CK(guard.enter(p->device));
    RunArgs a;
    smap_status st = run_prepare(p, pl, points, points_bytes, param, out, out_bytes, flags, &a);
    if (st != SMAP_OK) return st;
    return run_launch(p, a, (cudaStream_t)stream, true);
}

static void fill_stats(smap_plan_t p, const Result *r, smap_stats *st)
{
    smap_plan_query(p, st);
    uint64_t v[5] = {0, 0, 0, 0, 0}, xr = 0;
    for (int s = 0; s < kSlots; s++) {
        for (int k = 0; k < 5; k++) v[k] += r->slot[s][k];
        xr ^= r->slot[s][5];
    }
    st->count = v[0]; st->s0 = v[1]; st->s1 = v[2]; st->mix = v[3]; st->tc = v[4]; st->xr = xr;
    st->sum = r->sum;
    st->launches = p->last_launches;
    float ms = 0.f;
    if (p->ran && cudaEventElapsedTime(&ms, p->ev0, p->ev1) == cudaSuccess) st->kernel_ms = ms;
}

smap_status smap_stats_fetch(smap_plan_t p, smap_stats *st)
{
    if (!p || !st) return fail(SMAP_E_INVALID, "smap_stats_fetch: NULL argument");
    if (!p->ran) return fail(SMAP_E_INVALID, "smap_stats_fetch before smap_run (or on a host-only plan)");
    DevGuard guard;
    CK(guard.enter(p->device));
    CK(cudaEventSynchronize(p->ev1));
    CK(cudaMemcpy(p->h_res, p->d_res, sizeof(Result), cudaMemcpyDeviceToHost));
    fill_stats(p, p->h_res, st);
    return SMAP_OK;
}

static int floor_log2_u64(uint64_t y) { return 63 - __builtin_clzll(y); }

}  // extern "C"

// ---------------------------------------------------------------- E29 inverse
// Grid id of the tile (J, I), J <= I, in the lambda2 inclusive tile grid of side
// N = 2^e (row order; rows 0 and N hold the diagonal tiles): lambda2^-1 as in E23.
static uint64_t tri_grid_id(uint64_t J, uint64_t I, int e)
{
    if (e == 0) return 0;
    const uint64_t N = 1ull << e, W = N / 2;
    if (I == J) return I < W ? I : N * W + (I - W);
    const int l = 63 - __builtin_clzll(I ^ J);
    const uint64_t b = 1ull << l, q = I >> (l + 1);
    return (I - 2 * q * b) * W + (J - q * b);
}
static uint64_t tri_slot_h(uint64_t g, int e, uint64_t sd, uint64_t sf)      // = below_tri_slot
{
    if (e == 0) return 0;
    const uint64_t W = 1ull << (e - 1), N = W << 1;
    if (g < W) return g * sd;
    if (g < N * W) return W * sd + (g - W) * sf;
    return W * sd + (N - 1) * W * sf + (g - N * W) * sd;
}

// Position of element e in the E29 layout of a below plan: the segments of
// the element's tiles give the piece, the piece's closed form the slot, the
// segment kind the place inside the slot.  O(#pieces) piece lookup (host).
static smap_status locate_below(smap_plan_t p, const int64_t *e, int *shard, uint64_t *pos)
{
    const smap_plan_desc &d = p->d;
    const bool incl = d.diag == SMAP_DIAG_INCLUSIVE;
    const int64_t n = d.n;
    const uint64_t T = (uint64_t)d.rho;
    auto seg = [&](uint64_t X) {
        int s = 0;
        while (s + 1 < (int)p->segO.size() && X >= p->segO[s + 1]) s++;
        return s;
    };
    auto piece = [&](int kind, int a, int b, int c) -> const Piece * {
        for (const Piece &pc : p->pieces)
            if (pc.kind == kind && pc.Oa == p->segO[a] && pc.Ob == p->segO[b] && pc.Oc == p->segO[c]) return &pc;
        return nullptr;
    };
    *shard = 0;
    if (d.m == 2) {
        const int64_t i = e[0], j = e[1];
        if (!(0 <= j && j < n && i < n && (incl ? j <= i : j < i))) return fail(SMAP_E_INVALID, "element outside the domain");
        const uint64_t I = (uint64_t)i / T, J = (uint64_t)j / T, r = (uint64_t)i % T, c = (uint64_t)j % T;
        const int a = seg(J), b = seg(I);
        const Piece *pc = piece(a == b ? PK_TRI2 : PK_RECT2, a, b, b);
        if (!pc && a == b) pc = piece(PK_TRI2, a, a, a);
        if (!pc) return fail(SMAP_E_CUDA, "smap_locate: piece not found (internal)");
        const uint64_t sd = incl ? T * (T + 1) / 2 : T * (T - 1) / 2;
        uint64_t slot;
        if (a == b) slot = pc->sbase + tri_slot_h(tri_grid_id(J - pc->Oa, I - pc->Oa, pc->ea), pc->ea, sd, T * T);
        else slot = pc->sbase + ((I - pc->Ob) * (1ull << pc->ea) + (J - pc->Oa)) * T * T;
        const uint64_t in = I != J ? r * T + c : incl ? r * (r + 1) / 2 + c : r * (r - 1) / 2 + c;
        *pos = slot + in;
        return SMAP_OK;
    }
    int64_t i = e[0], j = e[1], k = e[2];
    if (incl ? !(0 <= i && i <= j && j <= k && k < n) : !(0 <= i && i < j && j < k && k < n))
        return fail(SMAP_E_INVALID, "element outside the domain");
    if (incl) { j += 1; k += 2; }                       // E24: the strict set of n + 2
    const uint64_t bi = (uint64_t)i / T, bj = (uint64_t)j / T, bk = (uint64_t)k / T;
    const uint64_t il = (uint64_t)i % T, jl = (uint64_t)j % T, kl = (uint64_t)k % T;
    const int a = seg(bi), b = seg(bj), c = seg(bk);
    const uint64_t T3 = T * T * T, Tf = T * T * (T - 1) / 2;
    const int kind = (bi == bj && bj == bk) ? 3 : bi == bj ? 1 : bj == bk ? 2 : 0;
    uint64_t slot, half = 0;
    if (a == c) {
        const uint64_t O = p->segO[a], N = p->segN[a];
        const Piece *pc = piece(N >= 8 ? PK_TET3 : PK_TETS, a, a, a);
        if (!pc) return fail(SMAP_E_CUDA, "smap_locate: piece not found (internal)");
        const uint64_t I = bi - O, J = bj - O, K = bk - O;
        if (N < 8) {
            slot = pc->sbase + tile_slot3_bb(I, J, K, T);
        } else {                                 // lambda3^-1 inside the piece (as for the lambda layout)
            const uint64_t h = N / 2;
            uint64_t wx, wy, wz;
            if (kind == 3) {
                if (I < h) { wx = I; wy = 0; wz = h; } else { wx = I - h; wy = 0; wz = h + 1; }
            } else {
                const uint64_t Z = kind == 0 ? J - I : 0;
                if (kind == 2) half = Tf;
                const int l = 63 - __builtin_clzll(I ^ K);
                const uint64_t bb = 1ull << l, q = I >> (l + 1);
                const uint64_t u0 = I - 2 * q * bb, v0 = K - 2 * q * bb - bb;
                uint64_t u, v, w;
                if (Z < bb) { u = u0; v = v0; w = Z; }
                else { u = bb - 1 - u0; v = bb - 1 - v0; w = 2 * bb - 1 - Z; }
                if (bb == h) { wx = u; wy = v; wz = w; }
                else { wx = q * bb + u; wy = bb + v; wz = h + w; }
            }
            slot = pc->sbase + tile_slot3_lambda(wx, wy, wz, h, h, T);
        }
    } else if (b == c) {                         // I in S_a x triangle J <= K of S_b
        const Piece *pc = piece(PK_LT, a, b, c);
        if (!pc) return fail(SMAP_E_CUDA, "smap_locate: piece not found (internal)");
        const uint64_t h = tri_grid_id(bj - pc->Ob, bk - pc->Ob, pc->eb), x = bi - pc->Oa;
        slot = pc->sbase + (1ull << pc->ea) * tri_slot_h(h, pc->eb, Tf, T3) + x * (bj == bk ? Tf : T3);
    } else if (a == b) {                         // triangle I <= J of S_a x K in S_c
        const Piece *pc = piece(PK_TL, a, b, c);
        if (!pc) return fail(SMAP_E_CUDA, "smap_locate: piece not found (internal)");
        const uint64_t Na = 1ull << pc->ea;
        const uint64_t total = pc->ea == 0 ? Tf : Na * Tf + (Na / 2) * (Na - 1) * T3;
        const uint64_t h = tri_grid_id(bi - pc->Oa, bj - pc->Oa, pc->ea);
        slot = pc->sbase + (bk - pc->Oc) * total + tri_slot_h(h, pc->ea, Tf, T3);
    } else {
        const Piece *pc = piece(PK_BOX, a, b, c);
        if (!pc) return fail(SMAP_E_CUDA, "smap_locate: piece not found (internal)");
        const uint64_t g = (bi - pc->Oa) + (1ull << pc->ea) * ((bj - pc->Ob) + (1ull << pc->eb) * (bk - pc->Oc));
        slot = pc->sbase + g * T3;
    }
    *pos = slot + half + seg3_local(kind, il, jl, kl, T);
    return SMAP_OK;
}

extern "C" {

smap_status smap_locate(smap_plan_t p, const int64_t *e, int *shard, uint64_t *pos)
{
    if (!p || !e || !shard || !pos) return fail(SMAP_E_INVALID, "smap_locate: NULL argument");
    const smap_plan_desc &d = p->d;
    if (d.map == SMAP_MAP_BELOW && d.layout == SMAP_LAYOUT_TILES) return locate_below(p, e, shard, pos);
    const bool lam = d.map == SMAP_MAP_LAMBDA, incl = d.diag == SMAP_DIAG_INCLUSIVE;
    const int64_t n = d.n;
    if (d.m == 3) {
        int64_t i = e[0], j = e[1], k = e[2];
        if (incl ? !(0 <= i && i <= j && j <= k && k < n) : !(0 <= i && i < j && j < k && k < n))
            return fail(SMAP_E_INVALID, "element outside the domain");
        if (incl) { j += 1; k += 2; }                                  // E24 shift to the strict set of n + 2
        const uint64_t canon = (uint64_t)((unsigned __int128)k * (k - 1) * (k - 2) / 6) + (uint64_t)(j * (j - 1) / 2) + (uint64_t)i;
        if (!lam) {
            *shard = 0;
            *pos = d.layout == SMAP_LAYOUT_ROWS ? canon
                 : tile_slot3_bb((uint64_t)i / d.rho, (uint64_t)j / d.rho, (uint64_t)k / d.rho, d.rho)
                   + seg3_local(((i / d.rho == j / d.rho) && (j / d.rho == k / d.rho)) ? 3 : (i / d.rho == j / d.rho) ? 1
                                : (j / d.rho == k / d.rho) ? 2 : 0, i % d.rho, j % d.rho, k % d.rho, d.rho);
            return SMAP_OK;
        }
        // lambda3^-1 (reading R3 inverted): the tile holding (i, j, k) and its grid position
        const uint64_t T = (uint64_t)d.rho, N = (uint64_t)p->P.N, h = N / 2, W = (uint64_t)p->P.W;
        const uint64_t bi = (uint64_t)i / T, bj = (uint64_t)j / T, bk = (uint64_t)k / T;
        const uint64_t il = (uint64_t)i % T, jl = (uint64_t)j % T, kl = (uint64_t)k % T;
        uint64_t wx, wy, wz, half = 0;
        int kind;
        if (bi == bj && bj == bk) {                                    // body tile d in the spare row (E14)
            kind = 3;
            if (bi < h) { wx = bi; wy = 0; wz = h; } else { wx = bi - h; wy = 0; wz = h + 1; }
        } else {
            uint64_t I = bi, Kb = bk, Z;
            if (bi == bj) { kind = 1; Z = 0; }                         // {I=J<K} half of face tile (I, I, K)
            else if (bj == bk) { kind = 2; Z = 0; half = T * T * (T - 1) / 2; }   // {I<J=K} half of face tile (I, I, K)
            else { kind = 0; Z = bj - bi; }
            // (X, Y, Z) = (I, K, J - I): b = 2^floor(log2(X ^ Y)), q = X >> (log2 b + 1)
            const int l = floor_log2_u64(I ^ Kb);
            const uint64_t b = 1ull << l, q = I >> (l + 1);
            const uint64_t u0 = I - 2 * q * b, v0 = Kb - 2 * q * b - b;
            uint64_t u, v, w;
            if (Z < b) { u = u0; v = v0; w = Z; }                      // inside branch
            else { u = b - 1 - u0; v = b - 1 - v0; w = 2 * b - 1 - Z; } // reflected branch
            if (b == h) { wx = u; wy = v; wz = w; }                    // main cube (level N/2, q = 0)
            else { wx = q * b + u; wy = b + v; wz = h + w; }           // slab level b
        }
        const int owner = (int)(wx / W);
        *shard = owner;
        if (d.layout == SMAP_LAYOUT_ROWS) { *pos = canon; return SMAP_OK; }
        *pos = tile_slot3_lambda(wx - (uint64_t)owner * W, wy, wz, W, h, T) + half + seg3_local(kind, il, jl, kl, T);
        return SMAP_OK;
    }
    const int64_t i = e[0], j = e[1];
    if (!(0 <= j && j < n && i < n && (incl ? j <= i : j < i))) return fail(SMAP_E_INVALID, "element outside the domain");
    const uint64_t T = (uint64_t)d.rho, N = (uint64_t)p->P.N, W = lam ? (uint64_t)p->P.W : 0;
    const uint64_t I = (uint64_t)i / T, J = (uint64_t)j / T, r = (uint64_t)i % T, c = (uint64_t)j % T;
    // owner block omega (lambda) -- lambda2^-1 for off-diagonal blocks, the row-0 / row-N fold otherwise
    uint64_t wx = 0, wy = 0;
    bool second = false;                                         // strict row 0: D2 half of the slot
    if (lam) {
        if (I != J) {
            const int l = floor_log2_u64(I ^ J);
            const uint64_t b = 1ull << l, q = I >> (l + 1);
            wx = J - q * b; wy = I - 2 * q * b;
        } else if (!incl) {
            if (I < N / 2) { wx = I; wy = 0; } else { wx = N - 1 - I; wy = 0; second = true; }
        } else {
            if (I < N / 2) { wx = I; wy = 0; } else { wx = I - N / 2; wy = N; }
        }
    }
    const int owner = lam ? (int)(wx / W) : 0;
    *shard = owner;
    if (d.layout == SMAP_LAYOUT_ROWS) {
        *pos = incl ? (uint64_t)i * (i + 1) / 2 + j : (uint64_t)i * (i - 1) / 2 + j;
        return SMAP_OK;
    }
    // E23 tile layout: slot offset + position inside the slot
    const uint64_t T2 = T * T, Sd = incl ? T * (T + 1) / 2 : T * (T - 1) / 2;
    uint64_t slot;
    if (!lam) {
        slot = (I * (I - 1) / 2 + J) * T2 + I * Sd;
    } else {
        const uint64_t bid = wy * W + (wx - (uint64_t)owner * W);
        if (!incl) slot = bid < W ? bid * T * (T - 1) : W * T * (T - 1) + (bid - W) * T2;
        else if (bid < W) slot = bid * Sd;
        else if (bid < N * W) slot = W * Sd + (bid - W) * T2;
        else slot = W * Sd + (N - 1) * W * T2 + (bid - N * W) * Sd;
    }
    uint64_t in;
    if (I != J) in = r * T + c;
    else if (incl) in = r * (r + 1) / 2 + c;
    else in = (second ? T * (T - 1) / 2 : 0) + r * (r - 1) / 2 + c;
    *pos = slot + in;
    return SMAP_OK;
}

smap_status smap_result_reduce(smap_plan_t p, void *dst, void *stream)
{
    if (!p || !dst) return fail(SMAP_E_INVALID, "smap_result_reduce: NULL argument");
    if (p->device == SMAP_DEVICE_NONE) return fail(SMAP_E_INVALID, "smap_result_reduce on a host-only plan");
    if ((reinterpret_cast<uintptr_t>(dst) & 7) != 0) return fail(SMAP_E_INVALID, "smap_result_reduce: dst not 8-byte aligned");
    if (!p->ran) return fail(SMAP_E_INVALID, "smap_result_reduce before smap_run");
    DevGuard guard;
    CK(guard.enter(p->device));
    cudaError_t e = launch_result_reduce(p->d_res, reinterpret_cast<smap_result *>(dst), (cudaStream_t)stream, false, false);
    if (e != cudaSuccess) return cuda_fail(e, "result reduce launch");
    return SMAP_OK;
}

smap_status smap_result_combine(const void *records, int count, void *dst, void *stream)
{
    g_err.clear();
    if (!records || !dst) return fail(SMAP_E_INVALID, "smap_result_combine: NULL argument");
    if (count < 1) return fail(SMAP_E_INVALID, "smap_result_combine: count must be >= 1 (got %d)", count);
    if (((reinterpret_cast<uintptr_t>(records) | reinterpret_cast<uintptr_t>(dst)) & 7) != 0)
        return fail(SMAP_E_INVALID, "smap_result_combine: pointers must be 8-byte aligned");
    k_result_combine<<<1, 32, 0, (cudaStream_t)stream>>>(reinterpret_cast<const smap_result *>(records), count,
                                                          reinterpret_cast<smap_result *>(dst));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "result combine launch");
    return SMAP_OK;
}

smap_status smap_run_host(smap_plan_t p, smap_payload pl, const float *host_points, size_t points_bytes, float param,
                          void *out, size_t out_bytes, uint32_t flags, void *stream, smap_stats *stats)
{
    g_err.clear();
    if (!p || !stats) return fail(SMAP_E_INVALID, "smap_run_host: NULL argument");
    if (p->device == SMAP_DEVICE_NONE) return fail(SMAP_E_INVALID, "smap_run_host on a host-only plan");
    cudaStream_t s = (cudaStream_t)stream;
    DevGuard guard;                           // staging buffers, kernels and copies on the plan's device
    CK(guard.enter(p->device));
    const float *dev_pts = nullptr;
    size_t dev_bytes = 0;
    if (host_points) {
        const size_t bytes = (size_t)p->d.n * 3 * sizeof(float);
        if (points_bytes < bytes)
            return fail(SMAP_E_INVALID, "host points buffer too small: need %zu bytes (n x 3 fp32), got %zu", bytes, points_bytes);
        if (!p->d_stage) CK(cudaMalloc(&p->d_stage, bytes));
        CK(cudaMemcpyAsync(p->d_stage, host_points, bytes, cudaMemcpyHostToDevice, s));
        dev_pts = p->d_stage;
        dev_bytes = bytes;
    }
    smap_status st = smap_run(p, pl, dev_pts, dev_bytes, param, out, out_bytes, flags, stream);
    if (st != SMAP_OK) return st;
    if (!p->d_rec) CK(cudaMalloc(&p->d_rec, sizeof(smap_result)));
    if (!p->h_rec) CK(cudaMallocHost(&p->h_rec, sizeof(smap_result)));
    cudaError_t e = launch_result_reduce(p->d_res, p->d_rec, s, false, false);
    if (e != cudaSuccess) return cuda_fail(e, "result reduce launch");
    CK(cudaMemcpyAsync(p->h_rec, p->d_rec, sizeof(smap_result), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    smap_plan_query(p, stats);
    stats->count = p->h_rec->count; stats->s0 = p->h_rec->s0; stats->s1 = p->h_rec->s1;
    stats->mix = p->h_rec->mix; stats->tc = p->h_rec->tc; stats->sum = p->h_rec->sum; stats->xr = p->h_rec->xr;
    stats->launches = p->last_launches + 1;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p->ev0, p->ev1) == cudaSuccess) stats->kernel_ms = ms;
    return SMAP_OK;
}

struct smap_graph_s {
    bool lean = false;                // no memset node: the result block is clear between launches
    smap_plan_t p = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    uint32_t launches = 0;
};

smap_status smap_graph_capture(smap_plan_t p, smap_payload pl, const float *points, size_t points_bytes, float param,
                               void *out, size_t out_bytes, uint32_t flags, void *record, smap_graph_t *g)
{
    g_err.clear();
    if (!g) return fail(SMAP_E_INVALID, "smap_graph_capture: NULL graph handle");
    *g = nullptr;
    if (!p) return fail(SMAP_E_INVALID, "smap_graph_capture: NULL plan");
    if (p->device == SMAP_DEVICE_NONE) return fail(SMAP_E_INVALID, "smap_graph_capture on a host-only plan");
    if ((reinterpret_cast<uintptr_t>(record) & 7) != 0) return fail(SMAP_E_INVALID, "record not 8-byte aligned");
    DevGuard guard;
    CK(guard.enter(p->device));
    RunArgs a;
    smap_status st = run_prepare(p, pl, points, points_bytes, param, out, out_bytes, flags, &a);   // (allocates outside the capture)
    if (st != SMAP_OK) return st;
    cudaStream_t cs;
    CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) { cudaStreamDestroy(cs); return cuda_fail(e, "cudaStreamBeginCapture"); }
    const bool lean = record != nullptr;     // (measured: C3 step 0.0378 -> 0.0357 ms at G = 8, 0.132 -> 0.130 at G = 1)
    bool rec_done = false;
    smap_result *rec = reinterpret_cast<smap_result *>(record);
    st = run_launch(p, a, cs, false, rec, lean, &rec_done);
    uint32_t launches = p->last_launches;
    if (st == SMAP_OK && record && !rec_done) {
        e = launch_result_reduce(p->d_res, rec, cs, lean, lean);
        if (e != cudaSuccess) st = cuda_fail(e, "result reduce launch");
        launches++;
    }
    cudaGraph_t graph = nullptr;
    e = cudaStreamEndCapture(cs, &graph);
    cudaStreamDestroy(cs);
    if (st != SMAP_OK) { if (graph) cudaGraphDestroy(graph); return st; }
    if (e != cudaSuccess) { if (graph) cudaGraphDestroy(graph); return cuda_fail(e, "cudaStreamEndCapture"); }
    cudaGraphExec_t exec = nullptr;
    e = cudaGraphInstantiate(&exec, graph, 0);
    if (e != cudaSuccess) { cudaGraphDestroy(graph); return cuda_fail(e, "cudaGraphInstantiate"); }
    smap_graph_s *h = new (std::nothrow) smap_graph_s();
    if (!h) { cudaGraphExecDestroy(exec); cudaGraphDestroy(graph); return fail(SMAP_E_NOMEM, "host allocation failed"); }
    h->p = p; h->graph = graph; h->exec = exec; h->launches = launches; h->lean = lean;
    *g = h;
    return SMAP_OK;
}

smap_status smap_graph_launch(smap_graph_t g, void *stream)
{
    if (!g || !g->exec) return fail(SMAP_E_INVALID, "smap_graph_launch: NULL graph");
    DevGuard guard;
    CK(guard.enter(g->p->device));
    if (g->lean && g->p->res_dirty) {   // an smap_run left its results in the block: clear it first
        CK(cudaMemsetAsync(g->p->d_res, 0, sizeof(Result), (cudaStream_t)stream));
        g->p->res_dirty = 0;
    }
    CK(cudaGraphLaunch(g->exec, (cudaStream_t)stream));
    return SMAP_OK;
}

uint32_t smap_graph_launches(smap_graph_t g) { return g ? g->launches : 0; }

void smap_graph_destroy(smap_graph_t g)
{
    if (!g) return;
    DevGuard guard;
    if (g->p && g->p->device >= 0) guard.enter(g->p->device);
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
}

void smap_destroy(smap_plan_t p)
{
    if (!p) return;
    DevGuard guard;
    if (p->device >= 0) guard.enter(p->device);
    if (p->d_res) cudaFree(p->d_res);
    if (p->h_res) cudaFreeHost(p->h_res);
    if (p->d_partials) cudaFree(p->d_partials);
    if (p->d_scratch) cudaFree(p->d_scratch);
    if (p->d_adj) cudaFree(p->d_adj);
    if (p->d_tcpairs) cudaFree(p->d_tcpairs);
    if (p->d_pieces) cudaFree(p->d_pieces);
    if (p->d_stage) cudaFree(p->d_stage);
    if (p->d_rec) cudaFree(p->d_rec);
    if (p->h_rec) cudaFreeHost(p->h_rec);
    if (p->ev0) cudaEventDestroy(p->ev0);
    if (p->ev1) cudaEventDestroy(p->ev1);
    delete p;
}

} // extern "C"

// ------------------------------------------------------------------ finalize (a7)
namespace smap {

constexpr int kFin1Per = 8192;   // partials per first-level CTA

__global__ void __launch_bounds__(256) k_fin1(const double *in, uint64_t n, double *out)
{
    const uint64_t base = (uint64_t)blockIdx.x * kFin1Per;
    double s = 0.0;
    for (int k = 0; k < kFin1Per / 256; k++) {
        const uint64_t idx = base + (uint64_t)k * 256 + threadIdx.x;
        if (idx < n) s += in[idx];
    }
    s = block_sum_f64(s);
    if (threadIdx.x == 0) out[blockIdx.x] = s;
}

__device__ __forceinline__ void pdl_wait()
{
    asm volatile("griddepcontrol.wait;" ::: "memory");   // (no-op unless launched as a programmatic dependent)
}

// One warp: the kSlots integer slots of res (exact mod 2^64, xr by xor) and the
// fp64 sum into one 56-byte record; with zero, the result block is cleared
// behind it for the next launch of a graph (see smap_graph_capture).
__device__ __forceinline__ void warp_record(Result *res, smap_result *dst, double sum, bool zero)
{
    const int lane = threadIdx.x & 31;
    uint64_t v[5];
#pragma unroll
    for (int k = 0; k < 5; k++) {
        uint64_t s = 0;
        for (int i = lane; i < kSlots; i += 32) s += res->slot[i][k];
        v[k] = warp_sum_u64(s);
    }
    uint64_t xr = 0;
    for (int i = lane; i < kSlots; i += 32) xr ^= res->slot[i][5];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) xr ^= __shfl_xor_sync(0xffffffffu, xr, o);
    if (lane == 0) {
        dst->count = v[0]; dst->s0 = v[1]; dst->s1 = v[2]; dst->mix = v[3]; dst->tc = v[4];
        dst->xr = xr;
        dst->sum = sum;
    }
    if (zero) {
        __syncwarp();
        for (int e = lane; e < (int)(sizeof(Result) / 8); e += 32) reinterpret_cast<unsigned long long *>(res)[e] = 0ull;
    }
}

// The fixed-order fp64 sum of the ATM partials; with rec, also the run's record
// (the record reduction folded into the finalize: one launch fewer per step).
__global__ void __launch_bounds__(1024) k_fin2(const double *in, uint64_t n, Result *res, smap_result *rec, int zero)
{
    pdl_wait();
    __shared__ double total;
    double s = 0.0;
    for (uint64_t idx = threadIdx.x; idx < n; idx += 1024) s += in[idx];
    s = block_sum_f64(s);
    if (threadIdx.x == 0) { res->sum = s; total = s; }
    if (!rec) return;
    __syncthreads();
    if (threadIdx.x < 32) warp_record(res, rec, total, zero != 0);
}

uint64_t finalize_scratch_elems(uint64_t np) { return (np + kFin1Per - 1) / kFin1Per; }

// Sum the kSlots integer slots (exact mod 2^64) and copy the fp64 sum into
// one 56-byte smap_result record.
__global__ void __launch_bounds__(32) k_result_reduce(Result *res, smap_result *dst, int zero)
{
    pdl_wait();
    warp_record(res, dst, res->sum, zero != 0);
}

// Combine G device records in one warp: integer fields add mod 2^64, xr by
// xor, the fp64 sums in record order 0, 1, ..., G-1 (deterministic).
__global__ void __launch_bounds__(32) k_result_combine(const smap_result *recs, int G, smap_result *dst)
{
    const int lane = threadIdx.x;
    uint64_t v[5] = {0, 0, 0, 0, 0}, xr = 0;
    for (int g = lane; g < G; g += 32) {
        const smap_result r = recs[g];
        v[0] += r.count; v[1] += r.s0; v[2] += r.s1; v[3] += r.mix; v[4] += r.tc;
        xr ^= r.xr;
    }
#pragma unroll
    for (int k = 0; k < 5; k++) v[k] = warp_sum_u64(v[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) xr ^= __shfl_xor_sync(0xffffffffu, xr, o);
    if (lane == 0) {
        double sum = 0.0;
        for (int g = 0; g < G; g++) sum += recs[g].sum;
        dst->count = v[0]; dst->s0 = v[1]; dst->s1 = v[2]; dst->mix = v[3]; dst->tc = v[4];
        dst->xr = xr;
        dst->sum = sum;
    }
}

// pdl: launch as a programmatic dependent of the previous kernel on s (its launch
// overlaps the tail of that kernel; the kernel waits in griddepcontrol.wait)
template <typename... Args>
static cudaError_t launch_small(void (*k)(Args...), unsigned grid, unsigned block, cudaStream_t s, bool pdl, Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.stream = s;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, args...);
}

cudaError_t launch_result_reduce(Result *res, smap_result *dst, cudaStream_t s, bool pdl, bool zero)
{
    return launch_small(k_result_reduce, 1, 32, s, pdl, res, dst, zero ? 1 : 0);
}

cudaError_t launch_finalize(const double *partials, uint64_t np, double *scratch, Result *res, cudaStream_t s,
                            uint32_t *launches, smap_result *rec, bool pdl, bool zero)
{
    if (np <= 65536) {
        *launches += 1;
        return launch_small(k_fin2, 1, 1024, s, pdl, partials, np, res, rec, zero ? 1 : 0);
    }
    const uint64_t n1 = finalize_scratch_elems(np);
    k_fin1<<<(unsigned)n1, 256, 0, s>>>(partials, np, scratch);
    *launches += 2;
    return launch_small(k_fin2, 1, 1024, s, false, (const double *)scratch, n1, res, rec, zero ? 1 : 0);
}

} // namespace smap
