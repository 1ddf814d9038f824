// smap_internal.h -- types shared by the C-ABI implementation (smap_api.cu)
// and the kernel translation units.  Not part of the public ABI.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace smap {

constexpr int kSlots = 64;   // spread the per-CTA integer atomics over 64 slots

// Device result block of one smap_run (zeroed on the stream before the kernel).
struct Result {
    unsigned long long slot[kSlots][6];  // per slot: count, s0, s1, mix, tc (added) and xr (xor-combined)
    double sum;                          // ATM, written by the finalize kernel
    double pad;
};

// Internal payload codes (the public smap_payload plus the index element width).
enum Pl { PL_IW32 = 0, PL_IW64, PL_EDM, PL_ATM, PL_TC, PL_MAPD, PL_HIT, PL_TDUMP, PL_EMPTY,
          PL_IWA32, PL_IWA64 };   // IWA: index write + ATM sum in one pass (C3)
// payload traits: writes packed indices / accumulates ATM terms / index element width
constexpr bool pl_iw(int pl) { return pl == PL_IW32 || pl == PL_IW64 || pl == PL_IWA32 || pl == PL_IWA64; }
constexpr bool pl_atm(int pl) { return pl == PL_ATM || pl == PL_IWA32 || pl == PL_IWA64; }
constexpr int pl_iw_width(int pl) { return (pl == PL_IW64 || pl == PL_IWA64) ? PL_IW64 : PL_IW32; }

// "Approach n from below" (reading E28): the M tiles per side are
// cut into the binary-digit segments of M; every piece of the decomposition
// is a power-of-two simplex mapped by lambda or a box at the identity.
enum PieceKind {
    PK_TRI2 = 0,   // m=2: triangle of segment a (lambda2 inclusive tile grid; N_a = 1: one diagonal tile)
    PK_RECT2,      // m=2: rectangle J in segment a x I in segment b, a < b (identity)
    PK_TET3,       // m=3: tetrahedron of segment a by lambda3 (R3), N_a >= 8
    PK_TETS,       // m=3: tetrahedron of segment a, N_a < 8: tiles I <= J <= K in colex order
    PK_LT,         // m=3: I in segment a  x  triangle J <= K of segment b (lambda2 grid)
    PK_TL,         // m=3: triangle I <= J of segment a (lambda2 grid)  x  K in segment c
    PK_BOX         // m=3: segments a < b < c at the identity
};
struct Piece {
    uint64_t start;            // first tile id of the piece (launch order)
    uint64_t sbase;            // first position of the piece in the tile-blocked layout (E29)
    uint32_t Oa, Ob, Oc;       // segment offsets (tiles)
    uint8_t kind, ea, eb, ec;  // PieceKind, log2 of the segment sizes
};

struct Params {
    int n;          // elements per side (any n; the grid covers N * rho >= n)
    int N;          // blocks (tiles) per side = n / rho
    int log2N;
    int rho;        // block side (THREAD) or tile side (TILE)
    int log2rho;
    int W;          // grid columns of this shard = N / (2G)   (BB: N)
    int log2W;
    int wx0;        // first column of this shard = rank * W
    int order;      // lambda2 launch order: 0 rows, 1 level squares
    int layout;     // m=2 output layout: 0 canonical packed rows (E16), 1 lambda-order tiles (E23)
    uint64_t nblocks;             // blocks / tiles in this shard's grid
    const float *pts;              // n x 3 fp32 AoS (EDM / ATM / TC)
    float param;                   // ATM eps^2, TC R
    void *out;
    Result *res;
    double *partials;              // ATM: one fp64 per CTA
    const uint32_t *adj;           // TC (TILE): pair-predicate bitmap, n rows of n/32 words
    const Piece *pieces;           // SMAP_MAP_BELOW: the decomposition, sorted by start
    int npieces;
    int fsqrt;                     // EDM (SMAP_RUN_FAST_SQRT): sqrt.approx on the vector tile path
    int tc64;                      // TC, T = 64: 64-thread CTAs (plans with >= 32 persistent CTAs per SM)
};

// ---------------------------------------------------------------- m=3 tile-blocked layout (E26)
// Slot offsets (elements, shard-local) of a T^3 tile in the tile-blocked
// layout: slots in launch order, sizes T^3 (interior), T^2(T-1) (lambda face
// tile: {I=J<K} then {I<J=K}), T^2(T-1)/2 (BB face tiles), C(T,3) (body),
// 0 (idle).  Shared by the kernels and smap_locate.
struct Slot3Sizes {
    uint64_t full, face, half, body;
};
__host__ __device__ __forceinline__ Slot3Sizes slot3_sizes(uint64_t T)
{
    Slot3Sizes s;
    s.full = T * T * T;
    s.half = T * T * (T - 1) / 2;
    s.face = 2 * s.half;
    s.body = T * (T - 1) * (T - 2) / 6;
    return s;
}

// lambda3, row launch order: tile at grid position (wx, wy, wz), x = wx - wx0,
// W columns per shard, h = N/2.  Main cube: layer wz = 0 is all face tiles,
// layers 1..h-1 all full.  Slab layer w = wz - h: row 0 holds body tiles for
// w <= 1 (idle otherwise); rows wy >= 1 are faces (w = 0), fillers
// (w >= 2^floor(log2 wy)), or full tiles -- i.e. full for wy >= r0(w) =
// 2^(floor(log2 w) + 1).
__host__ __device__ __forceinline__ uint64_t tile_slot3_lambda(uint64_t x, uint64_t wy, uint64_t wz, uint64_t W,
                                                                uint64_t h, uint64_t T)
{
    const Slot3Sizes z = slot3_sizes(T);
    if (wz == 0) return (wy * W + x) * z.face;
    if (wz < h) return h * W * z.face + ((wz - 1) * h * W + wy * W + x) * z.full;
    const uint64_t w = wz - h;
    uint64_t off = h * W * z.face + (h - 1) * h * W * z.full;         // the main cube
    if (w >= 1) off += W * z.body + (h - 1) * W * z.face;             // slab layer 0
    if (w >= 2) off += W * z.body + (h > 2 ? h - 2 : 0) * W * z.full; // slab layer 1 (full rows wy >= 2)
    for (uint64_t e = 1; ((uint64_t)1 << e) < w; e++) {               // layers [2^e, 2^(e+1)) below w: rows wy >= 2^(e+1)
        const uint64_t lo = (uint64_t)1 << e, hi = lo << 1;
        const uint64_t cnt = (w < hi ? w : hi) - lo, rows = h > hi ? h - hi : 0;
        off += cnt * rows * W * z.full;
    }
    if (wy == 0) return off + x * z.body;                             // body tile (w <= 1)
    if (w <= 1) off += W * z.body;
    if (w == 0) return off + ((wy - 1) * W + x) * z.face;
    uint64_t r0 = 2;
    while (r0 <= w) r0 <<= 1;                                         // 2^(floor(log2 w) + 1)
    return off + ((wy - r0) * W + x) * z.full;
}

// BB: tiles I <= J <= K in colex order (K outer, I inner).
__host__ __device__ __forceinline__ uint64_t tile_slot3_bb(uint64_t I, uint64_t J, uint64_t K, uint64_t T)
{
    const Slot3Sizes z = slot3_sizes(T);
    const uint64_t c3 = K * (K - 1) * (K - 2) / 6, c2 = K * (K - 1) / 2;   // (K < 3 / K < 2 give 0)
    const uint64_t base = (K >= 3 ? c3 : 0) * z.full + 2 * (K >= 2 ? c2 : 0) * z.half + K * z.body;
    if (J < K) return base + (J * (J - 1) / 2) * z.full + J * z.half + I * z.full;
    return base + c2 * z.full + K * z.half + I * z.half;
}

// position of element (il, jl, kl) inside a segment of kind 0 interior,
// 1 {I=J<K} (il < jl), 2 {I<J=K} (jl < kl), 3 body (il < jl < kl)
__host__ __device__ __forceinline__ uint64_t seg3_local(int kind, uint64_t il, uint64_t jl, uint64_t kl, uint64_t T)
{
    switch (kind) {
    case 0: return (kl * T + jl) * T + il;
    case 1: return kl * (T * (T - 1) / 2) + jl * (jl - 1) / 2 + il;
    case 2: return (kl * (kl - 1) / 2 + jl) * T + il;
    default: return kl * (kl - 1) * (kl - 2) / 6 + jl * (jl - 1) / 2 + il;
    }
}

// Kernel launchers (one per translation unit).  Return cudaErrorInvalidValue
// for a combination that has no instantiated kernel.
cudaError_t launch_thread2(const Params &P, int map, bool incl, int pl, int cs, cudaStream_t s);
cudaError_t launch_thread3(const Params &P, int map, int pl, int cs, cudaStream_t s);
cudaError_t launch_tile2(const Params &P, int T, int map, bool incl, int pl, int cs, unsigned ctas, cudaStream_t s);
cudaError_t launch_tile3(const Params &P, int T, int map, int pl, int cs, unsigned ctas, cudaStream_t s);
// TC pre-pass: adj[j * ceil(npad/32) + w] bit b <=> 32w + b < n, j < n and
// r2(32w + b, j) < R*R (the same fp32 predicate as the per-triple compare);
// npad = N * rho (rows j < npad, words rounded up).
// It also zeroes the run's result block (the main kernel follows in stream order).
// pairs (optional): the list of 32 x 32 block pairs (rb << 16 | cb, cb <= rb) to build
// (a sharded plan builds only what its tiles read); null = all of them.
cudaError_t launch_tc_adjacency(const float *pts, int n, int npad, float R, uint32_t *adj, Result *res,
                                const uint32_t *pairs, uint32_t npairs, cudaStream_t s);
uint64_t finalize_scratch_elems(uint64_t np);
}  // namespace smap

#include "smap.h"

namespace smap {
// Deterministic fixed-order fp64 reduction of partials[0..np) into res->sum;
// with rec, the same kernel also writes the run's record.  pdl: the last kernel
// is a programmatic dependent of the previous one on s; zero: it clears res
// behind the record.  Adds the number of kernels it launched to *launches.
cudaError_t launch_finalize(const double *partials, uint64_t np, double *scratch, Result *res, cudaStream_t s,
                            uint32_t *launches, smap_result *rec = nullptr, bool pdl = false, bool zero = false);
// res -> one record (pdl / zero as above)
cudaError_t launch_result_reduce(Result *res, smap_result *dst, cudaStream_t s, bool pdl, bool zero);

} // namespace smap
