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
enum Pl { PL_IW32 = 0, PL_IW64, PL_EDM, PL_ATM, PL_TC, PL_MAPD, PL_HIT, PL_TDUMP, PL_EMPTY };

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
};

// Kernel launchers (one per translation unit).  Return cudaErrorInvalidValue
// for a combination that has no instantiated kernel.
cudaError_t launch_thread2(const Params &P, int map, bool incl, int pl, int cs, cudaStream_t s);
cudaError_t launch_thread3(const Params &P, int map, int pl, int cs, cudaStream_t s);
cudaError_t launch_tile2(const Params &P, int T, bool lam, bool incl, int pl, int cs, unsigned ctas, cudaStream_t s);
cudaError_t launch_tile3(const Params &P, int T, bool lam, int pl, int cs, unsigned ctas, cudaStream_t s);
// TC pre-pass: adj[j * (npad/32) + w] bit b <=> 32w + b < n, j < n and
// r2(32w + b, j) < R*R (the same fp32 predicate as the per-triple compare);
// npad = N * rho, a multiple of 32.
cudaError_t launch_tc_adjacency(const float *pts, int n, int npad, float R, uint32_t *adj, cudaStream_t s);
// Deterministic fixed-order fp64 reduction of partials[0..np) into res->sum.
// Adds the number of kernels it launched to *launches.
cudaError_t launch_finalize(const double *partials, uint64_t np, double *scratch, Result *res,
                            cudaStream_t s, uint32_t *launches);
uint64_t finalize_scratch_elems(uint64_t np);
}  // namespace smap

#include "smap.h"

namespace smap {
cudaError_t launch_result_reduce(const Result *res, smap_result *dst, cudaStream_t s);

} // namespace smap
