// smap_thread3.cu -- m = 3, one element per thread, rho^3 threads per block
// (P:565-597 with reading R3).  The block triple is decoded once per block;
// face blocks (I = J < K) fold the {I=J<K} and {I<J=K} element sets, the
// spare slab row holds the N body-diagonal blocks (reading E14).  The BB
// baseline launches the N^3 box and filters i < j < k.
#include "smap_device.cuh"

namespace smap {

template <int MAP, int PL, int CS>
__global__ void __launch_bounds__(512) k_thread3(Params P)
{
    constexpr bool LAM = MAP == SMAP_MAP_LAMBDA;
    constexpr bool BEL = MAP == SMAP_MAP_BELOW;   // E28: lambda3 classes (0/1/2/3) plus BB-like faces 5/6
    constexpr bool LL = LAM || BEL;
    const uint64_t bid = blockIdx.x;
    const uint32_t a = threadIdx.x, bb = threadIdx.y, c = threadIdx.z, rho = (uint32_t)P.rho;
    const Blk3 B = decode3<MAP>(bid, P);

    if (PL == PL_MAPD) {
        if (a == 0 && bb == 0 && c == 0)
            reinterpret_cast<int4 *>(P.out)[bid] = make_int4((int)B.I, (int)B.J, (int)B.K, B.cls);
        return;
    }
    if (PL == PL_EMPTY) {
        if (B.cls != 3 && B.K > 0x7fffffffu) P.res->sum = 1.0;
        return;
    }
    // blocks with no element at all exit as a whole (lambda: idle spare/filler; BB: outside)
    if (PL != PL_TDUMP && ((LL && B.cls == 3) || (!LL && B.cls == 4))) {
        if (pl_atm(PL)) {                 // ATM writes one partial per block
            if (a == 0 && bb == 0 && c == 0) P.partials[bid] = 0.0;
        }
        return;
    }

    uint32_t i = 0, j = 0, k = 0;
    // element coordinates also as (slot, local) pairs: slot 0/1/2 = block I/J/K
    uint32_t si = 0, li = a, sj = 1, lj = bb, sk = 2, lk = c;
    bool valid;
    if (!LL || (BEL && (B.cls == 5 || B.cls == 6))) {   // identity + filter (BB; below's face blocks)
        i = B.I * rho + a; j = B.J * rho + bb; k = B.K * rho + c;
        valid = (B.cls != 4) && i < j && j < k;
    } else if (B.cls == 3) {
        valid = false;
    } else if (B.cls == 2) {              // body block d: a < b < c
        i = B.I * rho + a; j = B.I * rho + bb; k = B.I * rho + c;
        sj = 0; sk = 0;
        valid = a < bb && bb < c;
    } else if (B.I < B.J) {               // interior block I < J < K
        i = B.I * rho + a; j = B.J * rho + bb; k = B.K * rho + c;
        valid = true;
    } else {                              // face block I = J < K
        if (a < bb) { i = B.I * rho + a; j = B.I * rho + bb; k = B.K * rho + c; sj = 0; }
        else        { i = B.I * rho + c; j = B.K * rho + bb; k = B.K * rho + a; li = c; sj = 2; lk = a; }
        valid = a != bb;
    }
    valid = valid && k < (uint32_t)P.n;     // padded grid: k >= n filtered out (k is the largest)
    const uint64_t p = valid ? rank3(i, j, k) : 0;

    if (PL == PL_TDUMP) {
        reinterpret_cast<uint64_t *>(P.out)[(bid * rho + c) * rho * rho + bb * rho + a] = valid ? p : ~0ull;
        return;
    }

    if (pl_iw(PL) || PL == PL_HIT) {
        constexpr int WPL = pl_iw_width(PL);
        Acc<CS> acc;
        if (valid) {
            if (PL == PL_HIT) atomicAdd(reinterpret_cast<unsigned int *>(P.out) + p, 1u);
            else if (WPL == PL_IW32) { reinterpret_cast<uint32_t *>(P.out)[p] = (uint32_t)p; acc.add(p, p); }
            else { reinterpret_cast<uint64_t *>(P.out)[p] = p; acc.add(p, p); }
        }
        // IWA: the ATM half below counts the block's elements
        constexpr int MASK = pl_atm(PL) ? (cs_mask<CS>() & ~kMaskCount) : cs_mask<CS>();
        if (MASK != 0) block_add_slots<MASK>(acc.count, acc.s0, acc.s1, acc.mix, 0, P.res, bid, acc.xr);
        if (!pl_atm(PL)) return;
    }
    if (pl_atm(PL) || PL == PL_TC) {
        // stage the block's three point blocks (I, J, K) in shared memory once
        // (measured faster than per-thread loads: 9 scattered LDG per thread)
        __shared__ float4 sp[3 * 8];
        const uint32_t tid = a + rho * (bb + rho * c);
        if (tid < 3 * rho) {
            const uint32_t s = tid / rho, e = tid - s * rho;
            const uint32_t g = (s == 0 ? B.I : s == 1 ? B.J : B.K) * rho + e;
            sp[tid] = g < (uint32_t)P.n ? make_float4(__ldg(P.pts + 3 * g), __ldg(P.pts + 3 * g + 1), __ldg(P.pts + 3 * g + 2), 0.f)
                                        : make_float4(0.f, 0.f, 0.f, 0.f);   // padded index: never used
        }
        __syncthreads();
        const float4 pi = sp[si * rho + li], pj = sp[sj * rho + lj], pk = sp[sk * rho + lk];
        const float rij = r2_xyz(pi.x, pi.y, pi.z, pj.x, pj.y, pj.z);
        const float rjk = r2_xyz(pj.x, pj.y, pj.z, pk.x, pk.y, pk.z);
        const float rik = r2_xyz(pi.x, pi.y, pi.z, pk.x, pk.y, pk.z);
        // useful elements of this block in closed form (no second barrier)
        const uint32_t r3 = rho * rho * rho, face = rho * rho * (rho - 1), body = rho * (rho - 1) * (rho - 2) / 6;
        uint32_t cnt;
        if (LL && B.cls <= 2) cnt = B.cls == 2 ? body : (B.I < B.J ? r3 : face);
        else cnt = B.cls == 0 ? r3 : (B.cls == 2 ? body : face / 2);
        if ((B.K + 1) * rho > (uint32_t)P.n) cnt = __syncthreads_count(valid);   // block cut by n (block-uniform)
        if (pl_atm(PL)) {
            const double t = valid ? (double)atm_term(rij, rjk, rik, P.param) : 0.0;
            const double s = block_sum_f64(t);
            if (tid == 0) {
                P.partials[bid] = s;
                atomicAdd(&P.res->slot[bid % kSlots][0], (unsigned long long)cnt);
            }
        } else {
            // one block count (per-warp atomics measured slower: 16x more L2 atomics on the slots)
            const float R2 = __fmul_rn(P.param, P.param);
            const bool hit = valid && rij < R2 && rjk < R2 && rik < R2;
            const int hits = __syncthreads_count(hit);
            if (tid == 0) {
                atomicAdd(&P.res->slot[bid % kSlots][0], (unsigned long long)cnt);
                if (hits) atomicAdd(&P.res->slot[bid % kSlots][4], (unsigned long long)hits);
            }
        }
        return;
    }
}

template <int MAP, int PL, int CS>
static cudaError_t go3(const Params &P, cudaStream_t s)
{
    dim3 block(P.rho, P.rho, P.rho);
    k_thread3<MAP, PL, CS><<<(unsigned)P.nblocks, block, 0, s>>>(P);
    return cudaGetLastError();
}

template <int MAP>
static cudaError_t pick3(const Params &P, int pl, int cs, cudaStream_t s)
{
#define CS3(PLV)                                          \
    if (pl == PLV) {                                      \
        if (cs == 0) return go3<MAP, PLV, 0>(P, s);       \
        if (cs == 1) return go3<MAP, PLV, 1>(P, s);       \
        if (cs == 3) return go3<MAP, PLV, 3>(P, s);       \
        return go3<MAP, PLV, 2>(P, s);                    \
    }
    CS3(PL_IW32)
    CS3(PL_IW64)
    CS3(PL_IWA32)
    CS3(PL_IWA64)
#undef CS3
    if (pl == PL_ATM) return go3<MAP, PL_ATM, 0>(P, s);
    if (pl == PL_TC) return go3<MAP, PL_TC, 0>(P, s);
    if (pl == PL_MAPD) return go3<MAP, PL_MAPD, 0>(P, s);
    if (pl == PL_HIT) return go3<MAP, PL_HIT, 0>(P, s);
    if (pl == PL_TDUMP) return go3<MAP, PL_TDUMP, 0>(P, s);
    if (pl == PL_EMPTY) return go3<MAP, PL_EMPTY, 0>(P, s);
    return cudaErrorInvalidValue;
}

cudaError_t launch_thread3(const Params &P, int map, int pl, int cs, cudaStream_t s)
{
    if (map == SMAP_MAP_LAMBDA) return pick3<SMAP_MAP_LAMBDA>(P, pl, cs, s);
    if (map == SMAP_MAP_ENUM) return pick3<SMAP_MAP_ENUM>(P, pl, cs, s);
    if (map == SMAP_MAP_BELOW) return pick3<SMAP_MAP_BELOW>(P, pl, cs, s);
    return pick3<SMAP_MAP_BB>(P, pl, cs, s);
}

} // namespace smap
