// Legacy tensor-core rate on this GPU: back-to-back independent
// mma.sync.m16n8k32 u8 x u8 -> s32 (SASS IMMA.16832.U8.U8) per warp, 8 chains.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o imma_rate scripts/imma_rate.cu && ./imma_rate
// (round 2: ~1.14 POPS at 4-16 warps per CTA, 1-4 CTAs per SM; profiles/r02_imma_microbench.txt)
#include <cstdio>
#include <cstdint>
__global__ void k(const uint32_t *in, int *out, int iters) {
    uint32_t a0 = in[threadIdx.x], a1 = in[threadIdx.x + 1], a2 = in[threadIdx.x + 2], a3 = in[threadIdx.x + 3];
    uint32_t b0 = in[threadIdx.x + 4], b1 = in[threadIdx.x + 5];
    int d[8][4] = {};
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int u = 0; u < 8; u++)
            asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+r"(d[u][0]), "+r"(d[u][1]), "+r"(d[u][2]), "+r"(d[u][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    int s = 0;
    for (int u = 0; u < 8; u++) s += d[u][0] + d[u][1] + d[u][2] + d[u][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    uint32_t *in; int *out;
    cudaMalloc(&in, 4096); cudaMalloc(&out, 148 * 8 * 256 * 4 * 4); cudaMemset(in, 1, 4096);
    const int iters = 4096;
    for (int warps = 4; warps <= 16; warps *= 2)
        for (int cps = 1; cps <= 4; cps *= 2) {
            dim3 g(148 * cps), b(32 * warps);
            k<<<g, b>>>(in, out, 10); cudaDeviceSynchronize();
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0); k<<<g, b>>>(in, out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            const double ops = 2.0 * 16 * 8 * 32 * 8.0 * iters * (double)g.x * warps;
            printf("warps/CTA %d CTAs/SM %d: %.3f ms, %.1f TOPS\n", warps, cps, ms, ops / ms / 1e9);
        }
    return 0;
}
