/*
 * edm_c_api.c -- the C ABI of include/smap.h used from plain C (no Python, no
 * torch): plan the approach-from-below lambda2 tile map over any n points, run the EDM payload into a
 * device buffer, read the fused count + xor record, and locate one element.
 *
 *   gcc -O2 -I include examples/edm_c_api.c -L paper_1610_07394_b200 -lsmap \
 *       -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_1610_07394_b200 -o /tmp/edm_c_api
 *   /tmp/edm_c_api [n]
 *
 * Exit codes: 0 ok, 1 verification failure, 2 usage / library error.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "smap.h"

#define CHECK(call)                                                                  \
    do {                                                                             \
        smap_status s_ = (call);                                                     \
        if (s_ != SMAP_OK) {                                                         \
            fprintf(stderr, "%s: status %d: %s\n", #call, (int)s_, smap_last_error()); \
            return 2;                                                                \
        }                                                                            \
    } while (0)

int main(int argc, char **argv)
{
    const int64_t n = argc > 1 ? atoll(argv[1]) : 4096;
    smap_plan_desc d;
    memset(&d, 0, sizeof d);
    d.m = 2; d.n = n; d.rho = 128; d.map = SMAP_MAP_BELOW; d.diag = SMAP_DIAG_STRICT;   /* any n (E28) */
    d.granularity = SMAP_GRAN_TILE; d.shard_count = 1; d.device = -1; d.layout = SMAP_LAYOUT_TILES;
    smap_plan_t plan;
    CHECK(smap_plan(&d, &plan));

    /* points: a small deterministic cloud (x, y, z) = fractional parts of i * (golden ratios) */
    float *h = malloc((size_t)n * 3 * sizeof(float));
    for (int64_t i = 0; i < n; i++) {
        h[3 * i] = (float)fmod(i * 0.6180339887, 1.0);
        h[3 * i + 1] = (float)fmod(i * 0.7548776662, 1.0);
        h[3 * i + 2] = (float)fmod(i * 0.5698402910, 1.0);
    }
    float *dpts = NULL;
    void *dout = NULL;
    size_t nb = 0;
    CHECK(smap_out_bytes(plan, SMAP_PAYLOAD_EDM, &nb));
    if (cudaMalloc((void **)&dpts, (size_t)n * 3 * sizeof(float)) != cudaSuccess || cudaMalloc(&dout, nb) != cudaSuccess) {
        fprintf(stderr, "cudaMalloc failed\n");
        return 2;
    }
    cudaMemcpy(dpts, h, (size_t)n * 3 * sizeof(float), cudaMemcpyHostToDevice);

    smap_stats st;
    CHECK(smap_run(plan, SMAP_PAYLOAD_EDM, dpts, (size_t)n * 3 * sizeof(float), 0.0f, dout, nb, SMAP_RUN_XOR, NULL));
    CHECK(smap_stats_fetch(plan, &st));

    /* verify one distance through smap_locate, recomputed here in the stated fp32 order (E17) */
    const int64_t e[2] = {n - 1, n / 3};
    int shard;
    uint64_t pos;
    CHECK(smap_locate(plan, e, &shard, &pos));
    float got;
    cudaMemcpy(&got, (const char *)dout + pos * sizeof(float), sizeof got, cudaMemcpyDeviceToHost);
    const float dx = h[3 * e[1]] - h[3 * e[0]], dy = h[3 * e[1] + 1] - h[3 * e[0] + 1], dz = h[3 * e[1] + 2] - h[3 * e[0] + 2];
    const float want = sqrtf(fmaf(dz, dz, fmaf(dy, dy, dx * dx)));

    printf("n=%lld pairs=%llu count=%llu xor=%016llx kernel_ms=%.4f d(%lld,%lld)=%.9g (host %.9g)\n",
           (long long)n, (unsigned long long)st.useful_elems, (unsigned long long)st.count,
           (unsigned long long)st.xr, st.kernel_ms, (long long)e[0], (long long)e[1], got, want);
    const int ok = st.count == (uint64_t)n * (n - 1) / 2 && memcmp(&got, &want, sizeof got) == 0;
    cudaFree(dpts);
    cudaFree(dout);
    free(h);
    smap_destroy(plan);
    return ok ? 0 : 1;
}
