/*
 * smap.h -- C ABI of the B200-native (sm_100a) recursive simplex thread maps
 * of arXiv 1610.07394 (Navarro, Bustos, Hitschfeld, "Possibilities of Recursive
 * GPU Mapping for Discrete Orthogonal Simplices").
 *
 * Citations: "P:a-b" = PAPER.md lines a-b; "Ek" = reading k in DESIGN.md s.3.
 *
 * What the library computes (DESIGN.md s.1):
 *   a GPU launch over a compact orthotope of blocks is sent onto a discrete
 *   orthogonal m-simplex by the O(1) block-space map lambda (m=2: P:346-390;
 *   m=3: P:565-597, reading R3 = E11/E12), or -- the baseline -- by the
 *   bounding box f(x) = x plus a filter; every mapped
 *   element runs one payload of the paper's problem class (P:92-99,
 *   P:115-117; definitions E15) and the block results are reduced on device.
 *
 * Domains (E1, E13, E16) and their packed layouts (position in the nested-loop
 * enumeration; the kernels use the closed forms):
 *   m=2 strict     {(i,j): 0 <= j < i < n}         p = i(i-1)/2 + j   V = n(n-1)/2
 *   m=2 inclusive  {(i,j): 0 <= j <= i < n}        p = i(i+1)/2 + j   V = n(n+1)/2
 *   m=3 strict     {(i,j,k): 0 <= i < j < k < n}   p = C(k,3) + C(j,2) + i   V = C(n,3)
 *
 * Conventions of every entry point:
 *   - noexcept: errors are returned as smap_status codes, never thrown; the
 *     message of the last error on the calling thread is smap_last_error().
 *   - SMAP_E_INVALID is returned before any device work and has no side effect.
 *   - No CPU fallback exists: without a CUDA device smap_plan returns SMAP_E_CUDA.
 *   - Ownership: the caller owns `points`, `out` and the stream; a plan owns
 *     only its own scratch (result block, fp64 partials, staging buffers).
 *   - A plan may be used from one stream at a time (not re-entrant).
 *   - Devices: a plan lives on the device it was planned for (smap_plan_desc.device);
 *     every entry point taking a plan makes that device current for the call and
 *     restores the caller's current device before returning (also on errors).
 *     Streams and buffers passed with a plan must belong to its device.
 */
#ifndef SMAP_H
#define SMAP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SMAP_ABI_VERSION 2   /* 2: smap_run / smap_run_host take the points buffer size */

typedef enum {
    SMAP_OK = 0,
    SMAP_E_INVALID = 1,      /* bad arguments: nothing was done */
    SMAP_E_UNSUPPORTED = 2,  /* valid but not implemented for this combination */
    SMAP_E_CUDA = 3,         /* CUDA runtime error (message in smap_last_error) */
    SMAP_E_NOMEM = 4         /* device or pinned allocation failed */
} smap_status;

typedef enum {
    SMAP_MAP_BB = 0,         /* bounding box: identity + filter */
    SMAP_MAP_LAMBDA = 1,     /* lambda2 / lambda3 reading R3 */
    SMAP_MAP_ENUM = 2,       /* comparison baseline: the linear-enumeration map
                                g: Z^1 -> Z^m of P:166-174, block-space as in P:252-262, inverted by
                                the analytic root (fp32 sqrt for m=2, cbrt + sqrt for m=3, then an
                                exact integer correction).  A 1-D grid of the N(N+1)/2 blocks J<=I
                                (m=2) or the C(N+2,3) blocks I<=J<=K (m=3); diagonal blocks filter
                                like BB.  THREAD granularity, unsharded. */
    SMAP_MAP_BELOW = 3       /* "approach n from below" (reading E28): the M = ceil(n'/rho)
                                tiles per side are cut into the binary digits of M (segments
                                S_s = [O_s, O_s + N_s), N_0 > N_1 > ...); every piece is a power-of-two
                                simplex mapped by lambda (lambda2 inclusive tile grid, lambda3 for
                                N_s >= 8) or a box / small simplex at the identity, so every launched
                                tile holds elements (besides lambda3's own idle tiles).  Any n;
                                THREAD (blocks, the paper's launch) or TILE granularity, unsharded.  With SMAP_LAYOUT_TILES (reading E29) every
                                tile is one slot in launch order whose size depends on its class only
                                (T^m, diagonal/face, body); elements of a tile cut by n leave holes,
                                so smap_out_bytes may exceed V * sizeof(element).  smap_locate
                                inverts it (piece lookup + closed form, host). */
} smap_map;

typedef enum {
    SMAP_DIAG_STRICT = 0,    /* j < i  /  i < j < k */
    SMAP_DIAG_INCLUSIVE = 1  /* j <= i (the paper's Delta_n^2) / i <= j <= k (Delta_n^3,
                                P:559-563).  m=3 runs the strict set of n + 2 through the
                                rank-preserving bijection (i, j, k) -> (i, j+1, k+2) (reading E24);
                                no ATM / TC (defined on distinct triples) */
} smap_diag;

typedef enum {
    /* one element per thread, rho^m threads per block -- the paper's launch
     * (P:363-367); blocks at or next to the diagonal are folded (E6, E14).
     * rho^m <= 1024. */
    SMAP_GRAN_THREAD = 0,
    /* one rho^m TILE of elements per 256-thread CTA step: lambda is applied to
     * tiles (the same map, coarser blocks); threads loop over the tile rows
     * with lanes on the contiguous axis; diagonal tiles are clipped per row
     * instead of folded.  m=2: rho in {32,64,128,256,512}; m=3: rho in {8,16,32,64}
     * (ATM: rho <= 32). */
    SMAP_GRAN_TILE = 1
} smap_granularity;

typedef enum {
    SMAP_PAYLOAD_INDEX_WRITE = 0, /* out[p] = p; uint32 if V <= 2^32 else uint64 */
    SMAP_PAYLOAD_EDM = 1,         /* m=2 strict: out[p] = ||x_i - x_j||_2, fp32 (E15, E17) */
    SMAP_PAYLOAD_ATM = 2,         /* m=3: sum of Axilrod-Teller terms (E15), param = eps^2; result stats.sum */
    SMAP_PAYLOAD_TC = 3,          /* m=3: #{i<j<k: r_ij, r_jk, r_ik < R}, param = R; result stats.tc.  TILE plans
                                     allocate a pair-predicate bitmap of ~n'^2 / 8 bytes (32-row x 64-column
                                     blocks, n' rounded up to them) in the plan's scratch on the first TC run
                                     (n' = the grid's index range; SMAP_E_NOMEM if it does not fit) */
    SMAP_PAYLOAD_MAP_DUMP = 4,    /* int32[4] per grid block/tile in launch order (see below) */
    SMAP_PAYLOAD_HITCOUNT = 5,    /* uint32 out[p] += 1 per mapped element (caller zeroes out) */
    SMAP_PAYLOAD_THREAD_DUMP = 6, /* THREAD gran. only: uint64 per launched thread, p or UINT64_MAX */
    SMAP_PAYLOAD_EMPTY = 7,       /* decode only, no element work (block-scheduling microbenchmark) */
    SMAP_PAYLOAD_INDEX_WRITE_ATM = 8 /* m=3 strict, one pass (config C3, "index-write plus triple-interaction
                                        sum"): out[p] = p as INDEX_WRITE (same out buffer, layout, flags)
                                        AND the ATM sum of the same triples as ATM (param = eps^2,
                                        stats.sum); TILE rho <= 32 or THREAD */
} smap_payload;

#define SMAP_DEVICE_NONE (-2)      /* smap_plan_desc.device: host-only plan */

/* smap_run flags */
#define SMAP_RUN_CHECKSUM     0x1u /* INDEX_WRITE(_ATM)/EDM: accumulate s0, s1 (E21) */
#define SMAP_RUN_CHECKSUM_MIX 0x2u /* INDEX_WRITE(_ATM)/EDM: also accumulate mix (E21); implies CHECKSUM */
#define SMAP_RUN_XOR          0x4u /* INDEX_WRITE(_ATM)/EDM: count and xr only (the cheapest fused reduction, E21) */
#define SMAP_RUN_FAST_SQRT    0x8u /* EDM only: on the full tiles of a TILE rho >= 128 tile-blocked (E23) plan, the
                                    * distance is sqrt.approx.ftz (one MUFU.SQRT, relative error < 2^-22 -- inside the
                                    * north star's 1e-5, NOT bit-identical to the correctly rounded sqrt of E17);
                                    * every other tile, and any warp whose points include a nonzero coordinate below
                                    * 2^-40 in magnitude, keeps the exact path.  Fewer SM instructions per pair: for
                                    * the power-capped (sustained) regime. */

typedef struct smap_plan_s *smap_plan_t;

typedef struct {
    int     m;            /* 2 or 3 */
    int64_t n;            /* elements per side, any n in [m, 2^30] (m=3: every count of the plan, e.g.
                             8 * C(n,3), must fit in 64 bits, i.e. n <= ~2.6e6): the grid is built for
                             n' = 2^ceil(log2 n) and elements with an index >= n are filtered
                             ("approach n from above"); n' != n needs shard_count 1
                             and the canonical layout */
    int     rho;          /* block side (threads per axis for THREAD, elements per axis for TILE); power of two */
    int     map;          /* smap_map */
    int     diag;         /* smap_diag */
    int     granularity;  /* smap_granularity */
    int     persistent;   /* TILE only: 0 = one CTA per tile; k > 0 = k CTAs per SM looping over tiles
                           * (grid-stride; k above the resident limit launches the extra CTAs as
                           * others finish -- dynamic balance over tiles of unequal cost).
                           * CTAs have 256 threads, except TC at rho = 64: 128 threads, or 64 when
                           * k >= 32 (the sizes that fill an SM at 16 / 32 CTAs) */
    int     shard_rank;   /* 0 .. shard_count-1 */
    int     shard_count;  /* G: power of two dividing N/2 (lambda only); 1 = unsharded */
    int     device;       /* CUDA device ordinal; -1 = the calling thread's current device;
                             SMAP_DEVICE_NONE = host-only plan (validation + closed forms; cannot run) */
    int     order;        /* lambda2 launch order (smap_order); ignored otherwise */
    int     layout;       /* output layout (smap_layout); SMAP_LAYOUT_TILES needs TILE granularity (m=3
                             inclusive: BELOW plans only) */
} smap_plan_desc;

typedef enum {
    /* canonical packed rows (E16): out[p] at p = i(i-1)/2 + j (strict) / i(i+1)/2 + j;
     * a sharded plan writes its own positions of the FULL-size array */
    SMAP_LAYOUT_ROWS = 0,
    /* lambda-order tile-blocked layout (E23; the "succinct blocked" storage of
     * P:262-264): each T x T tile is one contiguous row-major slot, slots in row
     * launch order; a sharded plan writes a SHARD-LOCAL array of V/G elements.
     * Diagonal tiles are packed triangles (strict row 0: D1 then D2).
     * smap_locate gives the position of any element in O(1). */
    SMAP_LAYOUT_TILES = 1
} smap_layout;

typedef enum {
    SMAP_ORDER_ROWS = 0,    /* block-linear id = wy*W + (wx - wx0) */
    SMAP_ORDER_SQUARES = 1  /* level by level, one b x b copy square at a time (see the launch-order note) */
} smap_order;

typedef struct {
    /* closed forms of the plan (filled by smap_plan_query and smap_stats_fetch) */
    uint64_t grid_blocks;      /* blocks (THREAD) or tiles (TILE) of this shard's grid */
    uint64_t launched_threads; /* grid_blocks * rho^m: launched threads (THREAD) / element slots (TILE) */
    uint64_t useful_elems;     /* elements of the domain owned by this shard */
    uint64_t wasted_threads;   /* launched_threads - useful_elems */
    /* measured by the last smap_run (device results) */
    uint64_t count;            /* elements the kernel processed */
    uint64_t s0;               /* sum bits(v)            mod 2^64 (SMAP_RUN_CHECKSUM) */
    uint64_t s1;               /* sum (p+1) * bits(v)    mod 2^64 (SMAP_RUN_CHECKSUM) */
    uint64_t mix;              /* sum mix64(p ^ bits(v)*K) mod 2^64 (SMAP_RUN_CHECKSUM_MIX) */
    double   sum;              /* ATM: sum of terms (fp32 terms, fp32 per-thread, fp64 per CTA, fixed-order finalize) */
    uint64_t tc;               /* TC: triple count */
    uint64_t xr;               /* xor of bits(v) over the elements (SMAP_RUN_XOR) */
    float    kernel_ms;        /* device time of the last smap_run's kernels (CUDA events on its stream) */
    uint32_t launches;         /* number of kernels the last smap_run launched */
} smap_stats;

/* Validate `d`, derive the grid and the closed forms, and allocate the plan's
 * scratch on d->device.  Host math plus small cudaMalloc's; launches nothing.
 * SMAP_E_INVALID: m not in {2,3}; n outside [m, 2^30]; a plan count (volume x 8 bytes,
 * launched threads, dump bytes) that does not fit in 64 bits; rho not a power of two;
 * N = n'/rho too small (m=2: N >= 2; m=3 lambda: N >= 8, BB: N >= 1), with
 * n' = 2^ceil(log2 n) (2^ceil(log2 (n+2)) for m=3 inclusive); rho outside the
 * granularity's range; shard_count not a power of two or not dividing N/2, or
 * > 1 with BB / ENUM; persistent with THREAD granularity.
 * SMAP_E_UNSUPPORTED: n' != n with shard_count > 1 or the tile-blocked layout. */
smap_status smap_plan(const smap_plan_desc *d, smap_plan_t *out);

/* Fill the closed-form fields of *st (others zero).  Host only. */
smap_status smap_plan_query(smap_plan_t p, smap_stats *st);

/* Bytes `out` must hold for payload pl (0 for reduction-only payloads).
 * INDEX_WRITE/EDM/HITCOUNT index the FULL packed array of the domain even when
 * sharded (a shard writes only its own positions): V * sizeof(element).
 * MAP_DUMP: grid_blocks * 16.  THREAD_DUMP: launched_threads * 8. */
smap_status smap_out_bytes(smap_plan_t p, smap_payload pl, size_t *bytes);

/* Run payload pl over the plan's grid, asynchronously on `stream`
 * (cudaStream_t of the plan's device; NULL = legacy default stream).
 *   points:       DEVICE pointer to n x 3 fp32 (x,y,z) array-of-structs, 4-byte
 *                 aligned; required for EDM/ATM/TC, ignored otherwise (may be NULL).
 *   points_bytes: size of the points buffer; must be >= n * 12 when points are used.
 *   param:        ATM: eps^2 (softening); TC: R (distance threshold); else ignored.
 *   out:          DEVICE pointer of >= smap_out_bytes bytes, or NULL for ATM/TC/EMPTY;
 *                 16-byte aligned for SMAP_LAYOUT_TILES plans and MAP_DUMP (16-B vector
 *                 stores), else aligned to the element (4 B; 8 B for uint64 / THREAD_DUMP).
 *   flags:        SMAP_RUN_* bits.
 * The plan's result block is zeroed on the stream first; results are read with
 * smap_stats_fetch.  SMAP_E_INVALID (nothing launched): payload/m mismatch,
 * missing points/out, points_bytes or out_bytes too small, a misaligned buffer,
 * THREAD_DUMP with TILE granularity.
 * SMAP_E_UNSUPPORTED: ATM / INDEX_WRITE_ATM with TILE rho > 32; ATM / TC /
 * INDEX_WRITE_ATM on an inclusive plan. */
smap_status smap_run(smap_plan_t p, smap_payload pl, const float *points, size_t points_bytes, float param,
                     void *out, size_t out_bytes, uint32_t flags, void *stream);

/* End-to-end variant with a HOST point array: copies host_points (n x 3 fp32,
 * points_bytes >= n * 12; pinned memory recommended) to the plan's device
 * staging buffer on `stream`, runs like smap_run, reduces the result on the
 * device (smap_result_reduce), copies the 56-byte smap_result back to host and
 * synchronises the stream; *stats (required) receives the results.  `out`
 * stays a DEVICE buffer: the packed outputs (8.59 GB for C2) are consumed on
 * the device and are NOT copied to the host -- the host receives the
 * reductions (count, checksums / xor, ATM sum, TC count). */
smap_status smap_run_host(smap_plan_t p, smap_payload pl, const float *host_points, size_t points_bytes,
                          float param, void *out, size_t out_bytes, uint32_t flags, void *stream,
                          smap_stats *stats);

/* Synchronise the stream of the last smap_run and copy its results (a few
 * dozen bytes) into *stats, together with the plan's closed forms. */
smap_status smap_stats_fetch(smap_plan_t p, smap_stats *stats);

/* Device-side result record of one run (56 bytes). */
typedef struct {
    uint64_t count, s0, s1, mix, tc, xr;
    double   sum;
} smap_result;

/* Reduce the last smap_run's per-CTA results into one smap_result at the
 * DEVICE address `dst` (8-byte aligned), asynchronously on `stream` (one small
 * kernel, no host synchronisation) -- the input of a cross-GPU all-reduce:
 * count/s0/s1/mix/tc add exactly mod 2^64, xr combines by xor, sum adds in fp64. */
smap_status smap_result_reduce(smap_plan_t p, void *dst, void *stream);

/* Combine `count` smap_result records at the DEVICE address `records`
 * (contiguous, e.g. the output of an all-gather of every rank's record) into
 * one record at the DEVICE address `dst`, asynchronously on `stream` (one
 * one-warp kernel): count/s0/s1/mix/tc add mod 2^64, xr combines by xor, the
 * fp64 sums add in record order 0..count-1 (deterministic).  Both pointers
 * 8-byte aligned; dst may alias records[0].  SMAP_E_INVALID on NULL pointers,
 * misalignment or count < 1. */
smap_status smap_result_combine(const void *records, int count, void *dst, void *stream);

/* ---- CUDA graphs: one step without host enqueue gaps -------------------------------
 * smap_graph_capture records one step of plan p -- the kernels of smap_run(p, pl, points,
 * ..., flags) followed, when record != NULL, by smap_result_reduce(p, record) -- into a
 * CUDA graph on a private stream and instantiates it (validation and lazily allocated
 * scratch happen first, outside the capture; nothing runs).  smap_graph_launch replays it
 * on `stream` (of the plan's device): the step's 1-4 kernels run back to back with no host
 * work between them, which matters for steps of tens of microseconds (C3, C5).  Buffers
 * (points, out, record) and the plan are bound at capture time: they must outlive the
 * graph and not move.  Results of a replay are read from `record` (a device smap_result,
 * 8-byte aligned); smap_stats_fetch / kernel_ms describe the last smap_run only.  With a
 * record, the graph has no memset node: its last kernel (the record reduction, folded into
 * the ATM finalize for ATM payloads, launched as a programmatic dependent) clears the
 * plan's result block behind the record, and smap_graph_launch clears it first on `stream`
 * when an smap_run left its results there.  A plan's runs and replays must therefore be
 * stream-ordered (they share the result block).  Errors as smap_run; SMAP_E_CUDA if the
 * capture or instantiation fails. */
typedef struct smap_graph_s *smap_graph_t;
smap_status smap_graph_capture(smap_plan_t p, smap_payload pl, const float *points, size_t points_bytes, float param,
                               void *out, size_t out_bytes, uint32_t flags, void *record, smap_graph_t *g);
smap_status smap_graph_launch(smap_graph_t g, void *stream);
/* kernels one replay launches (0 for NULL) */
uint32_t smap_graph_launches(smap_graph_t g);
/* NULL-safe; the plan is not destroyed */
void smap_graph_destroy(smap_graph_t g);

/* Where element e lives (m=2: e = {i, j}, j < i (<= i inclusive); m=3: e = {i, j, k}):
 * *shard = the shard rank that writes it, *pos = its position in that shard's
 * `out` array (SMAP_LAYOUT_ROWS: the packed rank in the full-size array;
 * SMAP_LAYOUT_TILES: the position in the shard-local tile-blocked array).
 * Host only, O(1) (lambda2^-1 via b = 2^floor(log2(I xor J)), q = I >> (log2 b + 1);
 * lambda3^-1 via b = 2^floor(log2(I xor K)), q = I >> (log2 b + 1), inside iff J - I < b),
 * sharded plans included (the owner shard is omega_x / W).  BELOW plans: the E29 layout,
 * piece lookup + closed form.  SMAP_E_INVALID for an element outside the domain. */
smap_status smap_locate(smap_plan_t p, const int64_t *e, int *shard, uint64_t *pos);

/* Useful-element count V of a domain: C(n,2), n(n+1)/2 or C(n,3).  Host only. */
uint64_t smap_volume(int m, int64_t n, int diag);

/* Free the plan's scratch.  NULL-safe. */
void smap_destroy(smap_plan_t p);

/* Message of the last error on the calling thread ("" if none). */
const char *smap_last_error(void);

int smap_abi_version(void);

/* ---- Volume analysis of recursive orthotope sets (host only) ----------
 * The paper's analysis beyond the two maps: a set S_n^m of orthotopes built with scaling
 * factor r and arity beta, V(S_n^m) = (r n)^m + beta V(S_{r n}^m), whose
 * closed form is (n^m - beta^{log_{1/r} n}) / (1/r^m - beta) (Eq. generic-m);
 * r = 1/2, beta = 2 gives lambda2's n(n-1)/2 and lambda3's (n^3 - n)/6, beta = 3 the
 * arity-3 tetrahedral set (n^3 - 3^{log2 n})/5 (reading E8).  Readings E30
 * (r*) and E31 (n0) in DESIGN.md. */

/* V(S_n^m) by the recurrence, V(1) = 0, for r = 1/r_den and n a power of r_den; exact
 * (128-bit intermediates).  SMAP_E_INVALID: m outside [1,16], beta < 1, r_den < 2, n not
 * a power of r_den, or a result >= 2^64. */
smap_status smap_recursive_volume(int m, uint64_t n, int beta, int r_den, uint64_t *vol);

/* The same by the closed form of Eq. generic-m (beta = r_den^m: the degenerate sum
 * k (n/r_den)^m); same errors. */
smap_status smap_recursive_volume_closed(int m, uint64_t n, int beta, int r_den, uint64_t *vol);

/* lim_{n->inf} V(S_n^m) / V(Delta_n^m) - 1 = m! / (1/r^m - beta) - 1;
 * +inf when 1/r^m <= beta (the set grows faster than n^m); NaN for r outside (0,1). */
double smap_alpha_limit(int m, double r, int beta);

/* r* = (m! + beta)^{-1/m}: the scaling meeting the constraint 1/r^m - beta = m! (
 * the printed r = 1/(m^{-1/m}) is > 1, reading E30). */
double smap_r_star(int m, int beta);

/* n0 (reading E31): the smallest n in [2, n_max] such that the continuous
 * V(S_{n'}^m) >= V(Delta^m_{n'-1}) = C(n'+m-2, m) for every n' in [n, n_max]; *n0 = 0 when
 * the set does not cover at n_max.  *ratio_at_nmax (optional) = V(S)/V(Delta_{n-1}) there.
 * SMAP_E_INVALID: bad m / r / beta, n_max outside [2, 2^24]. */
smap_status smap_find_n0(int m, double r, int beta, uint64_t n_max, uint64_t *n0, double *ratio_at_nmax);

/* The paper's open optimisation for one beta: the smallest r -- i.e. the least
 * extra volume m!/(1/r^m - beta) - 1 -- whose set covers Delta^m_{n-1} for every n in
 * [n0, n_max] (continuous model, bisection between r* and the r of 1/r^m - beta = 1).
 * SMAP_E_UNSUPPORTED if even 1/r^m - beta = 1 does not cover; n_max <= 2^20. */
smap_status smap_r_cover(int m, int beta, uint64_t n0, uint64_t n_max, double *r);

/* MAP_DUMP record per grid block (THREAD) or tile (TILE), in launch order:
 *   int32 {x0, x1, x2, cls}
 * m=2 lambda: cls 0 off-diagonal block (x0,x1) = (J,I) = lambda2(w);
 *             cls 1 strict row-0 diagonal pair (x0,x1) = (D1,D2) = (wx, N-1-wx);
 *             cls 2 inclusive diagonal block x0 = D (row 0: wx, row N: wx + N/2).
 * m=2 BB:     (x0,x1) = (J,I) = (wx,wy); cls 0 J<I, 3 J==I, 4 J>I (filtered out).
 * m=3 lambda: (x0,x1,x2) = (I,J,K) sorted block triple; cls 0 inside branch,
 *             1 reflected branch; cls 2 body-diagonal block x0 = d; cls 3 idle.
 * m=3 BB:     (I,J,K) = (wx,wy,wz); cls 0 I<J<K, 5 I=J<K, 6 I<J=K, 2 I=J=K, 4 outside.
 * ENUM:       as BB (m=2 (J,I) cls 0/3; m=3 (I,J,K) cls 0/5/6/2), never outside.
 *
 * Launch order (block-linear id bid; W = N/(2G) columns per shard, wx0 = rank*W):
 *   lambda2, SMAP_ORDER_ROWS: bid = wy*W + (wx - wx0), wy in [0, N) strict / [0, N] inclusive
 *   lambda2, SMAP_ORDER_SQUARES: rows 0 and N as above; for row = bid/W in [b, 2b),
 *            t = bid - b*W; if b <= W: square s = t / b^2, r = t mod b^2,
 *            wy = b + r / b, wx = wx0 + s*b + r mod b; else wy = b + t / W, wx = wx0 + t mod W
 *   lambda3: bid = (wz*(N/2) + wy)*W + (wx - wx0), wz in [0, 3N/4)
 *   BB2:     bid = I*N + J;   BB3: bid = (K*N + J)*N + I
 *   ENUM2:   bid = I(I+1)/2 + J, J <= I;   ENUM3: bid = C(K+2,3) + C(J+1,2) + I, I <= J <= K
 *   BELOW:   pieces in order (m=2: for s = 0, 1, ...: triangle of S_s, then the rectangles
 *            S_a x S_s, a < s; m=3: segment triples a <= b <= c, c outer, then b, then a);
 *            inside a piece the lower-ranked coordinates vary fastest (rectangle: J, then I;
 *            a < b = c: the line I, then the lambda2 inclusive grid id in row order;
 *            a = b < c: the grid id, then K; box: I, J, K).  Records: m=2
 *            {J, I, 0, cls} with cls 0 off-diagonal, 2 diagonal tile; m=3 {I, J, K, cls}
 *            with cls 0/1/2/3 as lambda3 inside lambda3 pieces, else 0 interior,
 *            5 I=J<K, 6 I<J=K, 2 I=J=K.
 * Threads (THREAD_DUMP order): t = ty*rho + tx (m=2); t = (c*rho + b)*rho + a (m=3). */

#ifdef __cplusplus
}
#endif

#endif /* SMAP_H */
