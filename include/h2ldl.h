/*
 * h2ldl.h — C ABI of libh2ldl.so, the B200 (sm_100a) generalized-LDL^T
 * inertia engine for rank-structured (BLR2 / HSS / H2) symmetric matrices.
 *
 * This is the drop-in boundary for the reference's hot path:
 *
 *   h2l_inertia       replaces  gldl.generalized_ldl / gldl.inertia
 *                               (/root/reference/pkg/src/h2slice/gldl.py:605-633)
 *                               for s shifts at once; the Python shims in
 *                               paper_2311_08618_b200/ldl.py keep the retry
 *                               loop (gldl.py:615-633) and exceptions.
 *   h2l_upload        replaces  the per-origin skeleton caches
 *                               RankStructuredMatrix.skeleton_diag/_offdiag
 *                               (compress.py:99-127): the payload is uploaded
 *                               once and Q^T A Q is formed on the device.
 *   h2l_bk_factor     replaces  the native operator plug-in
 *                               _core.bk_factor (_core/_kernels.pyx:21-125),
 *                               bit-identical packed output and ipiv.
 *   h2l_bk_inertia    replaces  _core.bk_inertia (_kernels.pyx:128-168).
 *
 * Conventions
 *  - Every function returns H2L_OK (0) or a negative H2L_E* code; the last
 *    message is available from h2l_last_error(engine) (engine may be NULL for
 *    the engine-less entry points).
 *  - All matrices are row-major (C order) float64; host buffers are owned by
 *    the caller, device memory by the engine.  Calls are synchronous.
 *  - An engine is bound to one CUDA device and one stream; calls on one engine
 *    are not re-entrant.  Distinct engines may be driven from distinct host
 *    threads.
 *  - No C++ exception crosses this boundary; no CPU fallback exists: without
 *    a usable sm_100 device every compute entry point returns H2L_ENODEV.
 */
#ifndef H2LDL_H
#define H2LDL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    H2L_OK = 0,
    H2L_EINVAL = -1,   /* bad argument / inconsistent plan */
    H2L_ENODEV = -2,   /* no CUDA device / not sm_100 */
    H2L_ECUDA = -3,    /* CUDA runtime error */
    H2L_ENOMEM = -4,   /* device allocation failed */
    H2L_ESTATE = -5    /* call order violated (e.g. inertia before upload) */
};

/* per-shift status written by h2l_inertia */
enum {
    H2L_SHIFT_OK = 0,          /* factored; counts valid (zero count may be > 0) */
    H2L_SHIFT_SINGULAR = 1     /* a BK pivot block was singular (reference: ShiftHitEigenvalue) */
};

/* structure kinds: reference BlockStructure.kind (partition.py:122-157) */
enum { H2L_STRONG = 0, H2L_WEAK = 1, H2L_FLAT = 2 };

typedef struct h2l_engine h2l_engine;

/*
 * Static schedule + payload of one unshifted RankStructuredMatrix
 * (compress.py:24-56).  Clusters are numbered level-major: node id of
 * (level, i) is (1 << level) - 1 + i.  Offsets index `arena` (doubles).
 */
typedef struct h2l_plan {
    int32_t n;            /* matrix order */
    int32_t depth;        /* tree depth; leaves at level `depth` */
    int32_t kind;         /* H2L_STRONG / H2L_WEAK / H2L_FLAT */
    int32_t n_dense;      /* inadmissible leaf pairs (i < j) */
    int32_t n_lowrank;    /* classified low-rank pairs, all levels */
    int32_t n_deferred;   /* deferred non-leaf pairs, all levels */
    double eps;           /* construction tolerance; drop_tol = eps*(scale0+|mu|) */
    double scale0;        /* max |entry| of the leaf diagonal blocks (compress.py:71-82) */
    const int64_t *ranges;      /* [nodes][2]: index range [start, stop) */
    const int32_t *dense;       /* [n_dense][2] leaf cluster pairs */
    const int32_t *lowrank;     /* [n_lowrank][3] (level, i, j) */
    const int32_t *deferred;    /* [n_deferred][3] (level, i, j) */
    const int32_t *basis_rank;  /* [nodes] skeleton rank, -1 when the node has no basis */
    const int32_t *basis_dim;   /* [nodes] rows of the square basis [U_R | U_S] */
    const int64_t *basis_off;   /* [nodes] arena offset of [U_R | U_S] (dim x dim), -1 none */
    const int64_t *diag_off;    /* [leaves] arena offset of leaf_diag[i] (m_i x m_i) */
    const int64_t *dense_off;   /* [n_dense] arena offset of leaf_offdiag (m_i x m_j) */
    const int64_t *lowrank_off; /* [n_lowrank] arena offset of the coupling (r_i x r_j) */
    const double *arena;        /* all float64 payload */
    int64_t arena_len;          /* doubles in arena */
} h2l_plan;

/* structural statistics of the last h2l_inertia call (gldl.py:189-195) */
typedef struct h2l_stats {
    int64_t fill_blocks;
    int64_t recompressions;
    int64_t rank_added;
    int64_t max_front;
    double dropped_fro;   /* summed over shifts */
    double flops;         /* algorithmic fp64 flops of the call (all shifts, survey §8d) */
    double bytes;         /* algorithmic HBM bytes of the Schur updates (targets r+w, X/W reads) */
    double ms_total;      /* device time of the call (CUDA events) */
    double ms_schur;      /* device time inside the Schur-update GEMM launches */
    double ms_bk;         /* device time inside the BK launches */
    int64_t launches;     /* kernels launched by the call */
    double schur_flops;   /* algorithmic flops of the Schur updates (survey §8d formula) */
    double gemm_flops_exec; /* flops executed by all DMMA GEMM launches (2MNK) */
    double ms_kind[8];    /* device ms per launch kind (time_kernels=1): 0 panel GEMMs,
                             1 Schur GEMM, 2 rotation/merge GEMMs, 3 BK, 4 panel solve,
                             5 copies, 6 recompression Gram / energy products and tail
                             rank, 7 recompression ordering (pivoted QR, Q^T) */
    double ms_host;       /* wall-clock ms of the call on the host */
    double mem_peak;      /* bytes: high-water mark of the waves' device pools during the call */
    double elim_flops;    /* the elimination part of `flops` (BK + panel + Schur, live rows) */
    int64_t groups;       /* elimination groups (clusters eliminated together, one launch per
                             kernel kind) summed over levels and waves */
    int64_t paths[4];     /* cluster-steps through the large-front kernels: 0 BK in a
                             thread-block cluster (n_R > 224), 1 panel with L staged in
                             chunks (n_R > 160), 2 Gram ordering on a 16-CTA cluster,
                             3 Gram ordering beyond distributed shared memory (one CTA) */
} h2l_stats;

int h2l_create(h2l_engine **engine, int device);
int h2l_destroy(h2l_engine *engine);
const char *h2l_last_error(const h2l_engine *engine);

/* Upload the payload and build the shift-independent skeleton blocks. */
int h2l_upload(h2l_engine *engine, const h2l_plan *plan);

/*
 * Inertia of (A - mu[z] I) for z < s, all shifts in one batched sweep.
 * counts: [s][3] (neg, zero, pos); status: [s] H2L_SHIFT_*.
 * stats may be NULL.
 */
int h2l_inertia(h2l_engine *engine, const double *mu, int32_t s, int64_t *counts,
                int32_t *status, h2l_stats *stats);

/*
 * Same as h2l_inertia, but the result stays on the device: dev_counts is device
 * memory on the engine's device, [s][4] int64 rows (neg, zero, pos, status).
 * The multi-GPU drivers all-gather straight from this buffer (no host staging).
 */
int h2l_inertia_device(h2l_engine *engine, const double *mu, int32_t s, int64_t *dev_counts,
                       h2l_stats *stats);

/*
 * Multi-GPU in one process: one engine per device, each with
 * the same payload uploaded; a call shards the shifts over the engines in
 * contiguous slices (reference parallel.py:85-96), every engine factorizes its
 * slice on its own host thread, and the packed counts are exchanged by one NCCL
 * all-gather between the engines' device buffers (NCCL is dlopen'ed at
 * h2l_comm_init).  Counts are identical to h2l_inertia on any one engine.
 * stats (nullable): summed work, ms_total = max over the engines.
 */
typedef struct h2l_comm h2l_comm;
int h2l_comm_init(h2l_engine *const *engines, int ngpu, h2l_comm **comm);
int h2l_inertia_multi(h2l_comm *comm, const double *mu, int32_t s_total, int64_t *counts,
                      int32_t *status, h2l_stats *stats);
int h2l_comm_destroy(h2l_comm *comm);

/*
 * Tuning knobs (key, value):
 *  "max_batch"    shifts per device wave (default 64);
 *  "concurrency"  waves in flight on private streams (default 2);
 *  "time_kernels" 0 off, 1 CUDA-event timing of every launch kind (stats.ms_kind),
 *                 2 the Schur GEMM launches only (stats.ms_schur; negligible overhead);
 *  "borrow_arena" 1: a device-resident plan arena is used in place by h2l_upload
 *                 instead of being copied (it must then outlive the engine);
 *  "schedule"     0 one cluster at a time in the reference's ascending order;
 *                 1 (default) wavefronts of the ascending order's dependency DAG:
 *                 clusters whose eliminations touch disjoint blocks go out in one
 *                 launch per kernel kind, each shift factors what the ascending
 *                 sweep factors (up to the rounding of the complement basis under
 *                 "qr_budget");
 *                 2 colour classes of a greedy distance-2 colouring: a re-ordered
 *                 elimination with far fewer groups.  The factored matrix differs
 *                 from the ascending sweep's at the truncation tolerance (fills and
 *                 recompression ranks depend on the order), so counts agree with
 *                 the reference for shifts outside the tolerance band (tested on
 *                 the golden and production-size instances), not by construction;
 *                 3 colour classes of consecutive windows of "window" clusters
 *                 (default 64) of the order: batches like 2 while the eliminated
 *                 clusters stay a moving front (materialised blocks and fills stay
 *                 local, as in the ascending sweep); same caveat as 2;
 *  "group_mem_mb" cap on the temporaries of one group (default 8192);
 *  "group_max"    cap on the clusters of one group (default 512);
 *  "elim_order"   0 ascending (the reference), 1 low near-field degree first
 *                 (smaller fronts; a re-ordering with the same caveat as schedule 2);
 *  "qr_budget"    1 (default) order only ~1.5x the level's largest recompression
 *                 rank (+32) pivots, redone with all pivots when the rank reaches
 *                 the budget (same rank as the full ordering; the dropped
 *                 complement gets a different orthonormal basis), 0 full ordering;
 *  "block_cache"  how working blocks are allocated: 2 (default) from a host-side arena
 *                 (large slabs of the wave's pool, best-fit free list with coalescing),
 *                 1 from free lists of retired blocks per size class ("block_classes" 1:
 *                 8 classes per octave, 0: exact sizes; "block_cache_mb": cap, default
 *                 2048), 0 one stream-ordered pool call per block;
 *  "schur_arith"  arithmetic of the Schur update (the dominant kernel): 0 fp64 on the
 *                 DMMA pipe (mma.sync), 1 (default) fp64-accurate on the INT8 tensor cores
 *                 (tcgen05.mma.kind::i8): each row of X / Bg split into 8 exact
 *                 7-bit slices under a power-of-two row scale, the 36 slice-pair
 *                 products of weight >= 2^-63 summed exactly in int32 tensor memory,
 *                 the 8 group totals combined in fp64 (k_schur_oz.cu).
 * Unknown keys fail with H2L_EINVAL.
 */
int h2l_set_option(h2l_engine *engine, const char *key, int64_t value);

/*
 * Batched Bunch-Kaufman LDL^T on the device, the reference kernel's contract
 * (_kernels.pyx:21-125): `count` n x n row-major matrices in `a` (host,
 * overwritten with the packed factor, lower triangle), ipiv [count][n],
 * tol [count], info [count] (0 or k+1).  Bit-identical to the reference.
 */
int h2l_bk_factor(int device, double *a, int64_t n, int32_t count, int64_t *ipiv,
                  const double *tol, int64_t *info);

/* (neg, zero, pos) of packed BK factors, _kernels.pyx:128-168; counts [count][3]. */
int h2l_bk_inertia(int device, const double *a, int64_t n, int32_t count, const int64_t *ipiv,
                   const double *zero_tol, int64_t *counts);

/* Library version string, e.g. "h2ldl 0.1 sm_100a". */
const char *h2l_version(void);

#ifdef __cplusplus
}
#endif

#endif /* H2LDL_H */
