/*
 * aidw.h -- C ABI of the B200 AIDW hot path (arXiv 1511.02186, "GPU-accelerated
 * Adaptive IDW").  Implemented by paper_1511_02186_b200/libaidw.so (sm_100a).
 *
 * The path:
 *   aidw_create       S0  repack data to internal SoA, bbox area A, r_exp (Eq. 2)
 *   aidw_knn_robs     S1-S2  brute-force kNN per query (§3.1.2), r_obs (Eq. 3),
 *                          nearest squared distance, local {-min, max} of r_obs
 *   (caller)          S3  GLOBAL mode: allreduce(MAX) of {-min, max} across ranks
 *   aidw_alpha        S4  R (Eq. 4), mu_R (Eq. 5), alpha (Eq. 6)
 *   aidw_interpolate  S5  Shepard weighted average over ALL data points (Eq. 1)
 *   aidw_destroy
 *
 * Conventions (all entry points):
 *  - Every pointer argument documented "device" must be device memory of the
 *    handle's device (e.g. a torch CUDA tensor's data_ptr()).  The caller owns it
 *    and keeps it alive until `stream` has passed the call.
 *  - "T" below is the handle's dtype: float for AIDW_F32, double for AIDW_F64
 *    (the paper's REAL).  Arrays are dense, 1-D, contiguous.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *    asynchronous on it, except aidw_create, aidw_check and aidw_run_host, which
 *    synchronise it.
 *  - Argument errors are returned synchronously and nothing is enqueued.
 *    Per-query data errors (non-finite query coordinates) set a device flag
 *    holding the smallest failing query index; aidw_check() reports it
 *    (batch all-or-nothing).
 *  - No exceptions cross the ABI.  A handle is not thread-safe: use one handle
 *    per (device, stream) at a time.
 *  - nq == 0 is a successful no-op.  k must be in [1, 32], nd >= k.
 *  - Launch shape never changes a result: the kNN outputs are exact, and Z is
 *    bit-identical for any in-GPU split of the data range, query order or GPU count
 *    of the query-sharded path
 *    (DESIGN.md §4.6-4.7, §5).  The handle owns growable device scratch for the
 *    small-nq data split and the spatial query order (allocated on first use).  Handle
 *    memory comes from the device's stream-ordered pool (cudaMallocAsync, kept on
 *    destroy), so destroying and creating handles reuses it.
 *  - Tuning/testing environment variables (defaults are the measured best):
 *    AIDW_SPLIT=0|n (data split off / forced factor), AIDW_KNN_ORDER=0 (no
 *    spatial query order), AIDW_KNN_H16=0|1|2|3 (fp16 kNN pre-filter off / default /
 *    Q = 4 / register-capped shapes), AIDW_KNN_STRIP=0 (fp16 kernels without the strip
 *    pre-test), AIDW_KNN_PIPE=0 (fp16 tiles behind a CTA barrier instead of the
 *    mbarrier pipeline), AIDW_KNN_QSEED=0 (home-tile seeds instead of per-query seeds) and
 *    AIDW_EXP2_CLAMP=1 (always-clamped polynomial exp2) are read per call -- none
 *    changes a result; AIDW_ALPHA_CLASSES=0 (no
 *    exact-exponent weighting classes) and AIDW_KNN_VARIANT / AIDW_INTERP_VARIANT
 *    (tuning sweeps) once per process; AIDW_KNN_FILTER=0 (canonical kNN, no fp32
 *    filter, for either dtype) at aidw_create.  Spatially ordered kNN batches
 *    (>= 32768 queries) split the data range only with seeded lists (DESIGN.md
 *    §4.6); AIDW_SPLIT=n forces that factor (at most 8) too.
 */
#ifndef AIDW_H
#define AIDW_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define AIDW_API __attribute__((visibility("default")))
#else
#define AIDW_API
#endif

#define AIDW_ABI_VERSION 1
#define AIDW_KMAX 32

typedef struct aidw_ctx *aidw_t;

typedef enum {
    AIDW_OK = 0,
    AIDW_E_INVALID_ARG = 1,        /* null/negative/misaligned argument, bad enum, bad levels */
    AIDW_E_INSUFFICIENT_DATA = 2,  /* nd < k */
    AIDW_E_DEGENERATE_EXTENT = 3,  /* bbox area A == 0 */
    AIDW_E_INVALID_AREA = 4,       /* explicit area < 0 or non-finite */
    AIDW_E_INVALID_BOUNDS = 5,     /* FIXED r_min >= r_max */
    AIDW_E_NONFINITE_INPUT = 6,    /* NaN/Inf in data or query coordinates */
    AIDW_E_UNSUPPORTED = 7,        /* k > AIDW_KMAX, unknown dtype/layout */
    AIDW_E_CUDA = 8,               /* a CUDA runtime error (message in aidw_last_error) */
    AIDW_E_NOMEM = 9
} aidw_status;

/* REAL = float | double. */
typedef enum { AIDW_F32 = 0, AIDW_F64 = 1 } aidw_dtype;

/* Input layouts accepted at the boundary (Fig. 2).  Internally
 * the data is always repacked to SoA.
 *   SOA : x[nd], y[nd], z[nd] back to back
 *   AOS : (x, y, z) records, 3*nd values
 *   AOAS: (x, y, z, pad) records, 4*nd values (Array of aligned Structures) */
typedef enum { AIDW_SOA = 0, AIDW_AOS = 1, AIDW_AOAS = 2 } aidw_layout;

/* Source of R_min / R_max in Eq. 5 (reading R7).
 *   GLOBAL: min / max of R over all queries of the job (north star; across ranks
 *           after an allreduce(MAX) of {-min r_obs, max r_obs})
 *   FIXED : caller-given bounds; the paper's default is 0.0 / 2.0 */
typedef enum { AIDW_RB_GLOBAL = 0, AIDW_RB_FIXED = 1 } aidw_rbounds;

/* Argument of the cosine in Eq. 5 (reading R8).
 *   NORMALIZED: pi (R - Rmin) / (Rmax - Rmin)      (default; mu(Rmax) = 1)
 *   PRINTED   : pi / Rmax * (R - Rmin)             (as typeset) */
typedef enum { AIDW_MU_NORMALIZED = 0, AIDW_MU_PRINTED = 1 } aidw_muform;

AIDW_API int aidw_abi_version(void);
AIDW_API const char *aidw_status_string(aidw_status s);

/* Last error message of handle h (or of the calling thread's last failed
 * aidw_create when h == NULL).  Valid until the next call on that handle. */
AIDW_API const char *aidw_last_error(aidw_t h);

/*
 * aidw_create -- S0.  Copy the nd data points (x_i, y_i, z_i) -- the paper's
 * dx, dy, dz; z is the VALUE, geometry is 2-D -- into a
 * handle-owned SoA layout padded to the tile multiple, compute the study area
 * A and r_exp = 1 / (2 sqrt(nd / A)) (Eq. 2) in fp64.
 *   out      : receives the handle
 *   device   : CUDA device ordinal
 *   dt, lay  : dtype of data_xyz and its layout (see aidw_layout)
 *   data_xyz : device OR host pointer to the data in layout `lay`, dtype `dt`;
 *              may be freed once aidw_create returns
 *   nd       : number of data points, >= 1
 *   area     : > 0 explicit A; == 0 -> A = area of the data's axis-aligned bbox
 *              (R5); < 0 or non-finite -> AIDW_E_INVALID_AREA
 * Synchronises `stream` once (A == 0 must be reported synchronously:
 * AIDW_E_DEGENERATE_EXTENT).  Non-finite data -> AIDW_E_NONFINITE_INPUT.
 */
AIDW_API aidw_status aidw_create(aidw_t *out, int device, aidw_dtype dt, aidw_layout lay,
                        const void *data_xyz, int64_t nd, double area, void *stream);

/* Properties of a handle (host values). */
AIDW_API int64_t aidw_nd(aidw_t h);
AIDW_API double aidw_area(aidw_t h);
AIDW_API double aidw_r_exp(aidw_t h);
AIDW_API aidw_dtype aidw_dtype_of(aidw_t h);

/*
 * aidw_knn_robs -- S1 + S2.  For each query S0 = (qx[q], qy[q]), the k smallest
 * distances to ALL nd data points (brute force, §3.1.2 Steps 1-3,
 * PAPER.md:317-340; strict "<" as in Step 3) and r_obs = (1/k) sum_i d_i
 * (Eq. 3), summed in ascending order.
 * Distance arithmetic (R16), in T with round-to-nearest:
 *   dx = qx - px; dy = qy - py; s = fma(dx, dx, dy*dy); selection on s; d = sqrt(s).
 * (Both dtypes skip most pairs' canonical evaluation through an fp32 expanded-form
 * filter with a rigorous rounding margin; every pair that could enter the top-k is
 * re-evaluated with the sequence above, so the selected multiset is exactly the
 * unfiltered one -- DESIGN.md §4.1.)
 *   qx, qy      : device T[nq]
 *   k           : 1..AIDW_KMAX, nd >= k (else AIDW_E_INSUFFICIENT_DATA)
 *   r_obs       : device T[nq] out
 *   d1sq        : device T[nq] out, nullable: s of the nearest data point (used by
 *                 aidw_interpolate to scale weights and detect coincidence)
 *   robs_minmax : device T[2] out, nullable: {-min_q r_obs, max_q r_obs} over these
 *                 nq queries, ready for an allreduce(MAX); nq == 0 writes {-inf, -inf}
 *   knn_dists   : device T[nq*k] out, nullable: the k distances per query, ascending
 *                 (verification output of the same kernel)
 */
AIDW_API aidw_status aidw_knn_robs(aidw_t h, const void *qx, const void *qy, int64_t nq, int k,
                          void *r_obs, void *d1sq, void *robs_minmax, void *knn_dists,
                          void *stream);

/*
 * aidw_alpha -- S4.  Per query, in fp64: R = r_obs / r_exp (Eq. 4);
 * mu_R by Eq. 5 (`mf` selects the cosine argument; intervals
 * resolve first-match in printed order, R_max == R_min gives mu = 0); alpha by
 * Eq. 6 (first match in printed order).  alpha is rounded to T.
 *   r_obs       : device T[nq] (from aidw_knn_robs)
 *   alpha_lv    : HOST double[5], alpha_1..alpha_5, finite and > 0
 *   rb          : GLOBAL -> bounds from robs_minmax (device T[2] = {-min r_obs, max r_obs},
 *                 divided by r_exp); FIXED -> r_min < r_max (else AIDW_E_INVALID_BOUNDS)
 *   alpha       : device T[nq] out
 */
AIDW_API aidw_status aidw_alpha(aidw_t h, const void *r_obs, int64_t nq, const double *alpha_lv,
                       aidw_rbounds rb, double r_min, double r_max,
                       const void *robs_minmax, aidw_muform mf, void *alpha, void *stream);

/*
 * aidw_interpolate -- S5.  Z(S0) = sum_i w_i z_i / sum_i w_i over ALL nd data points,
 * w_i = d_i^-alpha (Eq. 1; all points).
 * Evaluated as w_i = 2^(-alpha/2 * log2(s_i / d1sq)) (scaled by the nearest
 * distance, which cancels in Eq. 1).  fp32: MUFU lg2/ex2, sums in fp32 within
 * 512-point tiles and fp64 across tiles; fp64: table + Taylor log2/exp2 (relative
 * error < 1e-15), fp64 sums.
 * Exact coincidence (d1sq == 0): Z = mean of z over the data points at distance 0
 * (R19).
 *   qx, qy : device T[nq];  alpha : device T[nq] (from aidw_alpha)
 *   d1sq   : device T[nq] from aidw_knn_robs, or NULL: computed internally (k = 1 pass)
 *   z_out  : device T[nq] out
 */
AIDW_API aidw_status aidw_interpolate(aidw_t h, const void *qx, const void *qy, int64_t nq,
                             const void *alpha, const void *d1sq, void *z_out, void *stream);

/*
 * aidw_run_fixed -- N1: S1..S5 with FIXED bounds in ONE launch -- the
 * paper's per-thread structure (kNN -> r_obs -> R -> mu -> alpha -> Eq. 1 in one kernel,
 * PAPER.md:407-438).  With caller-given R_min < R_max (paper default 0.0 / 2.0,
 * PAPER.md:221-223) no phase barrier is needed.  fp32 handles run one fused kernel; fp64
 * handles run the three stage kernels.  Results equal aidw_knn_robs + aidw_alpha(FIXED)
 * + aidw_interpolate.
 *   qx, qy     : device T[nq];  z_out : device T[nq] out
 *   r_obs_out, alpha_out : device T[nq] out, nullable (diagnostics)
 */
AIDW_API aidw_status aidw_run_fixed(aidw_t h, const void *qx, const void *qy, int64_t nq, int k,
                                    const double *alpha_lv, double r_min, double r_max, aidw_muform mf,
                                    void *z_out, void *r_obs_out, void *alpha_out, void *stream);

/*
 * aidw_idw -- N2: standard IDW (Eq. 1 with a user-specified constant power alpha for all
 * queries) on the same weighting kernel: one k = 1 pass for the
 * nearest distance (weight scaling, coincidence), then the weighting pass.
 *   alpha : finite, > 0;  qx, qy : device T[nq];  z_out : device T[nq] out
 */
AIDW_API aidw_status aidw_idw(aidw_t h, const void *qx, const void *qy, int64_t nq, double alpha,
                              void *z_out, void *stream);

/*
 * aidw_paper_baseline -- N3 (Table-1-shaped ablation): the paper's OWN
 * kernel designs recompiled for sm_100a, as the prior-art baseline the product kernels
 * are measured against (NOT the product path):
 *   variant 0 = naive (§3.2.1: registers + global memory only),
 *   variant 1 = tiled (§3.2.2: shared-memory tile = block size).
 * One thread per query: kNN buffer pass (Fig. 1), r_obs, R, mu, alpha in the thread with
 * FIXED bounds [r_min, r_max], then Eq. 1 with pow() and REAL accumulators.
 *   dt, lay : T and the data layout: AIDW_SOA (x[nd], y[nd], z[nd]) or AIDW_AOAS
 *   data    : device, in layout `lay`;  qx, qy : device T[nq];  z_out : device T[nq]
 *   area    : study area A > 0 (Eq. 2);  k : 1..AIDW_KMAX
 */
AIDW_API aidw_status aidw_paper_baseline(int variant, aidw_dtype dt, aidw_layout lay, const void *data,
                                         int64_t nd, const void *qx, const void *qy, int64_t nq, int k,
                                         const double *alpha_lv, double area, double r_min, double r_max,
                                         void *z_out, void *stream);

/*
 * N4 -- data-sharded mode: the DATA points are split across handles /
 * ranks (shard boundaries at multiples of 1024 points keep the fp32 tile sums identical),
 * every rank evaluates ALL queries against its shard, and the per-shard results are
 * combined exactly (kNN) or in a fixed rank order (Eq. 1 sums).  Sequence per rank:
 *   aidw_set_extent_bbox(h, nd_total, bbox) r_exp of the WHOLE data set (Eq. 2) from
 *                                           the job-wide bbox (MAX-allreduced aidw_bbox)
 *   aidw_knn_partial -> allgather lists    -> aidw_knn_merge (r_obs, d1sq, {-min, max})
 *   aidw_alpha (GLOBAL: the merged bounds already cover all queries)
 *   aidw_interpolate_partial -> allgather partials -> aidw_finalize (Z)
 * The merged k-lists, r_obs, d1sq and alpha are bit-identical to a single-device run.
 */
/* Set the data-set size and study area used for r_exp (Eq. 2); area > 0, nd_total >= 1. */
AIDW_API aidw_status aidw_set_extent(aidw_t h, int64_t nd_total, double area);

/* Bounding box of the handle's data: out[4] = {min x, max x, min y, max y} (host). */
AIDW_API aidw_status aidw_bbox(aidw_t h, double *out);

/* Eq. 2 for a data set split across handles: A = (x1 - x0)(y1 - y0)
 * from the JOB-WIDE bbox[4] = {min x, max x, min y, max y} (host; the MAX-allreduce of
 * every shard's {-min x, max x, -min y, max y}, R5), in fp64 exactly as
 * aidw_create computes it for one handle, then r_exp = 1/(2 sqrt(nd_total / A)).
 * AIDW_E_DEGENERATE_EXTENT if A == 0, AIDW_E_INVALID_AREA if non-finite. */
AIDW_API aidw_status aidw_set_extent_bbox(aidw_t h, int64_t nd_total, const double *bbox);

/* The k smallest SQUARED distances (ascending) of each query to this handle's data:
 * s_out device T[nq*k].  Same kernel and arithmetic as aidw_knn_robs (R16). */
AIDW_API aidw_status aidw_knn_partial(aidw_t h, const void *qx, const void *qy, int64_t nq, int k,
                                      void *s_out, void *stream);

/* Merge P partial lists (device T[P][nq][k], each ascending) into the k smallest, then
 * r_obs / d1sq / robs_minmax exactly as aidw_knn_robs (any of the three nullable). */
AIDW_API aidw_status aidw_knn_merge(aidw_t h, const void *lists, int P, int64_t nq, int k, void *r_obs,
                                    void *d1sq, void *robs_minmax, void *stream);

/* Eq. 1 partial sums over this handle's data: partial_out device double[nq][4] =
 * {sum w, sum w z, sum z (coincident points), count (coincident points)}; d1sq is the
 * merged (global) nearest squared distance. */
AIDW_API aidw_status aidw_interpolate_partial(aidw_t h, const void *qx, const void *qy, int64_t nq,
                                              const void *alpha, const void *d1sq, double *partial_out,
                                              void *stream);

/* Z from P partials (device double[P][nq][4]) summed in rank order: z_out device T[nq]. */
AIDW_API aidw_status aidw_finalize(aidw_t h, const double *partials, int P, int64_t nq, void *z_out,
                                   void *stream);

/*
 * Device-side GLOBAL-bounds exchange (SURVEY.md §8(f) N4 "device-initiated fused min/max
 * push").  Replaces the host-issued allreduce(MAX) of {-min, max} r_obs
 * between aidw_knn_robs and aidw_alpha (the north star's global R
 * bounds) by peer-memory stores: once connected, the LAST CTA of each kNN launch writes
 * its {-min, max} into every rank's exchange buffer over NVLink (CUDA IPC mappings,
 * system-scope release), and aidw_alpha(GLOBAL, robs_minmax = NULL) waits on the
 * device for all ranks of the same step (acquire loads), then takes the MAX.  Bounds
 * are bit-identical to the allreduce (MAX is exact).  Values of step e go to slot e mod 2
 * and each rank acks a step once its alpha launch has read it; a rank publishes step e
 * only after every rank acked step e - 2, so ranks may drift by one step without a
 * slower rank ever reading a newer step's bounds.  Every rank must call aidw_knn_robs
 * (with robs_minmax != NULL; nq == 0 pushes the MAX identity) and aidw_alpha in step;
 * a wait gives up after ~2 s: alpha (hence Z) of that step is NaN and aidw_check
 * returns AIDW_E_CUDA.  One process per GPU;
 * processes sharing a GPU also work (tests).  Not for aidw_run_host.
 *   aidw_exchange_setup  : allocate this rank's buffer; ipc_handle_out receives 64 bytes
 *                          (a cudaIpcMemHandle_t) to all-gather across ranks
 *   aidw_exchange_connect: ipc_handles = world x 64 bytes in rank order; maps the peers
 *   aidw_exchange_close  : unmap and free (also done by aidw_destroy)
 */
AIDW_API aidw_status aidw_exchange_setup(aidw_t h, int rank, int world, void *ipc_handle_out);
AIDW_API aidw_status aidw_exchange_connect(aidw_t h, const void *ipc_handles);
AIDW_API aidw_status aidw_exchange_close(aidw_t h);

/*
 * aidw_run_host -- the whole single-GPU path from HOST buffers: H2D of the
 * queries, knn_robs, (GLOBAL: local bounds = the job's bounds), alpha,
 * interpolate, D2H of Z; synchronises `stream` and reports deferred errors.
 *   qx_host, qy_host : host T[nq] (pinned memory gives asynchronous copies)
 *   z_host           : host T[nq] out
 * Other arguments as in aidw_knn_robs / aidw_alpha.  Device scratch is owned by
 * the handle and reused across calls.
 */
AIDW_API aidw_status aidw_run_host(aidw_t h, const void *qx_host, const void *qy_host, int64_t nq,
                          int k, const double *alpha_lv, aidw_rbounds rb, double r_min,
                          double r_max, aidw_muform mf, void *z_host, void *stream);

/* Synchronise `stream`, then report (and clear) deferred per-query errors:
 * AIDW_E_NONFINITE_INPUT with the first failing query index in aidw_last_error. */
AIDW_API aidw_status aidw_check(aidw_t h, void *stream);

/* Number of kernels the handle has launched since creation (launch accounting). */
AIDW_API int64_t aidw_launch_count(aidw_t h);

AIDW_API aidw_status aidw_destroy(aidw_t h);

#ifdef __cplusplus
}
#endif

#endif /* AIDW_H */
