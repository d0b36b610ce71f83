// knn_robs.cu -- S1 + S2 of the AIDW hot path on sm_100a.
//
// Per query: the k smallest squared distances to ALL data points (brute force,
// PAPER.md:317-340, §3.1.2 Steps 1-3 -- "if dist < the kth distance, then replace
// the kth distance", strict <), then r_obs = (1/k) sum d_i (Eq. 3),
// the nearest squared distance d1sq, and the {-min, max} of r_obs over the launch.
//
// B200 design -- the paper's "tiled" idea,
// rebuilt for sm_100a:
//  * data tiles stream through a shared-memory ring filled by the TMA engine
//    (cp.async.bulk, one elected thread, mbarrier complete_tx), decoupled from the
//    block size;
//  * every thread owns Q queries; a data point is read from smem once (LDS.128
//    broadcast, 4 points) and reused Q times from registers;
//  * the top-k list lives in registers (compile-time K; k < K handled by -inf
//    sentinels in the first K-k slots) and is updated by a branch-free min/max
//    network, entered only behind warp-uniform votes;
//  * fp32: an exact-safe expanded-form filter on packed FFMA2 (passes.cuh) screens the
//    pairs; fp64 (and AIDW_KNN_FILTER=0): the canonical distance per pair;
//  * the epilogue reduces min/max of r_obs with REDUX (fp32) / shuffles (fp64),
//    one atomic per warp, and the last CTA writes {-min, max} ready for an
//    allreduce(MAX) -- no extra launch.
#include "passes.cuh"

#include <climits>
#include <cmath>
#include <cstdlib>

namespace aidw {

template <typename T> struct KnnArgs {
    const T *px, *py;  // internal SoA, padded to ndp with +inf
    int64_t ndp;
    const T *qx, *qy;
    int64_t nq;
    int k;
    T *r_obs, *d1sq, *minmax, *dists;  // all nullable except where the caller needs them
    Scratch *sc;
    int dists_sq;  // 1: dists receives the k squared distances s (data-sharded partial lists)
    T *lists;      // split mode (gridDim.y = S > 1): per-split k smallest s, [S][nq][k] ascending
    const int *perm;  // nullable: launch slot i evaluates query perm[i] (spatial order, §4.7)
};

// Bounds exchange: wait until every rank acked epoch e - 2 (the last
// use of slot e & 1), values into val[e & 1][rank] of every rank's ExBuf, a system-scope
// fence, then the flags (release) -- P2P stores over NVLink.  A wait that exceeds ~2 s
// (a missing peer) sets ex_timeout (aidw_check reports it) and proceeds.
__device__ __forceinline__ void exchange_push(Scratch *sc, double v0, double v1)
{
    const unsigned long long ep = sc->ex_epoch + 1;
    sc->ex_epoch = ep;
    const int me = sc->ex_rank, n = sc->ex_world;
    if (ep > 2) {
        const ExBuf *own = sc->ex_peers[me];
        const long long t0 = clock64();
        for (int r = 0; r < n; ++r) {
            unsigned long long f;
            for (;;) {
                asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(f) : "l"(&own->ack[r]) : "memory");
                if (f + 2 >= ep) break;
                if (clock64() - t0 > 4000000000ll) {
                    atomicExch(&sc->ex_timeout, 1u);
                    break;
                }
                __nanosleep(100);
            }
        }
    }
    const int slot = (int)(ep & 1);
    for (int r = 0; r < n; ++r) {
        ExBuf *b = sc->ex_peers[r];
        b->val[slot][me][0] = v0;
        b->val[slot][me][1] = v1;
    }
    __threadfence_system();
    for (int r = 0; r < n; ++r)
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(&sc->ex_peers[r]->flag[me]), "l"(ep) : "memory");
}

__global__ void exchange_push_identity_kernel(Scratch *sc)
{
    exchange_push(sc, -__longlong_as_double(0x7ff0000000000000ll), -__longlong_as_double(0x7ff0000000000000ll));
}

int launch_exchange_push_identity(Scratch *sc, cudaStream_t st)
{
    exchange_push_identity_kernel<<<1, 1, 0, st>>>(sc);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// Query index of launch slot `pos` (identity without a permutation).
template <typename T> __device__ __forceinline__ int64_t query_of(const KnnArgs<T> &a, int64_t pos)
{
    return (a.perm && pos < a.nq) ? (int64_t)a.perm[pos] : pos;
}

// Split mode: this CTA scans data tiles [t0, t0 + nloc) (blockIdx.y of gridDim.y equal
// ranges); S = 1 covers everything.
struct TileRange {
    int t0, nloc;
};
__device__ __forceinline__ TileRange split_range(int ntiles)
{
    const int S = (int)gridDim.y, y = (int)blockIdx.y;
    const int t0 = (int)((long long)y * ntiles / S), t1 = (int)((long long)(y + 1) * ntiles / S);
    return {t0, t1 - t0};
}

// Split-mode epilogue: the CTA's ascending k smallest squared distances per query.
template <typename T, int K, int Q>
__device__ __forceinline__ void knn_write_split(const KnnArgs<T> &a, T (&buf)[Q][K], const bool (&valid)[Q],
                                                const int64_t (&qid)[Q], int k0)
{
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const int64_t idx = qid[q];
        if (!valid[q]) continue;
        T *o = a.lists + ((int64_t)blockIdx.y * a.nq + idx) * a.k;
#pragma unroll
        for (int i = 0; i < K; ++i)
            if (i >= k0) o[i - k0] = buf[q][i];
    }
}

template <typename T> __device__ __forceinline__ T from_bits(unsigned long long b);
template <> __device__ __forceinline__ float from_bits<float>(unsigned long long b) { return __uint_as_float((unsigned)b); }
template <> __device__ __forceinline__ double from_bits<double>(unsigned long long b) { return __longlong_as_double((long long)b); }

// Warp min/max of non-negative values via their (order-preserving) bit patterns.
__device__ __forceinline__ void warp_minmax(float v, bool valid, unsigned long long &mn, unsigned long long &mx)
{
    unsigned b = __float_as_uint(v);
    mn = __reduce_min_sync(0xffffffffu, valid ? b : 0xffffffffu);
    mx = __reduce_max_sync(0xffffffffu, valid ? b : 0u);
    if (mn == 0xffffffffu) mn = ~0ull;
}

__device__ __forceinline__ void warp_minmax(double v, bool valid, unsigned long long &mn, unsigned long long &mx)
{
    unsigned long long b = (unsigned long long)__double_as_longlong(v);
    mn = valid ? b : ~0ull;
    mx = valid ? b : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long a = __shfl_xor_sync(0xffffffffu, mn, o);
        unsigned long long c = __shfl_xor_sync(0xffffffffu, mx, o);
        mn = a < mn ? a : mn;
        mx = c > mx ? c : mx;
    }
}

// Query loads for the Q queries of this thread (strided by the block for coalescing),
// with the non-finite check (smallest failing index -> scratch).
template <typename T, int Q, int BLK = kBlock>
__device__ __forceinline__ void load_queries(const KnnArgs<T> &a, int64_t base, T (&qx)[Q], T (&qy)[Q],
                                             bool (&valid)[Q], int64_t (&qid)[Q])
{
    const T *qxp = a.qx, *qyp = a.qy;
    Scratch *sc = a.sc;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        valid[q] = base + q * BLK < a.nq;
        const int64_t idx = qid[q] = query_of(a, base + q * BLK);
        qx[q] = valid[q] ? qxp[idx] : T(0);
        qy[q] = valid[q] ? qyp[idx] : T(0);
        if (valid[q] && !(isfinite(qx[q]) && isfinite(qy[q]))) atomicMin(&sc->err_idx, (long long)idx);
    }
}

// Epilogue shared by the kNN kernels: r_obs (Eq. 3), d1sq, the k distances, and the
// {-min, max} of r_obs (warp reduce -> one atomic per warp -> last CTA publishes and
// resets the scratch).  Must be reached by all threads.
template <typename T, int K, int Q>
__device__ __forceinline__ void knn_epilogue(const KnnArgs<T> &a, T (&buf)[Q][K], const bool (&valid)[Q],
                                             const int64_t (&qid)[Q], int k0)
{
    const int tid = threadIdx.x, lane = tid & 31;
    T robs_l[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        T robs, d1;
        robs_of<T, K>(buf[q], k0, a.k, robs, d1);
        robs_l[q] = robs;
        const int64_t idx = qid[q];
        if (valid[q]) {
            if (a.r_obs) a.r_obs[idx] = robs;
            if (a.d1sq) a.d1sq[idx] = d1;
            if (a.dists) {
                T *o = a.dists + idx * a.k;
#pragma unroll
                for (int i = 0; i < K; ++i)
                    if (i >= k0) o[i - k0] = a.dists_sq ? buf[q][i] : sqrt_rn(buf[q][i]);
            }
        }
    }

    if (a.minmax) {
        unsigned long long mn = ~0ull, mx = 0ull;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            unsigned long long m0, m1;
            warp_minmax(robs_l[q], valid[q], m0, m1);
            mn = m0 < mn ? m0 : mn;
            mx = m1 > mx ? m1 : mx;
        }
        if (lane == 0) {
            if (mn != ~0ull) atomicMin(&a.sc->mn, mn);
            atomicMax(&a.sc->mx, mx);
            __threadfence();
        }
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            const unsigned ticket = atomicAdd(&a.sc->done, 1u);
            if (ticket == gridDim.x - 1) {  // last CTA: publish and reset the scratch
                __threadfence();
                const unsigned long long gmn = atomicAdd(&a.sc->mn, 0ull);
                const unsigned long long gmx = atomicAdd(&a.sc->mx, 0ull);
                a.minmax[0] = -from_bits<T>(gmn);
                a.minmax[1] = from_bits<T>(gmx);
                a.sc->mn = ~0ull;
                a.sc->mx = 0ull;
                a.sc->done = 0u;
                __threadfence();
                if (a.sc->ex_world > 0)  // N4 push: the bounds go straight to every peer
                    exchange_push(a.sc, (double)a.minmax[0], (double)a.minmax[1]);
            }
        }
    }
}

// ---------------------------------------------------------------------------------
// Canonical kernel: every pair evaluated with the R16 sequence (fp64 path; fp32 with
// AIDW_KNN_FILTER=0).  4 FP32/FP64 ops + 1 compare per pair.
template <typename T, int K, int Q, bool SPLIT>
__global__ void __launch_bounds__(kBlock) knn_robs_kernel(const KnnArgs<T> a)
{
    constexpr int TILE = kTileK, STAGES = kStagesK;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T *sx = reinterpret_cast<T *>(smem_raw);
    T *sy = sx + STAGES * TILE;
    Ring<STAGES> ring{reinterpret_cast<uint64_t *>(sy + STAGES * TILE),
                      reinterpret_cast<uint64_t *>(sy + STAGES * TILE) + STAGES};
    const TileRange tr = SPLIT ? split_range((int)(a.ndp / TILE)) : TileRange{0, (int)(a.ndp / TILE)};
    const int ntiles = tr.nloc;
    if (threadIdx.x == 0) ring.init();
    __syncthreads();

    auto issue = [&](int tile, int slot) {
        const int64_t off = (int64_t)(tr.t0 + tile) * TILE;
        mbar_arrive_expect_tx(&ring.full[slot], 2u * TILE * sizeof(T));
        bulk_g2s(sx + slot * TILE, a.px + off, TILE * sizeof(T), &ring.full[slot]);
        bulk_g2s(sy + slot * TILE, a.py + off, TILE * sizeof(T), &ring.full[slot]);
    };
    if (threadIdx.x == 0)
        for (int s = 0; s < STAGES && s < ntiles; ++s) issue(s, s);

    const int64_t base = (int64_t)blockIdx.x * (kBlock * Q) + threadIdx.x;
    T qx[Q], qy[Q];
    bool valid[Q];
    int64_t qid[Q];
    load_queries<T, Q>(a, base, qx, qy, valid, qid);

    // register top-K; slots [0, K-k) hold -inf sentinels (never displaced)
    T buf[Q][K];
    const int k0 = K - a.k;
#pragma unroll
    for (int q = 0; q < Q; ++q)
#pragma unroll
        for (int i = 0; i < K; ++i) buf[q][i] = (i < k0) ? -pos_inf<T>() : pos_inf<T>();

    for (int t = 0; t < ntiles; ++t) {
        ring.wait_full(t);
        const T *tx = sx + ring.slot(t) * TILE;
        const T *ty = sy + ring.slot(t) * TILE;
#pragma unroll 2
        for (int j = 0; j < TILE; j += 4) {
            const Vec4<T> X = lds4(tx + j), Y = lds4(ty + j);
            T s[Q][4];
            bool hit = false;
#pragma unroll
            for (int q = 0; q < Q; ++q)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    s[q][e] = dist_sq(qx[q], qy[q], X.v[e], Y.v[e]);
                    hit |= s[q][e] < buf[q][K - 1];
                }
            if (__any_sync(0xffffffffu, hit)) {
#pragma unroll
                for (int e = 0; e < 4; ++e)
#pragma unroll
                    for (int q = 0; q < Q; ++q) {
                        const bool h = s[q][e] < buf[q][K - 1];
                        if (__any_sync(0xffffffffu, h)) {
                            if (h) topk_insert<T, K>(buf[q], s[q][e]);
                        }
                    }
            }
        }
        ring.release(t, ntiles, issue);
    }
    if constexpr (SPLIT)
        knn_write_split<T, K, Q>(a, buf, valid, qid, k0);
    else
        knn_epilogue<T, K, Q>(a, buf, valid, qid, k0);
}

// ---------------------------------------------------------------------------------
// Filtered kernel (passes.cuh knn_f32_tile): smem tiles of the fp32 filter arrays
// (cx, cy, pp) and -- fp32 -- the coordinates (x, y) for the canonical re-check; fp64
// handles re-check from the global fp64 coordinates (rare path only) and keep their
// top-k in fp64.
// MINB = 0: no occupancy hint (an explicit minBlocks of 1 lets ptxas use up to 255
// registers and was measured slower: 113 vs 108 ms at C4).
template <typename T> __host__ __device__ constexpr int filter_arrays() { return sizeof(T) == 4 ? 5 : 3; }

// SPLIT: 0 = whole data range; 1 = a split (seeded from the home tile when the batch is
// spatially ordered); 2 = an unordered split with the per-query seed (seed_query).
// H16: spatially ordered batches -- the fp16 pre-filter (passes.cuh knn_h16_tile)
// replaces the fp32 main loop once every query of the CTA has a finite k-th distance
// (after the seed tile, or the first tile).  fp32 handles convert the tile's coordinates;
// fp64 handles (round 2) convert the centred fp32 filter coordinates cx = fl32(x - c), the
// CTA centre taken on the same centred scale, with the centring error in the margin.
template <typename T, int K, int Q, int G, int SPLIT, int MINB = 0, bool H16 = false, int BLK = kBlock>
__global__ void __launch_bounds__(BLK, MINB) knn_filter_kernel(const KnnArgs<T> a, const FilterArgs f)
{
    constexpr int TILE = kTileKF, STAGES = kStagesKF, NARR = filter_arrays<T>();
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float *scx = reinterpret_cast<float *>(smem_raw);
    float *scy = scx + STAGES * TILE;
    float *spp = scy + STAGES * TILE;
    float *spx = spp + STAGES * TILE;  // fp32 only
    float *spy = spx + STAGES * TILE;
    Ring<STAGES, BLK / 32> ring{reinterpret_cast<uint64_t *>(scx + NARR * STAGES * TILE),
                      reinterpret_cast<uint64_t *>(scx + NARR * STAGES * TILE) + STAGES};
    const int nt_all = (int)(a.ndp / TILE);
    const TileRange tr = SPLIT ? split_range(nt_all) : TileRange{0, nt_all};
    // Spatial order (§4.7): the CTA's queries are neighbours.  Its "home" tile is the
    // (Morton-sorted) data tile under its middle query.  Unsplit, the scan starts there
    // and wraps around, so the top-k is near-final after the first tiles and the filter
    // then rejects almost every group.  Split (seeded, §4.6), the CTA first scans the home
    // tile only to SEED its lists: the k-th smallest s over those k real points is an
    // upper bound of the query's true k-th distance, and filling the list with copies of
    // it (instead of +inf) lets the split's own range start filtered.  The merged
    // multiset is unchanged: every point below the seed is still inserted by the split
    // that owns it, and a seed copy survives the merge only where the true k-th distance
    // equals the seed value.
    int home = 0;
    if (a.perm) {
        const int64_t mid = min((int64_t)blockIdx.x * (BLK * Q) + BLK * Q / 2, a.nq - 1);
        const int64_t qm = a.perm[mid];
        home = (int)(f.cell_start[morton_cell((float)a.qx[qm], (float)a.qy[qm], f.grid)] / TILE);
        home = home >= nt_all ? nt_all - 1 : home;
    }
    // H16 kernels seed every query's lists from its own Morton cell instead (per-query seed,
    // f.sx / f.sx64 != null): no home tile to scan, and the fp16 loop starts on the first tile
    const bool qseed = H16 && a.perm != nullptr && (NARR == 5 ? f.sx != nullptr : f.sx64 != nullptr);
    const bool seed = SPLIT && a.perm != nullptr && !qseed;
    int start = 0;
    if (!SPLIT && a.perm) start = home == 0 ? nt_all - 1 : home - 1;
    const int ntiles = tr.nloc + (seed ? 1 : 0);
    auto tile_of = [&](int tile) {  // global tile index of ring tile `tile`
        if (SPLIT) return seed ? (tile == 0 ? home : tr.t0 + tile - 1) : tr.t0 + tile;
        const int pt = tile + start;
        return pt >= nt_all ? pt - nt_all : pt;
    };
    if (threadIdx.x == 0) ring.init();
    __syncthreads();

    auto issue = [&](int tile, int slot) {
        constexpr uint32_t B = TILE * sizeof(float);
        mbar_arrive_expect_tx(&ring.full[slot], (uint32_t)NARR * B);
        const int64_t off = (int64_t)tile_of(tile) * TILE;
        bulk_g2s(scx + slot * TILE, f.cx + off, B, &ring.full[slot]);
        bulk_g2s(scy + slot * TILE, f.cy + off, B, &ring.full[slot]);
        bulk_g2s(spp + slot * TILE, f.pp + off, B, &ring.full[slot]);
        if constexpr (NARR == 5) {
            bulk_g2s(spx + slot * TILE, f.px + off, B, &ring.full[slot]);
            bulk_g2s(spy + slot * TILE, f.py + off, B, &ring.full[slot]);
        }
    };
    if (threadIdx.x == 0)
        for (int s = 0; s < STAGES && s < ntiles; ++s) issue(s, s);

    const int64_t base = (int64_t)blockIdx.x * (BLK * Q) + threadIdx.x;
    T qx[Q], qy[Q];
    bool valid[Q];
    int64_t qid[Q];
    load_queries<T, Q, BLK>(a, base, qx, qy, valid, qid);
    const int k0 = K - a.k;
    KnnF32State<K, Q, T> st;
#pragma unroll
    for (int q = 0; q < Q; ++q) st.init(q, qx[q], qy[q], f, k0);
    if constexpr (SPLIT == 2) {  // unordered split: per-query seed (null pointers: off)
        if (!seed && (f.sx64 != nullptr || f.sx != nullptr)) {
#pragma unroll
            for (int q = 0; q < Q; ++q)
                if (valid[q]) st.seed_query(q, f, a.k, k0);
        }
    }
    if constexpr (H16) {  // ordered fp16 kernels: per-query seed
        if (qseed) {
#pragma unroll
            for (int q = 0; q < Q; ++q)
                if (valid[q]) st.seed_query(q, f, a.k, k0);
        }
    }

    // fp16 pre-filter state (H16): the CTA's query-bbox centre, the scale, per-query
    // coefficients and thresholds; enabled once every query has a finite k-th distance
    __shared__ __align__(16) __half2 hbuf[H16 ? 3 : 1][4][H16 ? TILE / 2 : 1];
    __shared__ __align__(8) uint64_t hbar[H16 ? 6 : 1];  // pipelined fp16 tiles: full[3], empty[3]
    __shared__ unsigned hrel[H16 ? STAGES : 1];          // pipelined: warps done with each ring slot
    __shared__ unsigned hred[4];
    __shared__ H16Frame hfr;
    KnnH16<Q> h16;
    float Cx = 0.f, Cy = 0.f, sig = 0.f;  // fp64 handles: C on the centred (cx, cy) scale
    float hq_x[H16 ? Q : 1], hq_y[H16 ? Q : 1];  // the queries on the scale of the converted points
    bool h16_on = false;
    int axis = -1;  // strip axis: the one along which the CTA's queries spread least
    if constexpr (H16) {
        // centre of the CTA's valid queries (order-preserving keys of the fp32 values)
        auto key = [](float v) { const unsigned b = __float_as_uint(v); return (b >> 31) ? ~b : b | 0x80000000u; };
        auto unkey = [](unsigned k) { return __uint_as_float((k >> 31) ? k & 0x7fffffffu : ~k); };
        if (threadIdx.x == 0) hred[0] = hred[2] = 0xffffffffu, hred[1] = hred[3] = 0u;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            hq_x[q] = NARR == 5 ? (float)qx[q] : centre_f32(qx[q], f.c_x);
            hq_y[q] = NARR == 5 ? (float)qy[q] : centre_f32(qy[q], f.c_y);
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < Q; ++q)
            if (valid[q] && isfinite(hq_x[q]) && isfinite(hq_y[q])) {
                atomicMin(&hred[0], key(hq_x[q]));
                atomicMax(&hred[1], key(hq_x[q]));
                atomicMin(&hred[2], key(hq_y[q]));
                atomicMax(&hred[3], key(hq_y[q]));
            }
        __syncthreads();
        if (hred[0] != 0xffffffffu) {
            Cx = 0.5f * unkey(hred[0]) + 0.5f * unkey(hred[1]);
            Cy = 0.5f * unkey(hred[2]) + 0.5f * unkey(hred[3]);
            if (f.strip) axis = unkey(hred[3]) - unkey(hred[2]) < unkey(hred[1]) - unkey(hred[0]) ? 1 : 0;
        }
        __syncthreads();  // hred is reused for the scale
    }

    // fp16 pre-filter setup once every list is finite: the CTA scale sigma (sigma m <= 16, m
    // the largest |q - C| and k-th distance over the CTA), per-query coefficients and
    // thresholds.  All threads; the result is CTA-uniform.
    auto h16_enable = [&]() -> bool {
        bool fin = true;
#pragma unroll
        for (int q = 0; q < Q; ++q) fin &= !valid[q] || st.buf[q][K - 1] < pos_inf<T>();
        if (!__syncthreads_and(fin)) return false;
        float m = 0.f;  // non-negative: float bits order like uint
#pragma unroll
        for (int q = 0; q < Q; ++q)
            if (valid[q]) {
                const float dx = hq_x[q] - Cx, dy = hq_y[q] - Cy;
                m = fmaxf(m, fmaxf(sqrtf(dx * dx + dy * dy), sqrtf((float)st.buf[q][K - 1])));
            }
        if (threadIdx.x == 0) hred[0] = 0u;
        __syncthreads();
        atomicMax(&hred[0], __float_as_uint(m * 1.001f));
        __syncthreads();
        const float mm = __uint_as_float(hred[0]);
        int e = 0;
        frexpf(kH16Radius / fmaxf(mm, 0x1p-100f), &e);  // 16/m = f 2^e, f in [0.5, 1)
        e = e - 1 < -100 ? -100 : (e - 1 > 100 ? 100 : e - 1);
        sig = ldexpf(1.0f, e);
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const float ax = -2.0f * __fmul_rn(__fsub_rn(hq_x[q], Cx), sig);
            const float by = -2.0f * __fmul_rn(__fsub_rn(hq_y[q], Cy), sig);
            // the strip axis' coefficient goes first (h16_convert swaps û, v̂ likewise)
            h16.A[q] = __float2half2_rn(axis == 1 ? by : ax);
            h16.B[q] = __float2half2_rn(axis == 1 ? ax : by);
        }
        if (threadIdx.x == 0) {
            const double ox = NARR == 5 ? 0.0 : (double)f.c_x, oy = NARR == 5 ? 0.0 : (double)f.c_y;
            hfr = H16Frame{ox + (double)Cx, oy + (double)Cy, ox, oy, NARR == 5 ? 0.0 : (double)f.r1, sig, NARR != 5};
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const T v = st.buf[q][K - 1];
            h16.T[q] = !valid[q] ? -pos_inf<float>()
                       : axis < 0 ? h16_threshold<false>(v, qx[q], qy[q], hfr, h16.A[q], h16.B[q])
                                  : h16_threshold<true>(v, qx[q], qy[q], hfr, h16.A[q], h16.B[q]);
        }
        return isfinite(mm) && sig > 0.f && isfinite(sig);
    };
    if constexpr (H16) {
        if (qseed) h16_on = h16_enable();  // seeded lists: fp16 from the first tile
    }

    // Pipelined fp16 tiles (round 2): with the fp16 stages on from the first
    // tile (per-query seeds) and the strip test, every warp converts its quarter of tile t+1
    // into one of three fp16 buffers before it processes tile t, and hands the buffers over
    // with mbarriers (full: all four quarters written; empty: all four warps done reading)
    // instead of a CTA barrier per tile -- a warp may run a tile ahead of the slowest one.
    // The converted values and the per-tile work are the same: results bit-identical.
    bool piped = false;
    if constexpr (H16) {
        piped = h16_on && axis >= 0 && f.pipe != 0;
        if (piped) {
            if (threadIdx.x == 0) {
                for (int b = 0; b < 6; ++b) mbar_init(&hbar[b], BLK);  // every thread arrives
                for (int b = 0; b < STAGES; ++b) hrel[b] = 0u;
                fence_mbar_init();
            }
            __syncthreads();
            auto convert = [&](int t) {  // this thread's 4 points of tile t -> buffer t % 3
                const int o = ring.slot(t) * TILE;
                __half2 *hb = &hbuf[t % 3][0][0];
                h16_convert<TILE>(NARR == 5 ? spx + o : scx + o, NARR == 5 ? spy + o : scy + o, hb, hb + TILE / 2,
                                  hb + TILE, hb + 3 * TILE / 2, axis, Cx, Cy, sig);
                mbar_arrive(&hbar[t % 3]);  // release: this thread's stores
            };
            ring.wait_full(0);
            convert(0);
            for (int t = 0; t < ntiles; ++t) {
                if (t + 1 < ntiles) {
                    ring.wait_full(t + 1);
                    if (t >= 2) mbar_wait(&hbar[3 + (t + 1) % 3], (uint32_t)((t - 2) / 3) & 1u);  // tile t-2 read
                    convert(t + 1);
                }
                mbar_wait(&hbar[t % 3], (uint32_t)(t / 3) & 1u);  // tile t converted by every warp
                const int o = ring.slot(t) * TILE;
                __half2 *hb = &hbuf[t % 3][0][0];
                const T *rpx, *rpy;
                if constexpr (NARR == 5) {
                    rpx = spx + o;
                    rpy = spy + o;
                } else {
                    const int64_t off = (int64_t)tile_of(t) * TILE;
                    rpx = f.px64 + off;
                    rpy = f.py64 + off;
                }
                knn_h16_tile<K, Q, G, TILE, true, 4, T>(st, h16, hb, hb + TILE / 2, hb + TILE, hb + 3 * TILE / 2,
                                                        scx + o, scy + o, spp + o, rpx, rpy, hfr);
                mbar_arrive(&hbar[3 + t % 3]);  // this thread has read buffer t % 3
                // the LAST warp to finish tile t refills its ring slot (no warp waits for the
                // others here; the slot's reads are ordered before the TMA write by the
                // acq_rel counter and the async-proxy fence)
                __syncwarp();
                if ((threadIdx.x & 31) == 0 && t + STAGES < ntiles) {
                    const int sl = ring.slot(t);
                    unsigned old;
                    asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                                 : "=r"(old) : "r"(smem_u32(&hrel[sl])) : "memory");
                    if (old == BLK / 32 - 1) {
                        hrel[sl] = 0u;
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        issue(t + STAGES, sl);
                    }
                }
            }
        }
    }

    for (int t = 0; t < (piped ? 0 : ntiles); ++t) {
        ring.wait_full(t);
        const int o = ring.slot(t) * TILE;
        if constexpr (H16) {
            if (h16_on) {
                __half2 *hb = &hbuf[t & 1][0][0];
                // fp32: the tile's coordinates; fp64: the centred filter coordinates
                h16_convert<TILE>(NARR == 5 ? spx + o : scx + o, NARR == 5 ? spy + o : scy + o, hb, hb + TILE / 2,
                                  hb + TILE, hb + 3 * TILE / 2, axis, Cx, Cy, sig);
                __syncthreads();
                const T *rpx, *rpy;  // the canonical re-check's coordinates (rare path)
                if constexpr (NARR == 5) {
                    rpx = spx + o;
                    rpy = spy + o;
                } else {
                    const int64_t off = (int64_t)tile_of(t) * TILE;
                    rpx = f.px64 + off;
                    rpy = f.py64 + off;
                }
                if (axis >= 0)  // strip groups of 4 G = 128 points (r02_tune_knn_strip_{d,e}.log)
                    knn_h16_tile<K, Q, G, TILE, true, 4, T>(st, h16, hb, hb + TILE / 2, hb + TILE, hb + 3 * TILE / 2,
                                                            scx + o, scy + o, spp + o, rpx, rpy, hfr);
                else
                    knn_h16_tile<K, Q, G, TILE, false, 1, T>(st, h16, hb, hb + TILE / 2, hb + TILE,
                                                             hb + 3 * TILE / 2, scx + o, scy + o, spp + o, rpx, rpy,
                                                             hfr);
            } else {  // warm-up tile (lists not yet finite): every group straight to the rare
                      // path -- with an infinite threshold the filter passes every pair anyway --
                      // so the kernel carries no fp32 main loop (registers)
                bool all[Q];
#pragma unroll
                for (int q = 0; q < Q; ++q) all[q] = true;
                if constexpr (NARR == 5) {
#pragma unroll 1
                    for (int j = 0; j < TILE; j += G)
                        knn_rare_group<K, Q, G>(st, all, scx + o, scy + o, spp + o, spx + o, spy + o, j);
                } else {
                    const int64_t off = (int64_t)tile_of(t) * TILE;
#pragma unroll 1
                    for (int j = 0; j < TILE; j += G)
                        knn_rare_group<K, Q, G>(st, all, scx + o, scy + o, spp + o, f.px64 + off, f.py64 + off, j);
                }
            }
        } else if constexpr (NARR == 5) {
            knn_f32_tile<K, Q, G, TILE>(st, scx + o, scy + o, spp + o, spx + o, spy + o);
        } else {
            const int64_t off = (int64_t)tile_of(t) * TILE;
            knn_f32_tile<K, Q, G, TILE, T>(st, scx + o, scy + o, spp + o, f.px64 + off, f.py64 + off);
        }
        if (seed && t == 0) st.seed_lists(k0);  // home tile scanned: lists := seed copies
        if constexpr (H16) {
            if (!h16_on && t + 1 < ntiles) h16_on = h16_enable();
        }
        ring.release(t, ntiles, issue);
    }
    if constexpr (SPLIT)
        knn_write_split<T, K, Q>(a, st.buf, valid, qid, k0);
    else
        knn_epilogue<T, K, Q>(a, st.buf, valid, qid, k0);
}

// ---------------------------------------------------------------------------------
// Small-nq data split: when the query grid leaves SMs idle, the data
// tiles are split across gridDim.y; each split writes its k smallest s and the merge
// kernel (N4's) forms the exact job-wide list and the usual epilogue.
template <typename T> static int dispatch_merge(const KnnArgs<T> &a, const T *lists, int P, cudaStream_t st);

template <typename T>
static int knn_split_factor(const void *kern, size_t smem, unsigned grid, int ntiles, KnnArgs<T> &a, SplitBuf *sp)
{
    a.lists = nullptr;
    if (!sp) return 1;
    const int S = choose_split(kern, kBlock, smem, grid, ntiles, 1);
    if (S <= 1) return 1;
    a.lists = static_cast<T *>(sp->reserve((size_t)S * (size_t)a.nq * (size_t)a.k * sizeof(T)));
    return a.lists ? S : 1;
}

// Seeded split of a spatially ordered batch: the factor S <= 8 (>= 128 tiles per split)
// minimising the waves per split, ceil(grid S / slots) / S, with each split's extra seed
// tile counted
// (C4: 2,000 CTAs on 592 slots -> S = 5, 17 waves of 1/5 instead of 4 of 1).
// AIDW_SPLIT=0 disables, AIDW_SPLIT=n forces n (tests).
template <typename T>
static int ordered_split_factor(const void *kern, size_t smem, unsigned grid, int ntiles, KnnArgs<T> &a, SplitBuf *sp,
                                int blk = kBlock)
{
    a.lists = nullptr;
    if (!sp) return 1;
    int S = 1;
    const char *e = getenv("AIDW_SPLIT");  // read per launch so tests can toggle it
    const int forced = e ? atoi(e) : -1;
    if (forced == 0) return 1;
    if (forced > 0) {
        S = forced < 8 ? forced : 8;
    } else {
        int dev = 0, sms = 148, occ = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, blk, smem) != cudaSuccess) {
            cudaGetLastError();
            return 1;
        }
        const double slots = (double)occ * sms;
        double best = 0.0;
        // each split keeps >= 128 tiles: shorter ranges lose more to the per-CTA fixed
        // costs (ring fill, seed tile, list write, merge) than the fuller wave gains
        // (C3, 200 tiles: unsplit 1.83 ms, S = 3 1.90, S = 7 1.96; C4, 2000 tiles: S = 5)
        for (int s = 1; s <= 8 && ntiles / s >= 128; ++s) {
            const double waves = std::ceil((double)grid * s / slots);
            const double cost = waves / s * (1.0 + (double)s / ntiles);
            if (s == 1 || cost < best * 0.995) {
                best = cost;
                S = s;
            }
        }
    }
    if (S <= 1) return 1;
    a.lists = static_cast<T *>(sp->reserve((size_t)S * (size_t)a.nq * (size_t)a.k * sizeof(T)));
    return a.lists ? S : 1;
}

template <typename T> static int knn_finish(const KnnArgs<T> &a, int S, cudaStream_t st)
{
    if (cudaPeekAtLastError() != cudaSuccess) return -1;
    if (S == 1) return 1;
    const int n = dispatch_merge<T>(a, a.lists, S, st);
    return n < 0 ? -1 : 1 + n;
}

// ---------------------------------------------------------------------------------
template <typename T, int K, int Q, int G, int SPLIT, int MINB, bool H16 = false, int BLK = kBlock>
static int set_filter_attrs(size_t smem)
{
    auto kern = knn_filter_kernel<T, K, Q, G, SPLIT, MINB, H16, BLK>;
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess &&
                   cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100) == cudaSuccess
               ? 0
               : -1;
}

// Query batches at least this large are spatially ordered first;
// AIDW_KNN_ORDER=0 disables (tests compare both).
static bool order_queries(int64_t nq)
{
    static int64_t min_q = -1;
    if (min_q < 0) {  // AIDW_KNN_ORDER_MIN: tuning knob for the threshold (tools/tune_knn.py)
        const char *m = getenv("AIDW_KNN_ORDER_MIN");
        min_q = m ? atoll(m) : 32768;
    }
    const char *e = getenv("AIDW_KNN_ORDER");
    return nq >= min_q && nq > 0 && nq <= INT_MAX && !(e && e[0] == '0');  // perm is int32
}

// Unordered split launches seed each query's lists from the sorted copy (§4.6);
// AIDW_KNN_SEED=0 disables (tests compare both).
static bool seed_unordered()
{
    const char *e = getenv("AIDW_KNN_SEED");
    return !(e && e[0] == '0');
}

// H16 (fp32, spatially ordered batches only): the fp16 pre-filter kernels; AIDW_KNN_H16=0
// turns them off (tests compare both).
// Ordered fp16 kernels seed lists per query (AIDW_KNN_QSEED=0: the home-tile seed).
static bool knn_qseed_enabled()
{
    const char *e = getenv("AIDW_KNN_QSEED");
    return !(e && e[0] == '0');
}

// AIDW_KNN_PIPE=0: the fp16 kernels convert each tile behind a CTA barrier (no mbarrier
// hand-off between warps).
static int knn_pipe_env()
{
    const char *e = getenv("AIDW_KNN_PIPE");
    return (e && e[0] == '0') ? 0 : 1;
}

// AIDW_KNN_STRIP=0: the fp16 kernels run the 2-D test on every group (no strip pre-test).
static int knn_strip_enabled()
{
    const char *e = getenv("AIDW_KNN_STRIP");
    return (e && e[0] == '0') ? 0 : 1;
}

static int knn_h16_mode()
{
    const char *e = getenv("AIDW_KNN_H16");
    // 0 off, 1 default (size-dependent shape, uncapped registers), 2 Q = 4 uncapped at every
    // size, 3 register-capped -- profiles/r02_tune_knn_h16.log, r02_tune_knn_shapes_qseed.log
    return e ? atoi(e) : 1;
}

template <int K, int Q, int G = 8, int MINB = 0, typename T = float, bool H16 = false, int BLK = kBlock>
static int launch_knn_filter_t(KnnArgs<T> a, const FilterArgs &f, cudaStream_t st, SplitBuf *sp,
                               FilterData *fd)
{
    const size_t smem =
        (size_t)filter_arrays<T>() * kStagesKF * kTileKF * sizeof(float) + 2 * kStagesKF * sizeof(uint64_t);
    if (set_filter_attrs<T, K, Q, G, 0, MINB>(smem) < 0) return -1;
    // A spatially ordered batch splits only with seeded lists (knn_filter_kernel), by the
    // factor that best fills the last wave (ordered_split_factor); an unordered one by
    // whole extra waves (knn_split_factor: its splits restart the top-k warm-up).
    const bool ordered = fd && fd->cell_start && order_queries(a.nq);
    const int blk = (H16 && ordered) ? BLK : kBlock;  // BLK: the fp16 kernels' CTA size
    const int64_t per_cta = (int64_t)blk * Q;
    const unsigned grid = (unsigned)((a.nq + per_cta - 1) / per_cta);
    if (ordered && set_filter_attrs<T, K, Q, G, 1, MINB, H16, (H16 ? BLK : kBlock)>(smem) < 0) return -1;
    const int S = ordered ? ordered_split_factor((const void *)knn_filter_kernel<T, K, Q, G, 1, MINB, H16, (H16 ? BLK : kBlock)>,
                                                 smem, grid, (int)(a.ndp / kTileKF), a, sp, blk)
                          : knn_split_factor((const void *)knn_filter_kernel<T, K, Q, G, 0, MINB>, smem, grid,
                                             (int)(a.ndp / kTileKF), a, sp);
    int pre = 0;
    FilterArgs fo = f;
    fo.strip = knn_strip_enabled();
    fo.pipe = knn_pipe_env();
    if (ordered) {
        pre = launch_order_queries(a.qx, a.qy, a.nq, fd, &fd->qorder, &a.perm, st);
        if (pre < 0) return -1;
        if (a.perm) {  // Morton-ordered copy of the data
            const float *c = static_cast<const float *>(fd->arrays);
            fo.cx = c + 3 * a.ndp;
            fo.cy = c + 4 * a.ndp;
            fo.pp = c + 5 * a.ndp;
            fo.px = c + 6 * a.ndp;
            fo.py = c + 7 * a.ndp;
            if (H16 && knn_qseed_enabled() && sizeof(T) == 4) {  // per-query seeds from the sorted copy
                fo.sx = fo.px;
                fo.sy = fo.py;
            }
            if (fd->coords64) {  // fp64 handles: the sorted fp64 coordinates for the re-check
                fo.px64 = fd->coords64;
                fo.py64 = fd->coords64 + a.ndp;
                if (H16 && knn_qseed_enabled()) {  // and for the per-query seeds
                    fo.sx64 = fo.px64;
                    fo.sy64 = fo.py64;
                }
            }
        }
    }
    if (S == 1) {
        if (H16 && ordered) {
            if (set_filter_attrs<T, K, Q, G, 0, MINB, H16, BLK>(smem) < 0) return -1;
            knn_filter_kernel<T, K, Q, G, 0, MINB, H16, BLK><<<grid, BLK, smem, st>>>(a, fo);
        } else {
            knn_filter_kernel<T, K, Q, G, 0, MINB><<<grid, kBlock, smem, st>>>(a, fo);
        }
    } else {
        if (!ordered && fd && fd->cell_start && seed_unordered()) {  // per-query seed (§4.6)
            const float *c = static_cast<const float *>(fd->arrays);
            if (fd->coords64) {
                fo.sx64 = fd->coords64;
                fo.sy64 = fd->coords64 + a.ndp;
            } else {
                fo.sx = c + 6 * a.ndp;
                fo.sy = c + 7 * a.ndp;
            }
        }
        if (ordered) {
            if (set_filter_attrs<T, K, Q, G, 1, MINB, H16, (H16 ? BLK : kBlock)>(smem) < 0) return -1;
            knn_filter_kernel<T, K, Q, G, 1, MINB, H16, (H16 ? BLK : kBlock)><<<dim3(grid, (unsigned)S), blk, smem, st>>>(a, fo);
        } else {
            if (set_filter_attrs<T, K, Q, G, 2, MINB>(smem) < 0) return -1;
            knn_filter_kernel<T, K, Q, G, 2, MINB><<<dim3(grid, (unsigned)S), kBlock, smem, st>>>(a, fo);
        }
    }
    const int n = knn_finish(a, S, st);
    return n < 0 ? -1 : n + pre;
}

static int knn_variant()
{
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("AIDW_KNN_VARIANT");
        v = e ? atoi(e) : 0;
    }
    return v;
}

// fp64 handles: the same fp32 filter, fp64 re-check and top-k (Q = 2, G = 16 for every K;
// the fp64 lists take twice the registers).
static int dispatch_filter_k(const KnnArgs<double> &a, const FilterArgs &f, cudaStream_t st, SplitBuf *sp,
                             FilterData *fd)
{
    const int k = a.k;
    if (k <= 1) return launch_knn_filter_t<1, 2, 16, 0, double>(a, f, st, sp, fd);
    if (k <= 2) return launch_knn_filter_t<2, 2, 16, 0, double>(a, f, st, sp, fd);
    if (k <= 4) return launch_knn_filter_t<4, 2, 16, 0, double>(a, f, st, sp, fd);
    if (k <= 8) return launch_knn_filter_t<8, 2, 16, 0, double>(a, f, st, sp, fd);
    if (k <= 10) {  // spatially ordered batches: the fp16 pre-filter with the strip test (round 2)
        if (fd && fd->cell_start && order_queries(a.nq) && a.nq >= 32768 && knn_h16_mode() != 0)
            return launch_knn_filter_t<10, 2, 32, 0, double, true>(a, f, st, sp, fd);
        return launch_knn_filter_t<10, 2, 16, 0, double>(a, f, st, sp, fd);
    }
    if (k <= 12) return launch_knn_filter_t<12, 2, 16, 0, double>(a, f, st, sp, fd);
    if (k <= 15) {  // C3-like ordered batches: the fp16 stages as for k = 10
        if (fd && fd->cell_start && order_queries(a.nq) && a.nq >= 32768 && knn_h16_mode() != 0)
            return launch_knn_filter_t<15, 2, 32, 0, double, true>(a, f, st, sp, fd);
        return launch_knn_filter_t<15, 2, 16, 0, double>(a, f, st, sp, fd);
    }
    if (k <= 16) return launch_knn_filter_t<16, 2, 16, 0, double>(a, f, st, sp, fd);
    if (k <= 24) return launch_knn_filter_t<24, 1, 16, 0, double>(a, f, st, sp, fd);
    return launch_knn_filter_t<32, 1, 16, 0, double>(a, f, st, sp, fd);
}

static int dispatch_filter_k(const KnnArgs<float> &a, const FilterArgs &f, cudaStream_t st, SplitBuf *sp,
                             FilterData *fd)
{
    const int k = a.k;
    if (k <= 10 && k > 8) {
        switch (knn_variant()) {  // tuning sweep (tools/tune_knn.py)
        case 2: return launch_knn_filter_t<10, 4, 8>(a, f, st, sp, fd);
        case 3: return launch_knn_filter_t<10, 2, 16>(a, f, st, sp, fd);
        case 4: return launch_knn_filter_t<10, 2, 8>(a, f, st, sp, fd);
        case 5: return launch_knn_filter_t<10, 3, 16>(a, f, st, sp, fd);
        case 6: return launch_knn_filter_t<10, 4, 16>(a, f, st, sp, fd);
        case 7: return launch_knn_filter_t<10, 2, 32>(a, f, st, sp, fd);
        case 8: return launch_knn_filter_t<10, 4, 32>(a, f, st, sp, fd);
        case 9: return launch_knn_filter_t<10, 3, 32>(a, f, st, sp, fd);
        case 10: return launch_knn_filter_t<10, 4, 32, 5>(a, f, st, sp, fd);
        case 11: return launch_knn_filter_t<10, 4, 16, 5>(a, f, st, sp, fd);
        case 12: return launch_knn_filter_t<10, 3, 32, 6>(a, f, st, sp, fd);
        case 13: return launch_knn_filter_t<10, 2, 32, 8>(a, f, st, sp, fd);
        case 14: return launch_knn_filter_t<10, 1, 16>(a, f, st, sp, fd);
        case 15: return launch_knn_filter_t<10, 1, 32>(a, f, st, sp, fd);
        case 24: return launch_knn_filter_t<10, 4, 16, 4, float, true>(a, f, st, sp, fd);  // fp16, G = 16
        case 25: return launch_knn_filter_t<10, 2, 32, 0, float, true>(a, f, st, sp, fd);  // fp16, Q = 2
        case 26: return launch_knn_filter_t<10, 2, 32, 6, float, true>(a, f, st, sp, fd);  // fp16, Q = 2, 6 CTAs/SM
        case 27: return launch_knn_filter_t<10, 3, 32, 5, float, true>(a, f, st, sp, fd);  // fp16, Q = 3
        case 28: return launch_knn_filter_t<10, 2, 32, 8, float, true>(a, f, st, sp, fd);  // fp16, Q = 2, 8 CTAs/SM
        case 29: return launch_knn_filter_t<10, 4, 32, 5, float, true>(a, f, st, sp, fd);  // fp16, Q = 4, 5 CTAs/SM
        case 30: return launch_knn_filter_t<10, 2, 32, 7, float, true>(a, f, st, sp, fd);  // fp16, Q = 2, 7 CTAs/SM
        case 31: return launch_knn_filter_t<10, 4, 32, 3, float, true>(a, f, st, sp, fd);  // fp16, Q = 4, 3 CTAs/SM
        case 32: return launch_knn_filter_t<10, 2, 32, 0, float, true, 256>(a, f, st, sp, fd);  // fp16, 256-thread CTAs
        default: break;
        }
    }
    // Q = 2 queries per thread, G = 16 points per warp vote (best measured, r01)
    if (k <= 1) return launch_knn_filter_t<1, 2, 16>(a, f, st, sp, fd);
    if (k <= 2) return launch_knn_filter_t<2, 2, 16>(a, f, st, sp, fd);
    if (k <= 4) return launch_knn_filter_t<4, 2, 16>(a, f, st, sp, fd);
    if (k <= 8) return launch_knn_filter_t<8, 2, 16>(a, f, st, sp, fd);
    if (k <= 10) {  // large (spatially ordered) batches: Q = 4, G = 32 (108 vs 115 ms at C4)
        if (order_queries(a.nq) && a.nq >= 32768) {
            switch (knn_h16_mode()) {
            case 1:  // with the strip pre-test in 128-point groups (round 2) Q = 2 uncapped wins
                     // at every size: C4 54.5 ms (Q = 4 at 3 CTAs/SM 58.0), 128,000 queries
                     // 8.2, 32,768 3.4 -- profiles/r02_tune_knn_strip_d.log
                return launch_knn_filter_t<10, 2, 32, 0, float, true>(a, f, st, sp, fd);
            case 3:  // the register-capped shapes (4 / 6 CTAs/SM), the round-2 default before the seeds
                if (a.nq < 393216) return launch_knn_filter_t<10, 2, 32, 6, float, true>(a, f, st, sp, fd);
                return launch_knn_filter_t<10, 4, 32, 4, float, true>(a, f, st, sp, fd);
            case 2: return launch_knn_filter_t<10, 4, 32, 0, float, true>(a, f, st, sp, fd);
            default: break;
            }
            return launch_knn_filter_t<10, 4, 32>(a, f, st, sp, fd);
        }
        return launch_knn_filter_t<10, 2, 16>(a, f, st, sp, fd);
    }
    if (k <= 12) return launch_knn_filter_t<12, 2, 16>(a, f, st, sp, fd);
    if (k > 12 && k <= 15) {
        switch (knn_variant()) {  // tuning sweep at C3 (tools/tune_knn.py, TUNE_CFG=C3)
        case 16: return launch_knn_filter_t<15, 4, 32>(a, f, st, sp, fd);
        case 17: return launch_knn_filter_t<15, 2, 32>(a, f, st, sp, fd);
        case 18: return launch_knn_filter_t<15, 1, 32>(a, f, st, sp, fd);
        case 19: return launch_knn_filter_t<15, 2, 8>(a, f, st, sp, fd);
        case 20: return launch_knn_filter_t<15, 1, 16>(a, f, st, sp, fd);
        case 21: return launch_knn_filter_t<15, 2, 32, 0, float, true>(a, f, st, sp, fd);  // fp16 pre-filter
        case 22: return launch_knn_filter_t<15, 4, 32, 4, float, true>(a, f, st, sp, fd);
        case 23: return launch_knn_filter_t<15, 2, 32, 6, float, true>(a, f, st, sp, fd);
        default: break;
        }
    }
    if (k <= 15) {  // C3: 1.95 vs 2.03 ms (G = 16); ordered batches with the fp16 pre-filter
                    // (Q = 2, uncapped): C3 kNN 1.82 -> 1.59 ms (profiles/r02_tune_knn_c3_h16.log)
        if (order_queries(a.nq) && a.nq >= 32768 && knn_h16_mode() != 0)
            return launch_knn_filter_t<15, 2, 32, 0, float, true>(a, f, st, sp, fd);
        return launch_knn_filter_t<15, 2, 32>(a, f, st, sp, fd);
    }
    if (k <= 16) return launch_knn_filter_t<16, 2, 16>(a, f, st, sp, fd);
    if (k <= 24) return launch_knn_filter_t<24, 2>(a, f, st, sp, fd);
    return launch_knn_filter_t<32, 2>(a, f, st, sp, fd);
}

// ---------------------------------------------------------------------------------
// N4 (data-sharded mode): merge P per-shard lists of the k smallest squared distances
// (each ascending, layout [P][nq][k]) into the job's k smallest -- the same register
// top-K insertion, so the merged multiset, r_obs and d1sq are bit-identical to a
// single-device run over the whole data -- then the usual epilogue.
template <typename T, int K>
__global__ void __launch_bounds__(kBlock) knn_merge_kernel(const KnnArgs<T> a, const T *__restrict__ lists, int P)
{
    constexpr int Q = 1;
    const int64_t base = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    bool valid[Q] = {base < a.nq};
    T buf[Q][K];
    const int k0 = K - a.k;
#pragma unroll
    for (int i = 0; i < K; ++i) buf[0][i] = (i < k0) ? -pos_inf<T>() : pos_inf<T>();
    if (valid[0]) {
        // a list's k values are loaded together (and the next list's while this one is
        // inserted), so the merge costs about one L2 latency per list, not per value;
        // the insertion sequence -- hence the merged multiset -- is unchanged
        T v[K], nx[K];
        const T *l = lists + base * a.k;
#pragma unroll
        for (int i = 0; i < K; ++i) nx[i] = i < a.k ? __ldg(l + i) : pos_inf<T>();
        for (int p = 0; p < P; ++p) {
#pragma unroll
            for (int i = 0; i < K; ++i) v[i] = nx[i];
            if (p + 1 < P) {
                const T *ln = lists + ((int64_t)(p + 1) * a.nq + base) * a.k;
#pragma unroll
                for (int i = 0; i < K; ++i) nx[i] = i < a.k ? __ldg(ln + i) : pos_inf<T>();
            }
#pragma unroll
            for (int i = 0; i < K; ++i)
                if (i < a.k && v[i] < buf[0][K - 1]) topk_insert<T, K>(buf[0], v[i]);
        }
    }
    const int64_t qid[Q] = {base};
    knn_epilogue<T, K, Q>(a, buf, valid, qid, k0);
}

template <typename T, int K>
static int launch_merge_k(const KnnArgs<T> &a, const T *lists, int P, cudaStream_t st)
{
    const unsigned grid = (unsigned)((a.nq + kBlock - 1) / kBlock);
    knn_merge_kernel<T, K><<<grid, kBlock, 0, st>>>(a, lists, P);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

template <typename T>
static int dispatch_merge(const KnnArgs<T> &a, const T *lists, int P, cudaStream_t st)
{  // a.lists is not read by the merge kernel
    const int k = a.k;
    if (k <= 1) return launch_merge_k<T, 1>(a, lists, P, st);
    if (k <= 2) return launch_merge_k<T, 2>(a, lists, P, st);
    if (k <= 4) return launch_merge_k<T, 4>(a, lists, P, st);
    if (k <= 8) return launch_merge_k<T, 8>(a, lists, P, st);
    if (k <= 10) return launch_merge_k<T, 10>(a, lists, P, st);
    if (k <= 12) return launch_merge_k<T, 12>(a, lists, P, st);
    if (k <= 15) return launch_merge_k<T, 15>(a, lists, P, st);
    if (k <= 16) return launch_merge_k<T, 16>(a, lists, P, st);
    if (k <= 24) return launch_merge_k<T, 24>(a, lists, P, st);
    return launch_merge_k<T, 32>(a, lists, P, st);
}

int launch_knn_merge(int dtype, int k, const void *lists, int P, int64_t nq, void *r_obs, void *d1sq,
                     void *minmax, Scratch *sc, cudaStream_t st)
{
    if (dtype == 0) {
        KnnArgs<float> a{nullptr, nullptr, 0, nullptr, nullptr, nq, k, (float *)r_obs, (float *)d1sq,
                         (float *)minmax, nullptr, sc, 0, nullptr, nullptr};
        return dispatch_merge(a, (const float *)lists, P, st);
    }
    KnnArgs<double> a{nullptr, nullptr, 0, nullptr, nullptr, nq, k, (double *)r_obs, (double *)d1sq,
                      (double *)minmax, nullptr, sc, 0, nullptr, nullptr};
    return dispatch_merge(a, (const double *)lists, P, st);
}

template <typename T> __global__ void minmax_identity_kernel(T *mm)
{
    mm[0] = -pos_inf<T>();
    mm[1] = -pos_inf<T>();
}

template <typename T, int K, int Q>
static int launch_knn_t(KnnArgs<T> a, cudaStream_t st, SplitBuf *sp)
{
    const size_t smem = (size_t)2 * kStagesK * kTileK * sizeof(T) + 2 * kStagesK * sizeof(uint64_t);
    if (cudaFuncSetAttribute(knn_robs_kernel<T, K, Q, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return -1;
    const int64_t per_cta = (int64_t)kBlock * Q;
    const unsigned grid = (unsigned)((a.nq + per_cta - 1) / per_cta);
    const int S =
        knn_split_factor((const void *)knn_robs_kernel<T, K, Q, false>, smem, grid, (int)(a.ndp / kTileK), a, sp);
    if (S == 1) {
        knn_robs_kernel<T, K, Q, false><<<grid, kBlock, smem, st>>>(a);
    } else {
        if (cudaFuncSetAttribute(knn_robs_kernel<T, K, Q, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem) != cudaSuccess)
            return -1;
        knn_robs_kernel<T, K, Q, true><<<dim3(grid, (unsigned)S), kBlock, smem, st>>>(a);
    }
    return knn_finish(a, S, st);
}

template <typename T>
static int dispatch_k(const KnnArgs<T> &a, cudaStream_t st, SplitBuf *sp)
{
    const int k = a.k;
    if (k <= 1) return launch_knn_t<T, 1, 2>(a, st, sp);
    if (k <= 2) return launch_knn_t<T, 2, 2>(a, st, sp);
    if (k <= 4) return launch_knn_t<T, 4, 2>(a, st, sp);
    if (k <= 8) return launch_knn_t<T, 8, 2>(a, st, sp);
    if (k <= 10) return launch_knn_t<T, 10, 2>(a, st, sp);
    if (k <= 12) return launch_knn_t<T, 12, 2>(a, st, sp);
    if (k <= 15) return launch_knn_t<T, 15, 2>(a, st, sp);
    if (k <= 16) return launch_knn_t<T, 16, 2>(a, st, sp);
    if (k <= 24) return launch_knn_t<T, 24, 1>(a, st, sp);
    return launch_knn_t<T, 32, 1>(a, st, sp);
}

int launch_knn(int dtype, int k, const void *data, int64_t ndp, const void *qx, const void *qy,
               int64_t nq, void *r_obs, void *d1sq, void *minmax, void *dists, Scratch *sc,
               FilterData *filt, cudaStream_t st, int dists_sq, SplitBuf *sp)
{
    if (dtype == 0) {
        const float *p = static_cast<const float *>(data);
        KnnArgs<float> a{p, p + ndp, ndp, (const float *)qx, (const float *)qy, nq, k,
                         (float *)r_obs, (float *)d1sq, (float *)minmax, (float *)dists, sc, dists_sq, nullptr, nullptr};
        if (filt && filt->arrays) {
            const float *c = static_cast<const float *>(filt->arrays);
            // caller's order (unordered launches); the Morton-ordered copy is selected in
            // launch_knn_filter_t when the query batch is ordered (§4.7)
            FilterArgs f{c, c + ndp, c + 2 * ndp, p, p + ndp, nullptr, nullptr, filt->c_x, filt->c_y, filt->r1,
                         filt->cell_start, filt->grid};
            return dispatch_filter_k(a, f, st, sp, filt);
        }
        return dispatch_k(a, st, sp);
    }
    const double *p = static_cast<const double *>(data);
    KnnArgs<double> a{p, p + ndp, ndp, (const double *)qx, (const double *)qy, nq, k,
                      (double *)r_obs, (double *)d1sq, (double *)minmax, (double *)dists, sc, dists_sq, nullptr, nullptr};
    if (filt && filt->arrays) {  // fp32 filter, fp64 re-check from the handle's data (caller's order)
        const float *c = static_cast<const float *>(filt->arrays);
        FilterArgs f{c, c + ndp, c + 2 * ndp, nullptr, nullptr, p, p + ndp, filt->c_x, filt->c_y, filt->r1,
                     filt->cell_start, filt->grid};
        return dispatch_filter_k(a, f, st, sp, filt);
    }
    return dispatch_k(a, st, sp);
}

int launch_minmax_identity(int dtype, void *minmax, cudaStream_t st)
{
    if (dtype == 0)
        minmax_identity_kernel<float><<<1, 1, 0, st>>>((float *)minmax);
    else
        minmax_identity_kernel<double><<<1, 1, 0, st>>>((double *)minmax);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace aidw
