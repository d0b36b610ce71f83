// knn_robs.cu -- S1 + S2 of the AIDW hot path on sm_100a.
//
// Per query: the k smallest squared distances to ALL data points (brute force,
// PAPER.md:317-340, §3.1.2 Steps 1-3 -- "if dist < the kth distance, then replace
// the kth distance", strict <), then r_obs = (1/k) sum d_i (Eq. 3),
// the nearest squared distance d1sq, and the {-min, max} of r_obs over the launch.
//
// B200 design -- the paper's "tiled" idea,
// rebuilt for sm_100a:
//  * data x/y tiles stream through a 4-stage shared-memory ring filled by the TMA
//    engine (cp.async.bulk, one elected thread, mbarrier complete_tx), decoupled
//    from the block size;
//  * every thread owns Q queries; a data point is read from smem once (LDS.128
//    broadcast, 4 points) and reused Q times from registers;
//  * the top-k list lives in registers (compile-time K; k < K handled by -inf
//    sentinels in the first K-k slots) and is updated by a branch-free min/max
//    network, entered only behind warp-uniform votes -- after the first few
//    thousand points insertions are rare, so the steady state is 4 FP32 ops +
//    1 compare per pair;
//  * the epilogue reduces min/max of r_obs with REDUX (fp32) / shuffles (fp64),
//    one atomic per warp, and the last CTA writes {-min, max} ready for an
//    allreduce(MAX) -- no extra launch.
#include "aidw_internal.h"
#include "device.cuh"
#include "packed.cuh"

#include <climits>
#include <cstdlib>

namespace aidw {

template <typename T> struct KnnArgs {
    const T *px, *py;  // internal SoA, padded to ndp with +inf
    int64_t ndp;
    const T *qx, *qy;
    int64_t nq;
    int k;
    T *r_obs, *d1sq, *minmax, *dists;
    Scratch *sc;
};

__device__ __forceinline__ unsigned long long ord_bits(float v) { return (unsigned long long)__float_as_uint(v); }
__device__ __forceinline__ unsigned long long ord_bits(double v) { return (unsigned long long)__double_as_longlong(v); }
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

// Sorted insertion of s into ascending b[0..K-1], dropping the largest:
// b'[i] = min(b[i], max(b[i-1], s)), b'[0] = min(b[0], s).  Equivalent to Step 3's
// replace-the-kth-then-bubble for s < b[K-1]; a no-op otherwise.
template <typename T, int K>
__device__ __forceinline__ void topk_insert(T (&b)[K], T s)
{
#pragma unroll
    for (int i = K - 1; i > 0; --i) b[i] = tmin(b[i], tmax(b[i - 1], s));
    b[0] = tmin(b[0], s);
}

// Epilogue shared by the kNN kernels: r_obs (Eq. 3, ascending sum then /k), d1sq,
// the k distances, and the {-min, max} of r_obs (warp reduce -> one atomic per warp ->
// last CTA publishes and resets the scratch).  Must be reached by all threads.
template <typename T, int K, int Q>
__device__ __forceinline__ void knn_epilogue(const KnnArgs<T> &a, T (&buf)[Q][K], const bool (&valid)[Q],
                                             int64_t base, int k0)
{
    const int tid = threadIdx.x, lane = tid & 31;
    T robs_l[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        T sum = T(0), d1 = buf[q][K - 1];
#pragma unroll
        for (int i = 0; i < K; ++i) {
            if (i >= k0) sum = add_rn(sum, sqrt_rn(buf[q][i]));  // ascending order
            if (i == k0) d1 = buf[q][i];
        }
        const T robs = div_rn(sum, (T)a.k);
        robs_l[q] = robs;
        const int64_t idx = base + q * kBlock;
        if (valid[q]) {
            a.r_obs[idx] = robs;
            if (a.d1sq) a.d1sq[idx] = d1;
            if (a.dists) {
                T *o = a.dists + idx * a.k;
#pragma unroll
                for (int i = 0; i < K; ++i)
                    if (i >= k0) o[i - k0] = sqrt_rn(buf[q][i]);
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
            }
        }
    }
}

template <typename T, int K, int Q>
__global__ void __launch_bounds__(kBlock) knn_robs_kernel(const KnnArgs<T> a)
{
    constexpr int TILE = kTileK, STAGES = kStagesK;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T *sx = reinterpret_cast<T *>(smem_raw);
    T *sy = sx + STAGES * TILE;
    uint64_t *full = reinterpret_cast<uint64_t *>(sy + STAGES * TILE);
    uint64_t *empty = full + STAGES;

    const int tid = threadIdx.x, lane = tid & 31;
    const int ntiles = (int)(a.ndp / TILE);

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();

    auto issue = [&](int tile, int slot) {
        mbar_arrive_expect_tx(&full[slot], 2u * TILE * sizeof(T));
        bulk_g2s(sx + slot * TILE, a.px + (int64_t)tile * TILE, TILE * sizeof(T), &full[slot]);
        bulk_g2s(sy + slot * TILE, a.py + (int64_t)tile * TILE, TILE * sizeof(T), &full[slot]);
    };
    if (tid == 0)
        for (int s = 0; s < STAGES && s < ntiles; ++s) issue(s, s);

    // ---- queries owned by this thread (strided by the block for coalescing)
    const int64_t base = (int64_t)blockIdx.x * (kBlock * Q) + tid;
    T qx[Q], qy[Q];
    bool valid[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const int64_t idx = base + q * kBlock;
        valid[q] = idx < a.nq;
        qx[q] = valid[q] ? a.qx[idx] : T(0);
        qy[q] = valid[q] ? a.qy[idx] : T(0);
        if (valid[q] && !(isfinite(qx[q]) && isfinite(qy[q])))
            atomicMin(&a.sc->err_idx, (long long)idx);
    }

    // ---- register top-K; slots [0, K-k) hold -inf sentinels (never displaced)
    T buf[Q][K];
    const int k0 = K - a.k;
#pragma unroll
    for (int q = 0; q < Q; ++q)
#pragma unroll
        for (int i = 0; i < K; ++i) buf[q][i] = (i < k0) ? -pos_inf<T>() : pos_inf<T>();

    for (int t = 0; t < ntiles; ++t) {
        const int slot = t % STAGES;
        const uint32_t par = (uint32_t)(t / STAGES) & 1u;
        mbar_wait(&full[slot], par);
        const T *tx = sx + slot * TILE;
        const T *ty = sy + slot * TILE;
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
                // points in index order; each query's list updated in order
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
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (tid == 0 && t + STAGES < ntiles) {
            mbar_wait(&empty[slot], par);
            issue(t + STAGES, slot);
        }
    }

    knn_epilogue<T, K, Q>(a, buf, valid, base, k0);
}


// ---------------------------------------------------------------------------------
// fp32 kNN with an exact-safe expanded-form filter.
//
// With centred coordinates p' = p - c, q' = q - c (c = bbox centre, fp32), the squared
// distance is s' = |q'|^2 + t,  t = |p'|^2 - 2 q'.p'.  t is evaluated with two packed
// FFMA2 per couple of points from per-point |p'|^2 (precomputed once per handle), i.e.
// 1 FMA-pipe op + 1 compare per pair instead of 4 + 1.  A pair can only enter the top-k
// if t <= thr_f, where thr_f is the current k-th canonical distance converted to the t
// scale with a rigorous rounding margin (thr_of below); pairs passing the filter are
// re-evaluated with the CANONICAL sequence (R16) on the original coordinates and the
// insertion decision is taken on that exact value, so the selected multiset is bit-for-
// bit the one of knn_robs_kernel / the oracle's float instantiation.
//
// Margin (all |.| bounds, n1 = |q'x| + |q'y|, R1 = max_p |p'x| + |p'y|, u = 2^-24):
//   |t~ - t| <= 4u (n1 + R1)^2         (pp rounding 2u|p'|^2, two FMA roundings u|t|)
//   canonical s >= D (1 - 4u), D the exact distance^2;  centring moves sqrt(s') by at
//   most 2u (n1 + R1).  Hence s < thr  =>  t~ < (sqrt(thr)(1+4u) + 4u(n1+R1))^2 - |q'|^2
//   + 8u(n1+R1)^2, evaluated in fp64 and rounded up to fp32 (factor-2 slack on each term).
struct FilterArgs {
    const float *cx, *cy, *pp;  // centred filter arrays, padded with +inf
    float c_x, c_y;             // centre
    float r1;                   // R1 bound (>= max |p'x| + |p'y|)
};

// thr_of: the filter threshold for the canonical k-th distance thr (see margin above),
// in fp32 with every rounding error covered: sqrt rounded up, (1 + 2^-20) and 2^-21
// slack terms absorb the <= 3 roundings of the remaining fp32 operations.
//   qq = |q'|^2 (rounded up), m = 4u(n1+R1) (centring), E = 16u(n1+R1)^2 + 4u qq.
__device__ __forceinline__ float thr_of(float thr, float qq, float m, float E)
{
    if (!(thr < pos_inf<float>())) return pos_inf<float>();
    const float r = __fmaf_ru(__fsqrt_ru(thr), 1.0f + 0x1p-20f, m);
    const float r2 = __fmul_ru(r, r);
    const float v = __fadd_ru(__fadd_ru(r2, -qq), E);
    return __fmaf_ru(0x1p-21f, r2 + qq + E, v);
}

template <int K, int Q, int G>
__global__ void __launch_bounds__(kBlock) knn_filter_kernel(const KnnArgs<float> a, const FilterArgs f)
{
    constexpr int TILE = kTileKF, STAGES = kStagesKF;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float *scx = reinterpret_cast<float *>(smem_raw);
    float *scy = scx + STAGES * TILE;
    float *spp = scy + STAGES * TILE;
    float *spx = spp + STAGES * TILE;
    float *spy = spx + STAGES * TILE;
    uint64_t *full = reinterpret_cast<uint64_t *>(spy + STAGES * TILE);
    uint64_t *empty = full + STAGES;

    const int tid = threadIdx.x, lane = tid & 31;
    const int ntiles = (int)(a.ndp / TILE);

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();

    auto issue = [&](int tile, int slot) {
        constexpr uint32_t B = TILE * sizeof(float);
        mbar_arrive_expect_tx(&full[slot], 5u * B);
        const int64_t off = (int64_t)tile * TILE;
        bulk_g2s(scx + slot * TILE, f.cx + off, B, &full[slot]);
        bulk_g2s(scy + slot * TILE, f.cy + off, B, &full[slot]);
        bulk_g2s(spp + slot * TILE, f.pp + off, B, &full[slot]);
        bulk_g2s(spx + slot * TILE, a.px + off, B, &full[slot]);
        bulk_g2s(spy + slot * TILE, a.py + off, B, &full[slot]);
    };
    if (tid == 0)
        for (int s = 0; s < STAGES && s < ntiles; ++s) issue(s, s);

    const int64_t base = (int64_t)blockIdx.x * (kBlock * Q) + tid;
    float qx[Q], qy[Q], thr[Q], qqf[Q], mf[Q], Ef[Q];
    f32x2 A2[Q], B2[Q];
    bool valid[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const int64_t idx = base + q * kBlock;
        valid[q] = idx < a.nq;
        qx[q] = valid[q] ? a.qx[idx] : 0.f;
        qy[q] = valid[q] ? a.qy[idx] : 0.f;
        if (valid[q] && !(isfinite(qx[q]) && isfinite(qy[q])))
            atomicMin(&a.sc->err_idx, (long long)idx);
        const float qcx = __fsub_rn(qx[q], f.c_x), qcy = __fsub_rn(qy[q], f.c_y);
        A2[q] = splat2(-2.0f * qcx);
        B2[q] = splat2(-2.0f * qcy);
        thr[q] = pos_inf<float>();
        {   // margin terms (fp64, rounded up to fp32)
            const double u = 0x1p-24;
            const double qq = (double)qcx * (double)qcx + (double)qcy * (double)qcy;
            const double n1r = fabs((double)qcx) + fabs((double)qcy) + (double)f.r1;
            qqf[q] = __double2float_ru(qq);
            mf[q] = __double2float_ru(8.0 * u * n1r);
            Ef[q] = __double2float_ru(16.0 * u * n1r * n1r + 4.0 * u * qq + 2.0 * u * qq);
        }
    }

    float buf[Q][K];
    const int k0 = K - a.k;
#pragma unroll
    for (int q = 0; q < Q; ++q)
#pragma unroll
        for (int i = 0; i < K; ++i) buf[q][i] = (i < k0) ? -pos_inf<float>() : pos_inf<float>();

    for (int t = 0; t < ntiles; ++t) {
        const int slot = t % STAGES;
        const uint32_t par = (uint32_t)(t / STAGES) & 1u;
        mbar_wait(&full[slot], par);
        const float *tcx = scx + slot * TILE, *tcy = scy + slot * TILE, *tpp = spp + slot * TILE;
        const float *tpx = spx + slot * TILE, *tpy = spy + slot * TILE;
#pragma unroll 1
        for (int j = 0; j < TILE; j += G) {
            // G points per warp vote; per query a min-tree of the G filter values
            float cxv[G], cyv[G], ppv[G];
#pragma unroll
            for (int g = 0; g < G; g += 4) {
                const float4 CX = *reinterpret_cast<const float4 *>(tcx + j + g);
                const float4 CY = *reinterpret_cast<const float4 *>(tcy + j + g);
                const float4 PP = *reinterpret_cast<const float4 *>(tpp + j + g);
                cxv[g] = CX.x; cxv[g + 1] = CX.y; cxv[g + 2] = CX.z; cxv[g + 3] = CX.w;
                cyv[g] = CY.x; cyv[g + 1] = CY.y; cyv[g + 2] = CY.z; cyv[g + 3] = CY.w;
                ppv[g] = PP.x; ppv[g + 1] = PP.y; ppv[g + 2] = PP.z; ppv[g + 3] = PP.w;
            }
            bool hit = false;
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                float tv[G];
#pragma unroll
                for (int h = 0; h < G / 2; ++h) {
                    const f32x2 tt = fma2(B2[q], pack2(cyv[2 * h], cyv[2 * h + 1]),
                                          fma2(A2[q], pack2(cxv[2 * h], cxv[2 * h + 1]),
                                               pack2(ppv[2 * h], ppv[2 * h + 1])));
                    unpack2(tt, tv[2 * h], tv[2 * h + 1]);
                }
#pragma unroll
                for (int w = 1; w < G; w *= 2)
#pragma unroll
                    for (int i = 0; i + w < G; i += 2 * w) tv[i] = fminf(tv[i], tv[i + w]);
                hit |= tv[0] <= thr[q];
            }
            if (__any_sync(0xffffffffu, hit)) {
                // rare path (a few % of groups): re-derive each pair's filter value from
                // smem (same RN fma as FFMA2), then the canonical distance on the original
                // coordinates decides the insertion
#pragma unroll 1
                for (int e = j; e < j + G; ++e) {
                    const float ce = tcx[e], de = tcy[e], pe = tpp[e];
#pragma unroll
                    for (int q = 0; q < Q; ++q) {
                        const float tq = __fmaf_rn(B2[q].x, de, __fmaf_rn(A2[q].x, ce, pe));
                        const bool h = tq <= thr[q];
                        if (__any_sync(0xffffffffu, h)) {
                            if (h) {
                                const float s = dist_sq(qx[q], qy[q], tpx[e], tpy[e]);
                                if (s < buf[q][K - 1]) {
                                    topk_insert<float, K>(buf[q], s);
                                    thr[q] = thr_of(buf[q][K - 1], qqf[q], mf[q], Ef[q]);
                                }
                            }
                        }
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (tid == 0 && t + STAGES < ntiles) {
            mbar_wait(&empty[slot], par);
            issue(t + STAGES, slot);
        }
    }
    knn_epilogue<float, K, Q>(a, buf, valid, base, k0);
}

template <int K, int Q, int G = 8>
static int launch_knn_filter_t(const KnnArgs<float> &a, const FilterArgs &f, cudaStream_t st)
{
    const size_t smem = (size_t)5 * kStagesKF * kTileKF * sizeof(float) + 2 * kStagesKF * sizeof(uint64_t);
    if (cudaFuncSetAttribute(knn_filter_kernel<K, Q, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return -1;
    const int64_t per_cta = (int64_t)kBlock * Q;
    const unsigned grid = (unsigned)((a.nq + per_cta - 1) / per_cta);
    knn_filter_kernel<K, Q, G><<<grid, kBlock, smem, st>>>(a, f);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// v2 of the filtered fp32 kNN: software-pipelined (the next group's smem loads are
// issued right after the current group's filter values are formed, so they overlap
// the warp vote), and a bitmask rare path that re-checks only the passing pairs.
// The insertion decision is unchanged (canonical s < k-th), so results are identical.
template <int K, int Q, int G>
__global__ void __launch_bounds__(kBlock) knn_filter2_kernel(const KnnArgs<float> a, const FilterArgs f)
{
    constexpr int TILE = kTileKF, STAGES = kStagesKF;
    static_assert(G % 4 == 0 && G <= 32 && TILE % G == 0, "group size");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float *scx = reinterpret_cast<float *>(smem_raw);
    float *scy = scx + STAGES * TILE;
    float *spp = scy + STAGES * TILE;
    float *spx = spp + STAGES * TILE;
    float *spy = spx + STAGES * TILE;
    uint64_t *full = reinterpret_cast<uint64_t *>(spy + STAGES * TILE);
    uint64_t *empty = full + STAGES;

    const int tid = threadIdx.x, lane = tid & 31;
    const int ntiles = (int)(a.ndp / TILE);

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();

    auto issue = [&](int tile, int slot) {
        constexpr uint32_t B = TILE * sizeof(float);
        mbar_arrive_expect_tx(&full[slot], 5u * B);
        const int64_t off = (int64_t)tile * TILE;
        bulk_g2s(scx + slot * TILE, f.cx + off, B, &full[slot]);
        bulk_g2s(scy + slot * TILE, f.cy + off, B, &full[slot]);
        bulk_g2s(spp + slot * TILE, f.pp + off, B, &full[slot]);
        bulk_g2s(spx + slot * TILE, a.px + off, B, &full[slot]);
        bulk_g2s(spy + slot * TILE, a.py + off, B, &full[slot]);
    };
    if (tid == 0)
        for (int s = 0; s < STAGES && s < ntiles; ++s) issue(s, s);

    const int64_t base = (int64_t)blockIdx.x * (kBlock * Q) + tid;
    float qx[Q], qy[Q], thr[Q], qqf[Q], mf[Q], Ef[Q], A[Q], B[Q];
    bool valid[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const int64_t idx = base + q * kBlock;
        valid[q] = idx < a.nq;
        qx[q] = valid[q] ? a.qx[idx] : 0.f;
        qy[q] = valid[q] ? a.qy[idx] : 0.f;
        if (valid[q] && !(isfinite(qx[q]) && isfinite(qy[q])))
            atomicMin(&a.sc->err_idx, (long long)idx);
        const float qcx = __fsub_rn(qx[q], f.c_x), qcy = __fsub_rn(qy[q], f.c_y);
        A[q] = -2.0f * qcx;
        B[q] = -2.0f * qcy;
        thr[q] = pos_inf<float>();
        const double u = 0x1p-24;
        const double qq = (double)qcx * (double)qcx + (double)qcy * (double)qcy;
        const double n1r = fabs((double)qcx) + fabs((double)qcy) + (double)f.r1;
        qqf[q] = __double2float_ru(qq);
        mf[q] = __double2float_ru(8.0 * u * n1r);
        Ef[q] = __double2float_ru(16.0 * u * n1r * n1r + 6.0 * u * qq);
    }

    float buf[Q][K];
    const int k0 = K - a.k;
#pragma unroll
    for (int q = 0; q < Q; ++q)
#pragma unroll
        for (int i = 0; i < K; ++i) buf[q][i] = (i < k0) ? -pos_inf<float>() : pos_inf<float>();

    for (int t = 0; t < ntiles; ++t) {
        const int slot = t % STAGES;
        const uint32_t par = (uint32_t)(t / STAGES) & 1u;
        mbar_wait(&full[slot], par);
        const float *tcx = scx + slot * TILE, *tcy = scy + slot * TILE, *tpp = spp + slot * TILE;
        const float *tpx = spx + slot * TILE, *tpy = spy + slot * TILE;

        float cxv[G], cyv[G], ppv[G];
        auto load = [&](int j) {
#pragma unroll
            for (int g = 0; g < G; g += 4) {
                const float4 CX = *reinterpret_cast<const float4 *>(tcx + j + g);
                const float4 CY = *reinterpret_cast<const float4 *>(tcy + j + g);
                const float4 PP = *reinterpret_cast<const float4 *>(tpp + j + g);
                cxv[g] = CX.x; cxv[g + 1] = CX.y; cxv[g + 2] = CX.z; cxv[g + 3] = CX.w;
                cyv[g] = CY.x; cyv[g + 1] = CY.y; cyv[g + 2] = CY.z; cyv[g + 3] = CY.w;
                ppv[g] = PP.x; ppv[g + 1] = PP.y; ppv[g + 2] = PP.z; ppv[g + 3] = PP.w;
            }
        };
        load(0);
#pragma unroll 1
        for (int j = 0; j < TILE; j += G) {
            float tv[Q][G];
#pragma unroll
            for (int q = 0; q < Q; ++q)
#pragma unroll
                for (int h = 0; h < G / 2; ++h) {
                    const f32x2 tt = fma2(splat2(B[q]), pack2(cyv[2 * h], cyv[2 * h + 1]),
                                          fma2(splat2(A[q]), pack2(cxv[2 * h], cxv[2 * h + 1]),
                                               pack2(ppv[2 * h], ppv[2 * h + 1])));
                    tv[q][2 * h] = tt.x;
                    tv[q][2 * h + 1] = tt.y;
                }
            load(j + G < TILE ? j + G : j);  // next group's loads overlap the vote below
            bool hit = false;
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                float m[G];
#pragma unroll
                for (int i = 0; i < G; ++i) m[i] = tv[q][i];
#pragma unroll
                for (int w = 1; w < G; w *= 2)
#pragma unroll
                    for (int i = 0; i + w < G; i += 2 * w) m[i] = fminf(m[i], m[i + w]);
                hit |= m[0] <= thr[q];
            }
            if (__any_sync(0xffffffffu, hit)) {
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    unsigned mask = 0;
#pragma unroll
                    for (int e = 0; e < G; ++e) mask |= (tv[q][e] <= thr[q]) ? (1u << e) : 0u;
                    while (__any_sync(0xffffffffu, mask != 0)) {
                        if (mask) {
                            const int e = __ffs(mask) - 1;
                            mask &= mask - 1;
                            const float s = dist_sq(qx[q], qy[q], tpx[j + e], tpy[j + e]);
                            if (s < buf[q][K - 1]) {
                                topk_insert<float, K>(buf[q], s);
                                thr[q] = thr_of(buf[q][K - 1], qqf[q], mf[q], Ef[q]);
                            }
                        }
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (tid == 0 && t + STAGES < ntiles) {
            mbar_wait(&empty[slot], par);
            issue(t + STAGES, slot);
        }
    }
    knn_epilogue<float, K, Q>(a, buf, valid, base, k0);
}

template <int K, int Q, int G = 8>
static int launch_knn_filter2_t(const KnnArgs<float> &a, const FilterArgs &f, cudaStream_t st)
{
    const size_t smem = (size_t)5 * kStagesKF * kTileKF * sizeof(float) + 2 * kStagesKF * sizeof(uint64_t);
    if (cudaFuncSetAttribute(knn_filter2_kernel<K, Q, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess ||
        cudaFuncSetAttribute(knn_filter2_kernel<K, Q, G>, cudaFuncAttributePreferredSharedMemoryCarveout, 100) !=
            cudaSuccess)
        return -1;
    const int64_t per_cta = (int64_t)kBlock * Q;
    const unsigned grid = (unsigned)((a.nq + per_cta - 1) / per_cta);
    knn_filter2_kernel<K, Q, G><<<grid, kBlock, smem, st>>>(a, f);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
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

static int dispatch_filter_k(const KnnArgs<float> &a, const FilterArgs &f, cudaStream_t st)
{
    const int k = a.k;
    if (k <= 10 && k > 8) {
        switch (knn_variant()) {
        case 1: return launch_knn_filter_t<10, 2, 8>(a, f, st);   // v1
        case 2: return launch_knn_filter2_t<10, 4, 8>(a, f, st);
        case 3: return launch_knn_filter2_t<10, 2, 16>(a, f, st);
        case 4: return launch_knn_filter2_t<10, 3, 8>(a, f, st);
        case 5: return launch_knn_filter2_t<10, 2, 4>(a, f, st);
        default: break;
        }
    }
    if (k <= 1) return launch_knn_filter_t<1, 2>(a, f, st);
    if (k <= 2) return launch_knn_filter_t<2, 2>(a, f, st);
    if (k <= 4) return launch_knn_filter_t<4, 2>(a, f, st);
    if (k <= 8) return launch_knn_filter_t<8, 2>(a, f, st);
    if (k <= 10) return launch_knn_filter2_t<10, 2>(a, f, st);
    if (k <= 12) return launch_knn_filter_t<12, 2>(a, f, st);
    if (k <= 15) return launch_knn_filter_t<15, 2>(a, f, st);
    if (k <= 16) return launch_knn_filter_t<16, 2>(a, f, st);
    if (k <= 24) return launch_knn_filter_t<24, 2>(a, f, st);
    return launch_knn_filter_t<32, 2>(a, f, st);
}

template <typename T> __global__ void minmax_identity_kernel(T *mm)
{
    mm[0] = -pos_inf<T>();
    mm[1] = -pos_inf<T>();
}

template <typename T, int K, int Q>
static int launch_knn_t(const KnnArgs<T> &a, cudaStream_t st)
{
    const size_t smem = (size_t)2 * kStagesK * kTileK * sizeof(T) + 2 * kStagesK * sizeof(uint64_t);
    if (cudaFuncSetAttribute(knn_robs_kernel<T, K, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return -1;
    const int64_t per_cta = (int64_t)kBlock * Q;
    const unsigned grid = (unsigned)((a.nq + per_cta - 1) / per_cta);
    knn_robs_kernel<T, K, Q><<<grid, kBlock, smem, st>>>(a);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

template <typename T>
static int dispatch_k(const KnnArgs<T> &a, cudaStream_t st)
{
    const int k = a.k;
    if (k <= 1) return launch_knn_t<T, 1, 2>(a, st);
    if (k <= 2) return launch_knn_t<T, 2, 2>(a, st);
    if (k <= 4) return launch_knn_t<T, 4, 2>(a, st);
    if (k <= 8) return launch_knn_t<T, 8, 2>(a, st);
    if (k <= 10) return launch_knn_t<T, 10, 2>(a, st);
    if (k <= 12) return launch_knn_t<T, 12, 2>(a, st);
    if (k <= 15) return launch_knn_t<T, 15, 2>(a, st);
    if (k <= 16) return launch_knn_t<T, 16, 2>(a, st);
    if (k <= 24) return launch_knn_t<T, 24, 1>(a, st);
    return launch_knn_t<T, 32, 1>(a, st);
}

int launch_knn(int dtype, int k, const void *data, int64_t ndp, const void *qx, const void *qy,
               int64_t nq, void *r_obs, void *d1sq, void *minmax, void *dists, Scratch *sc,
               const FilterData *filt, cudaStream_t st)
{
    if (dtype == 0) {
        const float *p = static_cast<const float *>(data);
        KnnArgs<float> a{p, p + ndp, ndp, (const float *)qx, (const float *)qy, nq, k,
                         (float *)r_obs, (float *)d1sq, (float *)minmax, (float *)dists, sc};
        if (filt && filt->arrays) {
            const float *c = static_cast<const float *>(filt->arrays);
            FilterArgs f{c, c + ndp, c + 2 * ndp, filt->c_x, filt->c_y, filt->r1};
            return dispatch_filter_k(a, f, st);
        }
        return dispatch_k(a, st);
    }
    const double *p = static_cast<const double *>(data);
    KnnArgs<double> a{p, p + ndp, ndp, (const double *)qx, (const double *)qy, nq, k,
                      (double *)r_obs, (double *)d1sq, (double *)minmax, (double *)dists, sc};
    return dispatch_k(a, st);
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
