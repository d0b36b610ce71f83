// passes.cuh -- the two O(nq*nd) passes of the AIDW hot path as per-tile device
// functions, shared by the stand-alone kernels (knn_robs.cu, interpolate.cu) and the
// fused FIXED-bounds kernel (fused.cu).  Also the TMA/mbarrier tile ring, the exact
// kNN epilogue pieces and the Eq. 4-6 map.
#pragma once

#include "aidw_internal.h"
#include "device.cuh"
#include "packed.cuh"
#include "f64_tables.h"

#include <cuda_fp16.h>

namespace aidw {

// ------------------------------------------------------------------ tile ring
// STAGES smem slots filled by the TMA engine (one elected producer thread), consumed
// by all warps.  Tile t lives in slot t % STAGES; full/empty barrier parity (t/S) & 1.
template <int STAGES, int WARPS = kWarps>
struct Ring {
    uint64_t *full, *empty;

    __device__ __forceinline__ void init()  // thread 0, then __syncthreads by the caller
    {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], WARPS);
        }
        fence_mbar_init();
    }
    __device__ __forceinline__ int slot(int t) const { return t % STAGES; }
    __device__ __forceinline__ uint32_t parity(int t) const { return (uint32_t)(t / STAGES) & 1u; }
    __device__ __forceinline__ void wait_full(int t) { mbar_wait(&full[slot(t)], parity(t)); }
    // every warp releases the slot; the producer refills it with tile t + STAGES
    template <class Issue>
    __device__ __forceinline__ void release(int t, int ntotal, Issue &&issue)
    {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[slot(t)]);
        if (threadIdx.x == 0 && t + STAGES < ntotal) {
            mbar_wait(&empty[slot(t)], parity(t));
            issue(t + STAGES, slot(t));
        }
    }
};

// ------------------------------------------------------------------ kNN pieces
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

// r_obs (Eq. 3: ascending sum of the k distances, then /k) and the nearest s of one
// query's register list (slots [0, k0) are -inf sentinels).
template <typename T, int K>
__device__ __forceinline__ void robs_of(const T (&b)[K], int k0, int k, T &robs, T &d1)
{
    T sum = T(0);
    d1 = b[K - 1];
#pragma unroll
    for (int i = 0; i < K; ++i) {
        if (i >= k0) sum = add_rn(sum, sqrt_rn(b[i]));
        if (i == k0) d1 = b[i];
    }
    robs = div_rn(sum, (T)k);
}

// ---------------------------------------------------------------------------------
// fp32 kNN with an exact-safe expanded-form filter.
//
// With centred coordinates p' = p - c, q' = q - c (c = bbox centre, fp32), the squared
// distance is s' = |q'|^2 + t,  t = |p'|^2 - 2 q'.p'.  t is evaluated with two packed
// FFMA2 per couple of points from per-point |p'|^2 (precomputed once per handle): 2 FMA
// + a share of a min-tree per pair instead of 4 FP32 + 1 compare.  A pair can only
// enter the top-k if t <= thr_f, where thr_f is the current k-th canonical distance
// converted to the t scale with a rigorous rounding margin (thr_of); passing pairs are
// re-evaluated with the CANONICAL sequence (R16) on the original coordinates and the
// insertion decision is taken on that exact value, so the selected multiset is bit-for-
// bit the one of the unfiltered kernel / the oracle's float instantiation.
//
// Margin (n1 = |q'x| + |q'y|, R1 >= max_p |p'x| + |p'y|, u = 2^-24):
//   |t~ - t| <= 4u (n1 + R1)^2         (pp rounding 2u|p'|^2, two FMA roundings u|t|)
//   canonical s >= D (1 - 4u), D the exact distance^2;  centring moves sqrt(s') by at
//   most 2u (n1 + R1).  Hence s < thr  =>  t~ < (sqrt(thr)(1+4u) + 4u(n1+R1))^2 - |q'|^2
//   + 8u(n1+R1)^2; the constants below double every term.
struct FilterArgs {
    const float *cx, *cy, *pp;  // centred filter arrays, padded with +inf (spatial order)
    const float *px, *py;       // the same points' coordinates (canonical re-check, fp32)
    const double *px64, *py64;  // fp64 handles: the same points' fp64 coordinates (global)
    float c_x, c_y;             // centre
    float r1;                   // R1 bound
    const int *cell_start;      // first sorted position of each Morton cell (§4.7)
    OrderGrid grid;
    // unordered split launches: the Morton-sorted coordinates for the per-query seed
    // (KnnF32State::seed_query); null = no seed
    const float *sx = nullptr, *sy = nullptr;
    const double *sx64 = nullptr, *sy64 = nullptr;
    int strip = 1;  // fp16 kernels: 1 = strip pre-test, 0 = the 2-D test only
    int pipe = 1;   // fp16 kernels: 1 = mbarrier-pipelined fp16 tiles, 0 = a CTA barrier per tile
};

// thr_of: the filter threshold for the canonical k-th distance thr, in fp32 with every
// rounding error covered: sqrt rounded up, (1 + 2^-20) and 2^-21 slack terms absorb
// the <= 3 roundings of the remaining fp32 operations.
//   qq = |q'|^2 (rounded up), m = 8u(n1+R1) (centring), E = 16u(n1+R1)^2 + 6u qq.
__device__ __forceinline__ float thr_of(float thr, float qq, float m, float E)
{
    if (!(thr < pos_inf<float>())) return pos_inf<float>();
    const float r = __fmaf_ru(__fsqrt_ru(thr), 1.0f + 0x1p-20f, m);
    const float r2 = __fmul_ru(r, r);
    const float v = __fadd_ru(__fadd_ru(r2, -qq), E);
    return __fmaf_ru(0x1p-21f, r2 + qq + E, v);
}

// Centred query coordinate in fp32: one rounding of q - c (fp32 queries: __fsub_rn; fp64
// queries: the fp64 difference rounded to fp32 -- relative error u(1 + 2^-29), inside the
// factor-2 slack of the centring term m).
__device__ __forceinline__ float centre_f32(float x, float c) { return __fsub_rn(x, c); }
__device__ __forceinline__ float centre_f32(double x, float c) { return __double2float_rn(x - (double)c); }
// The k-th canonical distance on the filter's fp32 scale, rounded up (fp64: s64 < thr64
// <= thr32 and the fp64 canonical s is within 4u64 << 4u of the exact distance, so the
// fp32 margin of thr_of covers it).
__device__ __forceinline__ float thr_f32(float v) { return v; }
__device__ __forceinline__ float thr_f32(double v) { return __double2float_ru(v); }

// Per-thread state of the filtered kNN for Q queries; T = working precision of the
// queries, the canonical re-check and the top-k (the filter itself is always fp32).
template <int K, int Q, typename T = float>
struct KnnF32State {
    T qx[Q], qy[Q];
    float thr[Q], qqf[Q], mf[Q], Ef[Q], A[Q], B[Q];
    T buf[Q][K];

    __device__ __forceinline__ void init(int q, T x, T y, const FilterArgs &f, int k0)
    {
        qx[q] = x;
        qy[q] = y;
        float qcx = centre_f32(x, f.c_x), qcy = centre_f32(y, f.c_y);
        const double u = 0x1p-24;
        double qq = (double)qcx * (double)qcx + (double)qcy * (double)qcy;
        const double n1r = fabs((double)qcx) + fabs((double)qcy) + (double)f.r1;
        const bool ok = n1r <= 0x1p60;  // else (far outside the fp32-safe range, or NaN)
        if (!ok) qcx = qcy = 0.f, qq = 0.0;  // unfiltered: t = pp <= +inf = thr for every point
        A[q] = opaque(-2.0f * qcx);  // opaque: keep in a register, never re-derived per group
        B[q] = opaque(-2.0f * qcy);
        thr[q] = pos_inf<float>();
        qqf[q] = __double2float_ru(qq);
        mf[q] = ok ? __double2float_ru(8.0 * u * n1r) : pos_inf<float>();  // m = +inf keeps thr at +inf
        Ef[q] = ok ? __double2float_ru(16.0 * u * n1r * n1r + 6.0 * u * qq) : 0.f;
#pragma unroll
        for (int i = 0; i < K; ++i) buf[q][i] = (i < k0) ? -pos_inf<T>() : pos_inf<T>();
    }
    // Seeded split (knn_filter_kernel): replace each list by k copies of its current
    // k-th value v (an upper bound of the query's k-th distance when the list holds k
    // real points; +inf otherwise) and filter against it.
    __device__ __forceinline__ void seed_lists(int k0)
    {
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const T v = buf[q][K - 1];
#pragma unroll
            for (int i = 0; i < K; ++i) buf[q][i] = (i < k0) ? -pos_inf<T>() : v;
            thr[q] = thr_of(thr_f32(v), qqf[q], mf[q], Ef[q]);
        }
    }
    // Per-query seed for unordered split launches: the k real points at
    // and after the query's Morton cell in the sorted copy (cell_start[kCells] = nd);
    // their largest canonical s, v, bounds the query's k-th distance from above, so the
    // list starts as k copies of v -- the argument of seed_lists.  A non-finite v (NaN or
    // far queries, nd < k) leaves the list unseeded.
    __device__ __forceinline__ void seed_query(int q, const FilterArgs &f, int k, int k0)
    {
        const T *sx, *sy;
        if constexpr (sizeof(T) == 4) {
            sx = f.sx;
            sy = f.sy;
        } else {
            sx = f.sx64;
            sy = f.sy64;
        }
        const int nd = f.cell_start[kCells];
        if (sx == nullptr || nd < k) return;
        int j0 = f.cell_start[morton_cell((float)qx[q], (float)qy[q], f.grid)];
        j0 = j0 > nd - k ? nd - k : j0;
        T v = T(0);
        for (int i = 0; i < k; ++i) {
            const T s = dist_sq(qx[q], qy[q], sx[j0 + i], sy[j0 + i]);
            v = (s > v || s != s) ? s : v;  // max, NaN-propagating
        }
        if (!(v < pos_inf<T>())) return;
#pragma unroll
        for (int i = 0; i < K; ++i) buf[q][i] = (i < k0) ? -pos_inf<T>() : v;
        thr[q] = thr_of(thr_f32(v), qqf[q], mf[q], Ef[q]);
    }
};

// Filter values t = pp + A cx + B cy of the 8 points at tile offset j for query q, as
// four packed couples (2 FFMA2 each).
template <int K, int Q, typename T>
__device__ __forceinline__ void filter8(const KnnF32State<K, Q, T> &st, int q, const float *__restrict__ tcx,
                                        const float *__restrict__ tcy, const float *__restrict__ tpp, int j,
                                        float (&t)[8])
{
#pragma unroll
    for (int g = 0; g < 8; g += 4) {
        const float4 CX = *reinterpret_cast<const float4 *>(tcx + j + g);
        const float4 CY = *reinterpret_cast<const float4 *>(tcy + j + g);
        const float4 PP = *reinterpret_cast<const float4 *>(tpp + j + g);
        const f32x2 a = fma2(splat2(st.B[q]), pack2(CY.x, CY.y), fma2(splat2(st.A[q]), pack2(CX.x, CX.y), pack2(PP.x, PP.y)));
        const f32x2 b = fma2(splat2(st.B[q]), pack2(CY.z, CY.w), fma2(splat2(st.A[q]), pack2(CX.z, CX.w), pack2(PP.z, PP.w)));
        t[g] = a.x;
        t[g + 1] = a.y;
        t[g + 2] = b.x;
        t[g + 3] = b.y;
    }
}

// Rare path of a G-point group: for every query some lane's filter
// flagged (hq), re-derive the group's fp32 filter values, build the bitmask of pairs that
// pass the exact-safe fp32 threshold and re-check only those with the CANONICAL distance
// on the original coordinates; the insertion is decided on that value.  One threshold
// update per group (all of the group's candidates were checked against the current k-th
// distance).  `on_thr` is called with the query slot after its threshold changed.
template <int K, int Q, int G, typename T, class OnThr>
__device__ __forceinline__ void knn_rare_group_impl(KnnF32State<K, Q, T> &st, const bool (&hq)[Q],
                                                    const float *__restrict__ tcx, const float *__restrict__ tcy,
                                                    const float *__restrict__ tpp, const T *__restrict__ tpx,
                                                    const T *__restrict__ tpy, int j, OnThr &&on_thr)
{
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        if (!__any_sync(0xffffffffu, hq[q])) continue;
        unsigned mask = 0;
        if (hq[q]) {
#pragma unroll
            for (int c = 0; c < G; c += 8) {
                float t[8];
                filter8(st, q, tcx, tcy, tpp, j + c, t);
#pragma unroll
                for (int e = 0; e < 8; ++e) mask |= (t[e] <= st.thr[q]) ? (1u << (c + e)) : 0u;
            }
        }
        bool inserted = false;
        while (__any_sync(0xffffffffu, mask != 0)) {
            if (mask) {
                const int e = __ffs(mask) - 1;
                mask &= mask - 1;
                const T s = dist_sq(st.qx[q], st.qy[q], tpx[j + e], tpy[j + e]);
                if (s < st.buf[q][K - 1]) {
                    topk_insert<T, K>(st.buf[q], s);
                    inserted = true;
                }
            }
        }
        if (inserted) {
            st.thr[q] = thr_of(thr_f32(st.buf[q][K - 1]), st.qqf[q], st.mf[q], st.Ef[q]);
            on_thr(q);
        }
    }
}

template <int K, int Q, int G, typename T>
__device__ __forceinline__ void knn_rare_group(KnnF32State<K, Q, T> &st, const bool (&hq)[Q],
                                               const float *__restrict__ tcx, const float *__restrict__ tcy,
                                               const float *__restrict__ tpp, const T *__restrict__ tpx,
                                               const T *__restrict__ tpy, int j)
{
    knn_rare_group_impl<K, Q, G>(st, hq, tcx, tcy, tpp, tpx, tpy, j, [](int) {});
}

// One smem tile of TILE points in groups of G points per warp vote.  The main loop keeps
// only a running 3-input-min per query (chunks of 8 points: 8 FFMA2 + 4 FMNMX3 per query,
// the smem loads shared by the Q queries); a group that passes for some lane re-derives
// its t values in the rare path, builds the bitmask of passing pairs and re-checks only
// those with the canonical distance.
// tpx, tpy: the tile's original coordinates for the canonical re-check -- the smem tile
// (fp32) or the global fp64 arrays at the tile's offset (fp64; read only in the rare path).
template <int K, int Q, int G, int TILE, typename T = float>
__device__ __forceinline__ void knn_f32_tile(KnnF32State<K, Q, T> &st, const float *__restrict__ tcx,
                                             const float *__restrict__ tcy, const float *__restrict__ tpp,
                                             const T *__restrict__ tpx, const T *__restrict__ tpy)
{
    static_assert(G % 8 == 0 && G <= 32 && TILE % G == 0, "group size");
    const uint32_t acx = smem_addr(tcx), acy = smem_addr(tcy), app = smem_addr(tpp);
#pragma unroll 1
    for (int j = 0; j < TILE; j += G) {
        float mn[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) mn[q] = pos_inf<float>();
#pragma unroll
        for (int c = 0; c < G; c += 8) {
            float cxv[8], cyv[8], ppv[8];
#pragma unroll
            for (int g = 0; g < 8; g += 4) {
                const uint32_t o = (uint32_t)(j + c + g) * 4u;
                const float4 CX = lds128(acx + o);
                const float4 CY = lds128(acy + o);
                const float4 PP = lds128(app + o);
                cxv[g] = CX.x; cxv[g + 1] = CX.y; cxv[g + 2] = CX.z; cxv[g + 3] = CX.w;
                cyv[g] = CY.x; cyv[g + 1] = CY.y; cyv[g + 2] = CY.z; cyv[g + 3] = CY.w;
                ppv[g] = PP.x; ppv[g + 1] = PP.y; ppv[g + 2] = PP.z; ppv[g + 3] = PP.w;
            }
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                float t[8];
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const f32x2 tt = fma2(splat2(st.B[q]), pack2(cyv[2 * h], cyv[2 * h + 1]),
                                          fma2(splat2(st.A[q]), pack2(cxv[2 * h], cxv[2 * h + 1]),
                                               pack2(ppv[2 * h], ppv[2 * h + 1])));
                    t[2 * h] = tt.x;
                    t[2 * h + 1] = tt.y;
                }
                mn[q] = fmin3(fmin3(t[0], t[1], t[2]), fmin3(t[3], t[4], t[5]), fmin3(t[6], t[7], mn[q]));
            }
        }
        bool hq[Q], hit = false;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            hq[q] = mn[q] <= st.thr[q];
            hit |= hq[q];
        }
        if (__any_sync(0xffffffffu, hit)) knn_rare_group<K, Q, G>(st, hq, tcx, tcy, tpp, tpx, tpy, j);
    }
}

// ---------------------------------------------------------------------------------
// fp16 pre-filter of the fp32 kNN (round 2).  The CTA's queries are
// spatial neighbours (Morton order, §4.7); with C their bbox centre and sigma a power of
// two, every data point of a tile is converted ONCE per CTA to fp16 û = fl16(sigma (x - C_x)),
// v̂ likewise, p̂p = fl16(û² + v̂²), and the main loop evaluates t̂ = p̂p + Â û + B̂ v̂ on
// HFMA2 (two points per instruction) with a packed HMNMX2 min tree -- 25 % more pairs per
// clock than the FFMA2 + FMNMX3 loop (tools/knn_loop_bench.cu).  A group flagged by the
// fp16 test goes to the SAME rare path as before (exact-safe fp32 filter, then the
// canonical re-check), so the fp16 stage only has to keep every true candidate: its
// threshold T (h16_threshold) is the k-th canonical distance on the t scale plus a
// rigorous bound of every rounding (coordinates, p̂p, the two fp16 FMAs, subnormals).
// Conversions clamp |û|, |v̂| <= 256 and p̂p <= 32768; sigma keeps |q̃| and the candidates'
// radius r within 16, so no candidate is clamped or overflows, and clamped far points
// land at t̂ >= 16384, far above T.
template <int Q> struct KnnH16 {
    __half2 A[Q], B[Q];  // splats of fl16(-2 sigma (q - C))
    float T[Q];          // STRIP threshold on the strip axis' t scale (fp32, rounded up; the
                         // 2-D threshold is derived from it, h16_t2d); -inf for empty slots
};

constexpr float kH16Clamp = 256.0f, kH16PPClamp = 32768.0f, kH16Radius = 16.0f;

// T for a canonical k-th distance v (DESIGN.md §4.1 "fp16 pre-filter margin"): a true
// candidate has s_canon < v, so sigma² s_exact <= r², r = sigma sqrt(v (1 + 2^-20)); with
// Q = sigma |q - C|, p = q + d (|d| <= r): |p̃| <= P = Q + r, the rounded coordinates move
// the pair by Delta <= up (2Q + r), |first FMA| <= (P + Delta)², |t̂| <= Q² + (r + Delta)²,
// and t̂ <= (r + Delta)² - |q̂|² + up (P + Delta)² + 1.002 u16 ((P + Delta)² + Q² + (r + Delta)²)
// + 2^-18 (absolute slack: fp16 subnormal coordinates and results, <= 2^-25 each; sigma
// keeps the candidates' scaled magnitudes O(1..32), so this is far below T).  |q̂|² is exact
// from the fp16 coefficients.
// Round 2 (the strip pre-test): the function returns the threshold of the ONE-axis test
// t̂1 = p̂s + Ŝ ŝ (ŝ = û for AXIS 0, v̂ for AXIS 1; p̂s = fl16(ŝ²)): a true candidate is
// within R = r + Delta of the query along that axis too, and every rounding term of the
// 2-D bound dominates its one-axis counterpart, so the same formula with |q̂|² replaced by
// the strip axis' share â² (A is the strip axis' coefficient) bounds t̂1.  The 2-D
// threshold is T1 - b̂², rounded up (h16_t2d).  !STRIP: the 2-D threshold itself.
// The CTA's fp16 frame (CTA-uniform, kept in shared memory: only the rare path reads it).
// The converted points are fl16(sigma (p' - C)) with p' the tile's coordinates: the data
// coordinates themselves (fp32 handles, o = 0) or the centred filter coordinates
// cx = fl32(x - c) of fp64 handles (o = c, `centred`).  In the latter each converted
// coordinate (point and query alike) carries the centring rounding, <= 2^-24 |x - c| per
// axis, so the displacement bound Delta grows by sigma 2^-23 (r1 + |q - c|_1) (r1 >= the
// data's largest |x - c|_1; factor 2 of slack).
struct H16Frame {
    double Cx, Cy;  // C in the data's coordinates (o + the centre on the converted scale)
    double ox, oy;  // o
    double r1;      // centred: r1; else 0
    float sig;
    int centred;
};

template <bool STRIP, typename T>
__device__ __forceinline__ float h16_threshold(T v, T qx, T qy, const H16Frame &fr, __half2 A, __half2 B)
{
    if (!(v < pos_inf<T>())) return pos_inf<float>();
    const double u16 = 0x1p-11, up = 0x1p-11 + 0x1p-22;
    const double sig = (double)fr.sig;
    const double dx = (double)qx - fr.Cx, dy = (double)qy - fr.Cy;
    const double Qn = sig * sqrt(dx * dx + dy * dy) * (1.0 + 0x1p-40);
    const double r = sig * sqrt((double)v * (1.0 + 0x1p-20));
    const double ah = 0.5 * (double)__low2float(A), bh = 0.5 * (double)__low2float(B);
    const double qq = ah * ah + bh * bh;  // |q̂|², exact
    const double Qb = fmax(Qn, sqrt(qq)) * (1.0 + up);
    const double ce = fr.centred ? sig * 0x1p-23 * (fr.r1 + fabs((double)qx - fr.ox) + fabs((double)qy - fr.oy)) * 1.001
                                 : 0.0;
    const double D = up * (2.0 * Qb + r) + ce;
    const double P = Qb + r + D, R = r + D;
    const double th = R * R - (STRIP ? ah * ah : qq) + up * P * P + 1.002 * u16 * (P * P + Qb * Qb + R * R) +
                      0x1p-18;
    return __double2float_ru(th);
}

// The 2-D test's threshold from the strip threshold T1: T1 - (B/2)², the product exact in
// fp32 (11-bit operands), one upward rounding.
__device__ __forceinline__ float h16_t2d(float T1, __half2 B)
{
    const float o = 0.5f * __low2float(B);
    return __fmaf_ru(-o, o, T1);
}

// One tile's fp16 copy: TILE/2 couples of (û, v̂, p̂p) and the strip squares p̂s = fl16(û²)
// (exact in fp32 before the rounding: 11-bit operands), all threads of the CTA.  With
// axis == 1 the CTA's strip axis is y: û and v̂ trade places (so do the query
// coefficients, knn_filter_kernel), t̂ is symmetric in the two.
template <int TILE>
__device__ __forceinline__ void h16_convert(const float *__restrict__ tpx, const float *__restrict__ tpy,
                                            __half2 *__restrict__ hu, __half2 *__restrict__ hv,
                                            __half2 *__restrict__ hp, __half2 *__restrict__ hs, int axis,
                                            float Cx, float Cy, float sig)
{
    const f32x2 C2x = splat2(Cx), C2y = splat2(Cy), S2 = splat2(sig);
    auto couple = [&](f32x2 xr, f32x2 yr, __half2 &U, __half2 &V, __half2 &Pp, __half2 &Ps) {
        // packed fp32x2 arithmetic: each lane is the IEEE round-to-nearest scalar op
        const f32x2 x = mul2(sub2(xr, C2x), S2);
        const f32x2 y = mul2(sub2(yr, C2y), S2);
        const float u0 = fminf(fmaxf(x.x, -kH16Clamp), kH16Clamp);
        const float u1 = fminf(fmaxf(x.y, -kH16Clamp), kH16Clamp);
        const float v0 = fminf(fmaxf(y.x, -kH16Clamp), kH16Clamp);
        const float v1 = fminf(fmaxf(y.y, -kH16Clamp), kH16Clamp);
        U = __floats2half2_rn(u0, u1);
        V = __floats2half2_rn(v0, v1);
        if (axis == 1) {  // the strip axis always goes first (the coefficients are swapped too)
            const __half2 w = U;
            U = V;
            V = w;
        }
        const f32x2 uf = __half22float2(U), vf = __half22float2(V);
        const f32x2 p = fma2(uf, uf, mul2(vf, vf));  // û² + v̂², exact (11-bit operands)
        const f32x2 q = mul2(uf, uf);                // û², exact
        Pp = __floats2half2_rn(fminf(p.x, kH16PPClamp), fminf(p.y, kH16PPClamp));
        Ps = __floats2half2_rn(fminf(q.x, kH16PPClamp), fminf(q.y, kH16PPClamp));
    };
    // four points per thread per pass: one LDS.128 per coordinate, 8-byte stores
    for (int i = threadIdx.x; i < TILE / 4; i += blockDim.x) {
        const float4 X = *reinterpret_cast<const float4 *>(tpx + 4 * i);
        const float4 Y = *reinterpret_cast<const float4 *>(tpy + 4 * i);
        __half2 U[2], V[2], Pp[2], Ps[2];
        couple(pack2(X.x, X.y), pack2(Y.x, Y.y), U[0], V[0], Pp[0], Ps[0]);
        couple(pack2(X.z, X.w), pack2(Y.z, Y.w), U[1], V[1], Pp[1], Ps[1]);
        *reinterpret_cast<uint2 *>(hu + 2 * i) = *reinterpret_cast<const uint2 *>(U);
        *reinterpret_cast<uint2 *>(hv + 2 * i) = *reinterpret_cast<const uint2 *>(V);
        *reinterpret_cast<uint2 *>(hp + 2 * i) = *reinterpret_cast<const uint2 *>(Pp);
        *reinterpret_cast<uint2 *>(hs + 2 * i) = *reinterpret_cast<const uint2 *>(Ps);
    }
}

// The fp16 main loop over one tile (same groups, votes and rare path as knn_f32_tile).
// STRIP (round 2, DESIGN.md §4.1 "strip pre-test"): every strip group of SGM * G points is
// first tested on ONE axis (the first, h16_convert), t̂1 = p̂s + Â û (one HFMA2 per couple
// instead of two: 1.6x the pairs per clock, tools/knn_loop_bench.cu) under one warp vote;
// a kept strip group runs the 2-D test per G-point group, and only a group that passes both
// reaches the rare path.  Both tests are necessary conditions of a true candidate, so the
// selected multiset is unchanged.  !STRIP: the 2-D test alone (AIDW_KNN_STRIP=0).
template <int K, int Q, int G, int TILE, bool STRIP, int SGM = 1, typename T = float>
__device__ __forceinline__ void knn_h16_tile(KnnF32State<K, Q, T> &st, KnnH16<Q> &h, const __half2 *hu,
                                             const __half2 *hv, const __half2 *hp, const __half2 *hs,
                                             const float *__restrict__ tcx, const float *__restrict__ tcy,
                                             const float *__restrict__ tpp, const T *__restrict__ tpx,
                                             const T *__restrict__ tpy, const H16Frame &fr)
{
    static_assert(G % 8 == 0 && G <= 32 && TILE % G == 0, "group size");
    const uint32_t au = smem_addr(hu), av = smem_addr(hv), ap = smem_addr(hp), aps = smem_addr(hs);
    // the 2-D test of group j: per-query flags (AND-ed into hq) and the warp vote
    auto test2d = [&](int j, bool (&hq)[Q]) -> bool {
        __half2 mn[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) mn[q] = __half2half2(__ushort_as_half((unsigned short)0x7c00));  // +inf
#pragma unroll
        for (int c = 0; c < G; c += 8) {
            const uint32_t o = (uint32_t)(j + c) * 2u;  // 8 points = 4 half2 = 16 bytes
            const float4 U4 = lds128(au + o), V4 = lds128(av + o), P4 = lds128(ap + o);
            const __half2 *u = reinterpret_cast<const __half2 *>(&U4);
            const __half2 *v = reinterpret_cast<const __half2 *>(&V4);
            const __half2 *pp = reinterpret_cast<const __half2 *>(&P4);
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                __half2 t[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) t[e] = __hfma2(h.B[q], v[e], __hfma2(h.A[q], u[e], pp[e]));
                mn[q] = __hmin2(__hmin2(__hmin2(t[0], t[1]), __hmin2(t[2], t[3])), mn[q]);
            }
        }
        bool hit = false;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const float2 m = __half22float2(mn[q]);
            const float T2 = STRIP ? h16_t2d(h.T[q], h.B[q]) : h.T[q];
            hq[q] = hq[q] && fminf(m.x, m.y) <= T2;
            hit |= hq[q];
        }
        return __any_sync(0xffffffffu, hit);
    };
    auto rare = [&](int j, const bool (&hq)[Q]) {
        knn_rare_group_impl<K, Q, G>(st, hq, tcx, tcy, tpp, tpx, tpy, j, [&](int q) {
            h.T[q] = h16_threshold<STRIP>(st.buf[q][K - 1], st.qx[q], st.qy[q], fr, h.A[q], h.B[q]);
        });
    };
    if constexpr (!STRIP) {
#pragma unroll 1
        for (int j = 0; j < TILE; j += G) {
            bool hq[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) hq[q] = true;
            if (test2d(j, hq)) rare(j, hq);
        }
    } else {
        // strip groups of SGM * G points per vote; a kept strip group runs the 2-D test per
        // G-point group
        constexpr int SG = SGM * G;
        static_assert(TILE % SG == 0, "strip group size");
#pragma unroll 1
        for (int j = 0; j < TILE; j += SG) {
            __half2 mn[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) mn[q] = __half2half2(__ushort_as_half((unsigned short)0x7c00));  // +inf
#pragma unroll
            for (int c = 0; c < SG; c += 8) {
                const uint32_t o = (uint32_t)(j + c) * 2u;
                const float4 S4 = lds128(au + o), P4 = lds128(aps + o);
                const __half2 *sv = reinterpret_cast<const __half2 *>(&S4);
                const __half2 *ps = reinterpret_cast<const __half2 *>(&P4);
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    __half2 t[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) t[e] = __hfma2(h.A[q], sv[e], ps[e]);
                    mn[q] = __hmin2(__hmin2(__hmin2(t[0], t[1]), __hmin2(t[2], t[3])), mn[q]);
                }
            }
            bool hs1[Q], hit = false;
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const float2 m = __half22float2(mn[q]);
                hs1[q] = fminf(m.x, m.y) <= h.T[q];
                hit |= hs1[q];
            }
            if (__any_sync(0xffffffffu, hit)) {
#pragma unroll 1
                for (int g = 0; g < SGM; ++g) {
                    bool hq[Q];
#pragma unroll
                    for (int q = 0; q < Q; ++q) hq[q] = hs1[q];
                    if (test2d(j + g * G, hq)) rare(j + g * G, hq);
                }
            }
        }
    }
}

// ------------------------------------------------------------------ fp64 log2 / exp2
// The fp64 weighting pass needs w to ~1e-12 relative (Z tolerance 1e-10), far below
// libdevice's cost (~90 FP64 ops per pair for log2 + exp2).  Both use a small table in
// shared memory (tools/gen_f64_tables.py) and a short Taylor polynomial:
//  log2(s) = e + LOGM[i] + log2(1 + t),  t = m * C[i] - 1, i = top 8 mantissa bits,
//            |t| <= 2^-9, degree kLog2Deg = 3 (truncation 5.2e-12); valid for normal s > 0.
//  exp2(x) = 2^j * T[k] * 2^r,  64x = 64j + k + 64r rounded, |r| <= 1/128, degree
//            kExp2Deg = 4 (truncation 3.8e-14); x clamped to >= -1000 (smaller weights vanish).
// (v11: 256/64-entry tables instead of 64/16 save 4 of ~29 FP64 ops per pair; round 2:
// the tolerance-driven degrees of DESIGN.md §4.9 save 3 more -- 21 FP64 ops per pair.)
__device__ __forceinline__ double log2_f64(double s, const double2 *__restrict__ tab)
{
    const unsigned long long bits = (unsigned long long)__double_as_longlong(s);
    const unsigned be = (unsigned)(bits >> 52) & 0x7ffu;
    const int i = (int)(bits >> (52 - kLog2TabBits)) & ((1 << kLog2TabBits) - 1);
    const double m = __longlong_as_double((long long)((bits & 0x000fffffffffffffull) | 0x3ff0000000000000ull));
    const double2 ci = tab[i];
    const double t = fma(m, ci.x, -1.0);
    double p = kLog2Poly[kLog2Deg - 1];
#pragma unroll
    for (int k = kLog2Deg - 2; k >= 0; --k) p = fma(p, t, kLog2Poly[k]);
    // exponent as double without a conversion: 2^52 + be, minus (2^52 + 1023)
    const double ed = __longlong_as_double((long long)(0x4330000000000000ull | be)) - (4503599627370496.0 + 1023.0);
    return ed + fma(p, t, ci.y);
}

__device__ __forceinline__ double exp2_f64(double x, const double *__restrict__ tab)
{
    constexpr double kM = 6755399441055744.0;  // 1.5 * 2^52
    x = fmax(x, -1000.0);
    constexpr double kN = (double)(1 << kExp2TabBits);
    const double t = fma(x, kN, kM);
    const double nd = t - kM;
    const double r = fma(nd, -1.0 / kN, x);
    const int n = (int)(unsigned)(unsigned long long)__double_as_longlong(t);
    double p = kExp2Poly[kExp2Deg];
#pragma unroll
    for (int k = kExp2Deg - 1; k >= 0; --k) p = fma(p, r, kExp2Poly[k]);
    const double y = tab[n & ((1 << kExp2TabBits) - 1)] * p;
    // multiply by 2^(n >> bits) through the exponent field (no overflow: y <= 2, n <= 0)
    return __longlong_as_double(__double_as_longlong(y) + ((long long)(n >> kExp2TabBits) << 52));
}

// ------------------------------------------------------------------ Eq. 4-6
struct Levels {
    double a[5];
};

// R = r_obs / r_exp (Eq. 4); mu (Eq. 5, first match
// in printed order, R8/R9/R10); alpha (Eq. 6, R12).  fp64 (R24).
__device__ __forceinline__ double alpha_eq(double robs, double r_exp, double rmin, double rmax, int mf,
                                           const Levels &lv)
{
    const double R = robs / r_exp;
    double mu;
    if (R <= rmin)
        mu = 0.0;
    else if (R <= rmax)
        mu = (mf == 0) ? 0.5 - 0.5 * cospi((R - rmin) / (rmax - rmin))
                       : 0.5 - 0.5 * cos(3.141592653589793 / rmax * (R - rmin));
    else
        mu = 1.0;
    if (mu <= 0.1) return lv.a[0];
    if (mu <= 0.3) return lv.a[0] * (1.0 - 5.0 * (mu - 0.1)) + 5.0 * lv.a[1] * (mu - 0.1);
    if (mu <= 0.5) return 5.0 * lv.a[2] * (mu - 0.3) + lv.a[1] * (1.0 - 5.0 * (mu - 0.3));
    if (mu <= 0.7) return lv.a[2] * (1.0 - 5.0 * (mu - 0.5)) + 5.0 * lv.a[3] * (mu - 0.5);
    if (mu <= 0.9) return 5.0 * lv.a[4] * (mu - 0.7) + lv.a[3] * (1.0 - 5.0 * (mu - 0.7));
    return lv.a[4];
}

// ------------------------------------------------------------------ weighting pass
// Per-thread state of the packed fp32 weighting pass for Q queries:
// w = 2^(c log2 s + b), c = -alpha/2, b = (alpha/2) log2(d1^2)  (R20).
template <int Q>
struct InterpF32State {
    f32x2 QX[Q], QY[Q], C[Q], B[Q];
    double SW[Q], SWZ[Q];  // job sums: block sums added in block order (R21)
    double BW[Q], BWZ[Q];  // current accumulation block

    __device__ __forceinline__ void init(int q, float x, float y, float alpha, float d1sq)
    {
        const float c = -0.5f * alpha;
        const float b = 0.5f * alpha * lg2_approx_noftz(d1sq);
        QX[q] = splat2(x);
        QY[q] = splat2(y);
        C[q] = splat2(c);
        B[q] = splat2(b);
        SW[q] = 0.0;
        SWZ[q] = 0.0;
        BW[q] = 0.0;
        BWZ[q] = 0.0;
    }
    __device__ __forceinline__ void end_block()
    {
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            SW[q] += BW[q];
            SWZ[q] += BWZ[q];
            BW[q] = 0.0;
            BWZ[q] = 0.0;
        }
    }
};



// One smem tile of the fp32 weighting pass with packed fp32x2 arithmetic.  Two
// consecutive data points of one query form a "couple" in one register pair; the fp32
// tile sums are {even, odd} partial sums folded into fp64 at the end of the tile (R21).
// The ex2 of couple (q, h) runs on the FMA pipe (exp2_poly2) when bit 2q+h of EMU is
// set, on the SFU otherwise.
template <int Q, unsigned HMASK, bool CLAMP = true>
__device__ __forceinline__ void interp_f32_group(InterpF32State<Q> &st, f32x2 (&sw)[Q], f32x2 (&swz)[Q],
                                                 const float *__restrict__ tx, const float *__restrict__ ty,
                                                 const float *__restrict__ tz)
{
    const float4 X = *reinterpret_cast<const float4 *>(tx);
    const float4 Y = *reinterpret_cast<const float4 *>(ty);
    const float4 Z = *reinterpret_cast<const float4 *>(tz);
    const f32x2 Xh[2] = {pack2(X.x, X.y), pack2(X.z, X.w)};
    const f32x2 Yh[2] = {pack2(Y.x, Y.y), pack2(Y.z, Y.w)};
    const f32x2 Zh[2] = {pack2(Z.x, Z.y), pack2(Z.z, Z.w)};
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const f32x2 dx = sub2(st.QX[q], Xh[h]);
            const f32x2 dy = sub2(st.QY[q], Yh[h]);
            const f32x2 s = fma2(dx, dx, mul2(dy, dy));
            const f32x2 l = pack2(lg2_approx(s.x), lg2_approx(s.y));
            const f32x2 e = fma2(st.C[q], l, st.B[q]);
            f32x2 w;
            const unsigned m = (HMASK >> (2 * h)) & 3u;
            if (m == 1u)
                w = exp2_poly2<CLAMP>(e);  // both lanes on the FMA pipe (packed)
            else if (m == 2u)
                w = pack2(ex2_approx(e.x), exp2_poly1<CLAMP>(e.y));  // split: SFU + FMA pipe
            else
                w = pack2(ex2_approx(e.x), ex2_approx(e.y));
            sw[q] = add2(sw[q], w);
            swz[q] = fma2(w, Zh[h], swz[q]);
        }
}

// One smem tile of the fp32 weighting pass with packed fp32x2 arithmetic.  Two
// consecutive data points of one query form a "couple" in one register pair; the fp32
// tile sums are {even, odd} partial sums folded into fp64 at the end of the tile (R21).
// The exp2 of couple h of 4-point group g (g = 0..3 within each 16 points) is chosen by
// the 2-bit field at bit 4g+2h of EMU: 0 = both lanes on the SFU, 1 = both on the FMA
// pipe (packed polynomial), 2 = split (lane x on the SFU, lane y on the FMA pipe)
// (DESIGN.md §4.3).  The choice depends on the data-point index only -- never on which register
// slot holds the query -- so every query's rounding is independent of its position in
// the launch (bit-identical results for any sharding).
template <int Q, unsigned EMU, int TILE, bool CLAMP = true>
__device__ __forceinline__ void interp_f32_tile(InterpF32State<Q> &st, const float *__restrict__ tx,
                                                const float *__restrict__ ty, const float *__restrict__ tz)
{
    static_assert(TILE % 16 == 0, "tile");
    f32x2 sw[Q], swz[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) sw[q] = swz[q] = make_float2(0.f, 0.f);
#pragma unroll 1
    for (int j = 0; j < TILE; j += 16) {
        interp_f32_group<Q, (EMU >> 0) & 15u, CLAMP>(st, sw, swz, tx + j, ty + j, tz + j);
        interp_f32_group<Q, (EMU >> 4) & 15u, CLAMP>(st, sw, swz, tx + j + 4, ty + j + 4, tz + j + 4);
        interp_f32_group<Q, (EMU >> 8) & 15u, CLAMP>(st, sw, swz, tx + j + 8, ty + j + 8, tz + j + 8);
        interp_f32_group<Q, (EMU >> 12) & 15u, CLAMP>(st, sw, swz, tx + j + 12, ty + j + 12, tz + j + 12);
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        st.BW[q] += (double)sw[q].x + (double)sw[q].y;
        st.BWZ[q] += (double)swz[q].x + (double)swz[q].y;
    }
}

// ---------------------------------------------------------------------------------
// Exact-exponent classes of the weighting pass: Eq. 6 is flat on
// mu <= 0.1 (alpha = alpha_1) and mu >= 0.9 (alpha = alpha_5), so whole ranges of queries
// share one power; when that power is 1, 2 or 3 the weight d^-alpha needs ONE SFU op
// instead of log2 + exp2:  alpha = 1: w = rsqrt(s);  2: w = rcp(s);  3: w = rsqrt(s)^3.
// (Unscaled by the nearest distance -- the factor cancels in Eq. 1 and these powers
// cannot overflow fp32 for distances >= 2^-42.)  A query's class depends only on its
// alpha VALUE, so its arithmetic never depends on which CTA or slot evaluates it.
enum : int { kClsGeneral = 0, kClsA1 = 1, kClsA2 = 2, kClsA3 = 3, kClsMixed = 4 };

// The unscaled special weights stay in fp32 range (no overflow of a 512-term tile sum,
// no underflow of the nearest weights) for 2^-78 <= d1sq <= 2^66; outside it the
// general, nearest-scaled formula is used.
__device__ __forceinline__ int alpha_class(float alpha, float d1sq)
{
    if (!(d1sq >= 0x1p-78f && d1sq <= 0x1p66f)) return kClsGeneral;
    return alpha == 1.0f ? kClsA1 : alpha == 2.0f ? kClsA2 : alpha == 3.0f ? kClsA3 : kClsGeneral;
}

template <int CLS>
__device__ __forceinline__ f32x2 special_w(f32x2 s)
{
    if (CLS == kClsA1) return pack2(rsqrt_approx(s.x), rsqrt_approx(s.y));
    if (CLS == kClsA2) return pack2(rcp_approx(s.x), rcp_approx(s.y));
    const f32x2 r = pack2(rsqrt_approx(s.x), rsqrt_approx(s.y));
    return mul2(mul2(r, r), r);
}

// One 4-point group for a CTA whose queries all have class CLS (A1/A2/A3), or, for
// CLS == kClsMixed, per-lane selection among the four formulas (rare: class boundaries).
template <int Q, int CLS, unsigned HMASK>
__device__ __forceinline__ void interp_f32_group_cls(InterpF32State<Q> &st, const int (&cls)[Q],
                                                     f32x2 (&sw)[Q], f32x2 (&swz)[Q], const float *__restrict__ tx,
                                                     const float *__restrict__ ty, const float *__restrict__ tz)
{
    const float4 X = *reinterpret_cast<const float4 *>(tx);
    const float4 Y = *reinterpret_cast<const float4 *>(ty);
    const float4 Z = *reinterpret_cast<const float4 *>(tz);
    const f32x2 Xh[2] = {pack2(X.x, X.y), pack2(X.z, X.w)};
    const f32x2 Yh[2] = {pack2(Y.x, Y.y), pack2(Y.z, Y.w)};
    const f32x2 Zh[2] = {pack2(Z.x, Z.y), pack2(Z.z, Z.w)};
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const f32x2 dx = sub2(st.QX[q], Xh[h]);
            const f32x2 dy = sub2(st.QY[q], Yh[h]);
            const f32x2 s = fma2(dx, dx, mul2(dy, dy));
            f32x2 w;
            if (CLS != kClsMixed) {
                w = special_w<CLS>(s);
            } else {
                const int c = cls[q];
                if (c == kClsA1)
                    w = special_w<kClsA1>(s);
                else if (c == kClsA2)
                    w = special_w<kClsA2>(s);
                else if (c == kClsA3)
                    w = special_w<kClsA3>(s);
                else {  // the general formula with the SAME offload choice as interp_f32_group
                    const f32x2 l = pack2(lg2_approx(s.x), lg2_approx(s.y));
                    const f32x2 e = fma2(st.C[q], l, st.B[q]);
                    const unsigned m = (HMASK >> (2 * h)) & 3u;
                    if (m == 1u)
                        w = exp2_poly2(e);
                    else if (m == 2u)
                        w = pack2(ex2_approx(e.x), exp2_poly1(e.y));
                    else
                        w = pack2(ex2_approx(e.x), ex2_approx(e.y));
                }
            }
            sw[q] = add2(sw[q], w);
            swz[q] = fma2(w, Zh[h], swz[q]);
        }
}

template <int Q, int CLS, unsigned EMU, int TILE>
__device__ __forceinline__ void interp_f32_tile_cls(InterpF32State<Q> &st, const int (&cls)[Q],
                                                    const float *__restrict__ tx, const float *__restrict__ ty,
                                                    const float *__restrict__ tz)
{
    static_assert(TILE % 16 == 0, "tile");
    f32x2 sw[Q], swz[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) sw[q] = swz[q] = make_float2(0.f, 0.f);
#pragma unroll 1
    for (int j = 0; j < TILE; j += 16) {
        interp_f32_group_cls<Q, CLS, (EMU >> 0) & 15u>(st, cls, sw, swz, tx + j, ty + j, tz + j);
        interp_f32_group_cls<Q, CLS, (EMU >> 4) & 15u>(st, cls, sw, swz, tx + j + 4, ty + j + 4, tz + j + 4);
        interp_f32_group_cls<Q, CLS, (EMU >> 8) & 15u>(st, cls, sw, swz, tx + j + 8, ty + j + 8, tz + j + 8);
        interp_f32_group_cls<Q, CLS, (EMU >> 12) & 15u>(st, cls, sw, swz, tx + j + 12, ty + j + 12, tz + j + 12);
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        st.BW[q] += (double)sw[q].x + (double)sw[q].y;
        st.BWZ[q] += (double)swz[q].x + (double)swz[q].y;
    }
}

// Exact coincidence (R19): the limit of Eq. 1 is the mean z of the data points at
// distance 0.  Rare; one extra pass over global memory for the calling lane.
template <typename T>
__device__ __forceinline__ void coincident_sums(T qx, T qy, const T *px, const T *py, const T *pz, int64_t nd,
                                                double &zc, double &cnt)
{
    zc = 0.0;
    cnt = 0.0;
    for (int64_t i = 0; i < nd; ++i)
        if (dist_sq(qx, qy, px[i], py[i]) == T(0)) {
            zc += (double)pz[i];
            cnt += 1.0;
        }
}

template <typename T>
__device__ __forceinline__ double coincident_mean(T qx, T qy, const T *px, const T *py, const T *pz, int64_t nd)
{
    double zc, cnt;
    coincident_sums<T>(qx, qy, px, py, pz, nd, zc, cnt);
    return zc / cnt;
}

// fp32 weighting with a SUBNORMAL nearest squared distance (0 < d1sq < 2^-126; tiny
// coordinates, or a query ~1e-19 from a data point near the origin): the packed loop's
// lg2.approx.ftz flushes subnormal s to -inf and its sums are not usable.  Rare; the lane
// re-evaluates Eq. 1 over global memory in fp64 with the same nearest-scaled weights
// w = (s / d1sq)^(-alpha/2) (R20), so data-sharded partials stay on one scale.
__device__ __forceinline__ void tiny_nearest_sums(float qx, float qy, const float *px, const float *py,
                                                  const float *pz, int64_t nd, double d1, double alpha,
                                                  double &SW, double &SWZ)
{
    SW = 0.0;
    SWZ = 0.0;
    for (int64_t i = 0; i < nd; ++i) {
        const double s = dist_sq((double)qx, (double)qy, (double)px[i], (double)py[i]);
        const double w = pow(s / d1, -0.5 * alpha);
        SW += w;
        SWZ += w * (double)pz[i];
    }
}

// Per-query result: Z (Eq. 1, or the coincidence mean R19), or -- in data-sharded mode --
// this shard's fp64 partials {sum w, sum w z, sum z_coincident, n_coincident}.
template <typename T>
__device__ __forceinline__ void write_result(T *z, double *partial, int64_t idx, double SW, double SWZ, T d1, T qx,
                                             T qy, const T *px, const T *py, const T *pz, int64_t nd, double alpha)
{
    double zc = 0.0, nc = 0.0;
    if (d1 == T(0)) coincident_sums<T>(qx, qy, px, py, pz, nd, zc, nc);
    if constexpr (sizeof(T) == 4)
        if (d1 > T(0) && d1 < 0x1p-126f) tiny_nearest_sums(qx, qy, px, py, pz, nd, (double)d1, alpha, SW, SWZ);
    if (partial) {
        partial[4 * idx] = SW;
        partial[4 * idx + 1] = SWZ;
        partial[4 * idx + 2] = zc;
        partial[4 * idx + 3] = nc;
    } else {
        z[idx] = (T)(d1 == T(0) ? zc / nc : SWZ / SW);
    }
}

}  // namespace aidw
