// interpolate.cu -- S5 of the AIDW hot path on sm_100a: the Shepard weighted
// average over ALL data points (Eq. 1; "calculate the distances
// to all the data points again") with the per-query alpha.
//
// Weights are evaluated as w = 2^(c*log2(s) + b) with s the squared distance,
// c = -alpha/2 and b = (alpha/2) log2(d1sq): w = (d/d1)^-alpha, i.e. Eq. 1's
// d^-alpha scaled by the (cancelling) factor d1^alpha so w is in (0, 1] for any
// coordinate scale.  fp32: MUFU lg2.approx / ex2.approx (2 SFU ops per pair, the
// binding pipe -- DESIGN.md §4.3); sums in fp32 within a kTileW-point tile and in
// fp64 across tiles (the paper's "two registers", made
// accurate for 1M-term sums).  fp64: libdevice log2/exp2, fp64 sums.
//
// Same smem ring as knn_robs.cu (TMA bulk copies of x, y, z tiles, mbarriers),
// Q queries per thread, every data point read once from smem per Q pairs.
#include "aidw_internal.h"
#include "device.cuh"
#include "packed.cuh"

#include <cstdlib>

namespace aidw {

template <typename T> struct InterpArgs {
    const T *px, *py, *pz;  // internal SoA padded with (+inf, +inf, 0)
    int64_t ndp, nd;
    const T *qx, *qy, *alpha, *d1sq;
    int64_t nq;
    T *z;
};

__device__ __forceinline__ float wlog2(float s) { return lg2_approx(s); }
__device__ __forceinline__ double wlog2(double s) { return log2(s); }
__device__ __forceinline__ float wexp2(float x) { return ex2_approx(x); }
__device__ __forceinline__ double wexp2(double x) { return exp2(x); }
__device__ __forceinline__ float log2_q(float s) { return lg2_approx_noftz(s); }
__device__ __forceinline__ double log2_q(double s) { return log2(s); }

template <typename T, int Q>
__global__ void __launch_bounds__(kBlock) interp_kernel(const InterpArgs<T> a)
{
    constexpr int TILE = kTileW, STAGES = kStagesW;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T *sx = reinterpret_cast<T *>(smem_raw);
    T *sy = sx + STAGES * TILE;
    T *sz = sy + STAGES * TILE;
    uint64_t *full = reinterpret_cast<uint64_t *>(sz + STAGES * TILE);
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
        mbar_arrive_expect_tx(&full[slot], 3u * TILE * sizeof(T));
        const int64_t off = (int64_t)tile * TILE;
        bulk_g2s(sx + slot * TILE, a.px + off, TILE * sizeof(T), &full[slot]);
        bulk_g2s(sy + slot * TILE, a.py + off, TILE * sizeof(T), &full[slot]);
        bulk_g2s(sz + slot * TILE, a.pz + off, TILE * sizeof(T), &full[slot]);
    };
    if (tid == 0)
        for (int s = 0; s < STAGES && s < ntiles; ++s) issue(s, s);

    const int64_t base = (int64_t)blockIdx.x * (kBlock * Q) + tid;
    T qx[Q], qy[Q], c[Q], b[Q], d1[Q];
    bool valid[Q];
    double SW[Q], SWZ[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const int64_t idx = base + q * kBlock;
        valid[q] = idx < a.nq;
        qx[q] = valid[q] ? a.qx[idx] : T(0);
        qy[q] = valid[q] ? a.qy[idx] : T(0);
        const T al = valid[q] ? a.alpha[idx] : T(1);
        d1[q] = valid[q] ? a.d1sq[idx] : T(1);
        c[q] = T(-0.5) * al;
        b[q] = T(0.5) * al * log2_q(d1[q]);
        SW[q] = 0.0;
        SWZ[q] = 0.0;
    }

    for (int t = 0; t < ntiles; ++t) {
        const int slot = t % STAGES;
        const uint32_t par = (uint32_t)(t / STAGES) & 1u;
        mbar_wait(&full[slot], par);
        const T *tx = sx + slot * TILE;
        const T *ty = sy + slot * TILE;
        const T *tz = sz + slot * TILE;
        T sw[Q], swz[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) sw[q] = swz[q] = T(0);
#pragma unroll 2
        for (int j = 0; j < TILE; j += 4) {
            const Vec4<T> X = lds4(tx + j), Y = lds4(ty + j), Z = lds4(tz + j);
#pragma unroll
            for (int e = 0; e < 4; ++e)
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    const T s = dist_sq(qx[q], qy[q], X.v[e], Y.v[e]);
                    const T w = wexp2(fma(c[q], wlog2(s), b[q]));
                    sw[q] += w;
                    swz[q] = fma(w, Z.v[e], swz[q]);
                }
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            SW[q] += (double)sw[q];
            SWZ[q] += (double)swz[q];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (tid == 0 && t + STAGES < ntiles) {
            mbar_wait(&empty[slot], par);
            issue(t + STAGES, slot);
        }
    }

#pragma unroll
    for (int q = 0; q < Q; ++q) {
        if (!valid[q]) continue;
        const int64_t idx = base + q * kBlock;
        double zq = SWZ[q] / SW[q];
        if (d1[q] == T(0)) {
            // Exact coincidence (R19): the limit of Eq. 1 is the mean z of
            // the data points at distance 0.  Rare; one extra pass for this lane.
            double zc = 0.0;
            long long cnt = 0;
            for (int64_t i = 0; i < a.nd; ++i)
                if (dist_sq(qx[q], qy[q], a.px[i], a.py[i]) == T(0)) {
                    zc += (double)a.pz[i];
                    ++cnt;
                }
            zq = zc / (double)cnt;
        }
        a.z[idx] = (T)zq;
    }
}

template <typename T, int Q>
static int launch_interp_t(const InterpArgs<T> &a, cudaStream_t st)
{
    const size_t smem = (size_t)3 * kStagesW * kTileW * sizeof(T) + 2 * kStagesW * sizeof(uint64_t);
    if (cudaFuncSetAttribute(interp_kernel<T, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return -1;
    const int64_t per_cta = (int64_t)kBlock * Q;
    const unsigned grid = (unsigned)((a.nq + per_cta - 1) / per_cta);
    interp_kernel<T, Q><<<grid, kBlock, smem, st>>>(a);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}


// ---------------------------------------------------------------------------------
// fp32 weighting pass with packed fp32x2 arithmetic (FADD2/FMUL2/FFMA2).  Two
// consecutive data points of one query form a "couple" evaluated in one packed
// register pair; the fp32 tile sums are kept as {even, odd} partial sums and folded
// into fp64 at every tile flush (R21).  The ex2 of couple (q, h) runs on
// the FMA pipe (exp2_poly2) when bit (2q + h) of EMU is set, on the SFU otherwise:
// this balances the SFU (8 issue-cycles per warp op) against the issue slot
// (DESIGN.md §4.3).
template <int Q, unsigned EMU>
__global__ void __launch_bounds__(kBlock) interp_f32x2_kernel(const InterpArgs<float> a)
{
    constexpr int TILE = kTileW, STAGES = kStagesW;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float *sx = reinterpret_cast<float *>(smem_raw);
    float *sy = sx + STAGES * TILE;
    float *sz = sy + STAGES * TILE;
    uint64_t *full = reinterpret_cast<uint64_t *>(sz + STAGES * TILE);
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
        mbar_arrive_expect_tx(&full[slot], 3u * TILE * sizeof(float));
        const int64_t off = (int64_t)tile * TILE;
        bulk_g2s(sx + slot * TILE, a.px + off, TILE * sizeof(float), &full[slot]);
        bulk_g2s(sy + slot * TILE, a.py + off, TILE * sizeof(float), &full[slot]);
        bulk_g2s(sz + slot * TILE, a.pz + off, TILE * sizeof(float), &full[slot]);
    };
    if (tid == 0)
        for (int s = 0; s < STAGES && s < ntiles; ++s) issue(s, s);

    const int64_t base = (int64_t)blockIdx.x * (kBlock * Q) + tid;
    float qx[Q], qy[Q], d1[Q];
    f32x2 QX[Q], QY[Q], C[Q], B[Q];
    bool valid[Q];
    double SW[Q], SWZ[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const int64_t idx = base + q * kBlock;
        valid[q] = idx < a.nq;
        qx[q] = valid[q] ? a.qx[idx] : 0.f;
        qy[q] = valid[q] ? a.qy[idx] : 0.f;
        const float al = valid[q] ? a.alpha[idx] : 1.f;
        d1[q] = valid[q] ? a.d1sq[idx] : 1.f;
        const float c = -0.5f * al;
        const float b = 0.5f * al * lg2_approx_noftz(d1[q]);
        QX[q] = splat2(qx[q]);
        QY[q] = splat2(qy[q]);
        C[q] = splat2(c);
        B[q] = splat2(b);
        SW[q] = 0.0;
        SWZ[q] = 0.0;
    }

    for (int t = 0; t < ntiles; ++t) {
        const int slot = t % STAGES;
        const uint32_t par = (uint32_t)(t / STAGES) & 1u;
        mbar_wait(&full[slot], par);
        const float *tx = sx + slot * TILE;
        const float *ty = sy + slot * TILE;
        const float *tz = sz + slot * TILE;
        f32x2 sw[Q], swz[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) sw[q] = swz[q] = make_float2(0.f, 0.f);
#pragma unroll 2
        for (int j = 0; j < TILE; j += 4) {
            const float4 X = *reinterpret_cast<const float4 *>(tx + j);
            const float4 Y = *reinterpret_cast<const float4 *>(ty + j);
            const float4 Z = *reinterpret_cast<const float4 *>(tz + j);
            const f32x2 Xh[2] = {pack2(X.x, X.y), pack2(X.z, X.w)};
            const f32x2 Yh[2] = {pack2(Y.x, Y.y), pack2(Y.z, Y.w)};
            const f32x2 Zh[2] = {pack2(Z.x, Z.y), pack2(Z.z, Z.w)};
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    const f32x2 dx = sub2(QX[q], Xh[h]);
                    const f32x2 dy = sub2(QY[q], Yh[h]);
                    const f32x2 s = fma2(dx, dx, mul2(dy, dy));
                    float s0, s1;
                    unpack2(s, s0, s1);
                    const f32x2 l = pack2(lg2_approx(s0), lg2_approx(s1));
                    const f32x2 e = fma2(C[q], l, B[q]);
                    f32x2 w;
                    if (EMU & (1u << (2 * q + h))) {
                        w = exp2_poly2(e);
                    } else {
                        float e0, e1;
                        unpack2(e, e0, e1);
                        w = pack2(ex2_approx(e0), ex2_approx(e1));
                    }
                    sw[q] = add2(sw[q], w);
                    swz[q] = fma2(w, Zh[h], swz[q]);
                }
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            float w0, w1, z0, z1;
            unpack2(sw[q], w0, w1);
            unpack2(swz[q], z0, z1);
            SW[q] += (double)w0 + (double)w1;
            SWZ[q] += (double)z0 + (double)z1;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (tid == 0 && t + STAGES < ntiles) {
            mbar_wait(&empty[slot], par);
            issue(t + STAGES, slot);
        }
    }

#pragma unroll
    for (int q = 0; q < Q; ++q) {
        if (!valid[q]) continue;
        const int64_t idx = base + q * kBlock;
        double zq = SWZ[q] / SW[q];
        if (d1[q] == 0.f) {  // exact coincidence (R19)
            double zc = 0.0;
            long long cnt = 0;
            for (int64_t i = 0; i < a.nd; ++i)
                if (dist_sq(qx[q], qy[q], a.px[i], a.py[i]) == 0.f) {
                    zc += (double)a.pz[i];
                    ++cnt;
                }
            zq = zc / (double)cnt;
        }
        a.z[idx] = (float)zq;
    }
}

template <int Q, unsigned EMU>
static int launch_interp_f32x2(const InterpArgs<float> &a, cudaStream_t st)
{
    const size_t smem = (size_t)3 * kStagesW * kTileW * sizeof(float) + 2 * kStagesW * sizeof(uint64_t);
    if (cudaFuncSetAttribute(interp_f32x2_kernel<Q, EMU>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return -1;
    const int64_t per_cta = (int64_t)kBlock * Q;
    const unsigned grid = (unsigned)((a.nq + per_cta - 1) / per_cta);
    interp_f32x2_kernel<Q, EMU><<<grid, kBlock, smem, st>>>(a);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// Variant selection for tuning (AIDW_INTERP_VARIANT); 0 = default.
static int interp_variant()
{
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("AIDW_INTERP_VARIANT");
        v = e ? atoi(e) : 0;
    }
    return v;
}

static int launch_interp_f32(const InterpArgs<float> &a, cudaStream_t st)
{
    switch (interp_variant()) {
    case 1: return launch_interp_t<float, 2>(a, st);         // scalar, all-SFU
    case 2: return launch_interp_f32x2<2, 0x0>(a, st);       // packed, all-SFU
    case 3: return launch_interp_f32x2<2, 0x5>(a, st);       // packed, 2 of 4 couples emulated
    case 4: return launch_interp_f32x2<2, 0x7>(a, st);       // 3 of 4
    case 5: return launch_interp_f32x2<2, 0xF>(a, st);       // 4 of 4
    case 6: return launch_interp_f32x2<4, 0x77>(a, st);      // Q=4, 6 of 8
    case 7: return launch_interp_f32x2<4, 0x7F>(a, st);      // Q=4, 7 of 8
    case 8: return launch_interp_f32x2<4, 0x55>(a, st);      // Q=4, 4 of 8
    case 9: return launch_interp_f32x2<4, 0x15>(a, st);      // Q=4, 3 of 8
    case 10: return launch_interp_f32x2<4, 0x57>(a, st);     // Q=4, 5 of 8
    case 11: return launch_interp_f32x2<2, 0x1>(a, st);      // Q=2, 1 of 4
    default: return launch_interp_f32x2<2, 0x5>(a, st);      // Q=2, 2 of 4 (best measured, r01)
    }
}

int launch_interp(int dtype, const void *data, int64_t ndp, int64_t nd, const void *qx,
                  const void *qy, int64_t nq, const void *alpha, const void *d1sq, void *z,
                  cudaStream_t st)
{
    if (dtype == 0) {
        const float *p = static_cast<const float *>(data);
        InterpArgs<float> a{p, p + ndp, p + 2 * ndp, ndp, nd, (const float *)qx, (const float *)qy,
                            (const float *)alpha, (const float *)d1sq, nq, (float *)z};
        return launch_interp_f32(a, st);
    }
    const double *p = static_cast<const double *>(data);
    InterpArgs<double> a{p, p + ndp, p + 2 * ndp, ndp, nd, (const double *)qx, (const double *)qy,
                         (const double *)alpha, (const double *)d1sq, nq, (double *)z};
    return launch_interp_t<double, 2>(a, st);
}

}  // namespace aidw
