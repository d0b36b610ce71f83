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

int launch_interp(int dtype, const void *data, int64_t ndp, int64_t nd, const void *qx,
                  const void *qy, int64_t nq, const void *alpha, const void *d1sq, void *z,
                  cudaStream_t st)
{
    if (dtype == 0) {
        const float *p = static_cast<const float *>(data);
        InterpArgs<float> a{p, p + ndp, p + 2 * ndp, ndp, nd, (const float *)qx, (const float *)qy,
                            (const float *)alpha, (const float *)d1sq, nq, (float *)z};
        return launch_interp_t<float, 2>(a, st);
    }
    const double *p = static_cast<const double *>(data);
    InterpArgs<double> a{p, p + ndp, p + 2 * ndp, ndp, nd, (const double *)qx, (const double *)qy,
                         (const double *)alpha, (const double *)d1sq, nq, (double *)z};
    return launch_interp_t<double, 2>(a, st);
}

}  // namespace aidw
