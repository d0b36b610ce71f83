// alpha_prep.cu -- S0 (repack + bounding box) and S4 (R, mu_R, alpha) kernels.
#include "passes.cuh"

namespace aidw {

// ------------------------------------------------------------------ S0: prep
// Order-preserving map double -> uint64 (for atomicMin/Max of signed values).
__device__ __forceinline__ unsigned long long ord_key(double v)
{
    unsigned long long u = (unsigned long long)__double_as_longlong(v);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long t = __shfl_xor_sync(0xffffffffu, v, o);
        v = t < v ? t : v;
    }
    return v;
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long t = __shfl_xor_sync(0xffffffffu, v, o);
        v = t > v ? t : v;
    }
    return v;
}

// Repack the user layout (SoA / AoS / AoaS) into the internal
// padded SoA; padding points are (+inf, +inf, 0): never selected by the kNN,
// weight 0 in Eq. 1.  Also the exact bbox min/max (for A, Eq. 2) and a
// non-finite count.
template <typename T>
__global__ void prep_kernel(const T *__restrict__ src, int layout, int64_t nd, int64_t ndp,
                            T *__restrict__ data, Scratch *sc)
{
    T *px = data, *py = data + ndp, *pz = data + 2 * ndp;
    unsigned long long kx0 = ~0ull, kx1 = 0, ky0 = ~0ull, ky1 = 0, bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ndp;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (i < nd) {
            T x, y, z;
            if (layout == 0) {
                x = src[i];
                y = src[nd + i];
                z = src[2 * nd + i];
            } else if (layout == 1) {
                x = src[3 * i];
                y = src[3 * i + 1];
                z = src[3 * i + 2];
            } else {
                x = src[4 * i];
                y = src[4 * i + 1];
                z = src[4 * i + 2];
            }
            px[i] = x;
            py[i] = y;
            pz[i] = z;
            if (!(isfinite(x) && isfinite(y) && isfinite(z))) ++bad;
            const unsigned long long a = ord_key((double)x), b = ord_key((double)y);
            kx0 = a < kx0 ? a : kx0;
            kx1 = a > kx1 ? a : kx1;
            ky0 = b < ky0 ? b : ky0;
            ky1 = b > ky1 ? b : ky1;
        } else {
            px[i] = pos_inf<T>();
            py[i] = pos_inf<T>();
            pz[i] = T(0);
        }
    }
    kx0 = warp_min_u64(kx0);
    ky0 = warp_min_u64(ky0);
    kx1 = warp_max_u64(kx1);
    ky1 = warp_max_u64(ky1);
    bad = __reduce_add_sync(0xffffffffu, (unsigned)bad);
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&sc->keys[0], kx0);
        atomicMax(&sc->keys[1], kx1);
        atomicMin(&sc->keys[2], ky0);
        atomicMax(&sc->keys[3], ky1);
        if (bad) atomicAdd(&sc->nonfinite, bad);
    }
}

int launch_prep(int dtype, int layout, const void *src, int64_t nd, int64_t ndp, void *data,
                Scratch *sc, cudaStream_t st)
{
    const int threads = 256;
    int64_t blocks = (ndp + threads - 1) / threads;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (dtype == 0)
        prep_kernel<float><<<(unsigned)blocks, threads, 0, st>>>((const float *)src, layout, nd, ndp,
                                                                  (float *)data, sc);
    else
        prep_kernel<double><<<(unsigned)blocks, threads, 0, st>>>((const double *)src, layout, nd, ndp,
                                                                   (double *)data, sc);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// Centred fp32 copies and |p'|^2 for the kNN filter (knn_robs.cu): cx = x - c_x,
// cy = y - c_y (RN), pp = fma(cx, cx, cy*cy); padding (+inf).
// ------------------------------------------------------------------ S4: alpha
// Eq. 4-6 per query in fp64 (passes.cuh alpha_eq); GLOBAL bounds read on the device.
// GLOBAL bounds from the peer-memory exchange: thread 0 of each CTA
// waits until every rank's flag in this rank's ExBuf reached the epoch the preceding kNN
// epilogue published (acquire loads), then takes the MAX over ranks of {-min, max} from
// slot epoch & 1.  The last CTA to have read (ticket) acks the epoch into every rank's
// buffer, releasing that slot for epoch + 2.  A wait that exceeds ~2 s (a missing peer)
// sets ex_timeout for aidw_check and makes the bounds NaN, so alpha and Z come out NaN
// instead of silently using stale bounds.
__device__ void exchange_wait(Scratch *sc, double &v0, double &v1)
{
    __shared__ double s0, s1;
    if (threadIdx.x == 0) {
        const int n = sc->ex_world, me = sc->ex_rank;
        const unsigned long long ep = *reinterpret_cast<const volatile unsigned long long *>(&sc->ex_epoch);
        const ExBuf *b = sc->ex_peers[me];
        const long long t0 = clock64();
        bool ok = true;
        for (int r = 0; r < n; ++r) {
            unsigned long long f;
            for (;;) {
                asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(f) : "l"(&b->flag[r]) : "memory");
                if (f >= ep) break;
                if (clock64() - t0 > 4000000000ll) {
                    ok = false;
                    break;
                }
                __nanosleep(100);
            }
            if (!ok) break;
        }
        double a0 = -__longlong_as_double(0x7ff0000000000000ll), a1 = a0;
        const int slot = (int)(ep & 1);
        for (int r = 0; r < n; ++r) {
            a0 = fmax(a0, *reinterpret_cast<const volatile double *>(&b->val[slot][r][0]));
            a1 = fmax(a1, *reinterpret_cast<const volatile double *>(&b->val[slot][r][1]));
        }
        if (!ok) {
            atomicExch(&sc->ex_timeout, 1u);
            a0 = a1 = __longlong_as_double(0x7ff8000000000000ll);
        }
        s0 = a0;
        s1 = a1;
        __threadfence();
        if (atomicAdd(&sc->ex_readers, 1u) == gridDim.x - 1) {  // every CTA has read: ack
            sc->ex_readers = 0;
            __threadfence_system();
            for (int r = 0; r < n; ++r)
                asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(&sc->ex_peers[r]->ack[me]), "l"(ep)
                             : "memory");
        }
    }
    __syncthreads();
    v0 = s0;
    v1 = s1;
}

template <typename T>
__global__ void alpha_kernel(const T *__restrict__ robs, int64_t nq, double r_exp, Levels lv, int rb,
                             double rmin, double rmax, const T *__restrict__ mm, int mf,
                             T *__restrict__ alpha, Scratch *ex_sc)
{
    if (rb == 0) {  // GLOBAL: bounds on r_obs -> bounds on R (division is monotone)
        double m0, m1;
        if (ex_sc) {
            exchange_wait(ex_sc, m0, m1);
        } else {
            m0 = (double)mm[0];
            m1 = (double)mm[1];
        }
        rmin = -m0 / r_exp;
        rmax = m1 / r_exp;
    }
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nq;
         i += (int64_t)gridDim.x * blockDim.x)
        alpha[i] = (T)alpha_eq((double)robs[i], r_exp, rmin, rmax, mf, lv);
}

int launch_alpha(int dtype, const void *r_obs, int64_t nq, double r_exp, const double *lvp, int rb,
                 double rmin, double rmax, const void *minmax, int mf, void *alpha, cudaStream_t st,
                 Scratch *ex_sc)
{
    Levels lv;
    for (int i = 0; i < 5; ++i) lv.a[i] = lvp[i];
    const int threads = 256;
    int64_t blocks = (nq + threads - 1) / threads;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;  // nq == 0 with the exchange: read + ack only
    if (dtype == 0)
        alpha_kernel<float><<<(unsigned)blocks, threads, 0, st>>>(
            (const float *)r_obs, nq, r_exp, lv, rb, rmin, rmax, (const float *)minmax, mf, (float *)alpha, ex_sc);
    else
        alpha_kernel<double><<<(unsigned)blocks, threads, 0, st>>>(
            (const double *)r_obs, nq, r_exp, lv, rb, rmin, rmax, (const double *)minmax, mf,
            (double *)alpha, ex_sc);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace aidw
