// paper_kernels.cu -- N3: the paper's own GPU designs, recompiled for
// sm_100a, as the prior-art baseline of the Table-1-shaped ablation.
//
//  * naive (§3.2.1): one thread per query, registers + global memory
//    only; the kNN buffer pass over all data points, R / mu / alpha in the thread, then
//    a second pass over all data points for Eq. 1 with pow(); the two sums in REAL.
//  * tiled (§3.2.2): the same, but "the tile size is directly set as
//    the same as the block size": each thread loads one data point of the tile into
//    shared memory, __syncthreads, every thread consumes the tile; both passes tiled.
//  * layouts SoA (dx[], dy[], dz[]) and AoaS ((x, y, z, pad) records).
//
// These kernels are NOT the product path (they are what the product path is measured
// against).  FIXED R bounds only (the paper's per-thread structure has no global phase).
// Kept deliberately plain: REAL accumulators, libm pow, per-thread branchy insertion.
#include "passes.cuh"

namespace aidw {

template <typename T> struct PaperArgs {
    const T *data;  // SoA: x[nd], y[nd], z[nd];  AoaS: (x, y, z, pad) * nd
    int64_t nd;
    const T *qx, *qy;
    int64_t nq;
    int k;
    double r_exp;
    Levels lv;
    double rmin, rmax;
    T *z;
};

template <typename T, bool AOAS>
__device__ __forceinline__ void load_point(const T *d, int64_t nd, int64_t i, T &x, T &y, T &z)
{
    if (AOAS) {
        x = d[4 * i];
        y = d[4 * i + 1];
        z = d[4 * i + 2];
    } else {
        x = d[i];
        y = d[nd + i];
        z = d[2 * nd + i];
    }
}

__device__ __forceinline__ float real_pow(float a, float b) { return powf(a, b); }
__device__ __forceinline__ double real_pow(double a, double b) { return pow(a, b); }

// Fig. 1 / Step 3: replace the k-th, then compare-and-swap neighbours down to the 1st.
template <typename T, int K>
__device__ __forceinline__ void paper_insert(T (&b)[K], int k, T d)
{
    if (d < b[k - 1]) {
        b[k - 1] = d;
#pragma unroll
        for (int i = K - 1; i > 0; --i)
            if (i < k && b[i] < b[i - 1]) {
                const T t = b[i];
                b[i] = b[i - 1];
                b[i - 1] = t;
            }
    }
}

template <typename T, int K>
__device__ __forceinline__ T paper_alpha(const T (&b)[K], int k, const PaperArgs<T> &a)
{
    T sum = T(0);
#pragma unroll
    for (int i = 0; i < K; ++i)
        if (i < k) sum += b[i];
    const T robs = sum / (T)k;
    return (T)alpha_eq((double)robs, a.r_exp, a.rmin, a.rmax, 0, a.lv);
}

template <typename T, int K, bool AOAS>
__global__ void __launch_bounds__(256) paper_naive_kernel(const PaperArgs<T> a)
{
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= a.nq) return;
    const T qx = a.qx[q], qy = a.qy[q];
    T buf[K];
#pragma unroll
    for (int i = 0; i < K; ++i) buf[i] = pos_inf<T>();
    for (int64_t i = 0; i < a.nd; ++i) {
        T x, y, z;
        load_point<T, AOAS>(a.data, a.nd, i, x, y, z);
        const T dx = qx - x, dy = qy - y;
        paper_insert<T, K>(buf, a.k, sqrt(dx * dx + dy * dy));
    }
    const T alpha = paper_alpha<T, K>(buf, a.k, a);
    T sw = T(0), swz = T(0), zc = T(0);
    int nc = 0;
    for (int64_t i = 0; i < a.nd; ++i) {
        T x, y, z;
        load_point<T, AOAS>(a.data, a.nd, i, x, y, z);
        const T dx = qx - x, dy = qy - y;
        const T d = sqrt(dx * dx + dy * dy);
        if (d == T(0)) {
            zc += z;
            ++nc;
            continue;
        }
        const T w = real_pow(d, -alpha);
        sw += w;
        swz += w * z;
    }
    a.z[q] = nc ? zc / (T)nc : swz / sw;
}

template <typename T, int K, bool AOAS>
__global__ void __launch_bounds__(256) paper_tiled_kernel(const PaperArgs<T> a)
{
    __shared__ T sx[256], sy[256], sz[256];
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = q < a.nq;
    const T qx = valid ? a.qx[q] : T(0), qy = valid ? a.qy[q] : T(0);
    T buf[K];
#pragma unroll
    for (int i = 0; i < K; ++i) buf[i] = pos_inf<T>();
    for (int64_t base = 0; base < a.nd; base += blockDim.x) {
        const int64_t i = base + threadIdx.x;
        T x = pos_inf<T>(), y = pos_inf<T>(), z = T(0);
        if (i < a.nd) load_point<T, AOAS>(a.data, a.nd, i, x, y, z);
        __syncthreads();
        sx[threadIdx.x] = x;
        sy[threadIdx.x] = y;
        __syncthreads();
        const int n = (int)min((int64_t)blockDim.x, a.nd - base);
        for (int j = 0; j < n; ++j) {
            const T dx = qx - sx[j], dy = qy - sy[j];
            paper_insert<T, K>(buf, a.k, sqrt(dx * dx + dy * dy));
        }
    }
    const T alpha = paper_alpha<T, K>(buf, a.k, a);
    T sw = T(0), swz = T(0), zc = T(0);
    int nc = 0;
    for (int64_t base = 0; base < a.nd; base += blockDim.x) {
        const int64_t i = base + threadIdx.x;
        T x = pos_inf<T>(), y = pos_inf<T>(), z = T(0);
        if (i < a.nd) load_point<T, AOAS>(a.data, a.nd, i, x, y, z);
        __syncthreads();
        sx[threadIdx.x] = x;
        sy[threadIdx.x] = y;
        sz[threadIdx.x] = z;
        __syncthreads();
        const int n = (int)min((int64_t)blockDim.x, a.nd - base);
        for (int j = 0; j < n; ++j) {
            const T dx = qx - sx[j], dy = qy - sy[j];
            const T d = sqrt(dx * dx + dy * dy);
            if (d == T(0)) {
                zc += sz[j];
                ++nc;
                continue;
            }
            const T w = real_pow(d, -alpha);
            sw += w;
            swz += w * sz[j];
        }
    }
    if (valid) a.z[q] = nc ? zc / (T)nc : swz / sw;
}

template <typename T, int K>
static int launch_paper_k(int variant, bool aoas, const PaperArgs<T> &a, cudaStream_t st)
{
    const unsigned grid = (unsigned)((a.nq + 255) / 256);
    if (variant == 0) {
        if (aoas)
            paper_naive_kernel<T, K, true><<<grid, 256, 0, st>>>(a);
        else
            paper_naive_kernel<T, K, false><<<grid, 256, 0, st>>>(a);
    } else {
        if (aoas)
            paper_tiled_kernel<T, K, true><<<grid, 256, 0, st>>>(a);
        else
            paper_tiled_kernel<T, K, false><<<grid, 256, 0, st>>>(a);
    }
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

template <typename T>
static int launch_paper_t(int variant, bool aoas, const PaperArgs<T> &a, cudaStream_t st)
{
    if (a.k <= 10) return launch_paper_k<T, 10>(variant, aoas, a, st);
    if (a.k <= 16) return launch_paper_k<T, 16>(variant, aoas, a, st);
    return launch_paper_k<T, 32>(variant, aoas, a, st);
}

int launch_paper(int variant, int dtype, int layout, const void *data, int64_t nd, const void *qx, const void *qy,
                 int64_t nq, int k, double r_exp, const double *lvp, double rmin, double rmax, void *z,
                 cudaStream_t st)
{
    Levels lv;
    for (int i = 0; i < 5; ++i) lv.a[i] = lvp[i];
    const bool aoas = layout == 2;
    if (dtype == 0) {
        PaperArgs<float> a{(const float *)data, nd, (const float *)qx, (const float *)qy, nq, k, r_exp, lv,
                           rmin, rmax, (float *)z};
        return launch_paper_t(variant, aoas, a, st);
    }
    PaperArgs<double> a{(const double *)data, nd, (const double *)qx, (const double *)qy, nq, k, r_exp, lv,
                        rmin, rmax, (double *)z};
    return launch_paper_t(variant, aoas, a, st);
}

}  // namespace aidw
