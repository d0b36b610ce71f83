// order.cu -- spatial (Morton) order for the fp32 kNN pass.
//
// The brute-force kNN (every pair evaluated) does not depend on the
// order in which data points are visited or queries are assigned to threads: the k
// smallest distances are a multiset.  Its COST does: a point that enters a query's
// top-k costs an insertion, and with random orders every warp keeps meeting points
// that are near one of its 64 queries.  So
//  * a second copy of the kNN filter data is counting-sorted by Morton cell at handle
//    creation (the weighting pass, and kNN launches without a query order -- small or
//    split batches, for which a sorted scan would insert far more -- keep the caller's
//    order);
//  * each large query batch is counting-sorted the same way into a permutation, so a
//    CTA's 256 queries are neighbours;
//  * the kNN CTA starts its scan at the sorted data under its queries and wraps around.
// Order within a cell follows atomics and may differ between runs; no result depends on
// it.  Each sort is three kernels: cell histogram, single-CTA exclusive scan, scatter.
#include "passes.cuh"

namespace aidw {

namespace {

// (fp64 coordinates pick their cell in fp32: any order is valid, only its cost changes)
template <typename T>
__global__ void cell_hist_kernel(const T *__restrict__ x, const T *__restrict__ y, int64_t n, OrderGrid g,
                                 unsigned *__restrict__ counts)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&counts[morton_cell((float)x[i], (float)y[i], g)], 1u);
}

// Exclusive scan of kCells counts by one CTA of 32 warps: warp w owns the contiguous
// chunk [w*2048, (w+1)*2048) and reads it coalesced into registers (64 per lane, all
// loads in flight at once); warp totals are scanned in shared memory.  Writes
// start[0..kCells] (start[kCells] = total) and a cursor copy for the scatter.
constexpr int kScanThreads = 1024;
__global__ void __launch_bounds__(kScanThreads) cell_scan_kernel(const unsigned *__restrict__ counts,
                                                                 int *__restrict__ start, int *__restrict__ cursor)
{
    constexpr int kWarps = kScanThreads / 32, chunk = kCells / kWarps, per = chunk / 32, batch = 16;
    __shared__ unsigned wtot[kWarps];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned *src = counts + w * chunk + lane;
    unsigned tot = 0;
    for (int i0 = 0; i0 < per; i0 += batch) {  // pass 1: warp total (batches of 16 loads in flight)
        unsigned v[batch];
#pragma unroll
        for (int i = 0; i < batch; ++i) v[i] = src[(i0 + i) * 32];
#pragma unroll
        for (int i = 0; i < batch; ++i) tot += v[i];
    }
    tot = __reduce_add_sync(0xffffffffu, tot);
    if (lane == 0) wtot[w] = tot;
    __syncthreads();
    if (w == 0) {  // exclusive scan of the warp totals
        const unsigned x = wtot[lane];
        unsigned incl = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        wtot[lane] = incl - x;
        if (lane == 31) start[kCells] = (int)incl;
    }
    __syncthreads();
    unsigned run = wtot[w];
    for (int i0 = 0; i0 < per; i0 += batch) {  // pass 2: re-read (L2) and scan
        unsigned v[batch];
#pragma unroll
        for (int i = 0; i < batch; ++i) v[i] = src[(i0 + i) * 32];
#pragma unroll
        for (int i = 0; i < batch; ++i) {
            unsigned incl = v[i];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const int c = w * chunk + (i0 + i) * 32 + lane;
            start[c] = (int)(run + incl - v[i]);
            if (cursor) cursor[c] = (int)(run + incl - v[i]);
            run += __shfl_sync(0xffffffffu, incl, 31);
        }
    }
}

// Data: the centred filter values in the caller's order (for unordered launches) and,
// with the coordinates, at sorted positions; padding slots [nd, ndp) get +inf.  fp64
// data: the centred values are the fp64 differences rounded once to fp32 (passes.cuh
// centre_f32), and the fp64 coordinates are also written in sorted order (s64).
__device__ __forceinline__ float centre_d(float x, float c) { return __fsub_rn(x, c); }
__device__ __forceinline__ float centre_d(double x, float c) { return __double2float_rn(x - (double)c); }

template <typename T>
__global__ void order_data_scatter_kernel(const T *__restrict__ px, const T *__restrict__ py, int64_t nd,
                                          int64_t ndp, OrderGrid g, float c_x, float c_y,
                                          int *__restrict__ cursor, float *__restrict__ out, double *__restrict__ s64)
{
    float *ux = out, *uy = out + ndp, *up = out + 2 * ndp;  // caller's order
    float *cx = out + 3 * ndp, *cy = out + 4 * ndp, *pp = out + 5 * ndp, *sx = out + 6 * ndp, *sy = out + 7 * ndp;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ndp;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (i < nd) {
            const T x = px[i], y = py[i];
            const int64_t o = atomicAdd(&cursor[morton_cell((float)x, (float)y, g)], 1);
            const float a = centre_d(x, c_x), b = centre_d(y, c_y);
            const float p2 = __fmaf_rn(a, a, __fmul_rn(b, b));
            ux[i] = cx[o] = a;
            uy[i] = cy[o] = b;
            up[i] = pp[o] = p2;
            sx[o] = (float)x;
            sy[o] = (float)y;
            if (s64) {
                s64[o] = (double)x;
                s64[ndp + o] = (double)y;
            }
        } else {
            ux[i] = uy[i] = up[i] = cx[i] = cy[i] = pp[i] = sx[i] = sy[i] = pos_inf<float>();
            if (s64) s64[i] = s64[ndp + i] = pos_inf<double>();
        }
    }
}

template <typename T>
__global__ void order_query_scatter_kernel(const T *__restrict__ qx, const T *__restrict__ qy, int64_t nq,
                                           OrderGrid g, int *__restrict__ cursor, int *__restrict__ perm)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nq; i += (int64_t)gridDim.x * blockDim.x)
        perm[atomicAdd(&cursor[morton_cell((float)qx[i], (float)qy[i], g)], 1)] = (int)i;
}

unsigned grid_for(int64_t n)
{
    int64_t b = (n + 255) / 256;
    if (b > 148 * 8) b = 148 * 8;
    return (unsigned)(b < 1 ? 1 : b);
}

}  // namespace

template <typename T> static int order_data_t(const T *px, int64_t ndp, int64_t nd, FilterData *fd, cudaStream_t st)
{
    const T *py = px + ndp;
    unsigned *counts = nullptr;
    int *cursor = nullptr;
    if (cudaMallocAsync(&counts, kCells * sizeof(unsigned), st) != cudaSuccess ||
        cudaMallocAsync(&cursor, kCells * sizeof(int), st) != cudaSuccess ||
        cudaMemsetAsync(counts, 0, kCells * sizeof(unsigned), st) != cudaSuccess)
        return -1;
    cell_hist_kernel<T><<<grid_for(nd), 256, 0, st>>>(px, py, nd, fd->grid, counts);
    cell_scan_kernel<<<1, kScanThreads, 0, st>>>(counts, fd->cell_start, cursor);
    order_data_scatter_kernel<T><<<grid_for(ndp), 256, 0, st>>>(px, py, nd, ndp, fd->grid, fd->c_x, fd->c_y, cursor,
                                                                static_cast<float *>(fd->arrays), fd->coords64);
    const bool ok = cudaPeekAtLastError() == cudaSuccess;
    cudaFreeAsync(counts, st);
    cudaFreeAsync(cursor, st);
    return ok ? 3 : -1;
}

int launch_order_data(int dtype, const void *data, int64_t ndp, int64_t nd, FilterData *fd, cudaStream_t st)
{
    return dtype == 0 ? order_data_t(static_cast<const float *>(data), ndp, nd, fd, st)
                      : order_data_t(static_cast<const double *>(data), ndp, nd, fd, st);
}

template <typename T>
static int order_queries_t(const T *qx, const T *qy, int64_t nq, const FilterData *fd, SplitBuf *buf,
                           const int **perm, cudaStream_t st)
{
    // buf layout: counts [kCells] | start [kCells + 1] | cursor [kCells] | perm [nq]
    const size_t head = (size_t)(3 * kCells + 1) * sizeof(int);
    char *b = static_cast<char *>(buf->reserve(head + (size_t)nq * sizeof(int)));
    if (!b) return 0;  // no memory: run unordered
    unsigned *counts = reinterpret_cast<unsigned *>(b);
    int *start = reinterpret_cast<int *>(b) + kCells;
    int *cursor = start + kCells + 1;
    int *p = cursor + kCells;
    if (cudaMemsetAsync(counts, 0, kCells * sizeof(unsigned), st) != cudaSuccess) return -1;
    cell_hist_kernel<T><<<grid_for(nq), 256, 0, st>>>(qx, qy, nq, fd->grid, counts);
    cell_scan_kernel<<<1, kScanThreads, 0, st>>>(counts, start, cursor);
    order_query_scatter_kernel<T><<<grid_for(nq), 256, 0, st>>>(qx, qy, nq, fd->grid, cursor, p);
    if (cudaPeekAtLastError() != cudaSuccess) return -1;
    *perm = p;
    return 3;
}

int launch_order_queries(const float *qx, const float *qy, int64_t nq, const FilterData *fd, SplitBuf *buf,
                         const int **perm, cudaStream_t st)
{
    return order_queries_t(qx, qy, nq, fd, buf, perm, st);
}

int launch_order_queries(const double *qx, const double *qy, int64_t nq, const FilterData *fd, SplitBuf *buf,
                         const int **perm, cudaStream_t st)
{
    return order_queries_t(qx, qy, nq, fd, buf, perm, st);
}

}  // namespace aidw
