// aidw_internal.h -- launchers shared by the C-ABI (aidw_api.cu) and the kernel
// translation units.  Not part of the public ABI.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace aidw {

// Data tiles.  kTileW is also the fp32 accumulation block of the
// weighting pass (fp32 sums within a tile, fp64 across tiles) -- part of the fp32
// result's rounding, fixed so results do not depend on launch shape or GPU count.
constexpr int kTileK = 1024;   // points per smem stage, kNN pass (x, y)
constexpr int kStagesK = 4;
constexpr int kTileW = 512;    // points per smem stage, weighting pass (x, y, z)
constexpr int kStagesW = 4;
constexpr int kTileKF = 512;   // points per smem stage, fp32 filtered kNN (cx, cy, pp, x, y)
constexpr int kStagesKF = 3;
constexpr int kPad = 1024;     // internal arrays padded to a multiple of both tiles

// The fp64 cross-tile sums of the weighting pass are formed per accumulation block of
// tiles (at most kAccBlocks per data set, boundaries depending only on nd) and the
// block sums are added in block order.  A launch that splits the data range across
// CTAs (small nq, "split mode") writes per-block sums and adds them in the same order
// afterwards, so split and unsplit launches give bit-identical Z.
constexpr int kAccBlocks = 16;
__host__ __device__ inline int acc_blocks(int ntiles) { return ntiles < kAccBlocks ? ntiles : kAccBlocks; }
__host__ __device__ inline int block_tile(int b, int ntiles, int nblk)
{
    return (int)((long long)b * ntiles / nblk);
}

// Device memory of handles and their scratch buffers: the device's default stream-ordered
// pool with an unlimited release threshold, so a destroy + create cycle (a serving
// process swapping data sets, bench.py e2e_full) reuses memory instead of paying
// cudaFree / cudaMalloc.  dev_malloc returns memory usable from any stream at once;
// callers synchronise the device before dev_free (as before with cudaFree).  The
// exchange buffer keeps cudaMalloc (CUDA IPC needs it).
cudaError_t dev_malloc(void **p, size_t n);
void dev_free(void *p);

// Growable device buffer for the small-nq data split (per-split kNN lists, per-block
// weighting sums).  reserve() grows it (device sync + free + malloc) and returns
// nullptr on allocation failure, in which case the launcher runs unsplit.
struct SplitBuf {
    void *p = nullptr;
    size_t bytes = 0;
    void *reserve(size_t n);
};

// Device-side GLOBAL-bounds exchange over peer memory (N4 push): every
// rank owns one ExBuf.  At epoch e rank r's kNN epilogue writes its {-min, max} into
// val[e & 1][r] of EVERY rank's buffer (NVLink P2P stores through CUDA-IPC-mapped
// pointers), then flag[r] = e (release); rank p's alpha kernel waits until every flag
// of its own buffer reached e, reads slot e & 1, and -- after its last CTA has read --
// stores ack[p] = e into every rank's buffer.  A publisher writes slot e & 1 only after
// every rank acked e - 2 (the previous use of that slot), so a rank that runs one epoch
// ahead never overwrites values a slower peer has not read yet.
constexpr int kExMaxRanks = 64;
struct ExBuf {
    unsigned long long flag[kExMaxRanks];  // epoch rank r last published into this buffer
    unsigned long long ack[kExMaxRanks];   // epoch rank r finished reading (its alpha kernel)
    double val[2][kExMaxRanks][2];         // [epoch parity][rank] {-min, max}
};

// Device scratch owned by a handle.
struct Scratch {
    unsigned long long mn;      // ordered bits of min r_obs (identity ~0ull)
    unsigned long long mx;      // ordered bits of max r_obs (identity 0)
    unsigned int done;          // CTA ticket for the last-CTA finalise
    unsigned int pad0;
    long long err_idx;          // smallest non-finite query index (LLONG_MAX = none)
    unsigned long long keys[4]; // bbox: ordered keys of min x, max x, min y, max y
    unsigned long long nonfinite;
    unsigned cls[8];            // weighting-pass class counts + cursors (launch_interp)
    // bounds exchange (zero = off): peers[r] = rank r's ExBuf (device pointers)
    ExBuf *const *ex_peers;
    int ex_rank, ex_world;
    unsigned long long ex_epoch;  // advanced by the kNN epilogue, read by the alpha kernel
    unsigned ex_timeout;          // set when a wait gave up (reported by aidw_check)
    unsigned ex_readers;          // alpha-kernel CTA ticket: the last reader sends the acks
};

// Spatial (Morton) order of points and queries for the fp32 kNN:
// 2^kOrderBits x 2^kOrderBits cells over the data bbox; cell(x, y) clamps outside points
// (and NaN) to the border, so any input maps to a cell.
constexpr int kOrderBits = 8;
constexpr int kCells = 1 << (2 * kOrderBits);
struct OrderGrid {
    float x0, y0, sx, sy;  // cell coordinate = (x - x0) * sx, clamped to [0, 2^bits - 1]
};
__host__ __device__ inline unsigned morton_cell(float x, float y, OrderGrid g)
{
    constexpr float top = (float)((1 << kOrderBits) - 1);
    const float fx = fminf(fmaxf((x - g.x0) * g.sx, 0.f), top);  // NaN -> 0
    const float fy = fminf(fmaxf((y - g.y0) * g.sy, 0.f), top);
    unsigned ix = (unsigned)fx, iy = (unsigned)fy, c = 0;
    for (int b = 0; b < kOrderBits; ++b) c |= ((ix >> b) & 1u) << (2 * b) | ((iy >> b) & 1u) << (2 * b + 1);
    return c;
}

// fp32 kNN filter data owned by a handle: [8][ndp] floats padded
// with +inf -- centred cx, cy, |p'|^2 in the caller's order, then the same three and
// x, y in Morton order -- the centre, the bound R1, the order grid and each cell's first
// sorted position.
struct FilterData {
    void *arrays = nullptr;
    double *coords64 = nullptr;  // fp64 handles: [2][ndp] x, y in Morton order (re-check)
    float c_x = 0.f, c_y = 0.f, r1 = 0.f;
    int *cell_start = nullptr;  // [kCells + 1]
    OrderGrid grid{0.f, 0.f, 0.f, 0.f};
    SplitBuf qorder;            // per-call query order: counts, cursors, perm
};

// Morton-sort the data into the filter arrays (3 launches) and order a query batch
// (perm[i] = query of launch slot i; 3 launches + a memset; scratch from `buf`).
int launch_order_data(int dtype, const void *data, int64_t ndp, int64_t nd, FilterData *fd, cudaStream_t st);
int launch_order_queries(const double *qx, const double *qy, int64_t nq, const FilterData *fd, SplitBuf *buf,
                         const int **perm, cudaStream_t st);
int launch_order_queries(const float *qx, const float *qy, int64_t nq, const FilterData *fd, SplitBuf *buf,
                         const int **perm, cudaStream_t st);

// Each launcher returns the number of kernels it launched (>= 0) or -1 on a
// launch error (cudaGetLastError is left set for the caller).
int launch_prep(int dtype, int layout, const void *src, int64_t nd, int64_t ndp, void *data,
                Scratch *sc, cudaStream_t st);

int launch_knn(int dtype, int k, const void *data, int64_t ndp, const void *qx, const void *qy,
               int64_t nq, void *r_obs, void *d1sq, void *minmax, void *dists, Scratch *sc,
               FilterData *filt, cudaStream_t st, int dists_sq = 0, SplitBuf *split = nullptr);

int launch_knn_merge(int dtype, int k, const void *lists, int P, int64_t nq, void *r_obs, void *d1sq,
                     void *minmax, Scratch *sc, cudaStream_t st);

int launch_finalize(int dtype, const double *partials, int P, int64_t nq, void *z, cudaStream_t st);

int launch_minmax_identity(int dtype, void *minmax, cudaStream_t st);

int launch_alpha(int dtype, const void *r_obs, int64_t nq, double r_exp, const double *lv,
                 int rb, double rmin, double rmax, const void *minmax, int mf, void *alpha,
                 cudaStream_t st, Scratch *ex_sc = nullptr);

// nq == 0 with an active exchange: push the MAX identity so peers do not wait.
int launch_exchange_push_identity(Scratch *sc, cudaStream_t st);

int launch_fused_fixed(const void *data, int64_t ndp, int64_t nd, FilterData *filt, const void *qx,
                       const void *qy, int64_t nq, int k, double r_exp, const double *lv, double rmin,
                       double rmax, int mf, void *z, void *r_obs, void *alpha, Scratch *sc, cudaStream_t st);

int launch_paper(int variant, int dtype, int layout, const void *data, int64_t nd, const void *qx, const void *qy,
                 int64_t nq, int k, double r_exp, const double *lv, double rmin, double rmax, void *z,
                 cudaStream_t st);

// alpha == nullptr -> every query uses alpha_const (standard IDW, Eq. 1 with a constant power).
// partial != nullptr -> write per-query fp64 {sum w, sum w z, sum z_coincident, n_coincident}
// over this handle's data (data-sharded mode) instead of z.
// perm (int32[nq]) + cls_counts (uint32[8]) != nullptr -> fp32: queries are grouped by
// exact-exponent class first (2 small kernels) so whole CTAs take the 1-SFU-op paths.
// Returns the number of kernels launched.
int launch_interp(int dtype, const void *data, int64_t ndp, int64_t nd, const void *qx,
                  const void *qy, int64_t nq, const void *alpha, double alpha_const, const void *d1sq, void *z,
                  cudaStream_t st, double *partial = nullptr, int *perm = nullptr,
                  unsigned *cls_counts = nullptr, SplitBuf *split = nullptr, const double *bbox = nullptr);

// Data-split factor for a launch of `grid` CTAs (small nq fills the GPU by splitting the
// data range across blockIdx.y); 1 = no split.
int choose_split(const void *kern, int block, size_t smem, int64_t grid, int maxs, int waves, bool full = false);

}  // namespace aidw
