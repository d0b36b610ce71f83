// interpolate.cu -- S5 of the AIDW hot path on sm_100a: the Shepard weighted
// average over ALL data points (Eq. 1; "calculate the distances
// to all the data points again") with the per-query alpha.
//
// Weights are evaluated as w = 2^(c*log2(s) + b) with s the squared distance,
// c = -alpha/2 and b = (alpha/2) log2(d1sq): w = (d/d1)^-alpha, i.e. Eq. 1's
// d^-alpha scaled by the (cancelling) factor d1^alpha so w is in (0, 1] for any
// coordinate scale.  fp32 (passes.cuh interp_f32_tile): packed FADD2/FMUL2/FFMA2,
// MUFU lg2.approx, ex2 split between MUFU ex2.approx and an FMA-pipe polynomial
// (DESIGN.md §4.3); sums in fp32 within a kTileW-point tile and in fp64 across tiles
// (the paper's "two registers", made accurate for 1M-term sums).
// fp64: libdevice log2/exp2, fp64 sums.
//
// Same smem ring as knn_robs.cu (TMA bulk copies of x, y, z tiles, mbarriers),
// Q queries per thread, every data point read once from smem per Q pairs.
#include "passes.cuh"

#include <limits>

#include <cstdlib>

namespace aidw {

template <typename T> struct InterpArgs {
    const T *px, *py, *pz;  // internal SoA padded with (+inf, +inf, 0)
    int64_t ndp, nd;
    const T *qx, *qy, *alpha, *d1sq;  // alpha nullable -> alpha_const for every query
    int64_t nq;
    T *z;
    T alpha_const;
    double *partial;  // nullable: data-sharded partial sums instead of z
    const int *perm;  // nullable: position i evaluates query perm[i] (class grouping)
    double2 *bpart;   // split mode: per-accumulation-block sums [nblk][nq] (gridDim.y > 1)
    float bb[4];      // data bbox {x0, x1, y0, y1} (fp32 kernel's clamp-free test); NaN: unknown
};

// fp32 general formula without the exp2 clamp (round 2): a query's
// exponents e = c lg2(s) + b over its REAL data points are >= c lg2(s_max) + b, s_max the
// squared distance to the farthest bbox corner (c < 0).  When that bound is >= -120 the
// polynomial exp2's clamp to -126 never fires, so dropping it (2 FMNMX per couple) leaves
// every weight bit-identical.  Coincident (d1 = 0), subnormal-nearest and far-outside
// queries fail the test and keep the clamp, as do the tiles holding padding points.
__device__ __forceinline__ bool exp2_clamp_free(float qx, float qy, float alpha, float d1sq, const float (&bb)[4])
{
    const float dxm = fmaxf(fabsf(qx - bb[0]), fabsf(qx - bb[1]));
    const float dym = fmaxf(fabsf(qy - bb[2]), fabsf(qy - bb[3]));
    const float smax = __fmul_ru(__fmaf_ru(dxm, dxm, __fmul_ru(dym, dym)), 1.0001f);
    const float e = 0.5f * alpha * (lg2_approx_noftz(d1sq) - lg2_approx_noftz(smax));
    return e >= -120.0f;  // false for NaN / -inf (coincident, unknown bbox, overflow)
}

// Weight math per precision: fp32 MUFU (scalar variant), fp64 table + polynomial
// (passes.cuh log2_f64 / exp2_f64; tables staged in shared memory).
struct F64Tabs {
    double2 lg[1 << kLog2TabBits];
    double ex[1 << kExp2TabBits];
};
__device__ __forceinline__ float wlog2(float s, const F64Tabs &) { return lg2_approx(s); }
__device__ __forceinline__ double wlog2(double s, const F64Tabs &t) { return log2_f64(s, t.lg); }
__device__ __forceinline__ float wexp2(float x, const F64Tabs &) { return ex2_approx(x); }
__device__ __forceinline__ double wexp2(double x, const F64Tabs &t) { return exp2_f64(x, t.ex); }
__device__ __forceinline__ float log2_q(float s) { return lg2_approx_noftz(s); }
__device__ __forceinline__ double log2_q(double s) { return log2(s); }

// Ring + smem tile layout shared by both kernels: x, y, z arrays of STAGES * TILE.
template <typename T, int TILE, int STAGES, int WARPS = kWarps>
struct XYZRing {
    T *sx, *sy, *sz;
    Ring<STAGES, WARPS> ring;
    __device__ __forceinline__ XYZRing(unsigned char *smem)
    {
        sx = reinterpret_cast<T *>(smem);
        sy = sx + STAGES * TILE;
        sz = sy + STAGES * TILE;
        ring.full = reinterpret_cast<uint64_t *>(sz + STAGES * TILE);
        ring.empty = ring.full + STAGES;
    }
    __device__ __forceinline__ void issue(const InterpArgs<T> &a, int tile, int slot)
    {
        mbar_arrive_expect_tx(&ring.full[slot], 3u * TILE * sizeof(T));
        const int64_t off = (int64_t)tile * TILE;
        bulk_g2s(sx + slot * TILE, a.px + off, TILE * sizeof(T), &ring.full[slot]);
        bulk_g2s(sy + slot * TILE, a.py + off, TILE * sizeof(T), &ring.full[slot]);
        bulk_g2s(sz + slot * TILE, a.pz + off, TILE * sizeof(T), &ring.full[slot]);
    }
    static constexpr size_t smem_bytes() { return (size_t)3 * STAGES * TILE * sizeof(T) + 2 * STAGES * 8; }
};

// Generic kernel: fp64 path (and the scalar fp32 variant, AIDW_INTERP_VARIANT=1).
template <typename T, int Q, bool SPLIT = false>
__global__ void __launch_bounds__(kBlock) interp_kernel(const InterpArgs<T> a)
{
    constexpr int TILE = kTileW, STAGES = kStagesW;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ F64Tabs tabs;
    XYZRing<T, TILE, STAGES> r(smem_raw);
    const int ntiles_all = (int)(a.ndp / TILE);
    // split mode (gridDim.y = S > 1, §4.6): this CTA covers accumulation blocks [b0, b1)
    const int nblk = acc_blocks(ntiles_all), S = SPLIT ? (int)gridDim.y : 1;
    const int b0 = SPLIT ? (int)blockIdx.y * nblk / S : 0, b1 = SPLIT ? ((int)blockIdx.y + 1) * nblk / S : nblk;
    const int t0 = block_tile(b0, ntiles_all, nblk), ntiles = block_tile(b1, ntiles_all, nblk) - t0;
    if (threadIdx.x == 0) r.ring.init();
    if (sizeof(T) == 8) {
        for (int i = threadIdx.x; i < (1 << kLog2TabBits); i += blockDim.x)
            tabs.lg[i] = make_double2(kLog2Tab[i][0], kLog2Tab[i][1]);
        for (int i = threadIdx.x; i < (1 << kExp2TabBits); i += blockDim.x) tabs.ex[i] = kExp2Tab[i];
    }
    __syncthreads();
    auto issue = [&](int tile, int slot) { r.issue(a, t0 + tile, slot); };
    if (threadIdx.x == 0)
        for (int s = 0; s < STAGES && s < ntiles; ++s) issue(s, s);

    const int64_t base = (int64_t)blockIdx.x * (kBlock * Q) + threadIdx.x;
    T qx[Q], qy[Q], c[Q], b[Q], d1[Q];
    bool valid[Q];
    double SW[Q], SWZ[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const int64_t idx = base + q * kBlock;
        valid[q] = idx < a.nq;
        qx[q] = valid[q] ? a.qx[idx] : T(0);
        qy[q] = valid[q] ? a.qy[idx] : T(0);
        const T al = valid[q] ? (a.alpha ? a.alpha[idx] : a.alpha_const) : T(1);
        d1[q] = valid[q] ? a.d1sq[idx] : T(1);
        c[q] = T(-0.5) * al;
        b[q] = T(0.5) * al * log2_q(d1[q]);
        SW[q] = 0.0;
        SWZ[q] = 0.0;
    }

    int blk = b0, bend = block_tile(b0 + 1, ntiles_all, nblk) - t0;
    double BW[Q], BWZ[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) BW[q] = BWZ[q] = 0.0;
    for (int t = 0; t < ntiles; ++t) {
        r.ring.wait_full(t);
        const int o = r.ring.slot(t) * TILE;
        const T *tx = r.sx + o, *ty = r.sy + o, *tz = r.sz + o;
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
                    const T w = wexp2(fma(c[q], wlog2(s, tabs), b[q]), tabs);
                    sw[q] += w;
                    swz[q] = fma(w, Z.v[e], swz[q]);
                }
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            BW[q] += (double)sw[q];
            BWZ[q] += (double)swz[q];
        }
        if (t + 1 == bend) {  // end of an accumulation block: block sums in block order
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                if constexpr (SPLIT) {
                    if (valid[q]) a.bpart[(int64_t)blk * a.nq + base + q * kBlock] = make_double2(BW[q], BWZ[q]);
                } else {
                    SW[q] += BW[q];
                    SWZ[q] += BWZ[q];
                }
                BW[q] = BWZ[q] = 0.0;
            }
            ++blk;
            bend = block_tile(blk + 1, ntiles_all, nblk) - t0;
        }
        r.ring.release(t, ntiles, issue);
    }

    if constexpr (!SPLIT) {
#pragma unroll
        for (int q = 0; q < Q; ++q)
            if (valid[q])
                write_result<T>(a.z, a.partial, base + q * kBlock, SW[q], SWZ[q], d1[q], qx[q], qy[q], a.px, a.py,
                                a.pz, a.nd, -2.0 * (double)c[q]);
    }
}

// Packed fp32 kernel (passes.cuh interp_f32_tile / interp_f32_tile_cls).  With a class
// permutation, a CTA whose queries all share an exact-exponent class runs the 1-SFU-op
// loop; a CTA mixing classes (only at class boundaries) selects per lane.
// CTAs per SM to target (register cap): 9 at Q = 2 (56 registers, the smem limit too).
constexpr int interp_min_blocks(int q) { return q == 1 ? 12 : q == 2 ? 9 : 6; }
// (the generic XYZRing is shared with the fp64 kernel; its stage count is a template
// parameter so the packed kernel can trade pipeline depth for occupancy)

template <int Q, unsigned EMU, int STAGES = kStagesW, int BLOCK = kBlock, bool SPLIT = false>
__global__ void __launch_bounds__(BLOCK, interp_min_blocks(Q) * kBlock / BLOCK)
    interp_f32x2_kernel(const InterpArgs<float> a)
{
    constexpr int TILE = kTileW;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    XYZRing<float, TILE, STAGES, BLOCK / 32> r(smem_raw);
    const int ntiles = (int)(a.ndp / TILE);
    // split mode (gridDim.y = S > 1): this CTA covers accumulation blocks [b0, b1)
    const int nblk = acc_blocks(ntiles), S = SPLIT ? (int)gridDim.y : 1;
    const int b0 = SPLIT ? (int)blockIdx.y * nblk / S : 0, b1 = SPLIT ? ((int)blockIdx.y + 1) * nblk / S : nblk;
    const int t0 = block_tile(b0, ntiles, nblk), nloc = block_tile(b1, ntiles, nblk) - t0;
    if (threadIdx.x == 0) r.ring.init();
    __syncthreads();
    auto issue = [&](int tile, int slot) { r.issue(a, t0 + tile, slot); };
    if (threadIdx.x == 0)
        for (int s = 0; s < STAGES && s < nloc; ++s) issue(s, s);

    const int64_t base = (int64_t)blockIdx.x * (BLOCK * Q) + threadIdx.x;
    float qx[Q], qy[Q], d1[Q];
    int64_t qid[Q];
    int cls[Q];
    bool valid[Q];
    unsigned present = 0;
    InterpF32State<Q> st;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const int64_t i = base + q * BLOCK;
        valid[q] = i < a.nq;
        qid[q] = valid[q] ? (a.perm ? (int64_t)a.perm[i] : i) : 0;
        qx[q] = valid[q] ? a.qx[qid[q]] : 0.f;
        qy[q] = valid[q] ? a.qy[qid[q]] : 0.f;
        d1[q] = valid[q] ? a.d1sq[qid[q]] : 1.f;
        const float al = valid[q] ? (a.alpha ? a.alpha[qid[q]] : a.alpha_const) : 1.f;
        st.init(q, qx[q], qy[q], al, d1[q]);
        cls[q] = a.perm ? alpha_class(al, d1[q]) : kClsGeneral;
        if (valid[q]) present |= 1u << cls[q];
    }
    // the exp2 clamp is needed only for queries whose far weights may drop below 2^-126
    // and on tiles holding padding points (s = +inf)
    bool unsafe = false;
#pragma unroll
    for (int q = 0; q < Q; ++q)
        if (valid[q])
            unsafe |= !exp2_clamp_free(qx[q], qy[q], -2.0f * st.C[q].x, d1[q], a.bb);
    // tiles from clamp_from on use the clamped exp2: all of them if some query needs it,
    // else those holding padding points
    const int clamp_from = __syncthreads_or(unsafe) ? 0 : (int)(a.nd / TILE);
    int cta_cls = kClsGeneral;
    if (a.perm) {
        const int any_g = __syncthreads_or(present & 1u), any_1 = __syncthreads_or(present & 2u);
        const int any_2 = __syncthreads_or(present & 4u), any_3 = __syncthreads_or(present & 8u);
        const int n = (any_g != 0) + (any_1 != 0) + (any_2 != 0) + (any_3 != 0);
        cta_cls = n > 1 ? kClsMixed : any_1 ? kClsA1 : any_2 ? kClsA2 : any_3 ? kClsA3 : kClsGeneral;
    }

    __shared__ double2 acc_s[Q][BLOCK];  // per-thread running sums over blocks (unsplit)
#pragma unroll
    for (int q = 0; q < Q; ++q) acc_s[q][threadIdx.x] = make_double2(0.0, 0.0);
    int blk = b0, bend = block_tile(b0 + 1, ntiles, nblk) - t0;
    for (int t = 0; t < nloc; ++t) {
        r.ring.wait_full(t);
        const int o = r.ring.slot(t) * TILE;
        switch (cta_cls) {  // CTA-uniform
        case kClsA1: interp_f32_tile_cls<Q, kClsA1, EMU, TILE>(st, cls, r.sx + o, r.sy + o, r.sz + o); break;
        case kClsA2: interp_f32_tile_cls<Q, kClsA2, EMU, TILE>(st, cls, r.sx + o, r.sy + o, r.sz + o); break;
        case kClsA3: interp_f32_tile_cls<Q, kClsA3, EMU, TILE>(st, cls, r.sx + o, r.sy + o, r.sz + o); break;
        case kClsMixed: interp_f32_tile_cls<Q, kClsMixed, EMU, TILE>(st, cls, r.sx + o, r.sy + o, r.sz + o); break;
        default:
            if (t0 + t >= clamp_from)
                interp_f32_tile<Q, EMU, TILE, true>(st, r.sx + o, r.sy + o, r.sz + o);
            else
                interp_f32_tile<Q, EMU, TILE, false>(st, r.sx + o, r.sy + o, r.sz + o);
            break;
        }
        if (t + 1 == bend) {  // end of an accumulation block
            if constexpr (SPLIT) {
#pragma unroll
                for (int q = 0; q < Q; ++q)
                    if (valid[q]) a.bpart[(int64_t)blk * a.nq + qid[q]] = make_double2(st.BW[q], st.BWZ[q]);
#pragma unroll
                for (int q = 0; q < Q; ++q) st.BW[q] = st.BWZ[q] = 0.0;
            } else {  // block sums accumulate in smem (registers are at the occupancy cap)
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    acc_s[q][threadIdx.x].x += st.BW[q];
                    acc_s[q][threadIdx.x].y += st.BWZ[q];
                    st.BW[q] = st.BWZ[q] = 0.0;
                }
            }
            ++blk;
            bend = block_tile(blk + 1, ntiles, nblk) - t0;
        }
        r.ring.release(t, nloc, issue);
    }

    if constexpr (!SPLIT) {
#pragma unroll
        for (int q = 0; q < Q; ++q)
            if (valid[q])
                write_result<float>(a.z, a.partial, qid[q], acc_s[q][threadIdx.x].x, acc_s[q][threadIdx.x].y, d1[q],
                                    qx[q], qy[q], a.px, a.py, a.pz, a.nd, -2.0 * (double)st.C[q].x);
    }
}

// Split mode: Z (or the data-sharded partials) from the per-block sums, added in block
// order exactly as an unsplit launch adds them.
template <typename T> __global__ void finalize_split_kernel(const InterpArgs<T> a, int nblk)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.nq; i += (int64_t)gridDim.x * blockDim.x) {
        double SW = 0.0, SWZ = 0.0;
        for (int b = 0; b < nblk; ++b) {
            const double2 v = a.bpart[(int64_t)b * a.nq + i];
            SW += v.x;
            SWZ += v.y;
        }
        write_result<T>(a.z, a.partial, i, SW, SWZ, a.d1sq[i], a.qx[i], a.qy[i], a.px, a.py, a.pz, a.nd,
                        (double)(a.alpha ? a.alpha[i] : a.alpha_const));
    }
}

// Class grouping (2 small kernels): counts per class, then a scatter into perm in the
// order alpha = 3, 2, 1, general: the class boundaries -- the only CTAs that mix classes
// and run slower -- fall in the first CTAs, never in the tail of the launch.
__device__ __forceinline__ int class_of(const InterpArgs<float> &a, int64_t i)
{
    return alpha_class(a.alpha ? a.alpha[i] : a.alpha_const, a.d1sq[i]);
}

__global__ void class_count_kernel(const InterpArgs<float> a, unsigned *counts)
{
    const int lane = threadIdx.x & 31;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < a.nq; i0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = i0 + threadIdx.x;
        const int c = i < a.nq ? class_of(a, i) : -1;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const unsigned m = __ballot_sync(0xffffffffu, c == k);
            if (lane == 0 && m) atomicAdd(&counts[k], __popc(m));
        }
    }
}

__global__ void class_scatter_kernel(const InterpArgs<float> a, unsigned *counts, int *perm)
{
    const int lane = threadIdx.x & 31;
    // offsets for classes 0 (general), 1, 2, 3 with the order 3, 2, 1, 0 in perm
    const unsigned off[4] = {counts[3] + counts[2] + counts[1], counts[3] + counts[2], counts[3], 0u};
    unsigned *cursor = counts + 4;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < a.nq; i0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = i0 + threadIdx.x;
        const int c = i < a.nq ? class_of(a, i) : -1;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const unsigned m = __ballot_sync(0xffffffffu, c == k);
            if (!m) continue;
            unsigned b = 0;
            if (lane == 0) b = atomicAdd(&cursor[k], __popc(m));
            b = __shfl_sync(0xffffffffu, b, 0);
            if (c == k) perm[off[k] + b + __popc(m & ((1u << lane) - 1u))] = (int)i;
        }
    }
}

// Split factor for a launch of `grid` CTAs: 1 when the grid already fills `waves`
// waves of resident CTAs, else enough data splits for ~`waves` waves (<= `maxs`), or
// `maxs` itself when `full`.  AIDW_SPLIT=0 disables,
// AIDW_SPLIT=n forces n (tests).
static int split_env()
{
    const char *e = getenv("AIDW_SPLIT");  // read per launch so tests can toggle it
    return e ? atoi(e) : -1;
}

int choose_split(const void *kern, int block, size_t smem, int64_t grid, int maxs, int waves, bool full)
{
    const int forced = split_env();
    if (forced == 0) return 1;
    if (forced > 0) return forced < maxs ? forced : maxs;
    int dev = 0, sms = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, block, smem) != cudaSuccess) {
        cudaGetLastError();
        return 1;
    }
    const int64_t slots = (int64_t)occ * sms, target = waves * slots;
    int64_t s = target / grid;  // floor: a partial extra wave costs more than it fills
    if (s < 2) return 1;
    if (full) return maxs;
    return (int)(s < maxs ? s : maxs);
}

template <typename T, int Q>
static int launch_interp_t(InterpArgs<T> a, cudaStream_t st, SplitBuf *split = nullptr)
{
    const size_t smem = XYZRing<T, kTileW, kStagesW>::smem_bytes();
    if (cudaFuncSetAttribute(interp_kernel<T, Q, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return -1;
    const int64_t per_cta = (int64_t)kBlock * Q;
    const unsigned grid = (unsigned)((a.nq + per_cta - 1) / per_cta);
    const int nblk = acc_blocks((int)(a.ndp / kTileW));
    int S = split ? choose_split((const void *)interp_kernel<T, Q, false>, kBlock, smem, grid, nblk, 16, true) : 1;
    a.bpart = S > 1 ? static_cast<double2 *>(split->reserve((size_t)nblk * (size_t)a.nq * sizeof(double2)))
                    : nullptr;
    if (!a.bpart) S = 1;
    if (S == 1) {
        interp_kernel<T, Q, false><<<grid, kBlock, smem, st>>>(a);
        return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
    }
    if (cudaFuncSetAttribute(interp_kernel<T, Q, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return -1;
    interp_kernel<T, Q, true><<<dim3(grid, (unsigned)S), kBlock, smem, st>>>(a);
    if (cudaPeekAtLastError() != cudaSuccess) return -1;
    int64_t blocks = (a.nq + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    finalize_split_kernel<T><<<(unsigned)blocks, 256, 0, st>>>(a, nblk);
    return cudaPeekAtLastError() == cudaSuccess ? 2 : -1;
}

template <int Q, unsigned EMU, int STAGES, int BLOCK, bool SPLIT> static int interp_attrs(size_t smem)
{
    auto kern = interp_f32x2_kernel<Q, EMU, STAGES, BLOCK, SPLIT>;
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess &&
                   cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100) == cudaSuccess
               ? 0
               : -1;
}

template <int Q, unsigned EMU, int STAGES = kStagesW, int BLOCK = kBlock>
static int launch_interp_f32x2(InterpArgs<float> a, cudaStream_t st, SplitBuf *split)
{
    const size_t smem = XYZRing<float, kTileW, STAGES>::smem_bytes();
    if (interp_attrs<Q, EMU, STAGES, BLOCK, false>(smem) < 0) return -1;
    const int64_t per_cta = (int64_t)BLOCK * Q;
    const unsigned grid = (unsigned)((a.nq + per_cta - 1) / per_cta);
    const int nblk = acc_blocks((int)(a.ndp / kTileW));
    // Weighting splits carry no per-split warm-up (unlike the kNN), so a full split into
    // the nblk accumulation blocks is used whenever the grid is under 16 waves: it also
    // removes the partial last wave (profiles/r01_split.jsonl).
    int S = split ? choose_split((const void *)interp_f32x2_kernel<Q, EMU, STAGES, BLOCK, false>, BLOCK, smem, grid,
                                 nblk, 16, true)
                  : 1;
    a.bpart = S > 1 ? static_cast<double2 *>(split->reserve((size_t)nblk * (size_t)a.nq * sizeof(double2)))
                    : nullptr;
    if (!a.bpart) S = 1;
    if (S == 1) {
        interp_f32x2_kernel<Q, EMU, STAGES, BLOCK, false><<<grid, BLOCK, smem, st>>>(a);
        return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
    }
    if (interp_attrs<Q, EMU, STAGES, BLOCK, true>(smem) < 0) return -1;
    interp_f32x2_kernel<Q, EMU, STAGES, BLOCK, true><<<dim3(grid, (unsigned)S), BLOCK, smem, st>>>(a);
    if (cudaPeekAtLastError() != cudaSuccess) return -1;
    int64_t blocks = (a.nq + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    finalize_split_kernel<float><<<(unsigned)blocks, 256, 0, st>>>(a, nblk);
    return cudaPeekAtLastError() == cudaSuccess ? 2 : -1;
}

// Variant selection for tuning (AIDW_INTERP_VARIANT; tools/tune_interp.py); 0 = default.
static int interp_variant()
{
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("AIDW_INTERP_VARIANT");
        v = e ? atoi(e) : 0;
    }
    return v;
}

// True when the Q = 2 grid, split into every accumulation block, has fewer than
// `per_sm` CTAs per SM (AIDW_INTERP_Q1=0 disables, =1 forces; tests).  fp32 (9 CTAs/SM
// resident): Q = 1 wins below ~5 waves (profiles/small/r01_q1_sweep_*.log, nd = 1M:
// 20,000 queries 11.1 -> 9.7 ms, 100,000 40.1 -> 39.2; 128,000 49.5 vs 50.3 with Q = 1);
// fp64: under one wave (C1, C2).
static bool small_grid(int64_t nq, int64_t ndp, int per_sm)
{
    const char *e = getenv("AIDW_INTERP_Q1");
    if (e) return e[0] == '1';
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t ctas = (nq + 2 * kBlock - 1) / (2 * kBlock) * acc_blocks((int)(ndp / kTileW));
    return ctas < (int64_t)sms * per_sm;
}

static int launch_interp_f32(const InterpArgs<float> &a, cudaStream_t st, SplitBuf *sp)
{
    // EMU: 2-bit mode per couple h of 4-point group g at bit 4g+2h (passes.cuh)
    switch (interp_variant()) {
    case 1: return launch_interp_t<float, 2>(a, st);        // scalar, all-SFU
    case 2: return launch_interp_f32x2<2, 0x0000>(a, st, sp);   // packed, all-SFU
    case 3: return launch_interp_f32x2<2, 0x1111>(a, st, sp);   // 4 of 8 couples on the FMA pipe
    case 4: return launch_interp_f32x2<2, 0xAAAA>(a, st, sp);   // every couple split (f = 1/2)
    case 5: return launch_interp_f32x2<2, 0x2A2A>(a, st, sp);   // f = 3/8, split
    case 6: return launch_interp_f32x2<2, 0x2222>(a, st, sp);   // f = 1/4, split
    case 7: return launch_interp_f32x2<2, 0x22A2>(a, st, sp);   // f = 5/16, split
    case 8: return launch_interp_f32x2<2, 0x1241>(a, st, sp);   // f = 3/8, packed + one split
    case 9: return launch_interp_f32x2<1, 0x0141>(a, st, sp);   // Q = 1
    case 10: return launch_interp_f32x2<3, 0x0141>(a, st, sp);  // Q = 3
    case 11: return launch_interp_f32x2<4, 0x0141>(a, st, sp);  // Q = 4
    case 12: return launch_interp_f32x2<1, 0x0141, 3>(a, st, sp);  // Q = 1, 3 stages (12 CTAs/SM)
    case 13: return launch_interp_f32x2<1, 0x0141, 2>(a, st, sp);  // Q = 1, 2 stages
    case 14: return launch_interp_f32x2<1, 0x1111, 3>(a, st, sp);  // Q = 1, 3 stages, f = 1/2
    case 15: return launch_interp_f32x2<2, 0x0141, 3>(a, st, sp);  // Q = 2, 3 stages
    case 16: return launch_interp_f32x2<2, 0x0141>(a, st, sp);  // Q = 2
    case 17: return launch_interp_f32x2<1, 0x0141, 4, 256>(a, st, sp);  // Q = 1, 256-thread CTAs
    case 18: return launch_interp_f32x2<1, 0x0141, 4, 512>(a, st, sp);  // Q = 1, 512-thread CTAs
    case 19: return launch_interp_f32x2<2, 0x0141, 4, 256>(a, st, sp);  // Q = 2, 256-thread CTAs
    case 20: return launch_interp_f32x2<1, 0x1111>(a, st, sp);  // Q = 1, f = 4/8
    case 21: return launch_interp_f32x2<1, 0x1115>(a, st, sp);  // Q = 1, f = 5/8
    case 22: return launch_interp_f32x2<1, 0x0155>(a, st, sp);  // Q = 1, f = 4/8 (first half)
    case 23: return launch_interp_f32x2<1, 0x2A2A>(a, st, sp);  // Q = 1, f = 3/8 split lanes
    case 24: return launch_interp_f32x2<1, 0xAAAA>(a, st, sp);  // Q = 1, f = 1/2 split lanes
    case 25: return launch_interp_f32x2<1, 0x4141>(a, st, sp);  // Q = 1, f = 4/8 (spread)
    case 26: return launch_interp_f32x2<2, 0x1115>(a, st, sp);  // Q = 2, f = 5/8
    case 27: return launch_interp_f32x2<2, 0x1111, 3>(a, st, sp);  // Q = 2, f = 4/8, 3 stages
    case 28: return launch_interp_f32x2<2, 0x4141>(a, st, sp);  // Q = 2, f = 4/8 (spread)
    case 29: return launch_interp_f32x2<2, 0x1111, 4, 256>(a, st, sp);  // Q = 2, f = 4/8, 256 threads
    case 30: return launch_interp_f32x2<3, 0x1111>(a, st, sp);  // Q = 3, f = 4/8
    case 31: return launch_interp_f32x2<2, 0x4141, 3>(a, st, sp);  // Q = 2, f = 4/8 spread, 3 stages
    case 32: return launch_interp_f32x2<2, 0x1414>(a, st, sp);  // Q = 2, f = 4/8 spread (odd)
    case 33: return launch_interp_f32x2<2, 0x4105>(a, st, sp);  // Q = 2, f = 4/8 (0, 1, 4, 7)
    case 34: return launch_interp_f32x2<2, 0x0141>(a, st, sp);  // Q = 2, f = 3/8
    case 35: return launch_interp_f32x2<1, 0x0141>(a, st, sp);  // Q = 1, f = 3/8 (default before v10)
    case 36: return launch_interp_f32x2<2, 0x4151>(a, st, sp);  // Q = 2, f = 5/8 spread (r02)
    case 37: return launch_interp_f32x2<2, 0x5151>(a, st, sp);  // Q = 2, f = 6/8 spread (r02)
    case 38: return launch_interp_f32x2<2, 0x4241>(a, st, sp);  // Q = 2, f = 9/16 (one split couple, r02)
    default: break;
    }
    // Q = 2, f = 4/8 spread (best measured, r01 v10); a grid of fewer than ~5 waves even
    // when fully split (small nq: C1-C3, a strong-scaled share, a serving batch) takes
    // Q = 1 for twice the CTAs -- same per-point offload pattern, so Z is bit-identical
    // (test_interp_q1_small_grid)
    if (small_grid(a.nq, a.ndp, 45)) return launch_interp_f32x2<1, 0x4141>(a, st, sp);
    return launch_interp_f32x2<2, 0x4141>(a, st, sp);
}

// N4: Z from P shards' partials [P][nq][4], summed in rank order (deterministic).
template <typename T>
__global__ void finalize_kernel(const double *__restrict__ part, int P, int64_t nq, T *__restrict__ z)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nq; i += (int64_t)gridDim.x * blockDim.x) {
        double sw = 0.0, swz = 0.0, zc = 0.0, nc = 0.0;
        for (int p = 0; p < P; ++p) {
            const double *r = part + 4 * ((int64_t)p * nq + i);
            sw += r[0];
            swz += r[1];
            zc += r[2];
            nc += r[3];
        }
        z[i] = (T)(nc > 0.0 ? zc / nc : swz / sw);
    }
}

int launch_finalize(int dtype, const double *partials, int P, int64_t nq, void *z, cudaStream_t st)
{
    int64_t blocks = (nq + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (dtype == 0)
        finalize_kernel<float><<<(unsigned)blocks, 256, 0, st>>>(partials, P, nq, (float *)z);
    else
        finalize_kernel<double><<<(unsigned)blocks, 256, 0, st>>>(partials, P, nq, (double *)z);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// Tuning/testing switch read per launch: the integer value of env var `name`, -1 if unset.
static int getenv_flag(const char *name)
{
    const char *e = getenv(name);
    return e ? atoi(e) : -1;
}

int launch_interp(int dtype, const void *data, int64_t ndp, int64_t nd, const void *qx,
                  const void *qy, int64_t nq, const void *alpha, double alpha_const, const void *d1sq, void *z,
                  cudaStream_t st, double *partial, int *perm, unsigned *cls_counts, SplitBuf *split,
                  const double *bbox)
{
    if (dtype == 0) {
        const float *p = static_cast<const float *>(data);
        InterpArgs<float> a{p, p + ndp, p + 2 * ndp, ndp, nd, (const float *)qx, (const float *)qy,
                            (const float *)alpha, (const float *)d1sq, nq, (float *)z, (float)alpha_const,
                            partial, nullptr, nullptr};
        const bool clamp_free = bbox && getenv_flag("AIDW_EXP2_CLAMP") != 1;
        for (int i = 0; i < 4; ++i)  // fp32 data: the bbox is exact in fp32
            a.bb[i] = clamp_free ? (float)bbox[i] : std::numeric_limits<float>::quiet_NaN();
        int launches = 0;
        if (perm && cls_counts && interp_variant() != 1) {
            if (cudaMemsetAsync(cls_counts, 0, 8 * sizeof(unsigned), st) != cudaSuccess) return -1;
            int64_t blocks = (nq + 255) / 256;
            if (blocks > 148 * 8) blocks = 148 * 8;
            class_count_kernel<<<(unsigned)blocks, 256, 0, st>>>(a, cls_counts);
            class_scatter_kernel<<<(unsigned)blocks, 256, 0, st>>>(a, cls_counts, perm);
            if (cudaPeekAtLastError() != cudaSuccess) return -1;
            launches = 2;
            a.perm = perm;
        }
        const int n = launch_interp_f32(a, st, split);
        return n < 0 ? -1 : n + launches;
    }
    const double *p = static_cast<const double *>(data);
    InterpArgs<double> a{p, p + ndp, p + 2 * ndp, ndp, nd, (const double *)qx, (const double *)qy,
                         (const double *)alpha, (const double *)d1sq, nq, (double *)z, alpha_const, partial,
                         nullptr, nullptr, {0.f, 0.f, 0.f, 0.f}};
    if (small_grid(nq, ndp, 8)) return launch_interp_t<double, 1>(a, st, split);
    return launch_interp_t<double, 2>(a, st, split);
}

}  // namespace aidw
