// fused.cu -- N1: FIXED-bounds AIDW in ONE kernel, the paper's
// per-thread structure (kNN -> r_obs -> R -> mu -> alpha -> weighting pass, PAPER.md
// :407-438, Fig. 3) rebuilt on the same sm_100a tile passes as the 3-kernel path.
//
// With caller-given R_min / R_max (Eq. 5's "in general 0.0 and 2.0")
// no query waits for any other, so there is no phase barrier: every CTA runs its kNN
// tiles, computes alpha in registers, and streams the data again for Eq. 1.  CTAs of
// the same SM are then at different phases, so the FMA/ALU-bound kNN pass and the
// SFU-bound weighting pass share the SM's pipes.  One TMA ring
// carries both passes: tiles 0..nt-1 are (cx, cy, pp, x, y) kNN tiles, tiles nt..2nt-1
// are (x, y, z) weighting tiles, so the weighting data is prefetched while the last
// kNN tiles are being consumed.  Results are identical to the 3-kernel path in FIXED
// mode (same tile functions, same operation order).
#include "passes.cuh"

#include <climits>

namespace aidw {

struct FusedArgs {
    const float *px, *py, *pz;  // internal SoA, padded
    int64_t ndp, nd;
    FilterArgs f;
    const float *qx, *qy;
    int64_t nq;
    int k;
    double r_exp;
    Levels lv;
    double rmin, rmax;
    int mf;
    float *z, *r_obs, *alpha;  // r_obs / alpha nullable
    Scratch *sc;
    const int *perm;  // nullable: launch slot i evaluates query perm[i] (spatial order, §4.7)
};

template <int K, int Q, int G, unsigned EMU>
__global__ void __launch_bounds__(kBlock) fused_fixed_kernel(const FusedArgs a)
{
    constexpr int TILE = kTileKF, STAGES = kStagesKF;
    static_assert(TILE == kTileW, "both passes use the same tile (fp32 sums are per kTileW)");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float *sm = reinterpret_cast<float *>(smem_raw);  // stage s at sm + s * 5 * TILE
    Ring<STAGES> ring{reinterpret_cast<uint64_t *>(sm + STAGES * 5 * TILE),
                      reinterpret_cast<uint64_t *>(sm + STAGES * 5 * TILE) + STAGES};
    const int nt = (int)(a.ndp / TILE);
    const int ntot = 2 * nt;
    // spatial order (§4.7): kNN tiles start under the CTA's queries and wrap around
    int start = 0;
    if (a.perm) {
        const int64_t mid = min((int64_t)blockIdx.x * (kBlock * Q) + kBlock * Q / 2, a.nq - 1);
        const int64_t qm = a.perm[mid];
        start = a.f.cell_start[morton_cell(a.qx[qm], a.qy[qm], a.f.grid)] / TILE - 1;
        start = start < 0 ? start + nt : (start >= nt ? nt - 1 : start);
    }
    if (threadIdx.x == 0) ring.init();
    __syncthreads();

    auto issue = [&](int gt, int slot) {
        constexpr uint32_t B = TILE * sizeof(float);
        float *d = sm + slot * 5 * TILE;
        if (gt < nt) {
            const int pt = gt + start < nt ? gt + start : gt + start - nt;
            const int64_t off = (int64_t)pt * TILE;
            mbar_arrive_expect_tx(&ring.full[slot], 5u * B);
            bulk_g2s(d, a.f.cx + off, B, &ring.full[slot]);
            bulk_g2s(d + TILE, a.f.cy + off, B, &ring.full[slot]);
            bulk_g2s(d + 2 * TILE, a.f.pp + off, B, &ring.full[slot]);
            bulk_g2s(d + 3 * TILE, a.f.px + off, B, &ring.full[slot]);
            bulk_g2s(d + 4 * TILE, a.f.py + off, B, &ring.full[slot]);
        } else {
            const int64_t off = (int64_t)(gt - nt) * TILE;
            mbar_arrive_expect_tx(&ring.full[slot], 3u * B);
            bulk_g2s(d, a.px + off, B, &ring.full[slot]);
            bulk_g2s(d + TILE, a.py + off, B, &ring.full[slot]);
            bulk_g2s(d + 2 * TILE, a.pz + off, B, &ring.full[slot]);
        }
    };
    if (threadIdx.x == 0)
        for (int s = 0; s < STAGES && s < ntot; ++s) issue(s, s);

    const int64_t base = (int64_t)blockIdx.x * (kBlock * Q) + threadIdx.x;
    float qx[Q], qy[Q];
    bool valid[Q];
    int64_t qid[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        valid[q] = base + q * kBlock < a.nq;
        const int64_t idx = qid[q] = (a.perm && valid[q]) ? (int64_t)a.perm[base + q * kBlock] : base + q * kBlock;
        qx[q] = valid[q] ? a.qx[idx] : 0.f;
        qy[q] = valid[q] ? a.qy[idx] : 0.f;
        if (valid[q] && !(isfinite(qx[q]) && isfinite(qy[q]))) atomicMin(&a.sc->err_idx, (long long)idx);
    }

    // ---- pass 1: kNN (S1), r_obs (S2)
    const int k0 = K - a.k;
    float d1[Q], al[Q];
    {
        KnnF32State<K, Q> st;
#pragma unroll
        for (int q = 0; q < Q; ++q) st.init(q, qx[q], qy[q], a.f, k0);
        for (int t = 0; t < nt; ++t) {
            ring.wait_full(t);
            const float *d = sm + ring.slot(t) * 5 * TILE;
            knn_f32_tile<K, Q, G, TILE>(st, d, d + TILE, d + 2 * TILE, d + 3 * TILE, d + 4 * TILE);
            ring.release(t, ntot, issue);
        }
        // ---- S4 in registers: R, mu, alpha (fp64) with the FIXED bounds
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            float robs;
            robs_of<float, K>(st.buf[q], k0, a.k, robs, d1[q]);
            al[q] = (float)alpha_eq((double)robs, a.r_exp, a.rmin, a.rmax, a.mf, a.lv);
            const int64_t idx = qid[q];
            if (valid[q]) {
                if (a.r_obs) a.r_obs[idx] = robs;
                if (a.alpha) a.alpha[idx] = al[q];
            }
        }
    }

    // ---- pass 2: weighting (S5)
    InterpF32State<Q> st2;
#pragma unroll
    for (int q = 0; q < Q; ++q) st2.init(q, qx[q], qy[q], al[q], d1[q]);
    const int nblk = acc_blocks(nt);
    int blk = 0, bend = nt + block_tile(1, nt, nblk);
    for (int t = nt; t < ntot; ++t) {
        ring.wait_full(t);
        const float *d = sm + ring.slot(t) * 5 * TILE;
        interp_f32_tile<Q, EMU, TILE>(st2, d, d + TILE, d + 2 * TILE);
        if (t + 1 == bend) {  // accumulation-block boundary, as in the weighting kernel
            st2.end_block();
            ++blk;
            bend = nt + block_tile(blk + 1, nt, nblk);
        }
        ring.release(t, ntot, issue);
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        if (!valid[q]) continue;
        write_result<float>(a.z, nullptr, qid[q], st2.SW[q], st2.SWZ[q], d1[q], qx[q], qy[q], a.px, a.py, a.pz,
                            a.nd, (double)al[q]);  // R19 coincidence, subnormal nearest
    }
}

template <int K, int Q = 2, int G = 16, unsigned EMU = 0x0141>
static int launch_fused_t(const FusedArgs &a, cudaStream_t st)
{
    const size_t smem = (size_t)5 * kStagesKF * kTileKF * sizeof(float) + 2 * kStagesKF * sizeof(uint64_t);
    if (cudaFuncSetAttribute(fused_fixed_kernel<K, Q, G, EMU>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess ||
        cudaFuncSetAttribute(fused_fixed_kernel<K, Q, G, EMU>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             100) != cudaSuccess)
        return -1;
    const int64_t per_cta = (int64_t)kBlock * Q;
    const unsigned grid = (unsigned)((a.nq + per_cta - 1) / per_cta);
    fused_fixed_kernel<K, Q, G, EMU><<<grid, kBlock, smem, st>>>(a);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

static int dispatch_fused(const FusedArgs &a, cudaStream_t st);

// Batches at least this large are spatially ordered (AIDW_KNN_ORDER=0 disables).
static bool order_fused(int64_t nq)
{
    const char *e = getenv("AIDW_KNN_ORDER");
    return nq >= 32768 && nq <= INT_MAX && !(e && e[0] == '0');  // perm is int32
}

int launch_fused_fixed(const void *data, int64_t ndp, int64_t nd, FilterData *filt, const void *qx,
                       const void *qy, int64_t nq, int k, double r_exp, const double *lvp, double rmin,
                       double rmax, int mf, void *z, void *r_obs, void *alpha, Scratch *sc, cudaStream_t st)
{
    const float *p = static_cast<const float *>(data);
    const float *c = static_cast<const float *>(filt->arrays);
    FusedArgs a;
    a.px = p;
    a.py = p + ndp;
    a.pz = p + 2 * ndp;
    a.ndp = ndp;
    a.nd = nd;
    a.f = FilterArgs{c, c + ndp, c + 2 * ndp, p, p + ndp, nullptr, nullptr, filt->c_x, filt->c_y, filt->r1, filt->cell_start,
                     filt->grid};  // caller's order
    a.qx = (const float *)qx;
    a.qy = (const float *)qy;
    a.nq = nq;
    a.k = k;
    a.r_exp = r_exp;
    for (int i = 0; i < 5; ++i) a.lv.a[i] = lvp[i];
    a.rmin = rmin;
    a.rmax = rmax;
    a.mf = mf;
    a.z = (float *)z;
    a.r_obs = (float *)r_obs;
    a.alpha = (float *)alpha;
    a.sc = sc;
    a.perm = nullptr;
    int pre = 0;
    if (filt->cell_start && order_fused(nq)) {  // spatial order (§4.7): Morton-sorted kNN copy
        pre = launch_order_queries((const float *)qx, (const float *)qy, nq, filt, &filt->qorder, &a.perm, st);
        if (pre < 0) return -1;
        if (a.perm) {
            a.f.cx = c + 3 * ndp;
            a.f.cy = c + 4 * ndp;
            a.f.pp = c + 5 * ndp;
            a.f.px = c + 6 * ndp;
            a.f.py = c + 7 * ndp;
        }
    }
    const int n = dispatch_fused(a, st);
    return n < 0 ? -1 : n + pre;
}

static int dispatch_fused(const FusedArgs &a, cudaStream_t st)
{
    const int k = a.k;
    if (k <= 1) return launch_fused_t<1>(a, st);
    if (k <= 2) return launch_fused_t<2>(a, st);
    if (k <= 4) return launch_fused_t<4>(a, st);
    if (k <= 8) return launch_fused_t<8>(a, st);
    if (k <= 10) return launch_fused_t<10>(a, st);
    if (k <= 12) return launch_fused_t<12>(a, st);
    if (k <= 15) return launch_fused_t<15>(a, st);
    if (k <= 16) return launch_fused_t<16>(a, st);
    if (k <= 24) return launch_fused_t<24>(a, st);
    return launch_fused_t<32>(a, st);
}

}  // namespace aidw
