// knn_loop_bench.cu -- microbenchmark of the kNN filter's main loop (passes.cuh
// knn_f32_tile) in isolation: one smem tile of (cx, cy, pp) read by every
// CTA, Q queries per thread, 8-point chunks of packed FFMA2 t = pp + A cx + B cy folded
// into a running 3-input minimum, one warp vote per group of G points (never taken:
// thr = -inf).  No TMA ring, no rare path, no epilogue -- the achievable pairs/clk/SM of
// the instruction mix alone, at a chosen number of resident CTAs per SM.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo tools/knn_loop_bench.cu -o knn_loop_bench
// Prints one JSON line per variant: pairs per clock per SM and the FMA-pipe fraction
// (1 FFMA2 = 2 FMA lanes per pair; 128 FMA lanes/clk/SM).
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

constexpr int TILE = 512;
constexpr int THREADS = 128;

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float fmin3f(float a, float b, float c)
{
    float d;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ float opaque(float x)
{
    asm volatile("" : "+f"(x));
    return x;
}

struct Clk {
    unsigned long long c0, c1;
};

// VAR 0: the product loop (3-input min tree per 8 points)
// VAR 1: 2-input min per couple (more ALU ops)
// VAR 2: FFMA2 only (t folded into a packed sum: no min; upper bound of the FMA rate)
// VAR 3: scalar FFMA for t (2 per pair, no packing) + the 3-input min tree
// VAR 4: FFMA2 for t + a direct compare per pair (hit |= t <= thr; FSETP)
// VAR 5: half the queries packed (FFMA2), half scalar (FFMA), + the min tree
template <int Q, int G, int VAR>
__global__ void __launch_bounds__(THREADS) knn_loop(const float *__restrict__ g, float *out, int reps, Clk *clk)
{
    extern __shared__ __align__(16) float sm[];
    float *scx = sm, *scy = sm + TILE, *spp = sm + 2 * TILE;
    for (int i = threadIdx.x; i < 3 * TILE; i += THREADS) sm[i] = g[i];
    __syncthreads();
    float A[Q], B[Q], thr[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        A[q] = opaque(-2.0f * (0.1f + 0.01f * q + 1e-6f * threadIdx.x));
        B[q] = opaque(-2.0f * (0.3f - 0.01f * q));
        thr[q] = opaque(-1e30f);
    }
    float acc = 0.f;
    float2 pacc[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) pacc[q] = make_float2(0.f, 0.f);
    unsigned long long c0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll 1
        for (int j = 0; j < TILE; j += G) {
            float mn[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) mn[q] = 3.0e38f;
#pragma unroll
            for (int c = 0; c < G; c += 8) {
                float cxv[8], cyv[8], ppv[8];
#pragma unroll
                for (int h = 0; h < 8; h += 4) {
                    const float4 CX = *reinterpret_cast<const float4 *>(scx + j + c + h);
                    const float4 CY = *reinterpret_cast<const float4 *>(scy + j + c + h);
                    const float4 PP = *reinterpret_cast<const float4 *>(spp + j + c + h);
                    cxv[h] = CX.x; cxv[h + 1] = CX.y; cxv[h + 2] = CX.z; cxv[h + 3] = CX.w;
                    cyv[h] = CY.x; cyv[h + 1] = CY.y; cyv[h + 2] = CY.z; cyv[h + 3] = CY.w;
                    ppv[h] = PP.x; ppv[h + 1] = PP.y; ppv[h + 2] = PP.z; ppv[h + 3] = PP.w;
                }
                bool hitv = false;
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    float t[8];
                    if (VAR == 3 || (VAR == 5 && q >= Q / 2)) {
#pragma unroll
                        for (int e = 0; e < 8; ++e) t[e] = fmaf(B[q], cyv[e], fmaf(A[q], cxv[e], ppv[e]));
                        mn[q] = fmin3f(fmin3f(t[0], t[1], t[2]), fmin3f(t[3], t[4], t[5]), fmin3f(t[6], t[7], mn[q]));
                        continue;
                    }
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        const float2 tt = ffma2(make_float2(B[q], B[q]), make_float2(cyv[2 * h], cyv[2 * h + 1]),
                                                ffma2(make_float2(A[q], A[q]), make_float2(cxv[2 * h], cxv[2 * h + 1]),
                                                      make_float2(ppv[2 * h], ppv[2 * h + 1])));
                        if (VAR == 2) {
                            pacc[q] = ffma2(tt, make_float2(1.0f, 1.0f), pacc[q]);
                        } else {
                            t[2 * h] = tt.x;
                            t[2 * h + 1] = tt.y;
                        }
                    }
                    if (VAR == 4) {
#pragma unroll
                        for (int e = 0; e < 8; ++e) hitv |= t[e] <= thr[q];
                    }
                    if (VAR == 0 || VAR == 5)
                        mn[q] = fmin3f(fmin3f(t[0], t[1], t[2]), fmin3f(t[3], t[4], t[5]), fmin3f(t[6], t[7], mn[q]));
                    else if (VAR == 1)
                        mn[q] = fminf(fminf(fminf(t[0], t[1]), fminf(t[2], t[3])),
                                      fminf(fminf(fminf(t[4], t[5]), fminf(t[6], t[7])), mn[q]));
                }
                if (VAR == 4) mn[0] = hitv ? -1.0f : mn[0];
            }
            bool hit = false;
#pragma unroll
            for (int q = 0; q < Q; ++q) hit |= mn[q] <= thr[q];
            if (__any_sync(0xffffffffu, hit)) acc += 1.f;  // never: thr = -1e30
        }
    }
    unsigned long long c1 = clock64();
#pragma unroll
    for (int q = 0; q < Q; ++q) acc += pacc[q].x + pacc[q].y;
    if (acc == 1234.5f) out[0] = acc;
    if (blockIdx.x == 0 && threadIdx.x == 0) *clk = Clk{c0, c1};
}

// VAR 6 (separate kernel): lanes = POINTS, the CTA's Q queries uniform across the CTA
// (coefficients from blockIdx only -> uniform registers): per couple of points 3 LDS.64,
// per query 2 FFMA2 with a uniform scalar operand and 1 FMNMX3 (min of the couple and
// the running minimum).
template <int Q, int G, int VAR>
__global__ void __launch_bounds__(THREADS) knn_loop_uni(const float *__restrict__ g, float *out, int reps, Clk *clk)
{
    extern __shared__ __align__(16) float sm[];
    float *scx = sm, *scy = sm + TILE, *spp = sm + 2 * TILE;
    for (int i = threadIdx.x; i < 3 * TILE; i += THREADS) sm[i] = g[i];
    __syncthreads();
    float A[Q], B[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        A[q] = -2.0f * (0.1f + 0.01f * q + 1e-6f * blockIdx.x);
        B[q] = -2.0f * (0.3f - 0.01f * q - 1e-6f * blockIdx.x);
    }
    const float thr = -1e30f;
    float acc = 0.f;
    unsigned long long c0 = clock64();
    for (int r = 0; r < reps; ++r) {
        float mn[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) mn[q] = 3.0e38f;
#pragma unroll 1
        for (int j = 2 * threadIdx.x; j < TILE; j += 2 * THREADS) {
            const float2 cx = *reinterpret_cast<const float2 *>(scx + j);
            const float2 cy = *reinterpret_cast<const float2 *>(scy + j);
            const float2 pp = *reinterpret_cast<const float2 *>(spp + j);
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const float2 t = ffma2(make_float2(B[q], B[q]), cy, ffma2(make_float2(A[q], A[q]), cx, pp));
                mn[q] = fmin3f(t.x, t.y, mn[q]);
            }
        }
        bool hit = false;
#pragma unroll
        for (int q = 0; q < Q; ++q) hit |= mn[q] <= thr;
        if (__any_sync(0xffffffffu, hit)) acc += 1.f;
    }
    unsigned long long c1 = clock64();
    if (acc == 1234.5f) out[0] = acc;
    if (blockIdx.x == 0 && threadIdx.x == 0) *clk = Clk{c0, c1};
}

// VAR 7 (separate kernel): the product loop's layout (lanes = queries, broadcast smem
// points) in fp16: t = pp + A cx + B cy on HFMA2 (2 points per instruction), a packed
// HMNMX2 min tree, 8-point chunks.  Tests whether the half2 pipes beat FFMA2 + FMNMX3.
template <int Q, int G, int VAR>
__global__ void __launch_bounds__(THREADS) knn_loop_h2(const float *__restrict__ g, float *out, int reps, Clk *clk)
{
    extern __shared__ __align__(16) float sm[];
    __half2 *hx = reinterpret_cast<__half2 *>(sm);  // TILE/2 couples each
    __half2 *hy = hx + TILE / 2, *hp = hy + TILE / 2;
    for (int i = threadIdx.x; i < TILE / 2; i += THREADS) {
        hx[i] = __floats2half2_rn(g[2 * i], g[2 * i + 1]);
        hy[i] = __floats2half2_rn(g[TILE + 2 * i], g[TILE + 2 * i + 1]);
        hp[i] = __floats2half2_rn(g[2 * TILE + 2 * i], g[2 * TILE + 2 * i + 1]);
    }
    __syncthreads();
    __half2 A[Q], B[Q];
    float thr[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        A[q] = __float2half2_rn(opaque(-2.0f * (0.1f + 0.01f * q + 1e-6f * threadIdx.x)));
        B[q] = __float2half2_rn(opaque(-2.0f * (0.3f - 0.01f * q)));
        thr[q] = opaque(-1e30f);
    }
    float acc = 0.f;
    unsigned long long c0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll 1
        for (int j = 0; j < TILE / 2; j += G / 2) {
            __half2 mn[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) mn[q] = __float2half2_rn(60000.f);
#pragma unroll
            for (int c = 0; c < G / 2; c += 4) {  // 8 points = 4 couples
                const uint4 X = *reinterpret_cast<const uint4 *>(hx + j + c);
                const uint4 Y = *reinterpret_cast<const uint4 *>(hy + j + c);
                const uint4 P = *reinterpret_cast<const uint4 *>(hp + j + c);
                const __half2 *xv = reinterpret_cast<const __half2 *>(&X);
                const __half2 *yv = reinterpret_cast<const __half2 *>(&Y);
                const __half2 *pv = reinterpret_cast<const __half2 *>(&P);
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    __half2 t[4];
#pragma unroll
                    for (int h = 0; h < 4; ++h) t[h] = __hfma2(B[q], yv[h], __hfma2(A[q], xv[h], pv[h]));
                    if (VAR == 8) {  // HFMA2 only: fold t into the running value with one more HFMA2
                        mn[q] = __hfma2(t[0], t[1], __hfma2(t[2], t[3], mn[q]));
                    } else if (VAR == 9) {  // compare per couple against the threshold (HSETP2) instead of a min tree
                        const __half2 th = __float2half2_rn(thr[q]);
                        const bool hh = __hble2(t[0], th) | __hble2(t[1], th) | __hble2(t[2], th) | __hble2(t[3], th);
                        if (hh) mn[q] = __float2half2_rn(-1.0f);
                    } else {
                        mn[q] = __hmin2(__hmin2(__hmin2(t[0], t[1]), __hmin2(t[2], t[3])), mn[q]);
                    }
                }
            }
            bool hit = false;
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const float2 m = __half22float2(mn[q]);
                hit |= fminf(m.x, m.y) <= thr[q];
            }
            if (__any_sync(0xffffffffu, hit)) acc += 1.f;
        }
    }
    unsigned long long c1 = clock64();
    if (acc == 1234.5f) out[0] = acc;
    if (blockIdx.x == 0 && threadIdx.x == 0) *clk = Clk{c0, c1};
}


// VAR 10-13 (round 2, separate kernel): the strip (1-D) pre-test and integer min trees.
// VAR 10: 1-D t = pu + A u (ONE HFMA2 per couple) + HMNMX2 tree (2 loads per 8 points)
// VAR 11: 1-D t on HFMA2 + packed int16 3-input min (VIMNMX3.S16x2) on the bit patterns
// VAR 12: 2-D t (two HFMA2 per couple, as VAR 7) + the VIMNMX3.S16x2 tree
__device__ __forceinline__ unsigned h2u(__half2 h) { return *reinterpret_cast<unsigned *>(&h); }
__device__ __forceinline__ unsigned vmin3(unsigned a, unsigned b, unsigned c)
{
    unsigned r;
    asm("min.s16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    asm("min.s16x2 %0, %1, %2;" : "=r"(r) : "r"(r), "r"(c));
    return r;
}
template <int Q, int G, int VAR>
__global__ void __launch_bounds__(THREADS) knn_loop_h1(const float *__restrict__ g, float *out, int reps, Clk *clk)
{
    extern __shared__ __align__(16) float sm[];
    __half2 *hx = reinterpret_cast<__half2 *>(sm);  // TILE/2 couples each
    __half2 *hy = hx + TILE / 2, *hp = hy + TILE / 2;
    for (int i = threadIdx.x; i < TILE / 2; i += THREADS) {
        hx[i] = __floats2half2_rn(g[2 * i], g[2 * i + 1]);
        hy[i] = __floats2half2_rn(g[TILE + 2 * i], g[TILE + 2 * i + 1]);
        hp[i] = __floats2half2_rn(g[2 * TILE + 2 * i], g[2 * TILE + 2 * i + 1]);
    }
    __syncthreads();
    __half2 A[Q], B[Q];
    float thr[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        A[q] = __float2half2_rn(opaque(-2.0f * (0.1f + 0.01f * q + 1e-6f * threadIdx.x)));
        B[q] = __float2half2_rn(opaque(-2.0f * (0.3f - 0.01f * q)));
        thr[q] = opaque(-1e30f);
    }
    float acc = 0.f;
    unsigned long long c0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll 1
        for (int j = 0; j < TILE / 2; j += G / 2) {
            __half2 mn[Q];
            unsigned mi[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                mn[q] = __float2half2_rn(60000.f);
                mi[q] = 0x7bff7bffu;
            }
#pragma unroll
            for (int c = 0; c < G / 2; c += 4) {  // 8 points = 4 couples
                const uint4 X = *reinterpret_cast<const uint4 *>(hx + j + c);
                const uint4 P = *reinterpret_cast<const uint4 *>(hp + j + c);
                const __half2 *xv = reinterpret_cast<const __half2 *>(&X);
                const __half2 *pv = reinterpret_cast<const __half2 *>(&P);
                uint4 Y = make_uint4(0, 0, 0, 0);
                if (VAR == 12) Y = *reinterpret_cast<const uint4 *>(hy + j + c);
                const __half2 *yv = reinterpret_cast<const __half2 *>(&Y);
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    __half2 t[4];
#pragma unroll
                    for (int h = 0; h < 4; ++h)
                        t[h] = VAR == 12 ? __hfma2(B[q], yv[h], __hfma2(A[q], xv[h], pv[h])) : __hfma2(A[q], xv[h], pv[h]);
                    if (VAR == 10)
                        mn[q] = __hmin2(__hmin2(__hmin2(t[0], t[1]), __hmin2(t[2], t[3])), mn[q]);
                    else
                        mi[q] = vmin3(h2u(t[0]), h2u(t[1]), vmin3(h2u(t[2]), h2u(t[3]), mi[q]));
                }
            }
            bool hit = false;
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                if (VAR == 10) {
                    const float2 m = __half22float2(mn[q]);
                    hit |= fminf(m.x, m.y) <= thr[q];
                } else {
                    const int lo = (int)(short)(mi[q] & 0xffffu), hi = (int)(short)(mi[q] >> 16);
                    hit |= (float)min(lo, hi) <= thr[q];
                }
            }
            if (__any_sync(0xffffffffu, hit)) acc += 1.f;
        }
    }
    unsigned long long c1 = clock64();
    if (acc == 1234.5f) out[0] = acc;
    if (blockIdx.x == 0 && threadIdx.x == 0) *clk = Clk{c0, c1};
}

template <int Q, int G, int VAR>
static void run(const char *name, int ctas_per_sm, const float *g, float *out, Clk *clk, int sms, double mhz_ref)
{
    auto k = (VAR >= 10) ? knn_loop_h1<Q, G, VAR> : (VAR >= 7) ? knn_loop_h2<Q, G, VAR> : VAR == 6 ? knn_loop_uni<Q, G, VAR> : knn_loop<Q, G, VAR>;
    // pad the dynamic smem so at most ctas_per_sm CTAs fit on an SM
    size_t smem = 3 * TILE * sizeof(float);
    const size_t per = (227 * 1024) / ctas_per_sm;
    if (per > smem) smem = per - 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, THREADS, smem);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k);
    const int reps = 200;
    const int grid = sms * occ;
    k<<<grid, THREADS, smem>>>(g, out, reps, clk);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<grid, THREADS, smem>>>(g, out, reps, clk);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    Clk h;
    cudaMemcpy(&h, clk, sizeof h, cudaMemcpyDeviceToHost);
    const double pairs = (double)grid * THREADS * Q * TILE * reps;
    // rate from the event time at the SM clock read during the run (block 0's clock64
    // span is not the kernel's: r02a showed CTAs finishing at different times)
    const double ppc = pairs / sms / (ms * 1e-3) / (mhz_ref * 1e6);
    printf("{\"variant\": \"%s\", \"Q\": %d, \"G\": %d, \"regs\": %d, \"ctas_per_sm\": %d, \"warps_per_sm\": %d, "
           "\"pairs_per_clk_sm\": %.2f, \"fma_lanes_frac\": %.3f, \"ms\": %.3f, \"mhz\": %.0f, \"err\": \"%s\"}\n",
           name, Q, G, fa.numRegs, occ, occ * THREADS / 32, ppc, ppc * 2.0 / 128.0, ms, mhz_ref,
           cudaGetErrorString(cudaGetLastError()));
}

int main()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *g, *out;
    Clk *clk;
    cudaMalloc(&g, 3 * TILE * sizeof(float));
    cudaMalloc(&out, 4);
    cudaMalloc(&clk, sizeof(Clk));
    float h[3 * TILE];
    for (int i = 0; i < 3 * TILE; ++i) h[i] = 0.001f * (float)(i % 997);
    cudaMemcpy(g, h, sizeof h, cudaMemcpyHostToDevice);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const double mhz = clk_khz / 1e3;  // max SM clock (the runs are checked against nvidia-smi)
    for (int c : {4, 8}) {
        run<4, 32, 0>("fmin3_q4", c, g, out, clk, sms, mhz);
        run<8, 32, 0>("fmin3_q8", c, g, out, clk, sms, mhz);
        run<4, 32, 1>("fmin2_q4", c, g, out, clk, sms, mhz);
        run<4, 32, 2>("ffma2_only_q4", c, g, out, clk, sms, mhz);
        run<4, 32, 3>("scalar_ffma_fmin3_q4", c, g, out, clk, sms, mhz);
        run<4, 32, 4>("ffma2_fsetp_q4", c, g, out, clk, sms, mhz);
        run<4, 32, 5>("half_packed_fmin3_q4", c, g, out, clk, sms, mhz);
        run<8, 32, 5>("half_packed_fmin3_q8", c, g, out, clk, sms, mhz);
        run<8, 32, 6>("uniform_queries_q8", c, g, out, clk, sms, mhz);
        run<16, 32, 6>("uniform_queries_q16", c, g, out, clk, sms, mhz);
        run<32, 32, 6>("uniform_queries_q32", c, g, out, clk, sms, mhz);
        run<4, 32, 7>("fp16_hfma2_hmin2_q4", c, g, out, clk, sms, mhz);
        run<8, 32, 7>("fp16_hfma2_hmin2_q8", c, g, out, clk, sms, mhz);
        run<4, 32, 8>("fp16_hfma2_only_q4", c, g, out, clk, sms, mhz);
        run<4, 32, 9>("fp16_hfma2_hsetp2_q4", c, g, out, clk, sms, mhz);
        run<4, 32, 10>("fp16_strip_hmin2_q4", c, g, out, clk, sms, mhz);
        run<8, 32, 10>("fp16_strip_hmin2_q8", c, g, out, clk, sms, mhz);
        run<4, 32, 11>("fp16_strip_vimnmx3_q4", c, g, out, clk, sms, mhz);
        run<8, 32, 11>("fp16_strip_vimnmx3_q8", c, g, out, clk, sms, mhz);
        run<4, 32, 12>("fp16_2d_vimnmx3_q4", c, g, out, clk, sms, mhz);
        run<8, 32, 12>("fp16_2d_vimnmx3_q8", c, g, out, clk, sms, mhz);
    }
    return 0;
}
