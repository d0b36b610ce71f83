// device.cuh -- sm_100a device helpers for the AIDW kernels: mbarrier + 1-D TMA
// bulk copies (cp.async.bulk, SASS UBLKCP) for the shared-memory data-tile ring,
// MUFU lg2/ex2, and exact (non-contracted) distance arithmetic.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace aidw {

constexpr int kBlock = 128;          // threads per CTA (4 warps)
constexpr int kWarps = kBlock / 32;

// ---------------------------------------------------------------- smem / mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(addr),
        "r"(parity)
        : "memory");
}

// 1-D bulk async copy global -> shared, completion signalled on `bar` (TMA engine).
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// ---------------------------------------------------------------- MUFU
__device__ __forceinline__ float lg2_approx(float x)
{
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float lg2_approx_noftz(float x)
{
    float y;
    asm("lg2.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float ex2_approx(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// A value the compiler cannot rematerialise from its inputs (it stays in a register).
__device__ __forceinline__ float opaque(float x)
{
    float r;
    asm volatile("mov.b32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// Three-input fp32 min (sm_100 FMNMX3; NaN inputs are ignored like fminf's).
__device__ __forceinline__ float fmin3(float a, float b, float c)
{
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

// Minimum of N values as a tree of 3-input mins (N = 16: 8 instructions, depth 3).
template <int N> __device__ __forceinline__ float min_tree3(const float (&t)[N])
{
    float v[N];
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = t[i];
    int n = N;
#pragma unroll
    for (int level = 0; level < 8; ++level) {
        if (n == 1) break;
        int o = 0;
#pragma unroll
        for (int i = 0; i < N; i += 3) {
            if (i >= n) break;
            if (i + 2 < n)
                v[o++] = fmin3(v[i], v[i + 1], v[i + 2]);
            else if (i + 1 < n)
                v[o++] = fminf(v[i], v[i + 1]);
            else
                v[o++] = v[i];
        }
        n = o;
    }
    return v[0];
}

__device__ __forceinline__ float rsqrt_approx(float x)
{
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float rcp_approx(float x)
{
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// ---------------------------------------------------------------- exact arithmetic
// Canonical distance sequence (R16), round-to-nearest, never contracted:
//   dx = qx - px; dy = qy - py; s = fma(dx, dx, dy*dy)
__device__ __forceinline__ float dist_sq(float qx, float qy, float px, float py)
{
    float dx = __fsub_rn(qx, px);
    float dy = __fsub_rn(qy, py);
    return __fmaf_rn(dx, dx, __fmul_rn(dy, dy));
}

__device__ __forceinline__ double dist_sq(double qx, double qy, double px, double py)
{
    double dx = __dsub_rn(qx, px);
    double dy = __dsub_rn(qy, py);
    return __fma_rn(dx, dx, __dmul_rn(dy, dy));
}

__device__ __forceinline__ float sqrt_rn(float s) { return __fsqrt_rn(s); }
__device__ __forceinline__ double sqrt_rn(double s) { return __dsqrt_rn(s); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }

template <typename T> __device__ __forceinline__ T pos_inf();
template <> __device__ __forceinline__ float pos_inf<float>() { return __int_as_float(0x7f800000); }
template <> __device__ __forceinline__ double pos_inf<double>() { return __longlong_as_double(0x7ff0000000000000LL); }

__device__ __forceinline__ float tmin(float a, float b) { return fminf(a, b); }
__device__ __forceinline__ float tmax(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ double tmin(double a, double b) { return fmin(a, b); }
__device__ __forceinline__ double tmax(double a, double b) { return fmax(a, b); }

// 4 consecutive values from shared memory (broadcast read: all lanes, same address).
// 16-byte shared-memory load from a 32-bit shared-window address (computed once per
// tile, so the loop does not re-derive the window base every iteration).
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ float4 lds128(uint32_t a)
{
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}

template <typename T> struct Vec4 { T v[4]; };

__device__ __forceinline__ Vec4<float> lds4(const float *p)
{
    float4 t = *reinterpret_cast<const float4 *>(p);
    return {{t.x, t.y, t.z, t.w}};
}

__device__ __forceinline__ Vec4<double> lds4(const double *p)
{
    double2 a = reinterpret_cast<const double2 *>(p)[0];
    double2 b = reinterpret_cast<const double2 *>(p)[1];
    return {{a.x, a.y, b.x, b.y}};
}

}  // namespace aidw
