// packed.cuh -- sm_100 packed fp32x2 arithmetic (PTX add/sub/mul/fma .rn.f32x2 ->
// SASS FADD2 / FMUL2 / FFMA2: two IEEE round-to-nearest fp32 operations per lane per
// issue slot) and a software exp2 on the FMA pipe used to offload part of the
// weighting pass's ex2 work from the SFU.
#pragma once

#include <cstdint>

namespace aidw {

typedef float2 f32x2;  // {lo, hi} fp32 pair in one 64-bit register pair

// CUDA 12.9 sm_100 builtins (crt/sm_100_rt.h): visible to the optimiser and the
// scheduler, unlike inline PTX.
__device__ __forceinline__ f32x2 pack2(float lo, float hi) { return make_float2(lo, hi); }
__device__ __forceinline__ void unpack2(f32x2 v, float &lo, float &hi) { lo = v.x; hi = v.y; }
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ f32x2 sub2(f32x2 a, f32x2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ f32x2 splat2(float v) { return make_float2(v, v); }

// 2^x for x <= ~0 on the FMA pipe: x clamped to [-126, +inf), j = rint(x) via the
// 1.5*2^23 magic constant, f = x - j in [-0.5, 0.5], 2^f by a degree-4 near-minimax
// polynomial (max relative error 2.7e-6 in fp32 Horner form; fitted offline, see
// tools/fit_exp2.py), exponent added as an integer: bits(2^f) + (j << 23).
// Results below 2^-126 are not produced (the clamp): such weights are < 1e-38 of the
// nearest point's weight (w is scaled to 1 at the nearest point) and vanish in the sums.
// CLAMP = false: the caller guarantees x >= -126 (round 2: tiles without
// padding points, CTAs whose queries' weights provably stay above 2^-126), saving the two
// FMNMX per couple; the result is then bit-identical to the clamped form.
template <bool CLAMP = true>
__device__ __forceinline__ f32x2 exp2_poly2(f32x2 a)
{
    constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
    float a0, a1;
    unpack2(a, a0, a1);
    if (CLAMP) {
        a0 = fmaxf(a0, -126.0f);
        a1 = fmaxf(a1, -126.0f);
    }
    const f32x2 x = pack2(a0, a1);
    const f32x2 t = add2(x, splat2(kMagic));
    const f32x2 j = sub2(t, splat2(kMagic));
    const f32x2 f = sub2(x, j);
    f32x2 p = fma2(splat2(0.009570101276040077f), f, splat2(0.05591785907745361f));
    p = fma2(p, f, splat2(0.240247443318367f));
    p = fma2(p, f, splat2(0.6931217908859253f));
    p = fma2(p, f, splat2(0.9999992847442627f));
    float t0, t1, p0, p1;
    unpack2(t, t0, t1);
    unpack2(p, p0, p1);
    const float r0 = __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23));
    const float r1 = __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23));
    return pack2(r0, r1);
}

// Scalar form of exp2_poly2 (same constants and operation order, per element).
template <bool CLAMP = true>
__device__ __forceinline__ float exp2_poly1(float a)
{
    constexpr float kMagic = 12582912.0f;
    const float x = CLAMP ? fmaxf(a, -126.0f) : a;
    const float t = __fadd_rn(x, kMagic);
    const float j = __fadd_rn(t, -kMagic);
    const float f = __fadd_rn(x, -j);
    float p = __fmaf_rn(0.009570101276040077f, f, 0.05591785907745361f);
    p = __fmaf_rn(p, f, 0.240247443318367f);
    p = __fmaf_rn(p, f, 0.6931217908859253f);
    p = __fmaf_rn(p, f, 0.9999992847442627f);
    return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

}  // namespace aidw
