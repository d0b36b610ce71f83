"""CPU property test of the fp16 kNN pre-filter's rounding margin (DESIGN.md §4.1,
passes.cuh h16_threshold / h16_convert / knn_h16_tile).

The fp16 stage may only drop pairs that cannot enter a query's list: every TRUE
candidate (canonical fp32 squared distance s < v, the list's k-th value) must give
t̂ <= T.  This test emulates the kernel's operations bit for bit on the CPU -- fp32
subtraction and scaling, fp16 rounding of the coordinates, p̂p rounded through fp32 to
fp16, the two fp16 FMAs (the exact product + sum of fp16 operands is exact in fp64, then
ONE rounding to fp16) -- and checks t̂ <= T on adversarial candidates: points just inside
the k-th distance, at every angle, for queries anywhere in the CTA's region, at the scales
the kernel picks (sigma m <= 16) and at extreme magnitudes (tiny and large coordinates,
subnormal fp16 values).  T is the margin formula of h16_threshold, restated here (the
GPU bit-identity tests exercise the CUDA code itself).
"""
import math
from fractions import Fraction

import numpy as np

f16, f32 = np.float16, np.float32
U16 = 2.0 ** -11
UP = 2.0 ** -11 + 2.0 ** -22


def fl32(x):
    return float(f32(x))


def fma32(a, b, c):
    """fp32 fma: the exact a*b + c rounded once (Fraction -> nearest fp64 is exact for
    these magnitudes only up to 53 bits, so round the exact value straight to fp32)."""
    ex = Fraction(a) * Fraction(b) + Fraction(c)
    lo = f32(float(ex))  # nearest fp64, then fp32: fix a possible double rounding below
    cand = [lo, np.nextafter(lo, f32(-np.inf)), np.nextafter(lo, f32(np.inf))]
    return float(min(cand, key=lambda z: (abs(Fraction(float(z)) - ex), int(np.float32(z).view(np.uint32)) & 1)))


def fl16(x):
    return float(f16(x))


def fma16(a, b, c):
    # a, b, c are fp16 values: a*b + c is exact in fp64, then one rounding
    return fl16(a * b + c)


def convert(x, y, cx, cy, sig):
    """h16_convert: fp32 x - C_x, times sigma (exact), clamp, fp16; p̂p via fp32."""
    u = fl16(min(max(fl32(fl32(x - cx) * sig), -256.0), 256.0))
    v = fl16(min(max(fl32(fl32(y - cy) * sig), -256.0), 256.0))
    pp = fl16(min(fma32(u, u, fl32(v * v)), 32768.0))
    return u, v, pp


def coeffs(qx, qy, cx, cy, sig):
    a = fl16(-2.0 * fl32(fl32(qx - cx) * sig))
    b = fl16(-2.0 * fl32(fl32(qy - cy) * sig))
    return a, b


def threshold(v, qx, qy, cx, cy, sig, a, b, strip=False):
    """h16_threshold<STRIP> (passes.cuh), restated: the 2-D threshold, or with strip=True
    the one-axis (strip) threshold of the axis whose coefficient is `a`."""
    if not v < math.inf:
        return math.inf
    dx, dy = qx - cx, qy - cy
    qn = sig * math.sqrt(dx * dx + dy * dy) * (1.0 + 2.0 ** -40)
    r = sig * math.sqrt(v * (1.0 + 2.0 ** -20))
    ah, bh = 0.5 * a, 0.5 * b
    qq = ah * ah + bh * bh
    qb = max(qn, math.sqrt(qq)) * (1.0 + UP)
    d = UP * (2.0 * qb + r)
    p = qb + r + d
    rr = r + d
    t = rr * rr - (ah * ah if strip else qq) + UP * p * p + 1.002 * U16 * (p * p + qb * qb + rr * rr) + 2.0 ** -18
    return ru32(t)  # __double2float_ru (upper bound)


def ru32(t):
    """fp64 -> fp32 rounded up (an upper bound of t)."""
    f = f32(t)
    return float(f) if float(f) >= t else float(np.nextafter(f, f32(np.inf)))


def t2d(T1, b):
    """h16_t2d: T1 - (b/2)^2, the product exact, ONE upward rounding to fp32."""
    ex = Fraction(T1) - Fraction(0.5 * b) ** 2
    lo = f32(float(ex))
    for z in (np.nextafter(lo, f32(-np.inf)), lo, np.nextafter(lo, f32(np.inf))):
        if Fraction(float(z)) >= ex:
            return float(z)
    raise AssertionError


def strip_convert(s):
    """h16_convert's strip square: p̂s = fl16(min(ŝ², 32768)) (ŝ² exact in fp32)."""
    return fl16(min(fl32(s * s), 32768.0))


def canon32(qx, qy, px, py):
    dx = fl32(qx - px)
    dy = fl32(qy - py)
    return fma32(dx, dx, fl32(dy * dy))


def check_case(rng, scale, n_q=40, n_p=60):
    """A CTA region of radius ~scale around C, queries inside, k-th distance ~ kth."""
    cx = fl32(rng.uniform(-3, 3) * scale * 50)
    cy = fl32(rng.uniform(-3, 3) * scale * 50)
    qs = [(fl32(cx + rng.uniform(-1, 1) * scale), fl32(cy + rng.uniform(-1, 1) * scale)) for _ in range(n_q)]
    kth = scale * 10 ** rng.uniform(-2.5, 0.3)  # k-th distance relative to the region
    vs = [fl32((kth * rng.uniform(0.5, 1.5)) ** 2) for _ in qs]
    m = max(max(math.hypot(qx - cx, qy - cy), math.sqrt(v)) for (qx, qy), v in zip(qs, vs)) * 1.001
    e = math.frexp(16.0 / m)[1] - 1
    sig = 2.0 ** max(-100, min(100, e))
    worst = -math.inf
    for (qx, qy), v in zip(qs, vs):
        a, b = coeffs(qx, qy, cx, cy, sig)
        T = threshold(v, qx, qy, cx, cy, sig, a, b)
        for _ in range(n_p):
            ang = rng.choice([0.0, 0.5 * math.pi, math.pi, 1.5 * math.pi]) if rng.uniform() < 0.3 else rng.uniform(0, 2 * math.pi)
            rad = math.sqrt(v) * (1.0 - 10 ** rng.uniform(-7, -0.3))  # just inside, mostly
            px, py = fl32(qx + rad * math.cos(ang)), fl32(qy + rad * math.sin(ang))
            if not canon32(qx, qy, px, py) < v:
                continue  # not a true candidate after rounding
            u, w, pp = convert(px, py, cx, cy, sig)
            t = fma16(b, w, fma16(a, u, pp))
            worst = max(worst, t - T)
            assert t <= T, (qx, qy, px, py, v, t, T)
            # the strip pre-test on either axis (knn_filter_kernel swaps the axes, and the
            # coefficients with them, when the strip axis is y) and its derived 2-D threshold
            for (c1, s1, c2, s2) in ((a, u, b, w), (b, w, a, u)):
                T1 = threshold(v, qx, qy, cx, cy, sig, c1, c2, strip=True)
                t1 = fma16(c1, s1, strip_convert(s1))
                assert t1 <= T1, (qx, qy, px, py, v, t1, T1)
                pp2 = fl16(min(fma32(s1, s1, fl32(s2 * s2)), 32768.0))
                t2 = fma16(c2, s2, fma16(c1, s1, pp2))
                assert t2 <= t2d(T1, c2), (qx, qy, px, py, v, t2, T1)
    return worst


def test_h16_margin_keeps_every_candidate():
    rng = np.random.default_rng(2024)
    for scale in (1e-2, 2e-2, 1.0, 3e-5, 7e3):
        for _ in range(12):
            check_case(rng, scale)


def test_h16_margin_is_not_vacuous():
    """The margin is tight enough to be useful: for a typical C4 CTA (region radius ~9
    k-th distances) T exceeds the exact scaled threshold by well under the threshold."""
    cx = cy = 0.5
    qx, qy = fl32(0.5 + 0.016), fl32(0.5)
    v = fl32(0.0018 ** 2)
    sig = 2.0 ** (math.frexp(16.0 / (0.016 * 1.001))[1] - 1)
    a, b = coeffs(qx, qy, cx, cy, sig)
    T = threshold(v, qx, qy, cx, cy, sig, a, b)
    exact = sig * sig * v - (0.5 * a) ** 2 - (0.5 * b) ** 2
    assert 0 < T - exact < 0.5 * sig * sig * v


def test_strip_margin_is_not_vacuous():
    """The strip threshold of a typical C4 CTA keeps only a thin strip: a point at 3 k-th
    distances from the query along the strip axis fails the one-axis test."""
    cx = cy = 0.5
    qx, qy = fl32(0.5 + 0.006), fl32(0.5 - 0.004)
    v = fl32(0.0018 ** 2)
    sig = 2.0 ** (math.frexp(16.0 / (0.011 * 1.001))[1] - 1)
    a, b = coeffs(qx, qy, cx, cy, sig)
    T1 = threshold(v, qx, qy, cx, cy, sig, a, b, strip=True)
    u, _, _ = convert(fl32(qx + 3 * 0.0018), qy, cx, cy, sig)
    assert fma16(a, u, strip_convert(u)) > T1


def test_strip_mutation_detected():
    """Dropping the margin terms from the strip threshold loses true candidates."""
    rng = np.random.default_rng(7)
    lost = 0
    for _ in range(400):
        cx, cy = 0.5, 0.5
        qx, qy = fl32(0.5 + rng.uniform(-0.01, 0.01)), fl32(0.5 + rng.uniform(-0.01, 0.01))
        v = fl32(0.0018 ** 2)
        sig = 2.0 ** (math.frexp(16.0 / (0.0142 * 1.001))[1] - 1)
        a, b = coeffs(qx, qy, cx, cy, sig)
        r = sig * math.sqrt(v)
        bare = r * r - (0.5 * a) ** 2  # no rounding terms
        rad = math.sqrt(v) * (1 - 1e-6)
        u, _, _ = convert(fl32(qx + rad * rng.choice([-1.0, 1.0])), qy, cx, cy, sig)
        lost += fma16(a, u, strip_convert(u)) > bare
    assert lost > 0


# ---------------------------------------------------------------------------------
# fp64 handles (round 2): the converted points are the centred fp32 filter coordinates
# cx = fl32(x - c) (c the fp32 data-bbox centre), the CTA centre C lives on the same
# centred scale, and the threshold adds the centring term of passes.cuh H16Frame:
# sigma 2^-23 (r1 + |q - c|_1) to the displacement bound.

def threshold_frame(v, qx, qy, Cxd, Cyd, ox, oy, r1, sig, a, b, strip, centred=True):
    """h16_threshold<STRIP, double> (passes.cuh), restated."""
    if not v < math.inf:
        return math.inf
    dx, dy = qx - Cxd, qy - Cyd
    qn = sig * math.sqrt(dx * dx + dy * dy) * (1.0 + 2.0 ** -40)
    r = sig * math.sqrt(v * (1.0 + 2.0 ** -20))
    ah, bh = 0.5 * a, 0.5 * b
    qq = ah * ah + bh * bh
    qb = max(qn, math.sqrt(qq)) * (1.0 + UP)
    ce = sig * 2.0 ** -23 * (r1 + abs(qx - ox) + abs(qy - oy)) * 1.001 if centred else 0.0
    d = UP * (2.0 * qb + r) + ce
    p = qb + r + d
    rr = r + d
    t = rr * rr - (ah * ah if strip else qq) + UP * p * p + 1.002 * U16 * (p * p + qb * qb + rr * rr) + 2.0 ** -18
    return ru32(t)


def canon64(qx, qy, px, py):
    """The fp64 canonical s = fma(dx, dx, dy*dy) (R16): one rounding of the exact value
    (int / int true division in Python rounds correctly)."""
    dx, dy = qx - px, qy - py
    ex = Fraction(dx) * Fraction(dx) + Fraction(dy * dy)
    return ex.numerator / ex.denominator


def check_case_f64(rng, region, kth, centred=True, n_q=30, n_p=50):
    """Data spread over [0, 1)^2 (r1 ~ 1), a CTA region of half-width `region` somewhere
    inside, k-th distances ~kth: the centring rounding (~2^-25 absolute) is then a
    sizeable share of the scaled margin when region and kth are small."""
    c_x, c_y = fl32(0.5 + 2.0 ** -30 * 3), fl32(0.5 - 2.0 ** -31 * 5)
    r1 = float(f32((0.5 + 0.5) * (1.0 + 1e-6)))
    ctr = (rng.uniform(0.1, 0.9), rng.uniform(0.1, 0.9))
    qs = [(ctr[0] + rng.uniform(-1, 1) * region, ctr[1] + rng.uniform(-1, 1) * region) for _ in range(n_q)]
    hq = [(fl32(qx - c_x), fl32(qy - c_y)) for qx, qy in qs]
    C = (fl32(0.5 * min(h[0] for h in hq)) + fl32(0.5 * max(h[0] for h in hq)),
         fl32(0.5 * min(h[1] for h in hq)) + fl32(0.5 * max(h[1] for h in hq)))
    C = (fl32(C[0]), fl32(C[1]))
    vs = [(kth * rng.uniform(0.5, 1.5)) ** 2 for _ in qs]
    m = max(max(math.hypot(h[0] - C[0], h[1] - C[1]), math.sqrt(v)) for h, v in zip(hq, vs)) * 1.001
    sig = 2.0 ** (math.frexp(16.0 / m)[1] - 1)
    lost = 0
    for (qx, qy), (hx, hy), v in zip(qs, hq, vs):
        a, b = coeffs(hx, hy, C[0], C[1], sig)
        for _ in range(n_p):
            ang = rng.choice([0.0, 0.5 * math.pi, math.pi, 1.5 * math.pi]) if rng.uniform() < 0.3 else rng.uniform(0, 2 * math.pi)
            rad = math.sqrt(v) * (1.0 - 10 ** rng.uniform(-9, -0.3))
            px, py = qx + rad * math.cos(ang), qy + rad * math.sin(ang)
            if not canon64(qx, qy, px, py) < v:
                continue
            cx, cy = fl32(px - c_x), fl32(py - c_y)
            u, w, pp = convert(cx, cy, C[0], C[1], sig)
            for (c1, s1, c2, s2) in ((a, u, b, w), (b, w, a, u)):
                T1 = threshold_frame(v, qx, qy, c_x + C[0], c_y + C[1], c_x, c_y, r1, sig, c1, c2, True, centred)
                t1 = fma16(c1, s1, strip_convert(s1))
                pp2 = fl16(min(fma32(s1, s1, fl32(s2 * s2)), 32768.0))
                t2 = fma16(c2, s2, fma16(c1, s1, pp2))
                ok = t1 <= T1 and t2 <= t2d(T1, c2)
                if centred:
                    assert ok, (qx, qy, px, py, v, t1, T1)
                lost += not ok
    return lost


def test_h16_margin_f64_centred_keeps_every_candidate():
    rng = np.random.default_rng(2025)
    for region, kth in ((1e-2, 2e-3), (2.0 ** -14, 2.0 ** -17), (2.0 ** -18, 2.0 ** -20), (1e-6, 3e-7), (1e-7, 2e-8)):
        for _ in range(6):
            check_case_f64(rng, region, kth)


def test_h16_margin_f64_centring_term_needed():
    """Mutation check: without the centring term the fp64 thresholds lose true candidates
    once the CTA region is small against the data extent."""
    rng = np.random.default_rng(5)
    assert check_case_f64(rng, 1e-6, 3e-7, centred=False, n_q=10, n_p=40) > 0
