"""Exact-arithmetic pins of the oracle's distance rounding sequence (R16).

The 2^-10-grid pin in test_oracle.py cannot tell ``fma(dx, dx, dy*dy)`` from
``dx*dx + dy*dy``: on that grid every operation is exact.  Here the expected values
come from exact rational arithmetic (``fractions.Fraction``) with ONE explicit
round-to-nearest-even per operation of the R16 sequence -- no libm, no numpy float
arithmetic, no oracle code -- on inputs where the fused and unfused sequences round
differently (the bench's 2^-24 grid for fp32, arbitrary doubles for fp64).  A dropped
fma, an extra rounding or a swapped operand fails them.

Fixture: tests/golden/fma_cases.json (the VERDICT r1 example, values by exact
arithmetic).
"""
import json
import math
import os
from fractions import Fraction

import numpy as np

F32 = (24, -126)   # (precision bits, minimum normal exponent)
F64 = (53, -1022)
CASES = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fma_cases.json")))


def rne(fr: Fraction, fmt) -> Fraction:
    """Round a rational to the nearest representable value of ``fmt``, ties to even."""
    p, emin = fmt
    if fr == 0:
        return Fraction(0)
    sign = -1 if fr < 0 else 1
    a = abs(fr)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    e = max(e, emin)
    scale = Fraction(2) ** (p - 1 - e)
    m = a * scale
    n = m.numerator // m.denominator
    r = m - n
    if r > Fraction(1, 2) or (r == Fraction(1, 2) and n % 2 == 1):
        n += 1
    return sign * Fraction(n) / scale


def sqrt_rn(s: Fraction, fmt) -> Fraction:
    """Correctly rounded square root of a non-negative rational (integer isqrt)."""
    p, _ = fmt
    if s == 0:
        return Fraction(0)
    e = (s.numerator.bit_length() - s.denominator.bit_length()) // 2
    # find e with 2^e <= sqrt(s) < 2^(e+1)
    while Fraction(2) ** (2 * e) > s:
        e -= 1
    while Fraction(2) ** (2 * e + 2) <= s:
        e += 1
    k = p - 1 - e
    t = s * Fraction(4) ** k             # sqrt(t) in [2^(p-1), 2^p)
    n = math.isqrt(t.numerator // t.denominator)
    h = Fraction(2 * n + 1, 2)           # midpoint n + 1/2
    if t > h * h or (t == h * h and n % 2 == 1):
        n += 1
    return Fraction(n) / Fraction(2) ** k


def r16(qx, qy, px, py, fmt):
    """R16 with one rounding per operation: dx, dy, dy*dy, fma, sqrt."""
    dx = rne(Fraction(qx) - Fraction(px), fmt)
    dy = rne(Fraction(qy) - Fraction(py), fmt)
    dy2 = rne(dy * dy, fmt)
    s = rne(dx * dx + dy2, fmt)
    return s, sqrt_rn(s, fmt)


def unfused(qx, qy, px, py, fmt):
    dx = rne(Fraction(qx) - Fraction(px), fmt)
    dy = rne(Fraction(qy) - Fraction(py), fmt)
    s = rne(rne(dx * dx, fmt) + rne(dy * dy, fmt), fmt)
    return s, sqrt_rn(s, fmt)


def test_rounding_helpers_against_known_values():
    # the helpers themselves, on values fixed by IEEE 754 / the decimal literals
    assert rne(Fraction(1, 3), F64) == Fraction(1 / 3)
    assert rne(Fraction(1, 3), F32) == Fraction(float(np.float32(1 / 3)))
    assert rne(Fraction(1) + Fraction(2) ** -24, F32) == 1           # tie -> even
    assert rne(Fraction(1) + Fraction(3, 2 ** 25), F32) == 1 + Fraction(2) ** -23
    assert sqrt_rn(Fraction(2), F64) == Fraction(1.4142135623730951)
    assert sqrt_rn(Fraction(25), F32) == 5
    assert sqrt_rn(Fraction(2), F32) == Fraction(float(np.float32(1.4142135)))


def test_verdict_example_fixture():
    """dx = -0.5729835033416748, dy = 0.6888355016708374 on the 2^-24
    grid: fused s = 0.8028044104576111, unfused 0.8028044700622559 (float32)."""
    for c in CASES["f32"]:
        s_f, _ = r16(c["qx"], c["qy"], c["px"], c["py"], F32)
        s_u, _ = unfused(c["qx"], c["qy"], c["px"], c["py"], F32)
        assert float(s_f) == c["s_fused"] and float(s_u) == c["s_unfused"], c["cite"]


def _grid_cases(seed, n, want):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < want:
        u = rng.integers(0, 1 << 24, size=(n, 4))
        for qx, qy, px, py in u / float(1 << 24):
            s_f, d_f = r16(qx, qy, px, py, F32)
            s_u, d_u = unfused(qx, qy, px, py, F32)
            if d_f != d_u:
                out.append((qx, qy, px, py, s_f, d_f, d_u))
        n = want
    return out[:want]


def test_knn_f32_fused_sequence_on_2m24_grid(orc):
    """oracle_knn_f32 returns d = sqrt_RN(fma_RN(dx, dx, RN(dy*dy))) and d1^2 = that s,
    exactly, on 2^-24-grid pairs whose unfused distance differs."""
    cases = _grid_cases(3, 400, 64)
    for qx, qy, px, py, s_f, d_f, d_u in cases:
        r, d, d1 = orc.knn_f32([px], [py], [qx], [qy], 1, want_dists=True, want_d1sq=True)
        assert Fraction(float(d[0, 0])) == d_f != d_u
        assert Fraction(float(d1[0])) == s_f
    # the same points as one data set: the k = 4 list is the 4 smallest R16 distances
    qx, qy = cases[0][0], cases[0][1]
    px = [c[2] for c in cases]
    py = [c[3] for c in cases]
    want = sorted(r16(qx, qy, a, b, F32)[1] for a, b in zip(px, py))[:4]
    _, d = orc.knn_f32(px, py, [qx], [qy], 4, want_dists=True)
    assert [Fraction(float(v)) for v in d[0]] == want


def test_knn_f64_fused_sequence_off_grid(orc):
    """fp64 oracle on arbitrary doubles: d = sqrt_RN(fma(dx, dx, dy*dy)), d1^2 = s."""
    rng = np.random.default_rng(5)
    n_diff = 0
    for _ in range(300):
        qx, qy, px, py = rng.random(4) * np.array([1.0, 1.0, 1.0, 1.0])
        s_f, d_f = r16(qx, qy, px, py, F64)
        s_u, d_u = unfused(qx, qy, px, py, F64)
        r, d, d1 = orc.knn_f64([px], [py], [qx], [qy], 1, want_dists=True, want_d1sq=True)
        assert Fraction(float(d[0, 0])) == d_f and Fraction(float(d1[0])) == s_f
        n_diff += d_f != d_u
    assert n_diff >= 10  # the sample discriminates fused from unfused


def test_r_obs_sum_order_f32(orc):
    """Eq. 3 in float (R17): ((d1 + d2) + ...) / k with one rounding per add and the
    division, on a list whose float sum depends on the order."""
    qx = qy = 0.0
    pts = [(1.0, 0.0), (2.0 ** -12, 0.0), (2.0 ** -12, 0.0), (2.0 ** -25 * 3, 0.0)]
    r, d = orc.knn_f32([p[0] for p in pts], [p[1] for p in pts], [qx], [qy], 4, want_dists=True)
    ds = sorted(Fraction(float(np.float32(p[0]))) for p in pts)
    acc = Fraction(0)
    for v in ds:
        acc = rne(acc + v, F32)
    assert Fraction(float(r[0])) == rne(acc / 4, F32)
