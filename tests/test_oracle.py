"""Pins for the CPU oracle (run without a GPU: ``-m "not gpu"``).

Each test pins one oracle function to something other than the oracle itself:
worked values (tests/golden/worked_values.json, cited), closed forms, integer-exact
brute force, statistical closed forms and invariants.
"""
import json
import math
import os

import numpy as np
import pytest

import datagen

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_values.json")))
LV = (1.0, 1.5, 2.0, 2.5, 3.0)


# ---------------------------------------------------------------- distances ---
def test_distance_worked_values(orc):
    for c in GOLD["distance"]:
        robs = orc.knn_f64([c["p"][0]], [c["p"][1]], [c["q"][0]], [c["q"][1]], 1)
        assert robs[0] == c["d"], c["cite"]


def _int_grid_cloud(seed, nd, nq, bits):
    rng = np.random.default_rng(seed)
    n = 1 << bits
    xi = rng.integers(0, n, nd)
    yi = rng.integers(0, n, nd)
    qi = rng.integers(0, n, nq)
    qj = rng.integers(0, n, nq)
    return xi, yi, qi, qj, float(n)


def test_knn_f64_vs_integer_bruteforce(orc):
    """100 seeded configs: the oracle's k nearest distances equal,
    bit for bit, sqrt of the k smallest EXACT integer squared distances (full sort)."""
    rng = np.random.default_rng(7)
    for cfg in range(100):
        nd = int(rng.integers(50, 2000))
        k = int([1, 5, 10, 50][cfg % 4])
        nq = 8
        xi, yi, qi, qj, n = _int_grid_cloud(cfg, nd, nq, 24)
        s_int = (qi[:, None] - xi[None, :]) ** 2 + (qj[:, None] - yi[None, :]) ** 2  # exact int64
        s_k = np.sort(s_int, axis=1)[:, :k]
        want = np.sqrt(s_k.astype(np.float64) * 2.0 ** -48)  # s < 2^49: exact in fp64
        robs, d = orc.knn_f64(xi / n, yi / n, qi / n, qj / n, k, want_dists=True)
        assert np.array_equal(d, want), cfg
        # Eq. 3: mean of the k distances, ascending summation
        acc = np.zeros(nq)
        for i in range(k):
            acc = acc + want[:, i]
        assert np.array_equal(robs, acc / k)


def test_knn_f32_vs_exact_bruteforce(orc):
    """fp32 instantiation on a 2^-10 grid, where every fp32 op of the canonical
    sequence is exact: distances are the correctly rounded float sqrt of the exact s."""
    rng = np.random.default_rng(11)
    for cfg in range(30):
        nd = int(rng.integers(20, 1500))
        k = int([1, 3, 10, 15, 32][cfg % 5])
        xi, yi, qi, qj, n = _int_grid_cloud(100 + cfg, nd, 6, 10)
        s_int = (qi[:, None] - xi[None, :]) ** 2 + (qj[:, None] - yi[None, :]) ** 2
        s_k = np.sort(s_int, axis=1)[:, :k]
        want = np.sqrt((s_k.astype(np.float64) * 2.0 ** -20).astype(np.float32))
        robs, d = orc.knn_f32(xi / n, yi / n, qi / n, qj / n, k, want_dists=True)
        assert d.dtype == np.float32 and np.array_equal(d, want), cfg
        acc = np.zeros(6, np.float32)
        for i in range(k):
            acc = (acc + want[:, i]).astype(np.float32)
        assert np.array_equal(robs, (acc / np.float32(k)).astype(np.float32))


def test_knn_insert_worked_values(orc):
    for c in GOLD["knn_insert"]:
        assert list(orc.knn_insert(c["buf"], c["dist"])) == c["out"], c["cite"]


def test_knn_spec_examples(orc):
    # SPEC.md:135-137, :154-157
    assert list(orc.knn_f64([1, 2, 3], [0, 0, 0], [0], [0], 3, True)[1][0]) == [1, 2, 3]
    assert list(orc.knn_f64([3, 1, 2], [0, 0, 0], [0], [0], 3, True)[1][0]) == [1, 2, 3]
    assert list(orc.knn_f64([1, 2, 3, 4, 5], [0] * 5, [0], [0], 2, True)[1][0]) == [1, 2]
    assert orc.knn_f64([0.5, 7], [0.5, 1], [0.5], [0.5], 1, True)[1][0][0] == 0.0  # Z4: no self-exclusion
    with pytest.raises(ValueError):
        orc.knn_f64([1, 2], [0, 0], [0], [0], 3)  # nd < k


def test_knn_permutation_robust(orc):
    x, y, z, qx, qy = datagen.random_cloud(5, 3000, 64)
    _, d1 = orc.knn_f64(x, y, qx, qy, 10, True)
    p = np.random.default_rng(0).permutation(3000)
    _, d2 = orc.knn_f64(x[p], y[p], qx, qy, 10, True)
    assert np.array_equal(d1, d2)


# ---------------------------------------------------------------- Eq. 2 / 3 / 4 --
def test_r_exp_closed_form(orc):
    for c in GOLD["r_exp"]:
        assert orc.r_exp(c["nd"], c["A"]) == c["r_exp"], c["cite"]
    for nd, A in [(10, 3.0), (1024000, 1.0), (7, 0.01)]:
        assert abs(orc.r_exp(nd, 4 * A) / orc.r_exp(nd, A) - 2.0) < 1e-15


def test_bbox_area(orc):
    assert orc.bbox_area([0, 2], [0, 3]) == 6.0
    assert orc.bbox_area([0, 1], [0, 0]) == 0.0  # degenerate


def test_r_obs_worked_values(orc):
    # Eq. 3: [1,2,3] -> 2, [5] -> 5, [0,0,0] -> 0
    assert orc.knn_f64([1, 2, 3, 9], [0, 0, 0, 0], [0], [0], 3)[0] == 2.0
    assert orc.knn_f64([5, 9], [0, 0], [0], [0], 1)[0] == 5.0
    assert orc.knn_f64([1, 1, 1, 9], [1, 1, 1, 0], [1], [1], 3)[0] == 0.0
    # k = nd: mean of all distances (integer-exact distances)
    xs = np.array([3.0, 0.0, 6.0, 8.0])
    ys = np.array([4.0, 5.0, 8.0, 6.0])  # all at distance 5 or 10 from the origin
    assert orc.knn_f64(xs, ys, [0], [0], 4)[0] == 7.5


def _expected_R(k):
    # Poisson pattern, no edge effects: E[d_j] = Gamma(j+1/2)/(Gamma(j) sqrt(pi lambda)),
    # r_exp = 1/(2 sqrt(lambda))  =>  E[R] = 2/(k sqrt(pi)) sum_j Gamma(j+1/2)/Gamma(j).
    s = sum(math.exp(math.lgamma(j + 0.5) - math.lgamma(j)) for j in range(1, k + 1))
    return 2.0 / (k * math.sqrt(math.pi)) * s


@pytest.mark.parametrize("k,want", [(1, 1.0), (2, 1.25), (10, 2.4668)])
def test_R_statistical_closed_form(orc, k, want):
    """Eq. 2-4 together: on a uniform (Poisson-like) pattern with interior queries, the
    mean of R equals the closed form (a dropped factor 2 in Eq. 2 or a wrong mean in
    Eq. 3 moves it by >= 2x)."""
    assert abs(_expected_R(k) - want) < 1e-4
    nd = 40000
    x, y = datagen.uniform_points(77, nd, datagen.S_DX, datagen.S_DY)
    qx, qy = datagen.uniform_points(78, 3000, datagen.S_QX, datagen.S_QY)
    qx, qy = 0.25 + 0.5 * qx, 0.25 + 0.5 * qy
    re = orc.r_exp(nd, orc.bbox_area(x, y))
    robs = orc.knn_f64(x, y, qx, qy, k)
    R = robs / re
    se = R.std() / math.sqrt(len(R))
    assert abs(R.mean() - _expected_R(k)) < 5 * se + 0.01, (R.mean(), _expected_R(k))


# ---------------------------------------------------------------- Eq. 5 -----
def test_mu_worked_values(orc):
    for c in GOLD["mu"]:
        assert abs(orc.mu(c["R"], c["rmin"], c["rmax"]) - c["mu"]) < 1e-15, c["cite"]
        assert abs(orc.mu(c["R"], c["rmin"], c["rmax"], orc.PRINTED) - c["mu"]) < 1e-15


def test_mu_forms_and_monotone(orc):
    Rs = np.linspace(-1, 5, 601)
    for rmin, rmax in [(0.0, 2.0), (1.1, 3.7)]:
        m = np.array([orc.mu(R, rmin, rmax) for R in Rs])
        assert np.all(np.diff(m) >= 0) and m.min() == 0.0 and m.max() == 1.0
        assert orc.mu(rmax, rmin, rmax) == 1.0  # NORMALIZED reaches 1 at R_max (R8)
        assert abs(orc.mu((rmin + rmax) / 2, rmin, rmax) - 0.5) < 1e-15
    # PRINTED equals NORMALIZED iff R_min = 0 (R8)
    for R in [0.3, 1.0, 1.7]:
        assert abs(orc.mu(R, 0, 2, orc.PRINTED) - orc.mu(R, 0, 2)) < 1e-15
    assert orc.mu(3.7, 1.1, 3.7, orc.PRINTED) < 1.0
    # R_max == R_min: row 1 wins, no division (R10)
    assert orc.mu(1.5, 1.5, 1.5) == 0.0


# ---------------------------------------------------------------- Eq. 6 -----
def test_alpha_worked_values(orc):
    for c in GOLD["alpha"]:
        assert abs(orc.alpha_of_mu(c["mu"], c["levels"]) - c["alpha"]) < 1e-15, c["cite"]


def test_alpha_continuity_and_constant(orc):
    rng = np.random.default_rng(3)
    for _ in range(20):
        lv = rng.uniform(0.5, 4.0, 5)
        for b in (0.1, 0.3, 0.5, 0.7, 0.9):
            lo = orc.alpha_of_mu(b - 1e-13, lv)
            hi = orc.alpha_of_mu(b + 1e-13, lv)
            assert abs(lo - hi) < 1e-11
        # nodes: alpha(0.1)=a1, alpha(0.3)=a2, ... alpha(0.9)=a5
        for b, a in zip((0.1, 0.3, 0.5, 0.7, 0.9), lv):
            assert abs(orc.alpha_of_mu(b, lv) - a) < 1e-12
    for c in (2.0, 0.7):
        for m in np.linspace(0, 1, 101):
            # the printed lerp a(1-5t) + 5at equals a up to rounding
            assert abs(orc.alpha_of_mu(m, [c] * 5) - c) <= 4e-16 * c


# ---------------------------------------------------------------- Eq. 1 -----
def test_idw_closed_forms(orc):
    # single sample -> its value, any alpha
    assert orc.idw([0.3], [0.2], [7.5], [0.9], [0.1], 2.3)[0] == 7.5
    # two samples equidistant -> mean
    assert abs(orc.idw([0, 2], [0, 0], [0, 10], [1], [5], 1.7)[0] - 5.0) < 1e-14
    # coincident query -> exact z
    assert orc.idw([0, 1, 2], [0, 1, 2], [3, 4, 5], [1], [1], 2)[0] == 4.0
    # d1 = 1, d2 = 2, alpha = 2 -> (z1 + z2/4) / 1.25
    z1, z2 = 3.0, 11.0
    assert abs(orc.idw([1, 0], [0, 2], [z1, z2], [0], [0], 2.0)[0] - (z1 + z2 / 4) / 1.25) < 1e-14
    # centre of the unit square's corners -> mean for any alpha
    for a in (0.5, 1, 2, 3.3):
        assert abs(orc.idw([0, 1, 0, 1], [0, 0, 1, 1], [1, 2, 3, 4], [0.5], [0.5], a)[0] - 2.5) < 1e-14


def test_idw_convexity_and_reproduction(orc):
    x, y, z, qx, qy = datagen.random_cloud(9, 500, 200)
    a = np.random.default_rng(1).uniform(1, 3, 200)
    Z = orc.idw(x, y, z, qx, qy, a)
    assert np.all(Z >= z.min()) and np.all(Z <= z.max())
    Zd = orc.idw(x, y, z, x[:50], y[:50], 2.0)
    assert np.array_equal(Zd, z[:50])  # exact reproduction at data locations


def test_aidw_constant_levels_is_idw(orc):
    """Eq. 6 collapses to IDW(c) when alpha1 = ... = alpha5 = c."""
    x, y, z, qx, qy = datagen.random_cloud(4, 800, 100)
    for mode in (orc.GLOBAL, orc.FIXED):
        Za = orc.aidw(x, y, z, qx, qy, 10, [2.0] * 5, mode=mode)
        assert np.max(np.abs(Za / orc.idw(x, y, z, qx, qy, 2.0) - 1)) < 1e-14


def test_appendix_a(orc):
    A = GOLD["appendix_a"]
    d = np.array(A["data"], float)
    for c in A["cases"]:
        Z, t = orc.aidw(d[:, 0], d[:, 1], d[:, 2], [c["q"][0]], [c["q"][1]], c["k"], A["levels"],
                        mode=c["mode"], r_min=c.get("rmin", 0), r_max=c.get("rmax", 2), trace=True)
        if c["mode"] == "global":
            # the global bounds are over all five Appendix-A queries
            qs = np.array([cc["q"] for cc in A["cases"] if cc["mode"] == "global"])
            Z_all, t = orc.aidw(d[:, 0], d[:, 1], d[:, 2], qs[:, 0], qs[:, 1], 2, A["levels"],
                                mode="global", trace=True)
            i = [tuple(q) for q in qs].index(tuple(c["q"]))
            assert abs(t["r_min"] - A["global_bounds_k2"][0]) < 1e-15
            assert abs(t["r_max"] - A["global_bounds_k2"][1]) < 1e-15
            Z, R, mu, al = Z_all[i:i + 1], t["R"][i], t["mu"][i], t["alpha"][i]
        else:
            R, mu, al = t["R"][0], t["mu"][0], t["alpha"][0]
        assert abs(t["r_exp"] - A["r_exp"]) < 1e-16
        for got, want in ((R, c["R"]), (mu, c["mu"]), (al, c["alpha"]), (Z[0], c["Z"])):
            assert abs(got - want) <= 1e-12 * max(1.0, abs(want)), (c, got, want)


def test_translation_invariance(orc):
    x, y, z, qx, qy = datagen.random_cloud(12, 400, 50)
    Z0 = orc.aidw(x, y, z, qx, qy, 10, LV)
    Z1 = orc.aidw(x + 1024.0, y - 512.0, z, qx + 1024.0, qy - 512.0, 10, LV)
    assert np.max(np.abs(Z1 - Z0) / Z0) < 1e-9


def test_power_of_two_scaling_bit_exact(orc):
    """R is scale-free; scaling every coordinate by 2^j is exact, so R is bit-identical."""
    x, y, z, qx, qy = datagen.random_cloud(13, 600, 60)
    _, t0 = orc.aidw(x, y, z, qx, qy, 10, LV, trace=True)
    _, t1 = orc.aidw(x * 8, y * 8, z, qx * 8, qy * 8, 10, LV, trace=True)
    assert np.array_equal(t0["R"], t1["R"]) and np.array_equal(t0["alpha"], t1["alpha"])


def test_thread_count_independent(orc):
    x, y, z, qx, qy = datagen.random_cloud(21, 700, 97)
    n0 = orc.num_threads()
    try:
        orc.set_num_threads(1)
        Z1 = orc.aidw(x, y, z, qx, qy, 10, LV)
        orc.set_num_threads(max(2, n0))
        Z2 = orc.aidw(x, y, z, qx, qy, 10, LV)
    finally:
        orc.set_num_threads(n0)
    assert np.array_equal(Z1, Z2)
