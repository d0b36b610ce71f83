"""Offline fit of the degree-4 polynomial for 2^f on [-0.5, 0.5] used by exp2_poly2
(paper_1511_02186_b200/csrc/packed.cuh): Lawson-weighted least squares on Chebyshev
nodes (near-minimax in RELATIVE error), then the fp32 Horner evaluation is checked."""
import numpy as np


def fit(n, iters=200):
    x = np.cos(np.pi * (np.arange(4000) + 0.5) / 4000) * 0.5
    y = 2.0 ** x
    w = np.ones_like(x)
    for _ in range(iters):
        A = np.vander(x, n + 1, increasing=True) / y[:, None]
        W = np.sqrt(w)
        c, *_ = np.linalg.lstsq(A * W[:, None], np.ones_like(x) * W, rcond=None)
        e = np.abs(A @ c - 1)
        w = w * e
        w /= w.sum()
    return c


if __name__ == "__main__":
    for n in (3, 4, 5):
        c = [np.float32(v) for v in fit(n)]
        xs = np.linspace(-0.5, 0.5, 200001).astype(np.float32)
        p = c[n]
        for k in range(n - 1, -1, -1):
            p = (p * xs + c[k]).astype(np.float32)
        rel = np.abs(p.astype(np.float64) / 2.0 ** xs.astype(np.float64) - 1)
        print(f"degree {n}: max rel err {rel.max():.3e}; coeffs (c0..c{n}) {[float(v) for v in c]}")
