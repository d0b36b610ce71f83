"""The seeded generators (datagen/) -- no method arithmetic, shared by both sides."""
import numpy as np

import datagen


def test_deterministic_and_counter_based():
    a = datagen.grid24(1004, 0, 1000)
    b = datagen.grid24(1004, 0, 1000)
    assert np.array_equal(a, b)
    # any slice can be regenerated independently (query sharding)
    c = datagen.grid24(1004, 0, 100, offset=450)
    assert np.array_equal(a[450:550], c)
    assert not np.array_equal(a, datagen.grid24(1004, 1, 1000))


def test_grid_exact_in_fp32():
    for name in ("C1", "C3"):
        x, y, z = datagen.make_data(name)
        for v in (x, y):
            assert np.all((v >= 0) & (v < 1))
            assert np.array_equal(v.astype(np.float32).astype(np.float64), v)
            assert np.array_equal(np.rint(v * 2 ** 24), v * 2 ** 24)
        assert np.array_equal(z.astype(np.float32).astype(np.float64), z)
        assert z.min() >= 0.75 and z.max() < 1.30


def test_clustered_is_clustered():
    x, y, _ = datagen.make_data("C3", nd=20000)
    h, _, _ = np.histogram2d(x, y, bins=32, range=[[0, 1], [0, 1]])
    # uniform would give ~19.5 per cell with small spread; blobs give heavy tails
    assert h.max() > 10 * h.mean()


def test_grid_queries():
    qx, qy = datagen.grid_queries()
    assert qx.shape == (4096 * 2000,)
    assert qx[0] == 0.5 / 4096 and qx[1] == 1.5 / 4096
    assert np.array_equal(np.rint(qy * 2 ** 24), qy * 2 ** 24)
    sl = datagen.make_queries("C5", nq=10, offset=4096)
    assert np.all(sl[1] == qy[4096])
