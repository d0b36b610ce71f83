"""CPU checks of bench.py's roofline model: the pipe-balanced
weighting bound against its closed form, and the exact-exponent class mix."""
import math

import pytest
import torch

import bench


def balanced(fp32, transc, poly=bench.POLY_FMA_PER_TRANSC, fma=bench.FMA_PER_CLK_SM, sfu=bench.MUFU_PER_CLK_SM):
    """Closed form: move f transcendentals to the FMA pipe so both pipes take equally long,
    (fp32 + poly f) / fma = (transc - f) / sfu, clamped to f in [0, transc]."""
    f = (transc * fma - fp32 * sfu) / (fma + poly * sfu)
    f = min(max(f, 0.0), transc)
    return max((fp32 + poly * f) / fma, (transc - f) / sfu)


@pytest.mark.parametrize("fp32,transc", [(7, 2), (6, 1), (8, 1), (4, 0), (0, 2)])
def test_weight_bound_closed_form(fp32, transc):
    assert bench.weight_clk_per_pair(fp32, transc) == pytest.approx(balanced(fp32, transc), rel=2e-3)


def test_weight_bound_values():
    # general formula: 7 FP32 + 2 transcendentals -> 0.0917 clk/pair/SM
    assert bench.weight_clk_per_pair() == pytest.approx(0.0917, abs=2e-4)
    # the SFU-only bound is slower, the FMA-only one too: balancing must beat both
    w = bench.weight_clk_per_pair()
    assert w < 2 / bench.MUFU_PER_CLK_SM and w < (7 + 2 * bench.POLY_FMA_PER_TRANSC) / bench.FMA_PER_CLK_SM


def test_class_fractions_and_mix():
    alpha = torch.tensor([1.0, 2.0, 3.0, 2.5, 1.0, 1.0, 3.0, 1.7])
    d1sq = torch.tensor([1e-6, 1e-6, 1e-6, 1e-6, 2.0 ** -80, 1e-6, 2.0 ** 70, 0.5])
    fr = bench.class_fractions(alpha, d1sq)
    # out-of-range d1sq falls back to the general formula (passes.cuh alpha_class)
    assert fr == pytest.approx({"a1": 2 / 8, "a2": 1 / 8, "a3": 1 / 8, "general": 4 / 8})
    mix = bench.weight_clk_mix(fr)
    expect = sum(f * bench.weight_clk_per_pair(*bench.CLASS_OPS[c]) for c, f in fr.items())
    assert mix == pytest.approx(expect)
    assert mix < bench.weight_clk_per_pair()  # exact-exponent classes only lower the bound
    assert math.isclose(bench.weight_clk_mix({"general": 1.0, "a1": 0, "a2": 0, "a3": 0}),
                        bench.weight_clk_per_pair())


@pytest.mark.parametrize("nq,world", [(1_024_000, 8), (1_024_000, 3), (7, 4), (0, 2), (5, 1)])
def test_query_blocks_strong(nq, world):
    # strong scaling: contiguous blocks that tile [0, nq) exactly, sizes differ by <= 1
    blocks = [bench.query_block(r, world, nq, True) for r in range(world)]
    assert all(t == nq for _, _, t in blocks)
    assert blocks[0][0] == 0
    for (a0, an, _), (b0, _, _) in zip(blocks, blocks[1:]):
        assert a0 + an == b0
    assert blocks[-1][0] + blocks[-1][1] == nq
    assert max(n for _, n, _ in blocks) - min(n for _, n, _ in blocks) <= 1


def test_query_blocks_weak():
    assert [bench.query_block(r, 4, 100, False) for r in range(4)] == [(r * 100, 100, 400) for r in range(4)]
