"""GPU index build (aqr_build_graph, NEXT-1; Alg1 l.16-22) against the oracle's graph
construction (or_build_graph, R28), byte for byte: levels, row offsets, every layer-0 and
upper row, the entry point and the top level -- with and without keepPrunedConnections, at the
fixtures' degree classes and widths (d = 7 ... 960, M = 6 ... 35, 128-d rows of C2)."""
import numpy as np
import pytest

import oracle
import synth
from tests._cases import case

pytestmark = pytest.mark.gpu


def _check(name, flags, batch_div=0):
    import torch
    from paper_2602_21600_b200 import graph as G
    c = case(name)
    g = c.graph
    d = c.w.x.shape[1]
    u = synth.level_draws(len(c.w.x), seed=c.w.seed, cfg="tiny")
    lv, uo, a0, au, e, ml = oracle.build_graph(c.codes, d, g.M, g.efc, u, flags=flags,
                                               batch_div=batch_div if batch_div else 32)
    gg = G.build_hnsw_gpu(torch.from_numpy(c.codes).cuda(), d, g.M, g.efc, u, flags=flags, batch_div=batch_div)
    np.testing.assert_array_equal(gg.levels, lv)
    np.testing.assert_array_equal(gg.upper_off, uo)
    np.testing.assert_array_equal(gg.adj0, a0, err_msg=f"{name} layer 0")
    np.testing.assert_array_equal(gg.adj_upper, au, err_msg=f"{name} upper layers")
    assert (gg.entry_point, gg.max_level) == (e, ml)


@pytest.mark.parametrize("name", ["tiny7", "tiny33", "grid", "tiny100ip", "tiny960", "c1small", "c4slice"])
@pytest.mark.parametrize("flags", [0, 1])
def test_gpu_build_equals_oracle(name, flags):
    _check(name, flags)


def test_gpu_build_sequential_waves():
    """batch_div huge: every wave is one node -- plain sequential insertion."""
    _check("tiny33", 1, batch_div=1 << 30)


def test_gpu_build_c2slice():
    """60k nodes of C2 (128-d, M = 20): ~450 waves, up to 1,875 nodes each."""
    _check("c2slice", 1)
