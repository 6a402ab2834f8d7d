"""Pins of the oracle's graph construction (Alg1 l.16-22; the oracle of the GPU index
build; wave order DESIGN.md R28):

* a hand-traced sequential build (tests/golden/hand_values.json "build_sequential"), with and
  without keepPrunedConnections, including a full row re-selected by the heuristic;
* byte equality with the host builder (csrc/hnsw_build.cpp: heap-form SEARCH-LAYER, threads),
  an independent implementation of the same semantics, on every fixture;
* structure: degree caps, no self-loops or repeated ids, rows packed, a node appears in
  layer L only if its level is >= L, the entry point has the top level, >= 99% of layer 0 reachable.
"""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from paper_2602_21600_b200 import graph as G
from tests._cases import case

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_values.json")))["build_sequential"]


def _codes(x):
    c = np.zeros((len(x), 16), np.uint8)
    c[:, 0] = x
    return c


def test_hand_traced_sequential_build():
    x = GOLD["codes"]
    lv, uo, a0, au, e, ml = oracle.build_graph(_codes(x), 1, GOLD["M"], GOLD["efc"], np.ones(len(x)), flags=0)
    np.testing.assert_array_equal(a0, GOLD["adj0_no_keep_pruned"])
    assert (e, ml) == (0, 0) and np.all(lv == 0) and len(au) == 0
    lv, uo, a0, au, e, ml = oracle.build_graph(_codes(x[:5]), 1, GOLD["M"], GOLD["efc"], np.ones(5), flags=1)
    np.testing.assert_array_equal(a0, GOLD["adj0_first5_keep_pruned"])


def test_levels_hand_values():
    """level(0.01) = 1, level(0.5) = 0 at M = 16 (floor(-ln u / ln M))."""
    np.testing.assert_array_equal(oracle.build_levels(np.array([0.01, 0.5, 1.0]), 16), [1, 0, 0])


@pytest.mark.parametrize("name", ["tiny7", "tiny33", "grid", "tiny100ip", "c1small"])
@pytest.mark.parametrize("flags", [0, 1])
def test_equals_host_builder(name, flags):
    c = case(name)
    g = c.graph
    u = synth.level_draws(len(c.w.x), seed=c.w.seed, cfg="tiny")
    lv, uo, a0, au, e, ml = oracle.build_graph(c.codes, c.w.x.shape[1], g.M, g.efc, u, flags=flags)
    h = G.build_hnsw(c.codes, g.M, g.efc, u, n_threads=4, flags=flags)
    np.testing.assert_array_equal(lv, h.levels)
    np.testing.assert_array_equal(uo, h.upper_off)
    np.testing.assert_array_equal(a0, h.adj0)
    np.testing.assert_array_equal(au, h.adj_upper)
    assert (e, ml) == (h.entry_point, h.max_level)


@pytest.mark.parametrize("name", ["tiny33", "c1small"])
def test_structure(name):
    c = case(name)
    g = c.graph
    u = synth.level_draws(len(c.w.x), seed=c.w.seed, cfg="tiny")
    lv, uo, a0, au, e, ml = oracle.build_graph(c.codes, c.w.x.shape[1], g.M, g.efc, u, flags=1)
    n = len(lv)
    assert lv[e] == ml == lv.max()
    for v in range(n):
        rows = [(0, a0[v])] + [(L, au[uo[v] + L - 1]) for L in range(1, lv[v] + 1)]
        for L, r in rows:
            k = int((r >= 0).sum())
            assert np.all(r[:k] >= 0) and np.all(r[k:] == -1)  # packed
            nb = r[:k]
            assert len(set(nb.tolist())) == k and v not in nb  # no repeats, no self-loop
            assert np.all(lv[nb] >= L)  # layer containment
    seen = np.zeros(n, bool)
    seen[e] = True
    front = [e]
    while front:
        nb = a0[front].ravel()
        nb = np.unique(nb[nb >= 0])
        nb = nb[~seen[nb]]
        seen[nb] = True
        front = list(nb)
    assert seen.mean() >= 0.99
