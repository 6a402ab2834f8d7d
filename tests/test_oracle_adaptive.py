"""Pins of the oracle's adaptive re-rank depth ("the system evaluates the spread of
asymmetric distances"; reading DESIGN.md R27): depth = the entries of A with
d^a <= (1 + tau_spread) d^a_k, at least k, at most N_rerank; tau_spread = +inf is the static N_rerank.

* hand values on the greedy_3layer fixture, where d^a = d^q are sums of two squares (golden);
* tau_spread = +inf reproduces the static path exactly;
* depth lies in [min(k, |A|), N_rerank] and grows with tau_spread; under the fill reading recall
  cannot drop as the depth grows."""
import numpy as np
import pytest

import oracle
from tests._cases import case
from tests._hand import hand_graph
from tests.test_oracle_greedy import _hand_index
import json
import os

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_values.json")))["adaptive_depth"]


@pytest.mark.parametrize("tau, depth", GOLD["cases"])
def test_hand_depths(tau, depth):
    ix, q, _ = _hand_index()
    _, _, tr = oracle.search(ix, q, k=GOLD["k"], ef=8, n_coarse=8, n_rerank=8, early_term=False, trace=True,
                             tau_spread=tau)
    assert tr["counters"][0, oracle.COUNTER_NAMES.index("depth")] == depth
    np.testing.assert_array_equal(tr["asym_ids"][0], [7, 5, 4, 6, 3, 2, 1, 0])


@pytest.mark.parametrize("name", ["tiny33", "c1small", "tiny100ip"])
def test_infinite_spread_is_static(name):
    c = case(name)
    p = dict(k=c.w.k, **oracle.ef_mapping(96, c.w.k))
    a = oracle.search(c.ix, c.w.q, trace=True, **p)
    b = oracle.search(c.ix, c.w.q, trace=True, tau_spread=float("inf"), **p)
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[2]["counters"], b[2]["counters"])


@pytest.mark.parametrize("name", ["c1small", "c2slice"])
def test_depth_bounds_and_monotone(name):
    c = case(name)
    k = c.w.k
    p = dict(k=k, **oracle.ef_mapping(192, k))
    p["n_rerank"] = p["n_coarse"]
    gt, _ = oracle.bruteforce(c.w.x, c.w.q, k, c.w.metric)
    prev_depth, prev_rec = None, None
    for tau in [0.0, 0.01, 0.05, 0.2, 1.0, float("inf")]:
        ids, _, tr = oracle.search(c.ix, c.w.q, trace=True, early_term=False, tau_spread=tau, **p)
        depth = tr["counters"][:, oracle.COUNTER_NAMES.index("depth")]
        nc = tr["counters"][:, oracle.COUNTER_NAMES.index("n_coarse")]
        assert np.all(depth >= np.minimum(k, nc)) and np.all(depth <= p["n_rerank"])
        rec = np.array([len(set(a) & set(b)) for a, b in zip(ids, gt)])
        if prev_depth is not None:
            assert np.all(depth >= prev_depth)
            assert np.all(rec >= prev_rec)  # per query: a deeper exact prefix never loses a true neighbour
        prev_depth, prev_rec = depth, rec
