"""Pins of the oracle's upper-layer greedy descent ("greedily traverses" the sparse upper
layers), independent of the oracle itself:

* a hand-built 3-layer graph whose descent was traced by hand (tests/golden/hand_values.json
  "greedy_3layer"): per-layer endpoints, counters, the layer-0 entry and the ef = 1 path.  It
  moves twice on one layer, needs the layer-L row of a node with two upper rows, and breaks a
  distance tie by id -- a one-step-per-layer bug, a wrong upper-row offset or a tie broken the
  other way each changes an endpoint;
* a property on generated graphs: every per-layer endpoint is a strict (d^q, id) local minimum of
  its own layer-L row (numpy reads the rows straight from the graph arrays), endpoints have
  level >= L, d^q never increases down the layers, and the layer-0 beam starts at the last one.
"""
import numpy as np
import pytest

import oracle
from tests._cases import case
from tests._hand import GOLD, hand_graph


def _hand_index():
    pts, q, g = hand_graph()
    d = pts.shape[1]
    quant = oracle.Quant(np.zeros(d, np.float32), np.full(d, 255, np.float32), np.ones(d, np.float32), 0.0, 0.0, 100.0)
    codes = oracle.encode(pts, quant)
    return oracle.Index(pts, codes, quant, g, "l2"), q, codes


def test_hand_codes_are_the_coordinates():
    ix, q, codes = _hand_index()
    np.testing.assert_array_equal(codes[:, :2], np.array(GOLD["points"]))
    dq = [oracle.dist_quantized(oracle.encode(q, ix.quant)[0], codes[v]) for v in range(len(codes))]
    assert dq == GOLD["dq_by_hand"]


@pytest.mark.parametrize("traversal", ["aqr", "fp32"])
def test_hand_traced_descent(traversal):
    ix, q, _ = _hand_index()
    ids, dist, tr = oracle.search(ix, q, k=1, ef=1, n_coarse=1, n_rerank=1, early_term=False, trace=True,
                                  traversal=traversal)
    np.testing.assert_array_equal(tr["upper_end"][0], GOLD["upper_end"])
    cnt = tr["counters"][0]
    assert cnt[oracle.COUNTER_NAMES.index("upper_exp")] == GOLD["upper_exp"]
    assert cnt[oracle.COUNTER_NAMES.index("upper_deg_sum")] == GOLD["upper_deg_sum"]
    assert cnt[oracle.COUNTER_NAMES.index("upper_evals")] == GOLD["upper_evals"]
    exp = tr["exp_ids"][0]
    assert exp[0] == GOLD["layer0_entry"]
    np.testing.assert_array_equal(exp[:len(GOLD["ef1_expansions"])], GOLD["ef1_expansions"])
    assert exp[len(GOLD["ef1_expansions"])] == -1
    assert ids[0, 0] == GOLD["ef1_result"]
    if traversal == "aqr":
        assert tr["coarse_dq"][0, 0] == GOLD["ef1_result_dq"]


def _dq_rows(codes, qc, ids):
    ids = np.asarray(ids)
    return ((codes[ids].astype(np.int64) - qc[None].astype(np.int64)) ** 2).sum(-1)


@pytest.mark.parametrize("name", ["tiny33", "c1small", "grid"])
def test_endpoints_are_strict_local_minima(name):
    c = case(name)
    g = c.graph
    if g.max_level < 1:
        pytest.skip("no upper layer")
    ids, dist, tr = oracle.search(c.ix, c.w.q, k=1, ef=8, n_coarse=8, n_rerank=8, early_term=False, trace=True)
    qcs = oracle.encode(c.w.q, c.quant)
    for qi in range(len(c.w.q)):
        qc = qcs[qi]
        ends = tr["upper_end"][qi]
        prev_d = None
        for t, L in enumerate(range(g.max_level, 0, -1)):
            e = int(ends[t])
            assert g.levels[e] >= L
            row = g.adj_upper[g.upper_off[e] + L - 1]
            row = row[row >= 0]
            de = int(_dq_rows(c.codes, qc, [e])[0])
            if len(row):
                dn = _dq_rows(c.codes, qc, row)
                assert np.all((dn > de) | ((dn == de) & (row > e))), (qi, L)
            if prev_d is not None:
                assert de <= prev_d
            prev_d = de
        assert tr["exp_ids"][qi, 0] == ends[-1]
