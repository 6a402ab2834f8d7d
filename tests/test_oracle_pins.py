"""Pins of the CPU oracle to things other than itself (-m "not gpu").

Each test checks an oracle function against a hand value (tests/golden/hand_values.json,
cited), a closed form, a library routine in a special case, brute force on a tiny input or
an invariant the paper's definitions imply -- chosen so that a dropped term, a wrong sign or
index, or a transposed operand fails one of them.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth
from paper_2602_21600_b200 import graph as G

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_values.json")))


# ------------------------------------------------------------------------------------------
# O2-O3: density and delta (Alg1 l.5-6)
# ------------------------------------------------------------------------------------------

def test_density_three_points_hand_value():
    g = GOLD["density_3pt"]
    x = np.array(g["points"], np.float32)
    rho = oracle.density(x, np.arange(3, dtype=np.int32), k=g["k"])
    assert rho[0] == pytest.approx(g["rho_of_point0"], rel=1e-12)
    # point (1,0): squared distances 1 and 2 -> mean 1.5 (a dropped square would give 1.207)
    assert rho[1] == pytest.approx(1.0 / (1.5 + 1e-6), rel=1e-12)


def test_density_exact_duplicates():
    x = np.zeros((12, 4), np.float32)
    x[11] = 5.0
    rho = oracle.density(x, np.arange(12, dtype=np.int32), k=10)
    assert rho[0] == pytest.approx(GOLD["density_dups"]["rho"], rel=1e-9)


def test_density_vs_bruteforce_pairwise_matrix():
    """densities equal a full pairwise-matrix computation to 1e-9 relative."""
    rng = np.random.default_rng(0)
    x = rng.normal(size=(300, 9)).astype(np.float32)
    sample = np.sort(rng.choice(300, 120, replace=False)).astype(np.int32)
    rho = oracle.density(x, sample, k=10)
    xs = x[sample].astype(np.float64)
    D = ((xs[:, None, :] - xs[None, :, :]) ** 2).sum(-1)
    np.fill_diagonal(D, np.inf)
    ref = 1.0 / (np.sort(D, axis=1)[:, :10].mean(1) + 1e-6)
    np.testing.assert_allclose(rho, ref, rtol=1e-9)


@pytest.mark.parametrize("key", ["delta_uniform", "delta_1_3"])
def test_delta_hand_values(key):
    g = GOLD[key]
    assert oracle.delta(np.array(g["rho"])) == pytest.approx(g["delta"], abs=1e-12)


def test_delta_extreme_and_range():
    g = GOLD["delta_extreme"]
    assert abs(oracle.delta(np.array(g["rho"])) - g["delta_approx"]) < g["tol"]
    rng = np.random.default_rng(1)
    for _ in range(20):
        r = rng.uniform(0.01, 100, size=50)
        d = oracle.delta(r)
        assert 0.0 <= d < 1.0
        # scale invariance up to eps effects (SPEC invariant)
        assert abs(d - oracle.delta(r * 7.0)) < 1e-6


# ------------------------------------------------------------------------------------------
# O4-O6: percentile window and quantizer training (Alg1 l.8-11)
# ------------------------------------------------------------------------------------------

@pytest.mark.parametrize("P", [0.0, 2.5, 5.0, 37.3, 50.0, 95.0, 97.5, 100.0])
def test_percentile_matches_numpy_linear(P):
    rng = np.random.default_rng(2)
    for n in [1, 2, 7, 1000, 1001]:
        s = np.sort(rng.normal(size=n))
        assert oracle.percentile_sorted(s, P) == pytest.approx(np.percentile(s, P, method="linear"), rel=1e-13, abs=1e-15)


@pytest.mark.parametrize("delta,pmax,pl,ph", GOLD["percentile_bounds"]["cases"])
def test_percentile_bounds(delta, pmax, pl, ph):
    x = np.random.default_rng(3).normal(size=(50, 3)).astype(np.float32)
    q = oracle.train(x, np.arange(50, dtype=np.int32), p_max=pmax, delta_override=delta)
    assert q.p_l == pytest.approx(pl) and q.p_h == pytest.approx(ph)


def test_train_delta0_is_minmax_sq8():
    """delta = 0 reduces to plain full-range min/max scalar quantization."""
    x = np.random.default_rng(4).normal(size=(500, 6)).astype(np.float32)
    q = oracle.train(x, np.arange(500, dtype=np.int32), delta_override=0.0)
    np.testing.assert_array_equal(q.min_f, x.min(0))
    np.testing.assert_array_equal(q.max_f, x.max(0))
    ref = (255.0 / ((x.max(0).astype(np.float64) - x.min(0)) + 1e-6)).astype(np.float32)
    np.testing.assert_array_equal(q.scale_f, ref)


def test_train_percentile_window_and_degenerate_dim():
    rng = np.random.default_rng(5)
    x = rng.normal(size=(2001, 4)).astype(np.float32)
    x[:, 2] = 3.25  # constant column -> degenerate
    q = oracle.train(x, np.arange(2001, dtype=np.int32), p_max=5.0, delta_override=0.6)
    for j in [0, 1, 3]:
        col = x[:, j].astype(np.float64)
        assert q.min_f[j] == np.float32(np.percentile(col, 3.0, method="linear"))
        assert q.max_f[j] == np.float32(np.percentile(col, 97.0, method="linear"))
    assert q.scale_f[2] == 1.0 and q.min_f[2] == np.float32(3.25)
    c = oracle.encode(x, q)
    assert (c[:, 2] == 0).all()


def test_train_full_pipeline_samples_only_density():
    """n > 10,000 uses the sample for delta but all n points for the percentiles."""
    rng = np.random.default_rng(6)
    x = rng.normal(size=(12000, 3)).astype(np.float32)
    s = synth.density_sample(12000, cfg="C2")
    assert len(s) == 5000 and (np.diff(s) > 0).all()
    q = oracle.train(x, s)
    rho = oracle.density(x, s)
    assert q.delta == oracle.delta(rho)
    assert q.min_f[0] == np.float32(np.percentile(x[:, 0].astype(np.float64), q.p_l, method="linear"))


# ------------------------------------------------------------------------------------------
# O7: encode / decode (Alg1 l.9, Alg2 l.11)
# ------------------------------------------------------------------------------------------

def _quant_from(mn, mx):
    mn = np.asarray(mn, np.float32)
    mx = np.asarray(mx, np.float32)
    sc = (255.0 / ((mx.astype(np.float64) - mn) + 1e-6)).astype(np.float32)
    return oracle.Quant(mn, mx, sc, 0.0, 0.0, 100.0)


def test_encode_hand_values():
    g = GOLD["encode_min0_max10"]
    q = _quant_from([g["min"]], [g["max"]])
    c = oracle.encode(np.array(g["x"], np.float32)[:, None], q)
    assert list(c[:, 0]) == g["codes"]


def test_decode_hand_value():
    g = GOLD["decode_255"]
    q = _quant_from([g["min"]], [g["max"]])
    assert oracle.decode(g["code"], float(q.scale_f[0]), g["min"]) == pytest.approx(g["value"], abs=1e-6)


def test_encode_rounding_half_away_not_floor_plus_half():
    """R5: roundf (half away from zero).  At v = 0.49999997f floor(v + 0.5f) gives 1, roundf 0;
    at v = 2.5 rint gives 2, roundf 3.  scale = 255/(254.999999 + 1e-6) rounds to 1.0f."""
    q = _quant_from([0.0], [254.999999])
    assert q.scale_f[0] == np.float32(1.0)
    x = np.array([[np.float32(0.49999997)], [2.5], [3.5], [254.5]], np.float32)
    assert list(oracle.encode(x, q)[:, 0]) == [0, 3, 4, 255]


def test_encode_monotone_and_roundtrip():
    rng = np.random.default_rng(7)
    x = rng.normal(size=(3000, 5)).astype(np.float32)
    q = oracle.train(x, np.arange(3000, dtype=np.int32), delta_override=0.4)
    c = oracle.encode(x, q)
    for j in range(5):
        o = np.argsort(x[:, j], kind="stable")
        assert (np.diff(c[o, j].astype(int)) >= 0).all()  # monotone
        inr = (x[:, j] >= q.min_f[j]) & (x[:, j] <= q.max_f[j])
        dec = np.array([oracle.decode(int(v), float(q.scale_f[j]), float(q.min_f[j])) for v in c[inr, j][:200]])
        err = np.abs(dec - x[inr, j][:200])
        assert (err <= 0.5 / q.scale_f[j] + 1e-5).all()  # round trip


# ------------------------------------------------------------------------------------------
# O8, O11, O13: distances
# ------------------------------------------------------------------------------------------

def test_distance_hand_values():
    g = GOLD["dist_quantized"]
    assert oracle.dist_quantized(g["q"], g["x"]) == g["d"]
    g = GOLD["dist_asym"]
    assert oracle.dist_asym(g["q"], g["xtilde_codes"], [0, 0], [1, 1]) == g["d"]
    g = GOLD["dist_exact"]
    assert oracle.dist_exact(g["q"], g["x"]) == g["d"]
    assert oracle.dist_exact([1, 2, 3], [4, 6, 3], metric="ip") == pytest.approx(1 - (4 + 12 + 9))


def test_distances_vs_numpy():
    rng = np.random.default_rng(8)
    for d in [7, 8, 128, 960]:
        a = rng.integers(0, 256, d).astype(np.uint8)
        b = rng.integers(0, 256, d).astype(np.uint8)
        assert oracle.dist_quantized(a, b) == int(((a.astype(np.int64) - b) ** 2).sum())
        q = rng.normal(size=d).astype(np.float32)
        mn = rng.normal(size=d).astype(np.float32)
        sc = rng.uniform(10, 100, size=d).astype(np.float32)
        xt = (b.astype(np.float32) / sc + mn).astype(np.float64)
        ref = ((q.astype(np.float64) - xt) ** 2).sum()
        assert oracle.dist_asym(q, b, mn, sc) == pytest.approx(ref, rel=1e-5)
        x = rng.normal(size=d).astype(np.float32)
        assert oracle.dist_exact(q, x) == pytest.approx(((q.astype(np.float64) - x) ** 2).sum(), rel=1e-5)
        assert oracle.dist_exact(q, x, "ip") == pytest.approx(1 - (q.astype(np.float64) * x).sum(), rel=1e-5, abs=1e-5)


# ------------------------------------------------------------------------------------------
# builder parameters (Alg1 l.17-18) -- fixture logic, pinned to hand values
# ------------------------------------------------------------------------------------------

@pytest.mark.parametrize("M0,efc0,delta,eta,M,efc", GOLD["adapt"]["cases"])
def test_adapt_params(M0, efc0, delta, eta, M, efc):
    assert G.adapt_params(M0, efc0, delta, eta) == (M, efc)


def test_eta_hand_values():
    assert G.eta_of(np.array([1.0, 3.0])) == pytest.approx(0.5)
    assert G.eta_of(np.array([2.0, 6.0])) == pytest.approx(0.5)
    assert G.eta_of(np.array([4.0, 4.0, 4.0])) == 0.0


def test_table3_and_ef_mapping():
    rows = GOLD["table3"]["rows"]
    top = rows[-1]
    assert top[0] == "0.97+" and top[2] == 28 and top[3] == 0.010 and top[4] == 1.008 and top[5] == 3
    g = GOLD["ef_search"]
    assert g["n_c"] * g["m_ef"] == g["ef"]
    m = oracle.ef_mapping(165, 10)
    assert m == dict(ef=165, n_coarse=55, n_rerank=28)
    m = oracle.ef_mapping(16, 10)
    assert m["n_coarse"] == 10 and m["n_rerank"] == 10 and m["ef"] == 16


def test_literal_density_weights():
    """NEXT-4 variant: w_j as printed in Alg1 l.12, (1/n) sum_i rho_i for every j, so
    sigma_w = 0, eta = 0 (Alg1 l.14), M_i = floor(M0 (1 + delta)) and ef_c = ef_0 (Alg1 l.17-18)."""
    from paper_2602_21600_b200 import graph as G
    rng = np.random.default_rng(4)
    x = rng.normal(size=(300, 17)).astype(np.float32)
    rho = rng.uniform(0.1, 3.0, size=300)
    w = G.density_weights(x, rho, literal=True)
    assert w.shape == (17,) and np.all(w == rho.mean())
    assert G.eta_of(w) == 0.0
    assert G.adapt_params(16, 200, 0.5, G.eta_of(w)) == (24, 200)
    assert G.eta_of(G.density_weights(x, rho)) > 0  # the SPEC reading (R16) varies with j
