"""Host-side arithmetic of bench.py (no GPU): the algorithmic-bytes formula behind the roofline
 and the ef -> (N_c, N_rerank) mapping (R13), which the product
binding and the oracle implement separately."""
import numpy as np
import pytest

import bench
import oracle
import paper_2602_21600_b200 as aqr


def _counters(exp, deg, ev, uexp, udeg, uev, nc, depth, fails=0):
    c = np.zeros(aqr.NCOUNT, np.int64)
    c[:11] = [exp, deg, ev, uexp, udeg, uev, nc, depth, 0, nc, fails]
    return c


def test_bytes_per_query_aqr():
    # 2 queries, d = 128, k = 10: per query 4d + 4(deg + exp) + 4(udeg + uexp) + d*(distinct evals + upper
    # evals) + d*N_c + 4d*depth + 8k
    c = _counters(exp=10, deg=100, ev=100, uexp=4, udeg=20, uev=24, nc=30, depth=8)
    d, k, nq, ratio = 128, 10, 2, 0.5
    want = (4 * d * nq + 4 * (100 + 10) + 4 * (20 + 4) + d * (100 * ratio + 24) + d * 30 + 4 * d * 8 + 8 * k * nq) / nq
    assert bench.bytes_per_query(c, nq, d, k, ratio) == pytest.approx(want)


def test_bytes_per_query_fp32_baseline():
    c = _counters(exp=10, deg=100, ev=100, uexp=4, udeg=20, uev=24, nc=10, depth=0)
    d, k, nq = 96, 10, 1
    want = 4 * d + 4 * (100 + 10) + 4 * (20 + 4) + 4 * d * (100 + 24) + 8 * k
    assert bench.bytes_per_query(c, nq, d, k, 1.0, "fp32") == pytest.approx(want)


@pytest.mark.parametrize("k", [1, 10, 100])
@pytest.mark.parametrize("ef", [1, 10, 16, 64, 128, 784, 4096])
def test_ef_mapping_product_matches_oracle(ef, k):
    if ef < k:
        ef = k
    assert aqr.ef_mapping(ef, k) == oracle.ef_mapping(ef, k)


def test_ef_mapping_table3_preset():
    # Table 3 "0.97+": m_ef = 3, N_rerank = 28 -> ef 784 gives N_c = 261, N_rerank = 28
    assert aqr.ef_mapping(784, 10) == {"ef": 784, "n_coarse": 261, "n_rerank": 28}
    assert aqr.ef_mapping(16, 10) == {"ef": 16, "n_coarse": 10, "n_rerank": 10}
