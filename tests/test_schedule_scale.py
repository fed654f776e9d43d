"""The native scheduler at the survey's scale.

The product builds the reference's O(s n^2) cost table (schedule.py:139-155)
with int32 saturation, a thread team and an AVX2 inner min
(csrc/schedule.cpp).  These tests pin it where the reference itself would
take hours:

* SURVEY §8(c) values computed from the reference's recurrence:
  cost(10^5, 10) = 877,123 and cost(n, 62) for n = 10^3 ... 10^5;
* the whole table against the plain C restatement (oracle/revolve_dp.c,
  int64, INF = 2^40, no tricks) on random (n, s) up to a (20000, 20) and a
  (3000, 200) table;
* _best_split (schedule.py:177-181, smallest argmin) against the oracle's
  first argmin on random (length, slots), including cases with several
  minimisers.
CPU only.
"""

import numpy as np
import pytest

from oracle import c_oracle
from paper_1806_01117_b200 import schedule as MS

pytestmark = pytest.mark.skipif(not c_oracle.available(), reason="make -C oracle first")


@pytest.mark.parametrize("n,s,cost", [
    (100_000, 10, 877_123),
    (1_000, 62, 1_955), (2_000, 62, 3_994), (5_000, 62, 13_037), (10_000, 62, 28_139),
    (20_000, 62, 58_393), (50_000, 62, 156_368), (100_000, 62, 357_400),
    (10_000, 999, 19_010), (10_000, 10, 60_960), (1_000, 10, 3_921),
])
def test_survey_costs_at_scale(n, s, cost):
    assert MS.forward_cost(n, s) == cost


@pytest.fixture(scope="module")
def tables():
    return {
        (20_000, 20): c_oracle.cost_table(20_000, 20),
        (3_000, 200): c_oracle.cost_table(3_000, 200),
    }


def _oracle_split(table, length, slots):
    # k in [1, length): k + c[slots-1][length-k] + c[slots][k], first argmin
    k = np.arange(1, length)
    v = k + table[slots - 1, length - k] + table[slots, k]
    return int(k[np.argmin(v)]), int(np.sum(v == v.min()))


@pytest.mark.parametrize("shape", [(20_000, 20), (3_000, 200)])
def test_cost_table_matches_c_oracle(tables, shape):
    t = tables[shape]
    n_max, s_max = shape
    rng = np.random.default_rng(n_max + s_max)
    for _ in range(300):
        s = int(rng.integers(1, s_max + 1))
        n = int(rng.integers(1, n_max + 1))
        assert MS.forward_cost(n, s) == t[s, n], (n, s)
    for s in (1, s_max // 2, s_max):  # whole rows at a few slot counts
        for n in np.linspace(1, n_max, 97).astype(int):
            assert MS.forward_cost(int(n), s) == t[s, n], (n, s)


@pytest.mark.parametrize("shape", [(20_000, 20), (3_000, 200)])
def test_best_split_first_argmin(tables, shape):
    t = tables[shape]
    n_max, s_max = shape
    rng = np.random.default_rng(7 * n_max + s_max)
    ties = 0
    for _ in range(400):
        slots = int(rng.integers(1, s_max + 1))
        length = int(rng.integers(slots + 2, n_max + 1))
        want, n_min = _oracle_split(t, length, slots)
        ties += n_min > 1
        assert MS.best_split(length, slots) == want, (length, slots)
    assert ties > 0, "no tie exercised: the smallest-argmin rule went untested"
