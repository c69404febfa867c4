"""Pin the C oracle (oracle/ebc_oracle.c) against the reference itself.

Golden vectors in tests/golden/reference_golden.json were produced by running
ebcsum 0.1.0's own naive backend (tests/golden/make_golden.py).  The oracle
must reproduce the selected indices bit-exactly and every value to 1e-12
relative; then it can stand in for the reference at sizes the reference cannot
reach (C2-C5).
"""

import os

import numpy as np
import pytest

import oracle
from conftest import case_sets, load_golden, max_scaled_diff, stored

GOLDEN = load_golden()
GREEDY = [c for c in GOLDEN["cases"] if c["kind"] == "greedy"]
MULTI = [c for c in GOLDEN["cases"] if c["kind"] == "multiset"]


@pytest.mark.parametrize("case", GREEDY, ids=[c["name"] for c in GREEDY])
def test_oracle_greedy_matches_reference(case):
    V = stored(case)
    sel, vals, gains, evals = oracle.greedy(V, case["k"], e0=case.get("e0"))
    assert sel == case["selected"]
    assert evals == case["evaluations"]
    np.testing.assert_allclose(vals, case["values"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(gains, case["gains"], rtol=1e-10, atol=1e-12)
    base, _ = oracle.baseline(V, case.get("e0"))
    assert base == pytest.approx(case["baseline"], rel=1e-14)


@pytest.mark.parametrize("case", MULTI, ids=[c["name"] for c in MULTI])
def test_oracle_multiset_matches_reference(case):
    V = stored(case)
    got = oracle.eval_multiset(V, case_sets(case), e0=case.get("e0"))
    assert max_scaled_diff(got, case["values"]) <= 1e-13


def test_known_answers():
    # test_ebc.py:41-67 / test_batched.py:86-91 / test_optimize.py:22-40 of the reference
    two = [[1.0, 0.0], [0.0, 1.0]]
    assert oracle.baseline(two)[0] == 1.0
    assert oracle.eval_multiset(two, [[0], [1], [0, 1], []]).tolist() == [0.5, 0.5, 1.0, 0.0]
    sel, vals, _, evals = oracle.greedy([[1.0, 0.0], [0.0, 1.0], [5.0, 5.0]], 2)
    assert sel[0] == 2 and vals[0] == pytest.approx(50.0 / 3.0, rel=1e-12) and evals == 5
    assert oracle.greedy([[3.0, 3.0], [1.0, 1.0], [3.0, 3.0]], 1)[0] == [0]


def test_oracle_index_error_names_set():
    with pytest.raises(IndexError, match="set 1: index 9 out of range for ground size 2"):
        oracle.eval_multiset([[1.0, 0.0], [0.0, 1.0]], [[0], [9]])


def test_oracle_thread_count_invariance():
    V = np.random.default_rng(3).standard_normal((300, 7))
    oracle.set_threads(1)
    a = oracle.greedy(V, 6)
    oracle.set_threads(max(2, os.cpu_count() or 2))
    b = oracle.greedy(V, 6)
    assert a[0] == b[0] and np.array_equal(a[1], b[1])


def test_step_values_consistent_with_greedy():
    V = np.random.default_rng(4).standard_normal((200, 5))
    sel, vals, _, _ = oracle.greedy(V, 4)
    v = oracle.step_values(V, sel[:3], [sel[3]])
    assert v[0] == vals[3]


def test_oracle_kmedoids_matches_reference():
    """k_medoids_loss (ebc.py:21-43): reference-produced losses on seeded inputs."""
    import json
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    import datasets
    want = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_kmedoids.json")))["losses"]
    store = {"fp32": np.float32, "fp16-storage": np.float16, "fp64": np.float64}
    for (prec, data, reps), w in zip(datasets.kmedoids_cases(), want):
        got = oracle.kmedoids_loss(data.astype(store[prec]).astype(np.float64), reps)
        assert abs(got - w) <= 1e-14 * max(1.0, abs(w)), (prec, data.shape, got, w)
