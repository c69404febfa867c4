"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container only (it imports /root/reference/pkg/src, which does
not exist on the GPU box):

    python tests/golden/make_golden.py            # writes tests/golden/reference_golden.json

Every value here comes from ``ebcsum`` 0.1.0 through its public API with the
exact-oracle backend ``naive`` (optimize.py:43-47, ebc.py:109-121); nothing is
computed by this repo's code.  The fixtures pin both the C oracle
(tests/test_oracle.py) and the CUDA path (tests/test_gpu_parity.py).
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, REF_SRC)

import datasets  # noqa: E402
from ebcsum import (EbcFunction, EvalMultiset, GroundMatrix, OptimizerBudget,  # noqa: E402
                    Precision, evaluate_multiset_naive, greedy_maximize)
from ebcsum.cli import SurrogateSpec, generate_surrogate  # noqa: E402


def _greedy_case(name, X, precision, k, recipe):
    t0 = time.perf_counter()
    f = EbcFunction(GroundMatrix(X, precision))
    s = greedy_maximize(f, OptimizerBudget(k=k, backend="naive"))
    vals = np.cumsum(s.gains).tolist()
    print(f"  {name}: {time.perf_counter() - t0:.1f}s selected={s.selected}", flush=True)
    return {"name": name, "kind": "greedy", "recipe": recipe, "precision": precision.value,
            "k": k, "baseline": f.baseline_loss, "selected": s.selected, "value": s.value,
            "gains": s.gains, "values": vals, "evaluations": s.evaluations}


def _random_instance(rng, precision, n_max, dims_max, l_max, size_max):
    # tests/conftest.py:35-47 of the reference
    n = int(rng.integers(2, n_max + 1))
    dims = int(rng.integers(1, dims_max + 1))
    l = int(rng.integers(1, l_max + 1))
    data = rng.random((n, dims))
    sets = []
    for _ in range(l):
        size = int(rng.integers(0, min(size_max, n) + 1))
        sets.append(rng.choice(n, size=size, replace=False).tolist())
    return data, sets


def main(out_path=os.path.join(HERE, "reference_golden.json")):
    cases = []
    print("known-answer fixtures")
    two = [[1.0, 0.0], [0.0, 1.0]]
    three = [[1.0, 0.0], [0.0, 1.0], [5.0, 5.0]]
    tie = [[3.0, 3.0], [1.0, 1.0], [3.0, 3.0]]
    f2 = EbcFunction(GroundMatrix(two))
    ms = [[0], [1], [0, 1], []]
    cases.append({"name": "two_point", "kind": "multiset", "data": two, "precision": "fp64",
                  "e0": None, "sets": ms, "baseline": f2.baseline_loss,
                  "values": evaluate_multiset_naive(f2, EvalMultiset(ms)).tolist()})
    for name, data, k in (("three_point_k1", three, 1), ("three_point_k2", three, 2),
                          ("three_point_k3", three, 3), ("tie_k1", tie, 1), ("tie_k3", tie, 3)):
        c = _greedy_case(name, np.asarray(data), Precision.FP64, k, {"data": data})
        c["data"] = data
        cases.append(c)

    print("custom anchor e0")
    rng = np.random.default_rng(7)
    data = rng.random((40, 3))
    e0 = [0.25, -0.5, 1.5]
    f = EbcFunction(GroundMatrix(data, Precision.FP32), e0=e0)
    sets = [[0], [1, 2], [], list(range(10)), [39, 0, 5]]
    cases.append({"name": "custom_e0_multiset", "kind": "multiset", "data": data.tolist(),
                  "precision": "fp32", "e0": e0, "sets": sets, "baseline": f.baseline_loss,
                  "values": evaluate_multiset_naive(f, EvalMultiset(sets)).tolist()})
    s = greedy_maximize(f, OptimizerBudget(k=5))
    cases.append({"name": "custom_e0_greedy", "kind": "greedy", "data": data.tolist(),
                  "precision": "fp32", "e0": e0, "k": 5, "baseline": f.baseline_loss,
                  "selected": s.selected, "value": s.value, "gains": s.gains,
                  "values": np.cumsum(s.gains).tolist(), "evaluations": s.evaluations})

    print("random multiset instances (reference conftest generator)")
    rng = np.random.default_rng(2024)
    for precision in (Precision.FP64, Precision.FP32, Precision.FP16_STORAGE):
        for i in range(12):
            data, sets = _random_instance(rng, precision, 200, 20, 50, 10)
            f = EbcFunction(GroundMatrix(data, precision))
            vals = evaluate_multiset_naive(f, EvalMultiset(sets))
            cases.append({"name": f"random_{precision.value}_{i}", "kind": "multiset",
                          "data": data.tolist(), "precision": precision.value, "e0": None,
                          "sets": sets, "baseline": f.baseline_loss, "values": vals.tolist()})

    print("random greedy instances")
    rng = np.random.default_rng(99)
    for precision in (Precision.FP64, Precision.FP32, Precision.FP16_STORAGE):
        for i in range(6):
            n = int(rng.integers(5, 120))
            d = int(rng.integers(1, 12))
            data = rng.random((n, d))
            k = int(rng.integers(1, min(8, n) + 1))
            c = _greedy_case(f"greedy_{precision.value}_{i}", data, precision, k, {})
            c["data"] = data.tolist()
            cases.append(c)

    print("BASELINE config C1 (Gaussian N=2000 d=16 seed 0, k=10) -- fp32 and fp16 storage")
    X = datasets.gaussian(2000, 16, 0)
    cases.append(_greedy_case("C1_fp32", X, Precision.FP32, 10,
                              {"generator": "gaussian", "n": 2000, "d": 16, "seed": 0}))
    cases.append(_greedy_case("C1_fp16", X, Precision.FP16_STORAGE, 10,
                              {"generator": "gaussian", "n": 2000, "d": 16, "seed": 0}))

    print("Gaussian d=100 (C2 shape, downscaled N=1200 k=15)")
    X = datasets.gaussian(1200, 100, 42)
    cases.append(_greedy_case("gauss_1200x100_fp32", X, Precision.FP32, 15,
                              {"generator": "gaussian", "n": 1200, "d": 100, "seed": 42}))
    cases.append(_greedy_case("gauss_1200x100_fp16", X, Precision.FP16_STORAGE, 15,
                              {"generator": "gaussian", "n": 1200, "d": 100, "seed": 42}))

    print("surrogate (C4 shape, downscaled): 5 and 50 regimes, d=32")
    for regimes, n in ((5, 2000), (50, 2500)):
        spec = SurrogateSpec(n_cycles=n, dims=32, n_regimes=regimes,
                             cycles_per_regime=n // regimes, noise_scale=0.01, seed=0)
        Xs, _ = generate_surrogate(spec)
        mine = datasets.surrogate(n, 32, regimes, 0.01, 0)
        assert np.array_equal(Xs, mine), "surrogate restatement drifted from cli.py"
        cases.append(_greedy_case(f"surrogate_{regimes}r_{n}x32_fp32", Xs.astype(np.float32),
                                  Precision.FP32, 20,
                                  {"generator": "surrogate", "n": n, "d": 32, "regimes": regimes,
                                   "noise": 0.01, "seed": 0}))

    print("work-matrix (C5 shape, downscaled N=4000 d=64, 128 sets x 10)")
    X, sets = datasets.c5_problem(n=4000, d=64, l=128, size=10, seed=5)
    f = EbcFunction(GroundMatrix(X, Precision.FP32))
    vals = evaluate_multiset_naive(f, EvalMultiset(sets))
    cases.append({"name": "c5_small", "kind": "multiset", "precision": "fp32", "e0": None,
                  "recipe": {"generator": "c5_problem", "n": 4000, "d": 64, "l": 128, "size": 10,
                             "seed": 5},
                  "baseline": f.baseline_loss, "values": vals.tolist()})

    with open(out_path, "w") as fh:
        json.dump({"generator": "ebcsum 0.1.0 (reference) via tests/golden/make_golden.py",
                   "numpy": np.__version__, "cases": cases}, fh)
    print("wrote", out_path, len(cases), "cases")


if __name__ == "__main__":
    main()
