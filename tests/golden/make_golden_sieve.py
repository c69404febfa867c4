"""Golden vectors for threshold-sieve streaming, produced by the REFERENCE
(ebcsum 0.1.0 sieve_stream_maximize, optimize.py:140-197).  Build container
only:  python tests/golden/make_golden_sieve.py  -> reference_sieve.json"""

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import datasets  # noqa: E402
from ebcsum import EbcFunction, GroundMatrix, Precision, sieve_stream_maximize  # noqa: E402


def main():
    cases = []
    rng = np.random.default_rng(77)
    for i in range(14):
        n = int(rng.integers(3, 160))
        d = int(rng.integers(1, 12))
        k = int(rng.integers(1, 9))
        eps = float(rng.choice([0.05, 0.1, 0.3]))
        prec = [Precision.FP64, Precision.FP32, Precision.FP16_STORAGE][i % 3]
        data = rng.standard_normal((n, d)) * float(rng.choice([0.5, 3.0]))
        stream = rng.permutation(n).tolist() if i % 2 else list(range(n))
        f = EbcFunction(GroundMatrix(data, prec))
        s = sieve_stream_maximize(stream, f, k, eps)
        cases.append({"name": f"sieve_{i}", "data": data.tolist(), "precision": prec.value, "k": k, "epsilon": eps,
                      "stream": stream, "selected": s.selected, "value": s.value, "gains": s.gains,
                      "evaluations": s.evaluations})
    t0 = time.perf_counter()
    X = datasets.gaussian(2000, 16, 0)
    f = EbcFunction(GroundMatrix(X, Precision.FP32))
    s = sieve_stream_maximize(range(2000), f, 10, 0.1)
    print("C1 sieve", time.perf_counter() - t0, s.selected)
    cases.append({"name": "C1_sieve", "recipe": {"generator": "gaussian", "n": 2000, "d": 16, "seed": 0},
                  "precision": "fp32", "k": 10, "epsilon": 0.1, "stream": "range", "selected": s.selected,
                  "value": s.value, "gains": s.gains, "evaluations": s.evaluations})
    with open(os.path.join(HERE, "reference_sieve.json"), "w") as fh:
        json.dump({"generator": "ebcsum 0.1.0 sieve_stream_maximize via make_golden_sieve.py", "cases": cases}, fh)


if __name__ == "__main__":
    main()
