"""Seeded synthetic datasets shared by the golden-vector script, the tests and
bench.py (SURVEY.md §8(d) 'Synthetic inputs').  Pure numpy; no reference code.

The injection-molding surrogate restates the reference generator
(cli.py:111-173: SurrogateSpec, _regime_curve, generate_surrogate) so that the
C4 workload can be built where /root/reference is absent; tests pin it against
the reference generator in this container.
"""

from __future__ import annotations

import os
import sys

import numpy as np

_ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

def gaussian(n: int, d: int, seed: int, dtype=np.float32) -> np.ndarray:
    """X = default_rng(seed).standard_normal((n, d)).astype(dtype)."""
    return np.random.default_rng(seed).standard_normal((n, d)).astype(dtype)


from paper_2105_12026_b200.surrogate import _regime_curve, surrogate  # noqa: E402,F401  (one implementation)


def random_sets(n: int, l: int, size: int, seed: int):
    """l sets of `size` distinct indices, rng.choice(n, size, replace=False) as bench.py:61-62."""
    rng = np.random.default_rng(seed)
    return [rng.choice(n, size=size, replace=False).tolist() for _ in range(l)]


# BASELINE.json configs
def config_data(name: str) -> np.ndarray:
    if name == "C1":
        return gaussian(2000, 16, 0)
    if name in ("C2", "C3"):
        x = gaussian(100_000, 100, 1)
        return x.astype(np.float16) if name == "C3" else x
    if name == "C4":
        return surrogate(500_000, 32, 5, 0.01, 0).astype(np.float32)
    if name == "C4S50":  # the 50-regime near-tie stress case of C4
        return surrogate(500_000, 32, 50, 0.01, 0).astype(np.float32)
    if name == "C5":
        return c5_problem()[0]
    raise KeyError(name)


def c5_problem(n: int = 200_000, d: int = 64, l: int = 4096, size: int = 10, seed: int = 5):
    """Work-matrix workload: one rng draws the ground matrix then the sets, like
    bench.generate_problem (bench.py:51-63) but Gaussian per BASELINE.json."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, d)).astype(np.float32)
    sets = [rng.choice(n, size=size, replace=False).tolist() for _ in range(l)]
    return x, sets


CONFIG_K = {"C1": 10, "C2": 50, "C3": 50, "C4": 20, "C4S50": 20}


def kmedoids_cases():
    """Seeded k_medoids_loss inputs (tests/golden/make_golden_kmedoids.py pairs
    each with the reference's loss): (precision name, data fp64, reps fp64)."""
    rng = np.random.default_rng(2105)
    precs = ["fp32", "fp16-storage", "fp64"]
    half = {"fp32": np.float32, "fp16-storage": np.float16, "fp64": np.float64}
    out = []
    for i in range(18):
        n = int(rng.integers(1, 3000))
        d = int(rng.integers(1, 70))
        r = int(rng.integers(1, 40))
        prec = precs[i % 3]
        scale = float(rng.choice([0.01, 1.0, 30.0]))
        data = rng.standard_normal((n, d)) * scale + float(rng.choice([0.0, 5.0]))
        if i % 4 == 0:  # representatives taken from the stored ground rows (exact zeros there)
            stored = data.astype(half[prec]).astype(np.float64)
            reps = stored[rng.choice(n, size=min(r, n), replace=False)]
        else:
            reps = rng.standard_normal((r, d)) * scale
        out.append((prec, data, reps))
    two = np.array([[0.0, 1.0], [0.0, -1.0]])
    out.append(("fp64", two, np.array([[0.0, 0.0]])))  # test_ebc.py:29-30: (1 + 1) / 2
    return out
