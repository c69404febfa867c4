"""Seeded synthetic datasets shared by the golden-vector script, the tests and
bench.py (SURVEY.md §8(d) 'Synthetic inputs').  Pure numpy; no reference code.

The injection-molding surrogate restates the reference generator
(cli.py:111-173: SurrogateSpec, _regime_curve, generate_surrogate) so that the
C4 workload can be built where /root/reference is absent; tests pin it against
the reference generator in this container.
"""

from __future__ import annotations

import numpy as np


def gaussian(n: int, d: int, seed: int, dtype=np.float32) -> np.ndarray:
    """X = default_rng(seed).standard_normal((n, d)).astype(dtype)."""
    return np.random.default_rng(seed).standard_normal((n, d)).astype(dtype)


def _regime_curve(dims: int, regime: int) -> np.ndarray:
    # cli.py:134-155
    t = np.linspace(0.0, 1.0, dims)
    peak = 1.0 + 0.3 * regime
    hold_end = 0.42 + 0.04 * regime
    plateau = 0.25 + 0.06 * regime
    curve = np.zeros(dims)
    rise = t < 0.12
    curve[rise] = peak * t[rise] / 0.12
    hold = (t >= 0.12) & (t < hold_end)
    curve[hold] = peak * (1.0 - 0.45 * (t[hold] - 0.12) / (hold_end - 0.12))
    plast = (t >= hold_end) & (t < 0.85)
    curve[plast] = plateau
    tail = t >= 0.85
    curve[tail] = plateau * np.exp(-(t[tail] - 0.85) / 0.05)
    return curve


def surrogate(n_cycles: int, dims: int, n_regimes: int, noise_scale: float = 0.01,
              seed: int = 0) -> np.ndarray:
    """generate_surrogate(SurrogateSpec(...)) rows, fp64 (cli.py:158-173)."""
    if n_cycles % n_regimes:
        raise ValueError("n_regimes must divide n_cycles")
    per = n_cycles // n_regimes
    rng = np.random.default_rng(seed)
    blocks = []
    for regime in range(n_regimes):
        base = _regime_curve(dims, regime)
        if noise_scale > 0:
            blocks.append(base[None, :] + rng.normal(0.0, noise_scale, size=(per, dims)))
        else:
            blocks.append(np.tile(base, (per, 1)))
    return np.vstack(blocks)


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


CONFIG_K = {"C1": 10, "C2": 50, "C3": 50, "C4": 20}
