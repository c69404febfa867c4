"""Injection-molding surrogate data (the paper's case-study shape, C4).

Restates the reference generator's contract (cli.py:111-173: SurrogateSpec,
_regime_curve, generate_surrogate): n_regimes blocks of identical noisy
pressure curves; seeded, fp64.  Pinned against the reference generator by
tests/test_oracle.py (in the container that has the reference).
"""

from __future__ import annotations

import numpy as np


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
