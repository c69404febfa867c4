"""Injection-molding surrogate data (the paper's case-study shape, C4).

Restates the reference generator's contract (cli.py:111-173: SurrogateSpec,
_regime_curve, generate_surrogate): n_regimes blocks of identical noisy
pressure curves; seeded, fp64.  Pinned against the reference generator by
tests/test_oracle.py (in the container that has the reference).
"""

from __future__ import annotations

from pathlib import Path
from typing import Tuple

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


def check_spec(n_cycles: int, dims: int, n_regimes: int, cycles_per_regime: int, noise_scale: float) -> None:
    """SurrogateSpec's validation and messages (cli.py:121-131)."""
    if min(n_cycles, dims, n_regimes, cycles_per_regime) < 1:
        raise ValueError("all surrogate counts must be >= 1")
    if n_regimes * cycles_per_regime != n_cycles:
        raise ValueError(f"n_regimes * cycles_per_regime must equal n_cycles "
                         f"({n_regimes} * {cycles_per_regime} != {n_cycles})")
    if noise_scale < 0:
        raise ValueError("noise_scale must be >= 0")


def labels(n_regimes: int, cycles_per_regime: int) -> np.ndarray:
    """Per-row regime labels of the regime-ordered blocks (cli.py:165)."""
    return np.repeat(np.arange(n_regimes), cycles_per_regime)


def labels_path(output: str) -> str:
    """The regime-label sidecar next to `output`: stem + "_labels" (cli.py:176-178)."""
    p = Path(output)
    return str(p.with_name(p.stem + "_labels" + (p.suffix or ".csv")))


def write(output: str, n_cycles: int, dims: int, n_regimes: int, cycles_per_regime: int,
          noise_scale: float = 0.01, seed: int = 0) -> Tuple[str, str]:
    """Surrogate CSV plus the regime-label sidecar (cli.py:181-187); returns both paths."""
    check_spec(n_cycles, dims, n_regimes, cycles_per_regime, noise_scale)
    X = surrogate(n_cycles, dims, n_regimes, noise_scale, seed)
    np.savetxt(output, X, delimiter=",", fmt="%.17g")
    lp = labels_path(output)
    np.savetxt(lp, labels(n_regimes, cycles_per_regime), fmt="%d")
    return output, lp


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
