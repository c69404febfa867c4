"""Optimizers and backend dispatch of the drop-in API (optimize.py:18-91).

``greedy_maximize`` keeps the reference's contract -- full frontier every step,
argmax with the 1e-12*max(1,|top|) tie window and lowest index, gains =
value - previous, evaluations = sum of frontier sizes -- but runs the whole k-step
loop on the device through ``ebc_greedy`` instead of materialising the
multiset S_multi = {S u {c}} on the host each step.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass
from typing import Tuple

import numpy as np

from . import _native
from .core import EvalMultiset, Summary
from .ebc import EbcFunction

BACKENDS = ("b200",)


def parse_backend_spec(text: str) -> Tuple[str, int]:
    """'b200' or 'b200:T' (bench.py:66-76 style).  T is accepted for API
    compatibility; the device evaluator has no host thread pool."""
    name, _, threads_part = text.partition(":")
    threads = 1
    if threads_part:
        threads = int(threads_part)
        if threads < 1:
            raise ValueError(f"thread count must be >= 1 in {text!r}")
    if name not in BACKENDS:
        raise ValueError(f"unknown backend {name!r}; expected one of {BACKENDS}")
    return name, threads


@dataclass
class OptimizerBudget:
    """How large a summary to build and which evaluator to drive (optimize.py:24-40)."""

    k: int
    backend: str = "b200"
    threads: int = 1

    def __post_init__(self):
        if self.k < 1:
            raise ValueError("k must be >= 1")
        if self.threads < 1:
            raise ValueError("threads must be >= 1")
        if self.backend not in BACKENDS:
            raise ValueError(f"unknown backend {self.backend!r}; expected one of {BACKENDS}")


def evaluate_multiset_batched(f: EbcFunction, multiset: EvalMultiset, threads: int = 1) -> np.ndarray:
    """Device work-matrix evaluation (batched.py:180-240 contract): fp64 values
    in multiset order, IndexError naming the first offending set."""
    if threads < 1:
        raise ValueError("threads must be >= 1")
    multiset.validate_indices(f.ground.n)
    return f.evaluate_multiset(multiset)


def evaluate_with_backend(f: EbcFunction, multiset: EvalMultiset, backend: str = "b200",
                          threads: int = 1) -> np.ndarray:
    """Dispatch a multiset evaluation to the named backend (optimize.py:43-57)."""
    if backend == "b200":
        return evaluate_multiset_batched(f, multiset, threads)
    raise ValueError(f"unknown backend {backend!r}; expected one of {BACKENDS}")


def greedy_maximize(f: EbcFunction, budget: OptimizerBudget) -> Summary:
    """Greedy summary construction on the device (optimize.py:60-91)."""
    n = f.ground.n
    if budget.k > n:
        raise ValueError(f"k={budget.k} exceeds ground size {n}")
    if budget.backend not in BACKENDS:
        raise ValueError(f"unknown backend {budget.backend!r}; expected one of {BACKENDS}")
    k = int(budget.k)
    sel = np.empty(k, dtype=np.int64)
    val = np.empty(k, dtype=np.float64)
    gain = np.empty(k, dtype=np.float64)
    evals = ctypes.c_int64()
    t0 = time.perf_counter()
    rc = f._lib.ebc_greedy(f.native_context, k, sel.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                           val.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                           gain.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(evals))
    _native.check(rc, f.native_context)
    runtime = time.perf_counter() - t0
    return Summary(selected=[int(s) for s in sel], value=float(val[-1]), gains=[float(g) for g in gain],
                   evaluations=int(evals.value), runtime_seconds=runtime)


def last_timings(f: EbcFunction):
    """Device milliseconds of the last call: (screen, refine+pick, update, total)."""
    out = np.zeros(4, dtype=np.float64)
    _native.check(f._lib.ebc_last_timings(f.native_context, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))),
                  f.native_context)
    return tuple(float(x) for x in out)


def last_stats(f: EbcFunction):
    """(sum of window sizes, max window, screen rung at the end, steps) of the last run."""
    out = np.zeros(4, dtype=np.int64)
    _native.check(f._lib.ebc_last_stats(f.native_context, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))),
                  f.native_context)
    return tuple(int(x) for x in out)


def last_launches(f: EbcFunction) -> int:
    return int(f._lib.ebc_last_launches(f.native_context))


def set_timing(f: EbcFunction, on: bool) -> None:
    _native.check(f._lib.ebc_set_timing(f.native_context, 1 if on else 0), f.native_context)
