"""Optimizers and backend dispatch of the drop-in API (optimize.py:18-91).

``greedy_maximize`` keeps the reference's contract -- full frontier every step,
argmax with the 1e-12*max(1,|top|) tie window and lowest index, gains =
value - previous, evaluations = sum of frontier sizes -- but runs the whole k-step
loop on the device through ``ebc_greedy`` instead of materialising the
multiset S_multi = {S u {c}} on the host each step.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass
from typing import List, Tuple

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
    # index validation (validate_indices, core.py:137-143) happens in the C-ABI
    # before any launch, with the reference's message for the first bad index
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


def last_lazy_stats(f: EbcFunction):
    """(lazy steps on, lazy steps, steps decided without a screen, candidates re-examined) of the last run."""
    out = np.zeros(4, dtype=np.int64)
    _native.check(f._lib.ebc_last_lazy_stats(f.native_context, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))),
                  f.native_context)
    return tuple(int(x) for x in out)


def last_screen_work(f: EbcFunction) -> int:
    """Point-candidate pairs the tensor screen evaluated in the last run (after pruning)."""
    out = np.zeros(1, dtype=np.int64)
    _native.check(f._lib.ebc_last_screen_work(f.native_context,
                                              out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))),
                  f.native_context)
    return int(out[0])


def screen_info(f: EbcFunction):
    """(mode, tensor tile points, tensor operand kind 1=BF16 split/0=TF32 split/2=FP16/-1, padded K)."""
    out = np.zeros(4, dtype=np.int64)
    _native.check(f._lib.ebc_screen_info(f.native_context, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))),
                  f.native_context)
    return tuple(int(x) for x in out)


def last_launches(f: EbcFunction) -> int:
    return int(f._lib.ebc_last_launches(f.native_context))


def set_timing(f: EbcFunction, on: bool) -> None:
    _native.check(f._lib.ebc_set_timing(f.native_context, 1 if on else 0), f.native_context)


class _SieveSlots:
    """Device slots of the live sieves (ebc_sieve_*): each holds the sieve's
    cached minima; commits of the previous element and resets of new sieves
    ride along with the next evaluation call (one round trip per element)."""

    def __init__(self, f: EbcFunction, cap: int):
        self.f = f
        self.cap = 0
        self.free: List[int] = []
        self.pending_e = -1
        self.pending_commit: List[int] = []
        self.pending_reset: List[int] = []
        self._grow(cap)

    def _grow(self, cap: int) -> None:
        if cap > self.cap:
            _native.check(self.f._lib.ebc_sieve_reserve(self.f.native_context, cap), self.f.native_context)
            self.free.extend(range(self.cap, cap))
            self.cap = cap

    def new_slot(self) -> int:
        if not self.free:  # the grid never holds more than log(2k)/log(1+eps) + 2 sieves
            raise RuntimeError("sieve slots exhausted")
        slot = self.free.pop()
        self.pending_reset.append(slot)
        return slot

    def release(self, slot: int) -> None:
        if slot in self.pending_reset:
            self.pending_reset.remove(slot)
        if slot in self.pending_commit:
            self.pending_commit.remove(slot)
        self.free.append(slot)

    def commit(self, slots: List[int], e: int) -> None:
        self.pending_e = e
        self.pending_commit = list(slots)

    def _arr(self, xs):
        return (ctypes.c_int32 * max(1, len(xs)))(*xs)

    def step(self, e: int, eval_slots: List[int]):
        ce = self.pending_e if self.pending_commit else -1
        out_single = ctypes.c_double()
        vals = (ctypes.c_double * max(1, len(eval_slots)))()
        rc = self.f._lib.ebc_sieve_step(self.f.native_context, ce, self._arr(self.pending_commit),
                                        len(self.pending_commit), self._arr(self.pending_reset),
                                        len(self.pending_reset), e, self._arr(eval_slots), len(eval_slots),
                                        ctypes.byref(out_single), vals)
        _native.check(rc, self.f.native_context)
        self.pending_e, self.pending_commit, self.pending_reset = -1, [], []
        return float(out_single.value), [float(vals[i]) for i in range(len(eval_slots))]


def sieve_stream_maximize(stream, f: EbcFunction, k: int, epsilon: float = 0.1) -> Summary:
    """Single-pass threshold-sieve maximization (optimize.py:140-197 contract).

    Thresholds live on the geometric grid (1+epsilon)^i covering [m, 2km],
    m = best singleton value seen so far; a sieve with threshold tau admits the
    streamed element e while it holds fewer than k elements and
    f(S+e) - f(S) >= (tau/2 - f(S)) / (k - |S|).  The best sieve is returned;
    an empty stream gives an empty summary of value 0.

    Device work per element (one host round trip, ebc_sieve_step): the previous
    element folded into the cached minima of the sieves that admitted it, the
    distance pass d(., e), f({e}) and f(S_r u {e}) for every live sieve that
    can still admit e -- O(N d + N R) instead of re-evaluating every member.
    The singleton value is needed before the live set is known (a new maximum
    moves the threshold grid), so every live sieve is evaluated with it and
    only those the reference would examine are used.
    """
    if k < 1:
        raise ValueError("k must be >= 1")
    if not 0.0 < epsilon < 1.0:
        raise ValueError("epsilon must lie in (0, 1)")
    t0 = time.perf_counter()
    log_base = math.log1p(epsilon)
    sieves: dict = {}      # exponent -> [threshold, selected, value, gains, slot]
    best_single = 0.0
    evaluations = 0
    n = f.ground.n
    slots = _SieveSlots(f, int(math.log(2.0 * k) / log_base) + 3)
    for raw in stream:
        e = int(raw)
        if not 0 <= e < n:
            raise IndexError(f"index {e} out of range for ground size {n}")
        cand = [ex for ex in sorted(sieves) if len(sieves[ex][1]) < k and e not in sieves[ex][1]]
        single, vals = slots.step(e, [sieves[ex][4] for ex in cand])
        evaluations += 1
        by_ex = dict(zip(cand, vals))
        if single > best_single:
            best_single = single
            lo = math.ceil(math.log(best_single) / log_base - 1e-12)
            hi = math.floor(math.log(2.0 * k * best_single) / log_base + 1e-12)
            for ex in [x for x in sieves if x < lo or x > hi]:
                slots.release(sieves.pop(ex)[4])
            for ex in range(lo, hi + 1):
                if ex not in sieves:
                    sieves[ex] = [(1.0 + epsilon) ** ex, [], 0.0, [], slots.new_slot()]
                    by_ex[ex] = single  # S = {} : f(S u {e}) = f({e}), bit for bit
        live = [ex for ex in sorted(sieves) if len(sieves[ex][1]) < k and e not in sieves[ex][1]]
        if not live:
            continue
        evaluations += len(live)
        admitted = []
        for ex in live:
            sv = sieves[ex]
            gain = float(by_ex[ex]) - sv[2]
            need = (sv[0] / 2.0 - sv[2]) / (k - len(sv[1]))
            if gain >= need:
                sv[1].append(e)
                sv[2] += gain
                sv[3].append(gain)
                admitted.append(sv[4])
        slots.commit(admitted, e)
    runtime = time.perf_counter() - t0
    if not sieves:
        return Summary(selected=[], value=0.0, gains=[], evaluations=evaluations, runtime_seconds=runtime)
    best = None
    for ex in sorted(sieves):
        if best is None or sieves[ex][2] > best[2]:
            best = sieves[ex]
    return Summary(selected=list(best[1]), value=best[2], gains=list(best[3]), evaluations=evaluations,
                   runtime_seconds=runtime)
