"""TEST INFRASTRUCTURE ONLY -- the parity checker for the B200 path.

ctypes wrapper over ``libebc_oracle.so``, a plain-C fp64 restatement of the
reference hot path (see ``ebc_oracle.c`` for the reference file:line each
function follows).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline legs may import this package, and only as the
checker or the timed CPU baseline -- never as a fallback for the product path
(``paper_2105_12026_b200`` does not import it).

Pinning: ``tests/test_oracle.py`` checks this restatement against the
reference package's own known-answer tests and against golden vectors produced
by the reference itself (``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libebc_oracle.so")
_lib = None

_f64p = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> str:
    """Compile the C restatement in place (gcc + OpenMP)."""
    src = os.path.join(_HERE, "ebc_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-C", _HERE, "-B" if force else "-s", "libebc_oracle.so"],
                       check=True, capture_output=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        lib.ebc_oracle_baseline.argtypes = [_f64p, ctypes.c_int64, ctypes.c_int, _f64p, _f64p, _f64p]
        lib.ebc_oracle_eval_multiset.argtypes = [_f64p, ctypes.c_int64, ctypes.c_int, _f64p, _i64p, _i64p,
                                                 ctypes.c_int64, _f64p, _i64p, _i64p]
        lib.ebc_oracle_greedy.argtypes = [_f64p, ctypes.c_int64, ctypes.c_int, _f64p, ctypes.c_int,
                                          _i64p, _f64p, _f64p, _i64p]
        lib.ebc_oracle_step_values.argtypes = [_f64p, ctypes.c_int64, ctypes.c_int, _f64p, _i64p, ctypes.c_int,
                                               _i64p, ctypes.c_int64, _f64p]
        lib.ebc_oracle_kmedoids.argtypes = [_f64p, ctypes.c_int64, ctypes.c_int, _f64p, ctypes.c_int64, _f64p]
        lib.ebc_oracle_set_threads.argtypes = [ctypes.c_int]
        lib.ebc_oracle_num_threads.restype = ctypes.c_int
        lib.ebc_oracle_sqdist.restype = ctypes.c_double
        _lib = lib
    return _lib


def _as64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a, t=_f64p):
    return a.ctypes.data_as(t)


def set_threads(n: int) -> None:
    _load().ebc_oracle_set_threads(int(n))


def num_threads() -> int:
    return int(_load().ebc_oracle_num_threads())


def _prep(V, e0):
    V64 = _as64(V)
    if V64.ndim == 1:
        V64 = V64.reshape(-1, 1)
    n, d = V64.shape
    e0 = np.zeros(d) if e0 is None else _as64(e0).ravel()
    return V64, n, d, e0


def baseline(V, e0=None) -> Tuple[float, np.ndarray]:
    """(L({e0}), e0-distances) -- ebc.py:72."""
    V64, n, d, e0 = _prep(V, e0)
    e0d = np.empty(n)
    out = ctypes.c_double()
    rc = _load().ebc_oracle_baseline(_p(V64), n, d, _p(e0), _p(e0d), ctypes.byref(out))
    if rc:
        raise ValueError("oracle baseline: invalid argument")
    return out.value, e0d


def eval_multiset(V, sets: Sequence[Sequence[int]], e0=None) -> np.ndarray:
    """f(S_j) for every set, fp64, in set order (ebc.py:109-121)."""
    V64, n, d, e0 = _prep(V, e0)
    lens = [len(s) for s in sets]
    offsets = np.zeros(len(sets) + 1, dtype=np.int64)
    offsets[1:] = np.cumsum(lens)
    idx = np.ascontiguousarray(np.fromiter((int(i) for s in sets for i in s), dtype=np.int64,
                                           count=int(offsets[-1])))
    if idx.size == 0:
        idx = np.zeros(1, dtype=np.int64)
    out = np.empty(len(sets))
    bad_set = ctypes.c_int64(-1)
    bad_idx = ctypes.c_int64(-1)
    rc = _load().ebc_oracle_eval_multiset(_p(V64), n, d, _p(e0), _p(offsets, _i64p), _p(idx, _i64p),
                                          len(sets), _p(out), ctypes.byref(bad_set), ctypes.byref(bad_idx))
    if rc == 2:
        raise IndexError(f"set {bad_set.value}: index {bad_idx.value} out of range for ground size {n}")
    if rc:
        raise ValueError("oracle eval_multiset: invalid argument")
    return out


def greedy(V, k: int, e0=None):
    """(selected, values, gains, evaluations) of reference Greedy (optimize.py:60-91)."""
    V64, n, d, e0 = _prep(V, e0)
    sel = np.empty(k, dtype=np.int64)
    val = np.empty(k)
    gain = np.empty(k)
    evals = ctypes.c_int64()
    rc = _load().ebc_oracle_greedy(_p(V64), n, d, _p(e0), int(k), _p(sel, _i64p), _p(val), _p(gain),
                                   ctypes.byref(evals))
    if rc:
        raise ValueError(f"oracle greedy: invalid argument (k={k}, n={n})")
    return sel.tolist(), val, gain, int(evals.value)


def step_values(V, selected: Sequence[int], candidates: Sequence[int], e0=None) -> np.ndarray:
    """f(S u {c}) for the listed candidates c, S = selected."""
    V64, n, d, e0 = _prep(V, e0)
    s = np.ascontiguousarray(np.asarray(list(selected) or [0], dtype=np.int64))
    c = np.ascontiguousarray(np.asarray(list(candidates), dtype=np.int64))
    out = np.empty(c.size)
    rc = _load().ebc_oracle_step_values(_p(V64), n, d, _p(e0), _p(s, _i64p), len(selected), _p(c, _i64p),
                                        c.size, _p(out))
    if rc:
        raise ValueError("oracle step_values: invalid argument")
    return out


def kmedoids_loss(V, reps) -> float:
    """k_medoids_loss(GroundMatrix(V), reps) of the reference (ebc.py:21-43), fp64."""
    V64 = _as64(V)
    n, d = V64.shape
    R = np.ascontiguousarray(np.atleast_2d(np.asarray(reps, dtype=np.float64)))
    out = ctypes.c_double()
    rc = _load().ebc_oracle_kmedoids(_p(V64), n, d, _p(R), R.shape[0], ctypes.byref(out))
    if rc:
        raise ValueError("oracle kmedoids_loss: invalid argument")
    return float(out.value)
