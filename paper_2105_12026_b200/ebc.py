"""EbcFunction on the B200: the objective object of ebc.py:46-106 backed by a
device context (libebc200.so) that holds V, d(., e0) and the cached minima.

Construction uploads the ground matrix once and computes the baseline loss
L({e0}) on the device (ebc.py:72, computed exactly once); every evaluation
goes through the C-ABI -- there is no host arithmetic on the hot path.
"""

from __future__ import annotations

import ctypes
import weakref
import os
from typing import Optional, Sequence

import numpy as np

from . import _native
from .core import Dissimilarity, EvalMultiset, GroundMatrix, Precision, SquaredEuclidean

_DTYPE = {Precision.FP32: _native.EBC_F32, Precision.FP16_STORAGE: _native.EBC_F16,
          Precision.FP64: _native.EBC_F64}


def default_device() -> int:
    """CUDA device for new contexts: $EBC200_DEVICE, else $LOCAL_RANK, else 0."""
    for var in ("EBC200_DEVICE", "LOCAL_RANK"):
        if os.environ.get(var, "").strip():
            return int(os.environ[var])
    return 0


_PIN_MIN_BYTES = 1 << 20


def _unregister(lib, data):
    lib.ebc_host_unregister(data.ctypes.data_as(ctypes.c_void_p))


def _host_rows(lib, ground: GroundMatrix) -> np.ndarray:
    """The ground's rows as the C-contiguous host buffer ebc_create uploads.
    Grounds of >= 1 MiB are page-locked once (ebc_host_register) at their first
    context and stay so for the GroundMatrix's lifetime, so every later context
    uploads them by one direct DMA (the bench's e2e contract: host inputs in
    pinned memory).  If the driver refuses, the buffer stays pageable and the
    library's staged upload is used."""
    data = np.ascontiguousarray(ground.data)
    if data is ground.data and data.nbytes >= _PIN_MIN_BYTES and not getattr(ground, "_b200_pinned", False):
        ok = lib.ebc_host_register(data.ctypes.data_as(ctypes.c_void_p), data.nbytes) == 0
        ground._b200_pinned = True  # tried once either way
        if ok:
            weakref.finalize(ground, _unregister, lib, data)
    return data


class EbcFunction:
    """Monotone submodular EBC objective f(S) = L({e0}) - L(S u {e0}).

    Same constructor and attributes as the reference (ebc.py:55-72).  Only the
    squared Euclidean distance is supported on the B200 path; any other
    ``distance`` raises ValueError.
    """

    def __init__(self, ground: GroundMatrix, e0: Optional[np.ndarray] = None,
                 distance: Optional[Dissimilarity] = None, device: Optional[int] = None):
        if distance is not None and not isinstance(distance, SquaredEuclidean):
            raise ValueError(f"the b200 backend only implements squared Euclidean distance, "
                             f"got {type(distance).__name__}")
        self.ground = ground
        self.distance = distance or SquaredEuclidean()
        if e0 is None:
            e0 = np.zeros(ground.dims, dtype=np.float64)
        else:
            e0 = np.array(e0, dtype=np.float64).ravel()
            if e0.shape[0] != ground.dims:
                raise ValueError(f"auxiliary vector has {e0.shape[0]} dims, ground has {ground.dims}")
            if not np.all(np.isfinite(e0)):
                raise ValueError("auxiliary vector must be finite")
        self.e0 = e0
        self.e0.setflags(write=False)
        self.device = default_device() if device is None else int(device)
        self._lib = _native.load()
        self._ctx = ctypes.c_void_p()
        data = _host_rows(self._lib, ground)
        rc = self._lib.ebc_create(data.ctypes.data_as(ctypes.c_void_p), ground.n, ground.dims,
                                  _DTYPE[ground.precision],
                                  self.e0.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                  self.device, ctypes.byref(self._ctx))
        _native.check(rc, None)
        out = ctypes.c_double()
        _native.check(self._lib.ebc_baseline(self._ctx, ctypes.byref(out)), self._ctx)
        self.baseline_loss = float(out.value)

    # -- device evaluation -------------------------------------------------
    def _eval_csr(self, offsets: np.ndarray, idx: np.ndarray, l: int) -> np.ndarray:
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        if idx.size == 0:
            idx = np.zeros(1, dtype=np.int64)
        out = np.empty(l, dtype=np.float64)
        bad_set = ctypes.c_int64(-1)
        bad_idx = ctypes.c_int64(-1)
        rc = self._lib.ebc_eval_multiset(self._ctx, offsets.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                         idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), l,
                                         out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                         ctypes.byref(bad_set), ctypes.byref(bad_idx))
        _native.check(rc, self._ctx)
        return out

    def evaluate_multiset(self, multiset: EvalMultiset) -> np.ndarray:
        """f(S_j) for every set, fp64, in multiset order."""
        offsets, idx = multiset.csr()
        return self._eval_csr(offsets, idx, multiset.l)

    def loss_of_indices(self, indices: Sequence[int]) -> float:
        """L(S u {e0}) (ebc.py:74-88)."""
        return self.baseline_loss - self.value(indices)

    def value(self, indices: Sequence[int]) -> float:
        """f(S) (ebc.py:90-92)."""
        self._check_indices(indices)
        idx = np.asarray([int(i) for i in indices], dtype=np.int64)
        return float(self._eval_csr(np.array([0, idx.size], dtype=np.int64), idx, 1)[0])

    def marginal_gain(self, indices: Sequence[int], e: int) -> float:
        """f(S + {e}) - f(S) (ebc.py:94-100)."""
        self._check_indices([e])
        if e in indices:
            return 0.0
        vals = self._eval_csr(*_two_sets(indices, e), 2)
        return float(vals[1] - vals[0])

    def _check_indices(self, indices: Sequence[int]) -> None:
        n = self.ground.n
        for i in indices:
            if not 0 <= int(i) < n:
                raise IndexError(f"index {i} out of range for ground size {n}")

    # -- context lifetime --------------------------------------------------
    @property
    def native_context(self):
        return self._ctx

    def close(self) -> None:
        if getattr(self, "_ctx", None) and self._ctx.value:
            self._lib.ebc_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def k_medoids_loss(ground: GroundMatrix, reps, distance: Optional[Dissimilarity] = None) -> float:
    """Mean distance of every ground observation to its nearest representative
    (ebc.py:21-43): ``reps`` are explicit vectors of the ground dimensionality,
    the loss is computed in fp64 on the device (exact direct distances from the
    stored values, per-row minimum from +inf, fixed-order sum, / n).  The ground
    keeps one device context for these calls (created on first use)."""
    reps_arr = np.atleast_2d(np.asarray(reps, dtype=np.float64))
    if reps_arr.size == 0:
        raise ValueError("the loss is undefined for an empty representative set")
    if reps_arr.shape[1] != ground.dims:
        raise ValueError(f"representative dimensionality {reps_arr.shape[1]} does not match "
                         f"ground dims {ground.dims}")
    if not np.all(np.isfinite(reps_arr)):
        raise ValueError("representatives must be finite")
    if distance is not None and not isinstance(distance, SquaredEuclidean):
        raise ValueError(f"the b200 backend only implements squared Euclidean distance, "
                         f"got {type(distance).__name__}")
    f = getattr(ground, "_b200_kmedoids", None)
    if f is None:
        f = EbcFunction(ground)
        ground._b200_kmedoids = f
    reps_arr = np.ascontiguousarray(reps_arr)
    out = ctypes.c_double()
    rc = f._lib.ebc_kmedoids_loss(f._ctx, reps_arr.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                  reps_arr.shape[0], ctypes.byref(out))
    _native.check(rc, f._ctx)
    return float(out.value)


def _two_sets(indices, e):
    base = [int(i) for i in indices]
    idx = np.asarray(base + base + [int(e)], dtype=np.int64)
    offsets = np.array([0, len(base), 2 * len(base) + 1], dtype=np.int64)
    return offsets, idx
