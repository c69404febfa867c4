"""Candidate-sharded Greedy across GPUs, one process per GPU.

V and the cached minima are replicated on every rank; rank r screens only the
candidates [c0, c1) of a contiguous partition of the ground indices.  Per
Greedy step:

  1. ``engine.local_step()`` -- on the device: fp32 screen of the local
     candidates, certified window, exact fp64 gains of the window.  Returns the
     local list (index, gain64) and f(S).
  2. ``allgather_candidates`` -- NCCL (or gloo) all-gather of those (index,
     gain) pairs; a handful of 16-byte records per rank.
  3. ``pick`` -- every rank applies the reference argmax rule (optimize.py:83-85)
     to the union; all ranks hold bit-identical inputs, so they agree.
  4. ``engine.commit(best)`` -- every rank folds the winner into its cached
     minima and recomputes f(S) with the fixed-order fp64 reduction.

Device exchange (the NCCL path, ``greedy_device_exchange``): the same step
runs without a host round trip -- each rank reduces its window to its local
tie set {c : value_c >= top_r - 1e-12 max(1,|top_r|)} (a superset of what the
global rule can pick, since top - window(top) is monotone in top) and that to
its index-ordered Pareto frontier (the only members the lowest-index rule can
need; exact duplicates collapse to one), writes at most ``ebc_tie_cap()``
16-byte records, one ``ncclAllGather`` inside the step exchanges them (128 B
per rank), and every rank runs the identical device pick; the k-step loop is
graph-captured (``ebc_greedy_sharded``) and ends with an all-gather of a hash of
the selection that fails the call if any rank disagrees.  Steps 1-4 above are
the host-driven fallback (gloo, NCCL missing, or a frontier beyond
``ebc_tie_cap()`` records).

Why the union of local windows gives the single-GPU answer: a local window
W_r = {c in shard r : ub_c >= max_{c' in shard r} lb_c' - margin} contains
every candidate of shard r whose exact value is within the reference tie
window of the global top, and each candidate's exact gain is
computed with the same point chunking on every rank.  So selections are
identical for any number of ranks.
"""

from __future__ import annotations

import ctypes
import time
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _native
from .core import Summary
from .optimize import OptimizerBudget


SHARD_ALIGN = 128  # candidate tile of the screens: shard starts stay tile aligned


def shard_range(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous candidate range of `rank`: ceil(n / world) indices per rank,
    rounded up to a multiple of the 128-candidate screen tile (so every rank
    can use the tensor-core screen, whose tiles need 8-aligned starts)."""
    per = (n + world - 1) // world
    per = (per + SHARD_ALIGN - 1) // SHARD_ALIGN * SHARD_ALIGN
    c0 = min(n, rank * per)
    return c0, min(n, c0 + per)


def pick(idx: np.ndarray, gain: np.ndarray, current: float, n: int) -> Tuple[int, float]:
    """Reference argmax rule over exact gains (optimize.py:83-85).

    value_c = f(S) + gain_c / n, computed with separately rounded fp64 ops
    exactly as the device pick kernel does; top = max value; window =
    1e-12 * max(1, |top|); the winner is the lowest index with value >= top - window.
    """
    if idx.size == 0:
        raise RuntimeError("no remaining candidate on any rank")
    inv_n = 1.0 / float(n)
    values = np.float64(current) + np.asarray(gain, dtype=np.float64) * np.float64(inv_n)
    top = float(values.max())
    window = 1e-12 * max(1.0, abs(top))
    ok = values >= top - window
    best = int(np.asarray(idx)[ok].min())
    return best, top


def allgather_candidates(idx: np.ndarray, gain: np.ndarray, group=None, device=None):
    """All-gather variable-length (index, gain) lists: one all_gather of the
    counts, one of the padded records.  `device` is where the collective's
    tensors live (a CUDA device for NCCL, CPU for gloo)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = torch.device("cpu") if device is None else torch.device(device)
    cnt = torch.tensor([idx.size], dtype=torch.int64, device=dev)
    counts = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    counts = [int(c.item()) for c in counts]
    m = max(1, max(counts))
    rec = torch.full((m, 2), float("nan"), dtype=torch.float64, device=dev)
    if idx.size:
        # indices < 2^53 are exact in fp64
        rec[: idx.size, 0] = torch.from_numpy(np.asarray(idx, dtype=np.float64)).to(dev)
        rec[: idx.size, 1] = torch.from_numpy(np.asarray(gain, dtype=np.float64)).to(dev)
    recs = [torch.empty_like(rec) for _ in range(world)]
    dist.all_gather(recs, rec, group=group)
    out_i: List[np.ndarray] = []
    out_g: List[np.ndarray] = []
    for c, r in zip(counts, recs):
        r = r[:c].cpu().numpy()
        out_i.append(r[:, 0].astype(np.int64))
        out_g.append(r[:, 1])
    return np.concatenate(out_i), np.concatenate(out_g)


class NativeShardEngine:
    """Device side of one rank (wraps ebc_shard_* of include/ebc200.h)."""

    def __init__(self, f, c0: int, c1: int):
        self.f = f
        self.lib = f._lib
        self.ctx = f.native_context
        _native.check(self.lib.ebc_shard_set_range(self.ctx, c0, c1), self.ctx)
        _native.check(self.lib.ebc_reset(self.ctx), self.ctx)
        self.cap = 64
        self._idx = np.empty(self.cap, dtype=np.int64)
        self._gain = np.empty(self.cap, dtype=np.float64)

    def local_step(self):
        count = ctypes.c_int64()
        cur = ctypes.c_double()
        while True:
            rc = self.lib.ebc_shard_step(self.ctx, self._idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                         self._gain.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), self.cap,
                                         ctypes.byref(count), ctypes.byref(cur))
            _native.check(rc, self.ctx)
            if count.value <= self.cap:
                break
            self.cap = int(count.value)
            self._idx = np.empty(self.cap, dtype=np.int64)
            self._gain = np.empty(self.cap, dtype=np.float64)
        m = int(count.value)
        return self._idx[:m].copy(), self._gain[:m].copy(), float(cur.value)

    def advance(self, commit_idx: int, run_step: bool):
        """Commit `commit_idx` (-1: none) and screen the next step, one host sync."""
        count = ctypes.c_int64()
        cur = ctypes.c_double()
        rc = self.lib.ebc_shard_advance(self.ctx, int(commit_idx), 1 if run_step else 0,
                                        self._idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                        self._gain.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), self.cap,
                                        ctypes.byref(count), ctypes.byref(cur))
        _native.check(rc, self.ctx)
        m = int(count.value)
        if m > self.cap:
            self.cap = m
            self._idx = np.empty(m, dtype=np.int64)
            self._gain = np.empty(m, dtype=np.float64)
            _native.check(self.lib.ebc_shard_fetch(self.ctx, self._idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                                   self._gain.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), m),
                          self.ctx)
        return self._idx[:m].copy(), self._gain[:m].copy(), float(cur.value)

    def commit(self, s: int) -> float:
        out = ctypes.c_double()
        _native.check(self.lib.ebc_shard_commit(self.ctx, int(s), ctypes.byref(out)), self.ctx)
        return float(out.value)

    def close(self):
        # restore the full candidate range for later single-device calls
        self.lib.ebc_shard_set_range(self.ctx, 0, self.f.ground.n)


def greedy_sharded_loop(engine, n: int, k: int, group=None, device=None) -> Summary:
    """Drive k sharded Greedy steps with any engine exposing
    advance(commit_idx, run_step) -> (idx, gain, f(S)): one device round trip
    and one all-gather per step."""
    t0 = time.perf_counter()
    selected: List[int] = []
    gains: List[float] = []
    current = 0.0
    evaluations = 0
    idx, gain, cur = engine.advance(-1, True)
    for step in range(k):
        all_idx, all_gain = allgather_candidates(idx, gain, group=group, device=device)
        best, _top = pick(all_idx, all_gain, cur, n)
        idx, gain, newval = engine.advance(best, step + 1 < k)
        cur = newval
        evaluations += n - step
        gains.append(newval - current)
        current = newval
        selected.append(best)
    check_ranks_agree(selected, gains, current, group=group)
    return Summary(selected=selected, value=current, gains=gains, evaluations=evaluations,
                   runtime_seconds=time.perf_counter() - t0)


def selection_digest(selected: Sequence[int], gains: Sequence[float], value: float) -> bytes:
    """Digest of a Greedy result (indices and the exact bits of gains and value)."""
    import hashlib
    h = hashlib.sha256()
    h.update(np.asarray(selected, dtype=np.int64).tobytes())
    h.update(np.asarray(gains, dtype=np.float64).tobytes())
    h.update(np.float64(value).tobytes())
    return h.digest()


def check_ranks_agree(selected, gains, value, group=None) -> None:
    """End-of-run guard of the host-driven exchange: every rank must hold the
    same result; raises RuntimeError (never returns rank-dependent results)."""
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    mine = selection_digest(selected, gains, value)
    all_d = [None] * dist.get_world_size(group)
    dist.all_gather_object(all_d, mine, group=group)
    if any(d != all_d[0] for d in all_d):
        bad = [r for r, d in enumerate(all_d) if d != all_d[0]]
        raise RuntimeError(f"sharded Greedy: ranks {bad} disagree with rank 0 on the selection")


def _ensure_device_comm(f, group) -> bool:
    """NCCL communicator of the library for this EbcFunction (rank 0 makes the
    unique id, torch.distributed broadcasts it).  False if NCCL is unavailable
    on any rank -- then every rank uses the host exchange."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    key = (id(group), world, rank, f.device)
    if getattr(f, "_comm_key", None) == key:
        return True
    lib = f._lib
    if _COMM_READY.get(key):  # the device's communicator exists: attach, no collective init
        _native.check(lib.ebc_comm_attach(f.native_context), f.native_context)
        f._comm_key = key
        return True
    nb = int(lib.ebc_comm_id_bytes())
    payload = None
    if rank == 0:
        buf = ctypes.create_string_buffer(nb)
        if lib.ebc_comm_unique_id(buf, nb) == _native.EBC_OK:
            payload = buf.raw
    obj = [payload]
    src = dist.get_global_rank(group, 0) if group is not None else 0
    dist.broadcast_object_list(obj, src=src, group=group)
    if obj[0] is None:
        return False
    _native.check(lib.ebc_comm_init(f.native_context, obj[0], nb, world, rank), f.native_context)
    _COMM_READY.clear()  # a new init replaces the device's communicator
    _COMM_READY[key] = True
    f._comm_key = key
    return True


_COMM_READY: dict = {}  # (group, world, rank, device) -> the library holds a communicator for it


def greedy_device_exchange(f, k: int, c0: int, c1: int) -> Summary:
    """k sharded Greedy steps with the exchange on the device (ebc_greedy_sharded):
    one call, no host round trip per step."""
    lib = f._lib
    ctx = f.native_context
    t0 = time.perf_counter()
    _native.check(lib.ebc_shard_set_range(ctx, c0, c1), ctx)
    sel = np.empty(k, dtype=np.int64)
    val = np.empty(k, dtype=np.float64)
    gain = np.empty(k, dtype=np.float64)
    evals = ctypes.c_int64()
    try:
        _native.check(lib.ebc_greedy_sharded(ctx, k, sel.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                              val.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                              gain.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                              ctypes.byref(evals)), ctx)
    finally:
        lib.ebc_shard_set_range(ctx, 0, f.ground.n)
    return Summary(selected=[int(x) for x in sel], value=float(val[-1]), gains=[float(x) for x in gain],
                   evaluations=int(evals.value), runtime_seconds=time.perf_counter() - t0)


def greedy_maximize_sharded(f, budget: OptimizerBudget, group=None) -> Summary:
    """Greedy over all ranks of `group` (torch.distributed must be initialised;
    each rank passes its own EbcFunction built on its own GPU from the same data).

    With an NCCL process group the whole k-step loop runs on the devices
    (ebc_greedy_sharded: NCCL all-gather of fixed-size tie-set records inside
    the step, graph-captured); otherwise -- gloo, NCCL unavailable,
    EBC200_DEVICE_EXCHANGE=0, or a tie set larger than ebc_tie_cap() -- the
    host drives the exchange one step at a time (greedy_sharded_loop)."""
    import os

    import torch
    import torch.distributed as dist

    n = f.ground.n
    if budget.k > n:
        raise ValueError(f"k={budget.k} exceeds ground size {n}")
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    c0, c1 = shard_range(n, rank, world)
    nccl = dist.get_backend(group) == "nccl"
    if nccl and os.environ.get("EBC200_DEVICE_EXCHANGE", "1") != "0" and _ensure_device_comm(f, group):
        try:
            return greedy_device_exchange(f, int(budget.k), c0, c1)
        except _native.CommError:
            flags = ctypes.c_int32()
            _native.check(f._lib.ebc_comm_status(f.native_context, ctypes.byref(flags)), f.native_context)
            if flags.value & 2:
                raise  # the ranks disagree: a bug, never papered over by a fallback
            # a frontier overflow (every rank sees the same records): host exchange below
    engine = NativeShardEngine(f, c0, c1)
    device = f"cuda:{torch.cuda.current_device()}" if nccl else None
    try:
        return greedy_sharded_loop(engine, n, int(budget.k), group=group, device=device)
    finally:
        engine.close()


# ---------------------------------------------------------------- work-matrix sharding (C5)
# the sets of a multiset are independent units.  Rank r
# evaluates a contiguous range of sets [j0, j1) on its own GPU (V replicated),
# the fp64 values are all-gathered in rank order.  A set's value is a
# fixed-order reduction over the points that does not depend on which rank (or
# how many) evaluates it, so the gathered vector is bit-identical to the
# single-GPU call (batched.py:180-240 evaluates the same sets in one process).

def set_range(offsets: np.ndarray, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous set range of `rank`, balanced by work: each set weighs its
    member count + 1 (a set costs one pass over the points per member; the +1
    keeps runs of empty sets from piling onto one rank)."""
    offsets = np.asarray(offsets, dtype=np.int64)
    l = offsets.size - 1
    w = np.diff(offsets) + 1
    cum = np.concatenate([[0], np.cumsum(w)])
    total = int(cum[-1])
    bounds = [int(np.searchsorted(cum, (r * total + world - 1) // world, side="left")) for r in range(world + 1)]
    bounds[0], bounds[-1] = 0, l
    j0 = min(l, bounds[rank])
    j1 = min(l, max(j0, bounds[rank + 1]))
    return j0, j1


def _first_bad_index(offsets: np.ndarray, idx: np.ndarray, n: int):
    """(set, index) of the first out-of-range member in set order, or None."""
    bad = np.nonzero((idx < 0) | (idx >= n))[0]
    if bad.size == 0:
        return None
    p = int(bad[0])
    j = int(np.searchsorted(offsets, p, side="right") - 1)
    return j, int(idx[p])


def evaluate_multiset_sharded(f, multiset, group=None, evaluate=None) -> np.ndarray:
    """f(S_j) for every set, fp64, in multiset order, the sets split across the
    ranks of `group` (torch.distributed must be initialised; every rank passes
    the same multiset and its own EbcFunction on its own GPU).  Out-of-range
    indices raise the reference's IndexError (core.py:140-143) on every rank,
    before any device work.  ``evaluate(offsets, idx, l)`` overrides the local
    evaluator (tests); default: the rank's device (ebc_eval_multiset)."""
    import torch
    import torch.distributed as dist

    offsets, idx = multiset.csr()
    offsets = np.asarray(offsets, dtype=np.int64)
    idx = np.asarray(idx, dtype=np.int64)
    n = f.ground.n if f is not None else None
    if n is not None:
        bad = _first_bad_index(offsets, idx, n)
        if bad is not None:
            raise IndexError(f"set {bad[0]}: index {bad[1]} out of range for ground size {n}")
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    l = offsets.size - 1
    ranges = [set_range(offsets, r, world) for r in range(world)]
    j0, j1 = ranges[rank]
    if evaluate is None:
        evaluate = f._eval_csr
    local = np.zeros(0)
    if j1 > j0:
        lo = offsets[j0:j1 + 1] - offsets[j0]
        local = np.asarray(evaluate(lo, idx[offsets[j0]:offsets[j1]], j1 - j0), dtype=np.float64)
    nccl = dist.get_backend(group) == "nccl"
    dev = torch.device(f"cuda:{torch.cuda.current_device()}") if nccl else torch.device("cpu")
    m = max(b - a for a, b in ranges) or 1
    buf = torch.zeros(m, dtype=torch.float64, device=dev)
    if local.size:
        buf[: local.size] = torch.from_numpy(local).to(dev)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    out = np.empty(l, dtype=np.float64)
    for r, (a, b) in enumerate(ranges):
        out[a:b] = parts[r][: b - a].cpu().numpy()
    return out
