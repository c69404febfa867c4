"""Multi-rank Greedy driver on CPU: world_size 2 (and 3) over gloo.

The device engine of each rank is replaced by a small exact fp64 numpy engine
defined here (test scaffolding, not the oracle): it reports every unselected
candidate of its shard with its exact gain, which is a superset of the
device's certified window.  What is under test is the product code around it
-- the candidate sharding, the NCCL/gloo all-gather of (index, gain) records
and the reference argmax rule applied to the union -- which must reproduce the
single-process Greedy selection of the oracle bit-exactly.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2105_12026_b200.sharded import greedy_sharded_loop, shard_range


class ExactShardEngine:
    def __init__(self, V, c0, c1):
        self.V = np.asarray(V, dtype=np.float64)
        self.n = self.V.shape[0]
        self.c0, self.c1 = c0, c1
        self.e0d = np.einsum("ij,ij->i", self.V, self.V)
        self.cm = self.e0d.copy()
        self.taken = np.zeros(self.n, dtype=bool)
        self.cur = 0.0

    def local_step(self):
        idx = np.array([c for c in range(self.c0, self.c1) if not self.taken[c]], dtype=np.int64)
        gains = np.empty(idx.size)
        for a, c in enumerate(idx):
            d = ((self.V - self.V[c]) ** 2).sum(axis=1)
            gains[a] = np.maximum(self.cm - d, 0.0).sum()
        return idx, gains, self.cur

    def advance(self, commit_idx, run_step):
        cur = self.commit(commit_idx) if commit_idx >= 0 else self.cur
        if not run_step:
            return np.zeros(0, dtype=np.int64), np.zeros(0), cur
        return self.local_step()

    def commit(self, s):
        d = ((self.V - self.V[s]) ** 2).sum(axis=1)
        self.cm = np.minimum(self.cm, d)
        self.taken[s] = True
        self.cur = float((self.e0d - self.cm).sum() / self.n)
        return self.cur


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, V, k, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c0, c1 = shard_range(V.shape[0], rank, world)
        s = greedy_sharded_loop(ExactShardEngine(V, c0, c1), V.shape[0], k)
        q.put((rank, s.selected, s.value, s.gains, s.evaluations))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_greedy_matches_single_process(world):
    rng = np.random.default_rng(17)
    V = rng.standard_normal((300, 4))
    V[200] = V[7]  # exact duplicate across shards: the lowest index must win
    k = 6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, V, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sel, vals, gains, evals = oracle.greedy(V, k)
    for rank, selected, value, g, ev in res:
        assert selected == sel, f"rank {rank}"
        assert ev == evals
        assert value == pytest.approx(vals[-1], rel=1e-12)
        np.testing.assert_allclose(np.cumsum(g), vals, rtol=1e-12)
    # all ranks agree exactly
    assert len({tuple(r[1]) for r in res}) == 1 and len({r[2] for r in res}) == 1


# ---------------------------------------------------------------- work-matrix (C5) sharding

class _StubFunction:
    """Carries the ground size for the sharded multiset driver's index check;
    the device evaluator is replaced by the oracle on the rank's slice."""

    class _G:
        def __init__(self, n):
            self.n = n

    def __init__(self, n):
        self.ground = self._G(n)


def _ms_worker(rank, world, port, V, sets, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2105_12026_b200 import EvalMultiset
        from paper_2105_12026_b200.sharded import evaluate_multiset_sharded

        def local_eval(offsets, idx, l):
            return oracle.eval_multiset(V, [idx[offsets[j]:offsets[j + 1]].tolist() for j in range(l)])

        ms = EvalMultiset(sets)
        vals = evaluate_multiset_sharded(_StubFunction(V.shape[0]), ms, evaluate=local_eval)
        err = None
        try:
            evaluate_multiset_sharded(_StubFunction(V.shape[0]), EvalMultiset(sets + [[0, V.shape[0] + 3]]),
                                      evaluate=local_eval)
        except IndexError as e:
            err = str(e)
        q.put((rank, vals.tolist(), err))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_multiset_matches_single_process(world):
    rng = np.random.default_rng(23)
    V = rng.standard_normal((400, 5))
    sets = [rng.choice(400, size=int(rng.integers(0, 12)), replace=False).tolist() for _ in range(37)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ms_worker, args=(r, world, port, V, sets, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = oracle.eval_multiset(V, sets)
    for rank, vals, err in res:
        assert np.array_equal(np.asarray(vals), want), f"rank {rank}"  # bit-identical to one process
        assert err == f"set {len(sets)}: index {V.shape[0] + 3} out of range for ground size {V.shape[0]}"
