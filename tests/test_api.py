"""Host-side logic of the drop-in API and the C-ABI boundary (no GPU needed).

Mirrors the reference's own validation tests (test_core.py, test_optimize.py
TestBudget, test_batched.py index errors) for the B200 package, checks that
libebc200.so exports every symbol include/ebc200.h declares, and that the
product path refuses to run without a GPU instead of falling back to the CPU.
"""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2105_12026_b200 as eb
from paper_2105_12026_b200 import _native
from paper_2105_12026_b200.sharded import pick, shard_range

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ebc200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ebc_[a-z0-9_]+)\s*\(", text)))


# ---------------------------------------------------------------- C-ABI library

def test_library_exports_every_declared_symbol():
    lib = _native.load()
    syms = declared_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), f"libebc200.so lacks {s}"
    assert set(syms) == set(_native.SIGNATURES), "ctypes table out of sync with include/ebc200.h"


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_version_string():
    assert "sm_100a" in _native.version()


@pytest.mark.skipif(_native.device_count() > 0, reason="a GPU is visible")
def test_no_cpu_fallback_without_gpu():
    g = eb.GroundMatrix([[1.0, 0.0], [0.0, 1.0]])
    with pytest.raises(RuntimeError, match="CUDA|device"):
        eb.EbcFunction(g)


def test_create_rejects_bad_arguments():
    lib = _native.load()
    ctx = ctypes.c_void_p()
    x = np.zeros((2, 2), dtype=np.float32)
    rc = lib.ebc_create(x.ctypes.data_as(ctypes.c_void_p), 0, 2, 0, None, 0, ctypes.byref(ctx))
    assert rc == _native.EBC_EINVAL
    rc = lib.ebc_create(x.ctypes.data_as(ctypes.c_void_p), 2, 2, 7, None, 0, ctypes.byref(ctx))
    assert rc == _native.EBC_EINVAL
    assert "dtype" in _native.last_error(None)


# ---------------------------------------------------------------- core types

def test_ground_matrix_validation():
    with pytest.raises(ValueError, match="2-D"):
        eb.GroundMatrix(np.zeros((2, 2, 2)))
    with pytest.raises(ValueError, match="at least 1x1"):
        eb.GroundMatrix(np.zeros((0, 3)))
    with pytest.raises(ValueError, match="row 1, column 0"):
        eb.GroundMatrix([[1.0], [np.nan]])
    g = eb.GroundMatrix([1.0, 2.0, 3.0])
    assert (g.n, g.dims) == (3, 1)
    assert not g.data.flags.writeable


def test_fp16_storage_rounding_table():
    # test_core.py:49-61 of the reference
    g = eb.GroundMatrix([[0.1, np.pi, 1.0, 65504.0]], eb.Precision.FP16_STORAGE)
    assert g.data.dtype == np.float16
    assert g.as_float64().tolist()[0] == [0.0999755859375, 3.140625, 1.0, 65504.0]


def test_precision_parse():
    assert eb.Precision.parse("fp16-storage") is eb.Precision.FP16_STORAGE
    with pytest.raises(ValueError, match="unknown precision"):
        eb.Precision.parse("bf16")


def test_multiset_validation_and_csr():
    with pytest.raises(ValueError, match="at least one set"):
        eb.EvalMultiset([])
    with pytest.raises(IndexError, match="set 1 contains a negative index"):
        eb.EvalMultiset([[0], [-1]])
    ms = eb.EvalMultiset([[3, 1], [], [2]])
    off, idx = ms.csr()
    assert off.tolist() == [0, 2, 2, 3] and idx.tolist() == [3, 1, 2]
    assert eb.EvalMultiset.from_csr(off, idx).sets == [[3, 1], [], [2]]
    with pytest.raises(IndexError, match="set 0: index 3 out of range for ground size 3"):
        ms.validate_indices(3)


def test_multiset_sets_are_read_only():
    """The CSR arrays are built once; the sets they mirror cannot change under them."""
    ms = eb.EvalMultiset([[3, 1], [2]])
    off, idx = ms.csr()
    for mutate in (lambda: ms.sets[0].append(5), lambda: ms.sets.__setitem__(0, [0]),
                   lambda: ms.sets[1].__setitem__(0, 0), lambda: ms.sets.append([1])):
        with pytest.raises(TypeError, match="read-only"):
            mutate()
    assert ms.sets == [[3, 1], [2]] and ms.csr()[1] is idx
    assert ms.sets[0] + [7] == [3, 1, 7]  # building a new list from a set still works
    with pytest.raises(ValueError):
        idx[0] = 9


def test_ground_compute_view():
    """GroundMatrix.compute_view (reference core.py:82-92): widened to the
    arithmetic dtype, cached, read-only."""
    X = np.arange(6, dtype=np.float64).reshape(3, 2) / 3
    g16 = eb.GroundMatrix(X, eb.Precision.FP16_STORAGE)
    v = g16.compute_view()
    assert v.dtype == np.float32 and v is g16.compute_view() and not v.flags.writeable
    np.testing.assert_array_equal(v, g16.data.astype(np.float32))
    g64 = eb.GroundMatrix(X)
    assert g64.compute_view() is g64.data


def test_budget_validation():
    # test_optimize.py:11-18 of the reference
    with pytest.raises(ValueError):
        eb.OptimizerBudget(k=0)
    with pytest.raises(ValueError):
        eb.OptimizerBudget(k=1, threads=0)
    with pytest.raises(ValueError, match="backend"):
        eb.OptimizerBudget(k=1, backend="gpu")
    assert eb.OptimizerBudget(k=3).backend == "b200"


def test_backend_spec():
    assert eb.parse_backend_spec("b200") == ("b200", 1)
    assert eb.parse_backend_spec("b200:4") == ("b200", 4)
    with pytest.raises(ValueError):
        eb.parse_backend_spec("b200:0")
    with pytest.raises(ValueError, match="unknown backend"):
        eb.parse_backend_spec("batched")


def test_auxiliary_vector():
    g = eb.GroundMatrix([[2.0], [4.0]])
    assert eb.make_auxiliary_vector(1, "mean", g).tolist() == [3.0]
    assert eb.make_auxiliary_vector(3).tolist() == [0.0, 0.0, 0.0]
    with pytest.raises(ValueError):
        eb.make_auxiliary_vector(0)


# ---------------------------------------------------------------- pick rule / sharding

def test_pick_rule_lowest_index_in_window():
    # values = 1 + gain/n; gains at 5 and 9 tie exactly -> lowest index wins
    idx = np.array([9, 5, 7])
    gain = np.array([4.0, 4.0, 3.0])
    assert pick(idx, gain, 1.0, 2)[0] == 5
    # within the 1e-12 relative window counts as tied (optimize.py:84-85)
    gain = np.array([4.0, 4.0 - 1e-13, 3.0])
    assert pick(idx, gain, 1.0, 2)[0] == 5
    gain = np.array([4.0, 4.0 - 1e-6, 3.0])
    assert pick(idx, gain, 1.0, 2)[0] == 9


def test_shard_ranges_partition():
    for n in (1, 7, 100, 101):
        for world in (1, 2, 3, 8):
            cover = []
            for r in range(world):
                c0, c1 = shard_range(n, r, world)
                cover.extend(range(c0, c1))
            assert cover == list(range(n))


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"), reason="reference not mounted")
def test_surrogate_restatement_matches_reference_generator():
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    from ebcsum.cli import SurrogateSpec, generate_surrogate
    import datasets
    X, _ = generate_surrogate(SurrogateSpec(n_cycles=600, dims=32, n_regimes=5, cycles_per_regime=120,
                                            noise_scale=0.01, seed=0))
    assert np.array_equal(X, datasets.surrogate(600, 32, 5, 0.01, 0))


def test_kmedoids_validation_before_any_device_work():
    """k_medoids_loss raises the reference's ValueErrors (ebc.py:31-40) on the host."""
    g = eb.GroundMatrix(np.zeros((3, 2)), eb.Precision.FP64)
    with pytest.raises(ValueError, match="empty representative set"):
        eb.k_medoids_loss(g, np.empty((0, 2)))
    with pytest.raises(ValueError, match="representative dimensionality 3 does not match ground dims 2"):
        eb.k_medoids_loss(g, [[1.0, 2.0, 3.0]])
    with pytest.raises(ValueError, match="representatives must be finite"):
        eb.k_medoids_loss(g, [[1.0, np.nan]])


def test_set_ranges_partition_in_order():
    from paper_2105_12026_b200.sharded import set_range
    rng = np.random.default_rng(3)
    for _ in range(50):
        lens = rng.integers(0, 20, size=int(rng.integers(1, 60)))
        off = np.concatenate([[0], np.cumsum(lens)])
        for world in (1, 2, 3, 5, 8, 13):
            rs = [set_range(off, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == len(lens)
            for (a, b), (c, _) in zip(rs, rs[1:]):
                assert a <= b == c
