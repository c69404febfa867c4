"""Test configuration: the `gpu` marker, repo paths and shared helpers.

`-m "not gpu"` tests run on the CPU build container (oracle vs golden vectors,
host logic, C-ABI symbol checks, gloo world_size-2 sharding); `-m gpu` tests
need a B200 and call the CUDA path through the C-ABI.
"""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, GOLDEN_DIR):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 GPU and the built libebc200.so")


def load_golden(name="reference_golden.json"):
    with open(os.path.join(GOLDEN_DIR, name)) as fh:
        return json.load(fh)


def max_scaled_diff(a, b):
    """max |a-b| / max(1, max|a|, max|b|) -- the reference's tolerance metric
    (tests/conftest.py:66-71 of ebcsum)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = max(1.0, float(np.max(np.abs(a))), float(np.max(np.abs(b))))
    return float(np.max(np.abs(a - b))) / scale


def case_data(case):
    """Rebuild a golden case's ground matrix (explicit data or seeded recipe)."""
    import datasets
    if "data" in case:
        return np.asarray(case["data"], dtype=np.float64)
    r = case["recipe"]
    if r["generator"] == "gaussian":
        return datasets.gaussian(r["n"], r["d"], r["seed"])
    if r["generator"] == "surrogate":
        return datasets.surrogate(r["n"], r["d"], r["regimes"], r["noise"], r["seed"]).astype(np.float32)
    if r["generator"] == "c5_problem":
        return datasets.c5_problem(r["n"], r["d"], r["l"], r["size"], r["seed"])[0]
    raise KeyError(r["generator"])


def case_sets(case):
    import datasets
    if "sets" in case:
        return case["sets"]
    r = case["recipe"]
    return datasets.c5_problem(r["n"], r["d"], r["l"], r["size"], r["seed"])[1]


STORAGE = {"fp64": np.float64, "fp32": np.float32, "fp16-storage": np.float16}


def stored(case):
    """The values the reference stored (GroundMatrix rounds to the storage dtype)."""
    return case_data(case).astype(STORAGE[case["precision"]]).astype(np.float64)
