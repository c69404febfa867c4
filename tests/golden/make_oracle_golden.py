"""Full-size golden vectors for the BASELINE.json configs, from the C oracle.

The reference itself cannot run these sizes (~12 h for C2, ~20-50 h
for C4 on 8 cores), so the oracle -- pinned bit-exact against the reference's
own outputs by tests/test_oracle.py -- produces them:

    python tests/golden/make_oracle_golden.py C2 C5 C3 C4   # one JSON per config

Data come from tests/golden/datasets.py (seeded; no files needed on the GPU box).
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, HERE)
sys.path.insert(0, ROOT)

import datasets  # noqa: E402
import oracle  # noqa: E402


def run(name: str, threads: int) -> None:
    oracle.set_threads(threads)
    out = os.path.join(HERE, f"oracle_{name}.json")
    t0 = time.perf_counter()
    if name == "C5":
        X, sets = datasets.c5_problem()
        vals = oracle.eval_multiset(X.astype(np.float64), sets)
        base, _ = oracle.baseline(X.astype(np.float64))
        rec = {"name": name, "kind": "multiset", "recipe": "datasets.c5_problem()", "baseline": base,
               "values": vals.tolist()}
    else:
        X = datasets.config_data(name)
        k = datasets.CONFIG_K[name]
        sel, vals, gains, evals = oracle.greedy(X.astype(np.float64), k)
        base, _ = oracle.baseline(X.astype(np.float64))
        rec = {"name": name, "kind": "greedy", "recipe": f"datasets.config_data({name!r})", "k": k,
               "baseline": base, "selected": sel, "values": vals.tolist(), "gains": gains.tolist(),
               "evaluations": evals}
    rec["oracle_seconds"] = time.perf_counter() - t0
    rec["threads"] = threads
    with open(out, "w") as fh:
        json.dump(rec, fh)
    print(f"{name}: {rec['oracle_seconds']:.0f}s -> {out}", flush=True)


if __name__ == "__main__":
    threads = int(os.environ.get("ORACLE_THREADS", "6"))
    for name in sys.argv[1:]:
        run(name, threads)
