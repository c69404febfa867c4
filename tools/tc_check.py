"""Smoke test of the tensor-core screen (mode 3) against the oracle."""
import os, sys, time
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests/golden")
import oracle
import paper_2105_12026_b200 as eb
from paper_2105_12026_b200 import optimize
for (n, d, k, seed) in [(700, 32, 4, 1), (3000, 100, 6, 2), (2500, 64, 5, 3), (5000, 40, 5, 4)]:
    X = np.random.default_rng(seed).standard_normal((n, d)).astype(np.float32)
    f = eb.EbcFunction(eb.GroundMatrix(X, eb.Precision.FP32))
    optimize.set_timing(f, True)
    t0 = time.time()
    s = eb.greedy_maximize(f, eb.OptimizerBudget(k=k))
    t = optimize.last_timings(f)
    sel, vals, _, _ = oracle.greedy(X.astype(np.float64), k)
    st = optimize.last_stats(f)
    print(n, d, k, st, "ok" if s.selected == sel else f"MISMATCH {s.selected} vs {sel}",
          f"rel {abs(s.value - vals[-1]) / abs(vals[-1]):.2e}", f"screen {t[0]:.2f} ms refine {t[1]:.2f} ms", flush=True)
