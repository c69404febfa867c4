"""C5 work-matrix timing: dense vs sparse path (device ms)."""
import os, sys, time
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests/golden")
import datasets
import paper_2105_12026_b200 as eb
from paper_2105_12026_b200 import optimize
X, sets = datasets.c5_problem()
ms = eb.EvalMultiset(sets)
res = {}
for mode in ("1", "2", "0"):
    os.environ["EBC200_MULTISET_MODE"] = mode
    f = eb.EbcFunction(eb.GroundMatrix(X, eb.Precision.FP32))
    for rep in range(3):
        t0 = time.perf_counter(); v = eb.evaluate_with_backend(f, ms); t1 = time.perf_counter()
    dev = optimize.last_timings(f)[3]
    res[mode] = v
    pe = 200_000 * sum(len(s) for s in sets)
    print(f"mode {mode}: device {dev:.2f} ms, wall {1e3*(t1-t0):.2f} ms, point-element evals/s {pe/(dev*1e-3):.3e}, launches {optimize.last_launches(f)}")
print("bit-identical:", res["0"].tolist() == res["1"].tolist() == res["2"].tolist())
