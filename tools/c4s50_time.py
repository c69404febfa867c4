import os, sys, time
sys.path.insert(0, "."); sys.path.insert(0, "tests/golden")
import numpy as np, datasets
import paper_2105_12026_b200 as eb
from paper_2105_12026_b200 import optimize
X = datasets.config_data("C4S50")
f = eb.EbcFunction(eb.GroundMatrix(X, eb.Precision.FP32))
for r in range(3):
    s = eb.greedy_maximize(f, eb.OptimizerBudget(k=20))
    print(r, f"{s.runtime_seconds*1e3:.1f} ms", optimize.last_stats(f), optimize.last_lazy_stats(f), s.selected[:4], flush=True)
