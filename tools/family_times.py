"""Per-family device times of graph replays (timing mode): selection (lazy
batch + undecided part) vs cached-min update, per step.  python tools/family_times.py C2"""
import os, sys
import numpy as np
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests", "golden"))
import datasets
import paper_2105_12026_b200 as eb
from paper_2105_12026_b200 import optimize
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
X = datasets.config_data(name); k = datasets.CONFIG_K[name]
f = eb.EbcFunction(eb.GroundMatrix(X, eb.Precision.FP32))
optimize.set_timing(f, True)
for _ in range(4):
    eb.greedy_maximize(f, eb.OptimizerBudget(k=k))
t = optimize.last_timings(f)
print(f"{name}: total {t[3]:.3f} ms; selection {t[0]:.3f} (incl. step-0 screen), refine(step 0) {t[1]:.3f}, "
      f"update {t[2]:.3f} ms = {1e3 * t[2] / k:.1f} us/step")
optimize.set_timing(f, False)
for _ in range(3):
    s = eb.greedy_maximize(f, eb.OptimizerBudget(k=k))
print(f"untimed replay {s.runtime_seconds * 1e3:.2f} ms wall")
