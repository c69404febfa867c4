"""Greedy runs of a config for ncu launch lists of the graph REPLAY (the bench's
timed path): run 1 eager, run 2 capture + first replay, run 3 replay.
    python tools/profile_replay.py C2 [runs]"""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import datasets
import paper_2105_12026_b200 as eb

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 3
X = datasets.config_data(name)
k = datasets.CONFIG_K[name]
prec = eb.Precision.FP16_STORAGE if X.dtype == np.float16 else eb.Precision.FP32
f = eb.EbcFunction(eb.GroundMatrix(X, prec))
for r in range(runs):
    s = eb.greedy_maximize(f, eb.OptimizerBudget(k=k))
    print(name, r, s.selected[:5], s.value, f"{s.runtime_seconds * 1e3:.2f} ms", flush=True)
