"""One Greedy run of a BASELINE config, for ncu launch lists / full captures.
    python tools/profile_run.py C2 [k]"""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import datasets
import paper_2105_12026_b200 as eb

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
X = datasets.config_data(name)
k = int(sys.argv[2]) if len(sys.argv) > 2 else datasets.CONFIG_K[name]
prec = eb.Precision.FP16_STORAGE if X.dtype == np.float16 else eb.Precision.FP32
f = eb.EbcFunction(eb.GroundMatrix(X, prec))
s = eb.greedy_maximize(f, eb.OptimizerBudget(k=k))
print(name, k, s.selected[:5], s.value, s.runtime_seconds)
