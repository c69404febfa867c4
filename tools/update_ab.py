"""A/B of the cached-min update (K4): per-step device time of the update family,
fused one-launch kernel vs the split two-kernel form.
    python tools/update_ab.py C2 "fused split"   ('split' = two-kernel K4)"""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import datasets
import paper_2105_12026_b200 as eb
from paper_2105_12026_b200 import optimize

name = sys.argv[1]
X = datasets.config_data(name)
k = datasets.CONFIG_K[name]
prec = eb.Precision.FP16_STORAGE if X.dtype == np.float16 else eb.Precision.FP32
ref = None
for spec in sys.argv[2].split():
    if spec == "split":
        os.environ["EBC200_UPDATE_FUSED"] = "0"
    else:
        os.environ["EBC200_UPDATE_FUSED"] = "1"
    f = eb.EbcFunction(eb.GroundMatrix(X, prec))
    optimize.set_timing(f, True)
    us = []
    for i in range(5):
        s = eb.greedy_maximize(f, eb.OptimizerBudget(k=k))
        if i >= 2:
            us.append(optimize.last_timings(f)[2] / k * 1e3)
    if ref is None:
        ref = (s.selected, s.gains)
    assert (s.selected, s.gains) == ref, spec
    print(f"{name} {spec:6s} update {np.median(us):7.2f} us/step  total {optimize.last_timings(f)[3]:8.2f} ms", flush=True)
    f.close()
