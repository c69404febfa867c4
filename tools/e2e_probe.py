"""Break the e2e C2 path into create / first greedy / second greedy / close (wall clock)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
if os.environ.get("PROBE_TORCH"):
    import torch
    torch.cuda.init()
import paper_2105_12026_b200 as eb
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden"))
from datasets import config_data

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
X = config_data(cfg)
k = {"C1": 10, "C2": 50, "C3": 50, "C4": 20}[cfg]
prec = eb.Precision.FP16_STORAGE if X.dtype == np.float16 else eb.Precision.FP32
g = eb.GroundMatrix(X, prec)
f0 = eb.EbcFunction(g); eb.greedy_maximize(f0, eb.OptimizerBudget(k=k))
if not os.environ.get("PROBE_KEEP"):
    f0.close()
for rep in range(3):
    t0 = time.perf_counter(); f = eb.EbcFunction(g); t1 = time.perf_counter()
    s = eb.greedy_maximize(f, eb.OptimizerBudget(k=k)); t2 = time.perf_counter()
    s = eb.greedy_maximize(f, eb.OptimizerBudget(k=k)); t3 = time.perf_counter()
    s = eb.greedy_maximize(f, eb.OptimizerBudget(k=k)); t4 = time.perf_counter()
    f.close(); t5 = time.perf_counter()
    print(f"{cfg} create {1e3*(t1-t0):.1f} ms  greedy#1 {1e3*(t2-t1):.1f}  #2(capture) {1e3*(t3-t2):.1f}  #3(graph) {1e3*(t4-t3):.1f}  close {1e3*(t5-t4):.1f}")
