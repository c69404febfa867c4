"""A/B device timing of compile-time variants: python tools/ab_libs.py lib1.so lib2.so ...
Each variant runs in a subprocess (one library per process): C2 k=10, C3 k=10, C4 k=5."""
import os, subprocess, sys
code = r'''
import sys, os
sys.path.insert(0, "."); sys.path.insert(0, "tests/golden")
import numpy as np, datasets
import paper_2105_12026_b200 as eb
from paper_2105_12026_b200 import optimize
for name, k, prec in (("C2", 10, eb.Precision.FP32), ("C3", 10, eb.Precision.FP16_STORAGE), ("C4", int(os.environ.get("AB_C4K", "5")), eb.Precision.FP32)):
    X = datasets.config_data(name)
    f = eb.EbcFunction(eb.GroundMatrix(X, prec))
    optimize.set_timing(f, True)
    s = eb.greedy_maximize(f, eb.OptimizerBudget(k=k))
    best = None
    for _ in range(3):
        s = eb.greedy_maximize(f, eb.OptimizerBudget(k=k))
        t = optimize.last_timings(f)
        best = t if best is None or t[3] < best[3] else best
    print(f"  {name} k={k}: total {best[3]:.2f} ms screen {best[0]:.2f} refine {best[1]:.2f} update {best[2]:.2f} stats {optimize.last_stats(f)} sel {s.selected[:3]}", flush=True)
    f.close()
'''
for lib in sys.argv[1:]:
    env = dict(os.environ)
    if lib != "default":
        env["EBC200_LIB_PATH"] = os.path.abspath(lib)
    print(lib, flush=True)
    subprocess.run([sys.executable, "-c", code], env=env, timeout=600)
