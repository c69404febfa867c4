import os, sys
sys.path.insert(0, "."); sys.path.insert(0, "tests/golden")
import numpy as np, datasets
import paper_2105_12026_b200 as eb
X = datasets.config_data(sys.argv[1] if len(sys.argv) > 1 else "C2")
g = eb.GroundMatrix(X, eb.Precision.FP32)
f = eb.EbcFunction(g)
s = eb.greedy_maximize(f, eb.OptimizerBudget(k=2))
