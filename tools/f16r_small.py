"""Small fast-rung (and fp16-storage) Greedy runs, for compute-sanitizer."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2105_12026_b200 as eb
rng = np.random.default_rng(0)
for prec, dt in ((eb.Precision.FP32, np.float32), (eb.Precision.FP16_STORAGE, np.float16)):
    X = rng.standard_normal((3000, 100)).astype(dt)
    f = eb.EbcFunction(eb.GroundMatrix(X, prec))
    s = eb.greedy_maximize(f, eb.OptimizerBudget(k=4))
    print(prec, s.selected, flush=True)
    f.close()
