import sys, time
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests/golden")
import datasets, oracle
import paper_2105_12026_b200 as eb
from paper_2105_12026_b200 import optimize
import torch
for name, n, d, k in [("C1", 2000, 16, 10), ("g", 20000, 48, 8)]:
    X = datasets.gaussian(n, d, 0)
    f = eb.EbcFunction(eb.GroundMatrix(X, eb.Precision.FP32))
    st = torch.cuda.ExternalStream(f._lib.ebc_stream(f.native_context))
    res = []
    for rep in range(6):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st); s = eb.greedy_maximize(f, eb.OptimizerBudget(k=k)); e1.record(st); torch.cuda.synchronize()
        res.append((s.selected, s.gains, e0.elapsed_time(e1), optimize.last_launches(f)))
    ref = oracle.greedy(X.astype(np.float64), k)[0]
    print(name, "eager ms %.3f" % res[0][2], "graph ms", ["%.3f" % r[2] for r in res[1:]], "launches", [r[3] for r in res],
          "same", all(r[0] == res[0][0] and r[1] == res[0][1] for r in res), "oracle", res[0][0] == ref)
