"""One C5 work-matrix evaluation (for ncu launch lists)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import datasets
import paper_2105_12026_b200 as eb
X, sets = datasets.c5_problem()
f = eb.EbcFunction(eb.GroundMatrix(X, eb.Precision.FP32))
ms = eb.EvalMultiset(sets)
for _ in range(2):
    v = eb.evaluate_with_backend(f, ms)
print("c5", v[:3])
