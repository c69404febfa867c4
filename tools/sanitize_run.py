"""Small runs of every device path, for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import numpy as np
import datasets
import paper_2105_12026_b200 as eb

rng = np.random.default_rng(0)
runs = [("surrogate-anchored-pruned", datasets.surrogate(4000, 32, 5, 0.01, 0).astype(np.float32), eb.Precision.FP32),
        ("gaussian-bf16", rng.standard_normal((3000, 100)).astype(np.float32), eb.Precision.FP32),
        ("gaussian-fp16", rng.standard_normal((3000, 100)).astype(np.float16), eb.Precision.FP16_STORAGE),
        ("gaussian-d16-direct", rng.standard_normal((3000, 16)).astype(np.float32), eb.Precision.FP32)]
for name, X, prec in runs:
    f = eb.EbcFunction(eb.GroundMatrix(X, prec))
    s = eb.greedy_maximize(f, eb.OptimizerBudget(k=6))
    s2 = eb.greedy_maximize(f, eb.OptimizerBudget(k=6))  # captured graph
    s3 = eb.greedy_maximize(f, eb.OptimizerBudget(k=6))  # replay (decided lazy steps without conditional nodes)
    assert s.selected == s2.selected == s3.selected
    sets = [rng.choice(X.shape[0], size=10, replace=False).tolist() for _ in range(64)]
    v = eb.evaluate_with_backend(f, eb.EvalMultiset(sets))
    print(name, s.selected, float(v[0]))
    f.close()
print("sanitize run ok")
