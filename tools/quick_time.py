"""Quick device timing of Greedy steps at a BASELINE shape (development aid)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests/golden")
import paper_2105_12026_b200 as eb
from paper_2105_12026_b200 import optimize
import datasets

def run(name, n, d, k, prec=eb.Precision.FP32, gen="gaussian"):
    if gen == "gaussian":
        X = datasets.gaussian(n, d, 1)
    else:
        X = datasets.surrogate(n, d, 5, 0.01, 0).astype(np.float32)
    f = eb.EbcFunction(eb.GroundMatrix(X, prec))
    optimize.set_timing(f, True)
    s = eb.greedy_maximize(f, eb.OptimizerBudget(k=k))
    t = optimize.last_timings(f)
    pairs = sum(n * (n - s_) for s_ in range(k))
    ops = pairs * 2 * d
    peak = 148 * 128 * 1.965e9
    print(f"{name}: n={n} d={d} k={k} total {t[3]:.2f} ms screen {t[0]:.2f} refine {t[1]:.2f} update {t[2]:.2f}"
          f" | screen {ops / (t[0] * 1e-3) / peak:.3f} of FMA peak, whole {ops / (t[3] * 1e-3) / peak:.3f}"
          f" evals/s {pairs / (t[3] * 1e-3):.3e} launches {optimize.last_launches(f)} stats {optimize.last_stats(f)} sel {s.selected[:3]}")
    optimize.set_timing(f, False)
    t0 = time.perf_counter(); s2 = eb.greedy_maximize(f, eb.OptimizerBudget(k=k)); t1 = time.perf_counter()
    print(f"   untimed run wall {1e3 * (t1 - t0):.2f} ms, same selection {s2.selected == s.selected}")

if __name__ == "__main__":
    run("C1", 2000, 16, 10)
    run("C2-k5", 100000, 100, 5)
    run("C4-k3", 500000, 32, 3, gen="surrogate")
    run("C3-k5", 100000, 100, 5, prec=eb.Precision.FP16_STORAGE)
