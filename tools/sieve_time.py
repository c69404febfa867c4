"""Sieve streaming timing (development): the cached-minima device sieve on a
C4-shaped stream, next to the set-by-set work-matrix sieve for a prefix.
    python tools/sieve_time.py [stream_len] [k]"""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests", "golden")); sys.path.insert(0, os.path.join(ROOT, "tests"))
import datasets
import paper_2105_12026_b200 as eb

L = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 20
X = datasets.config_data("C4")
f = eb.EbcFunction(eb.GroundMatrix(X, eb.Precision.FP32))
stream = np.random.default_rng(0).permutation(X.shape[0])[:L].tolist()
eb.sieve_stream_maximize(stream[:200], f, k)  # warm-up
t0 = time.perf_counter()
s = eb.sieve_stream_maximize(stream, f, k)
dt = time.perf_counter() - t0
print(f"cached-minima sieve: {L} elements, k={k}: {dt:.2f} s ({dt / L * 1e6:.1f} us/element), "
      f"evaluations {s.evaluations}, value {s.value:.6g}, |S|={len(s.selected)}")
from test_gpu_parity import _sieve_by_multisets  # noqa: E402
P = min(L, 2000)
t0 = time.perf_counter()
_sieve_by_multisets(stream[:P], f, k, 0.1)
dt2 = time.perf_counter() - t0
print(f"set-by-set work-matrix sieve: first {P} elements {dt2:.2f} s ({dt2 / P * 1e6:.1f} us/element)")
