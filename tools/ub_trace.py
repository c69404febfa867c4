"""Phase stamps of the fused update + batch (k_update_batch) per Greedy step,
from a -DEBC200_TRACE build:
    bash tools/build_variant.sh trace -DEBC200_TRACE
    EBC200_LIB_PATH=paper_2105_12026_b200/libebc200_trace.so python tools/ub_trace.py C2"""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import datasets
import paper_2105_12026_b200 as eb
from paper_2105_12026_b200 import _native

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
X = datasets.config_data(name)
k = datasets.CONFIG_K[name]
f = eb.EbcFunction(eb.GroundMatrix(X, eb.Precision.FP32))
lib = _native.load()
fn = lib.ebc_debug_ub_trace
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
buf = (ctypes.c_ulonglong * (64 * 8 + 8192 * 4 + 64 * 4))()
for rep in range(3):
    fn(None, 1)
    eb.greedy_maximize(f, eb.OptimizerBudget(k=k))
    fn(buf, 0)
allb = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
a = allb[:512].reshape(64, 8)
blk = allb[512:512 + 8192 * 4].reshape(8192, 4)
tk = allb[512 + 8192 * 4:].reshape(64, 4)
nb = int(np.count_nonzero(blk[:, 0]))
if nb:
    b = blk[:nb].copy()
    t0 = b[:, 0].min()
    st, ld, mn = (b[:, 0] - t0) / 1e3, (b[:, 1] - b[:, 0]) / 1e3, (b[:, 2] - b[:, 1]) / 1e3
    print(f"step 10: {nb} blocks; start quantiles", np.round(np.quantile(st, [0, .25, .5, .75, 1]), 2))
    print("  load us quantiles", np.round(np.quantile(ld, [0, .25, .5, .75, .9, 1]), 2))
    print("  compute us quantiles", np.round(np.quantile(mn, [0, .25, .5, .75, .9, 1]), 2))
    w1 = st < 0.5
    print(f"  first-wave blocks {w1.sum()}: load med {np.median(ld[w1]):.2f} compute med {np.median(mn[w1]):.2f};"
          f" later: load med {np.median(ld[~w1]) if (~w1).any() else 0:.2f} compute med {np.median(mn[~w1]) if (~w1).any() else 0:.2f}")
    sms = b[:, 3]
    print("  blocks per SM max", np.bincount(sms).max(), "SMs used", len(np.unique(sms)))
names = ["last block start", "first load done(max)", "main done(max)", "final start", "sums done", "finalize done"]
rows = []
for st in range(64):
    if a[st, 0] <= 0 or a[st, 0] >= 2**62 or a[st, 6] == 0:
        continue
    rel = (a[st, 1:7] - a[st, 0]) / 1e3
    rows.append(rel)
    if len(rows) <= 6:
        print(st, " ".join(f"{x:7.2f}" for x in rel))
r = np.median(np.array(rows), axis=0)
print("median us from first block start:", dict(zip(names, np.round(r, 2))))

tr = []
for st in range(64):
    if 0 < tk[st, 0] < 2**62 and tk[st, 3] > 0:
        tr.append((tk[st, 1:4] - tk[st, 0]) / 1e3)
        # gap from the topk end to the update's first block (step st is the update's step + 1)
if tr:
    print("k_lazy_topk median us from its first block:", dict(zip(["scan done", "last block", "end (pack done)"],
                                                               np.round(np.median(np.array(tr), axis=0), 2))))
    gaps = [(a[st - 1, 0] - tk[st, 3]) / 1e3 for st in range(1, 64)
            if 0 < tk[st, 0] < 2**62 and tk[st, 3] > 0 and 0 < a[st - 1, 0] < 2**62]
    # update(s) is followed by step s+1's select (conditional node) and then
    # run_update_batch(s+1), whose top-k is traced as step s+2
    gaps2 = [(tk[st + 2, 0] - a[st, 6]) / 1e3 for st in range(0, 62)
             if 0 < tk[st + 2, 0] < 2**62 and 0 < a[st, 6] < 2**62]
    if gaps:
        print("median gap topk end -> update start (us):", round(float(np.median(gaps)), 2),
              " update end -> next topk start (us):", round(float(np.median(gaps2)), 2) if gaps2 else None)
