"""Probe (development only): how many candidates a lazy (Minoux) Greedy would have
to re-screen per step on a config, using torch fp32 gains on the GPU.

Lazy rule simulated: ub[c] = the gain of c at the last step it was screened
(+inf before); at step s the lower bound lb = gain of argmax ub; re-screen
{c : ub[c] >= lb * (1 - slack)}; pick the argmax of the fresh gains.
Submodularity makes every stale ub a valid upper bound of the current gain.

usage: python tools/lazy_probe.py C4 [slack]
"""
import os
import sys
import time

import numpy as np
import torch

_R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(_R, "tests", "golden"))
sys.path.insert(0, _R)
from datasets import CONFIG_K, config_data  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False


def gains(V, vn, cm, cidx, chunk=2048):
    out = torch.empty(cidx.numel(), dtype=torch.float64, device=V.device)
    for a in range(0, cidx.numel(), chunk):
        c = V[cidx[a:a + chunk]]
        d = vn[:, None] + (c * c).sum(1)[None, :] - 2.0 * (V @ c.T)
        out[a:a + chunk] = torch.clamp(cm[:, None] - d, min=0).sum(0, dtype=torch.float64)
    return out


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C4"
    slack = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-3
    X = torch.from_numpy(config_data(name).astype(np.float32)).cuda()
    k = CONFIG_K[name]
    n = X.shape[0]
    vn = (X * X).sum(1)
    cm = vn.clone()  # e0 = 0
    ub = torch.full((n,), float("inf"), dtype=torch.float64, device="cuda")
    sel = []
    t0 = time.time()
    total = 0
    for s in range(k):
        u = ub.clone()
        if sel:
            u[torch.tensor(sel, device="cuda")] = -1
        top = int(torch.argmax(u))
        lb = float(gains(X, vn, cm, torch.tensor([top], device="cuda"))[0]) if s else 0.0
        scr = torch.nonzero(u >= lb * (1 - slack)).flatten()
        g = gains(X, vn, cm, scr)
        ub[scr] = g
        best = int(scr[int(torch.argmax(g))])
        sel.append(best)
        total += scr.numel()
        # block-level view: how many 128-candidate blocks hold a screened candidate
        blocks = torch.unique(scr // 128).numel()
        print(f"step {s:2d} screened {scr.numel():8d} ({scr.numel()/n:.4f}) blocks {blocks:5d}/{(n+127)//128} "
              f"pick {best} gain {float(g.max()):.6g}", flush=True)
        d = vn + vn[best] - 2.0 * (X @ X[best])
        cm = torch.minimum(cm, torch.clamp(d, min=0))
    print(f"{name}: screened {total} of {n*k} candidate-steps ({total/(n*k):.4f}); {time.time()-t0:.1f}s; sel head {sel[:5]}")


if __name__ == "__main__":
    main()
