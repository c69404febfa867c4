"""Probe (development only): classify (candidate block, point tile) pairs of a
Greedy run as prunable / all-positive / mixed under two geometric tests:
  anchor : the screen's test through the block's FPS anchor mu (rho_t = min |v - mu|,
           rhomax_t = max |v - mu|, R_b = max |c - mu|)
  center : block center mu_b / radius R_b against tile center mu_t / radius R_t
           (gap = |mu_b - mu_t| - R_b - R_t, span = |mu_b - mu_t| + R_b + R_t)
prunable: gap > 0 and gap^2 > max cm(tile); all-positive: span^2 < min cm(tile).
Uses the oracle golden selection to replay cm.  usage: prune_probe.py C4 [steps]
"""
import json
import os
import sys

import numpy as np
import torch

_R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(_R, "tests", "golden"))
sys.path.insert(0, _R)
from datasets import config_data  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
X = torch.from_numpy(config_data(name).astype(np.float32)).double().cuda()
sel = json.load(open(os.path.join(_R, "tests", "golden", f"oracle_{name}.json")))["selected"]
n, d = X.shape
T = (n + 127) // 128
pad = T * 128 - n
Xp = torch.cat([X, X[-1:].expand(pad, d)]) if pad else X
tiles = Xp.view(T, 128, d)
mu = tiles.mean(1)                                     # T x d
rad = (tiles - mu[:, None]).norm(dim=2).max(1).values  # T
# FPS anchors like the library (32, first = origin)
na = 32
anchors = [torch.zeros(d, dtype=X.dtype, device=X.device)]
dmin = (X - anchors[0]).norm(dim=1)
for _ in range(na - 1):
    i = int(torch.argmax(dmin))
    anchors.append(X[i].clone())
    dmin = torch.minimum(dmin, (X - X[i]).norm(dim=1))
A = torch.stack(anchors)                                # na x d
dta = torch.cdist(tiles.reshape(-1, d), A).view(T, 128, na)   # |v - mu_a|
rho = dta.min(1).values                                  # T x na
rhomax = dta.max(1).values
Rb_a = dta.max(1).values                                 # block radius per anchor (blocks = tiles)
banc = torch.argmin(Rb_a, dim=1)                         # block anchor = min radius
Rb = Rb_a.gather(1, banc[:, None])[:, 0]
cdist = torch.cdist(mu, mu)                               # T x T center distances
gap_c = cdist - rad[:, None] - rad[None, :]
span_c = cdist + rad[:, None] + rad[None, :]
rho_b = rho[:, banc].T                                    # [block, tile] rho of block's anchor
rhx_b = rhomax[:, banc].T
gap_a = rho_b - Rb[:, None]
span_a = rhx_b + Rb[:, None]
cm = (X * X).sum(1)
tot = T * T
for s in range(steps):
    cmp_ = torch.cat([cm, cm[-1:].expand(pad)]) if pad else cm
    cmx = cmp_.view(T, 128).max(1).values
    cmn = cmp_.view(T, 128).min(1).values
    out = []
    for gap, span in ((gap_a, span_a), (gap_c, span_c)):
        prun = (gap > 0) & (gap * gap > cmx[None, :])
        allp = (~prun) & (span * span < cmn[None, :])
        mixed = ~(prun | allp)
        out.append((prun.sum().item() / tot, allp.sum().item() / tot, mixed.sum().item() / tot))
    print(f"step {s:2d} anchor prune {out[0][0]:.3f} allpos {out[0][1]:.3f} mixed {out[0][2]:.4f} | "
          f"center prune {out[1][0]:.3f} allpos {out[1][1]:.3f} mixed {out[1][2]:.4f}", flush=True)
    c = sel[s]
    cm = torch.minimum(cm, ((X - X[c]) ** 2).sum(1))
print("mean tile radius", float(rad.mean()), "mean block radius (anchor)", float(Rb.mean()))
