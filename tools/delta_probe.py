"""Probe (development only): per Greedy step, the fraction of 128-point tiles
whose cached minimum changes when the step's winner is folded in (what an
incremental screen over changed tiles would have to re-screen).
    python tools/delta_probe.py C4"""
import json, os, sys
import numpy as np
import torch
_R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(_R, "tests", "golden")); sys.path.insert(0, _R)
from datasets import config_data  # noqa: E402
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
X = torch.from_numpy(config_data(name).astype(np.float32)).double().cuda()
sel = json.load(open(os.path.join(_R, "tests", "golden", f"oracle_{name}.json")))["selected"]
n = X.shape[0]
T = (n + 127) // 128
cm = (X * X).sum(1)
for s, c in enumerate(sel):
    d = ((X - X[c]) ** 2).sum(1)
    ch = d < cm
    pad = T * 128 - n
    chp = torch.cat([ch, torch.zeros(pad, dtype=torch.bool, device=ch.device)]) if pad else ch
    tiles = chp.view(T, 128).any(1)
    print(f"step {s:2d}: points changed {ch.float().mean().item():.4f}  tiles changed {tiles.float().mean().item():.4f}")
    cm = torch.minimum(cm, d)
