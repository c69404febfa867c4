"""Helper for test_gpu_parity.py: greedy_maximize_sharded over a one-rank NCCL
process group (the device-exchange path a torchrun job takes), two
EbcFunctions in a row (the second attaches to the device's communicator)."""
import os
import socket
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_12026_b200 as eb  # noqa: E402
from paper_2105_12026_b200 import sharded  # noqa: E402

s = socket.socket()
s.bind(("127.0.0.1", 0))
port = s.getsockname()[1]
s.close()
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
X = np.random.default_rng(5).standard_normal((5000, 48)).astype(np.float32)
g = eb.GroundMatrix(X, eb.Precision.FP32)
ref = eb.greedy_maximize(eb.EbcFunction(g), eb.OptimizerBudget(k=8))
for _ in range(2):
    f = eb.EbcFunction(g)
    got = sharded.greedy_maximize_sharded(f, eb.OptimizerBudget(k=8))
    assert got.selected == ref.selected and got.gains == ref.gains, (got.selected, ref.selected)
    assert f._comm_key is not None
dist.destroy_process_group()
print("nccl one-rank ok", got.selected)
