set -x
timeout 900 python -m pytest tests -m gpu -q -x -k "device_exchange or device_pick or one_rank_nccl" 2>&1 | tail -15
