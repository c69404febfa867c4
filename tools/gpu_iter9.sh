set -x
timeout 900 python -m pytest tests -m gpu -q -x -k "device_exchange or device_pick" 2>&1 | tail -15
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
