set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
EBC200_SCREEN_MODE=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
EBC200_SCREEN_MODE=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for M in 0 1 2; do EBC200_SCREEN_MODE=$M python tools/quick_time.py 2>&1 | grep -v untimed; done
