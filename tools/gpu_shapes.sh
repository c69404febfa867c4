set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for S in 0 1 2; do EBC200_SCREEN=$S python tools/quick_time.py 2>&1 | grep -v untimed; done
