set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for M in ${MODES:-0 2}; do EBC200_SCREEN_MODE=$M python tools/quick_time.py 2>&1 | grep -v untimed; done
