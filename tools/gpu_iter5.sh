set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python tools/quick_time.py 2>&1 | grep -v untimed
EBC200_TC_ANCHORS=1 timeout 300 python tools/quick_time.py 2>&1 | grep -v untimed | grep C4
timeout 600 python -m pytest tests -m gpu -q -x -k "full_config" 2>&1 | tail -2
