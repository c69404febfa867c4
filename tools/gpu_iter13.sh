set -x
timeout 900 python -m pytest tests -m gpu -q -x -k "multiset or sparse or full_config or c5 or cli" 2>&1 | tail -3
timeout 300 python tools/c5_time.py
