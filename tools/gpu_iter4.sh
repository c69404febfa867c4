set -x
timeout 900 python -m pytest tests -m gpu -q -x -k "every_screen or full_config or random_instances or golden or matches_reference" 2>&1 | tail -3
timeout 300 python tools/quick_time.py 2>&1 | grep -v untimed
