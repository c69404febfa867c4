set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python tools/e2e_probe.py C2
timeout 300 python tools/e2e_probe.py C4
timeout 900 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('C2 bench', d['ms_per_step'], d['e2e'])"
