set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for C in C4 C3 C2; do
timeout 600 python bench.py --config $C --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$C', d['ms_per_step'], d['roofline']['tmem_read']['frac'], d['clocks']['sm_mhz'], d['window'])"
done
