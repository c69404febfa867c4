set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python tools/quick_time.py 2>&1 | grep -v untimed
for C in C4 C3 C2; do
timeout 600 python bench.py --config $C --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$C bench', d['ms_per_step'], d['roofline']['tmem_read']['frac'], d['window'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c4.csv python tools/profile_run.py C4 20 > /dev/null 2>&1; wc -l gpurun_out/launches_c4.csv
