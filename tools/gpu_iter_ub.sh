# Iteration check for the per-step kernels: GPU suite, C2/C4 bench lines,
# launch list of the per-step kernels (C2).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/it_tests.log 2>&1; tail -2 gpurun_out/it_tests.log
for c in ${CONFIGS:-C2 C4}; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/it_bench_$c.json 2> gpurun_out/it_bench_$c.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/it_bench_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3), 'upd_us', round(d['update_roofline']['us_per_step'],2), d['selected_head'], d['clocks']['sm_mhz'])"
done
CONFIG=C2 SKIP=20 bash tools/gpu_prof_ub.sh
