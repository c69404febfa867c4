# Round-2 (session 3) final measurements on one B200: suite, smoke, bench lines
# C2 (default) / C4 / C1 / C5 / C4S50, the reference arm, C2 launch list and a
# --set full capture of k_update_batch.
mkdir -p gpurun_out/final5
O=gpurun_out/final5
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 1200 python -m pytest tests -m gpu -q -x --durations=8 > $O/gpu_tests.txt 2>&1; tail -3 $O/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for c in C2 C4 C1 C5 C4S50; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
for f in $O/bench_*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', d.get('ms_per_step'), (d.get('e2e') or {}).get('ms_per_step'), (d.get('update_roofline') or {}).get('frac'), (d.get('roofline') or {}).get('frac'), d.get('selected_head'))
" 2>&1 | tail -1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  python tools/profile_run.py C2 > $O/launches_c2.csv 2> $O/launches_c2.err
python tools/launch_summary.py $O/launches_c2.csv > $O/launches_c2_summary.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_update_batch -s 20 -c 1 \
  -o $O/ub_full_c2 -f python tools/profile_run.py C2 > $O/ub_full.log 2>&1
EBC200_LIB_PATH=paper_2105_12026_b200/libebc200_trace.so python tools/ub_trace.py C2 > $O/ub_trace_c2.txt 2>&1
EBC200_LIB_PATH=paper_2105_12026_b200/libebc200_trace.so python tools/ub_trace.py C4 > $O/ub_trace_c4.txt 2>&1
