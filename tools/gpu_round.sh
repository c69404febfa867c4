# Full round check: gpu tests, every config's bench line, C5 timing, ncu captures.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for C in C2 C3 C4 C1; do
  timeout 900 python bench.py --config $C --no-cpu-baseline 2>gpurun_out/bench_err_$C.log > gpurun_out/bench_$C.json
  tail -2 gpurun_out/bench_err_$C.log
done
timeout 300 python tools/c5_time.py
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_screen_tc -s 12 -c 1 -o gpurun_out/screen_tc_C4 python tools/profile_run.py C4 10 > gpurun_out/ncu_C4.log 2>&1; tail -1 gpurun_out/ncu_C4.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python tools/profile_run.py C2 5 > /dev/null 2>&1; wc -l gpurun_out/launches_c2.csv
