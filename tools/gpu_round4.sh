# Round evidence (folded seeds + ladder-pruned graphs): tests, smoke, every bench line,
# reference arm, launch lists, ncu full of the C2 rung-0 screen, sanitizers on small runs.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py 2>gpurun_out/bench_err_C2.log > gpurun_out/bench_C2.json
for C in C3 C4 C1; do
  timeout 900 python bench.py --config $C --no-cpu-baseline 2>gpurun_out/bench_err_$C.log > gpurun_out/bench_$C.json
done
timeout 300 python tools/c5_time.py > gpurun_out/c5_time.txt 2>&1
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref_C2.json 2>gpurun_out/bench_err_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c2.csv python tools/profile_run.py C2 50 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_screen_tc -s 2 -c 1 -o gpurun_out/screen_ms_C2 python tools/profile_run.py C2 4 > gpurun_out/ncu_ms_C2.log 2>&1
for T in memcheck racecheck; do
  timeout 900 compute-sanitizer --tool $T --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/sanitizer_$T.log 2>&1; echo "$T rc=$?"; tail -2 gpurun_out/sanitizer_$T.log
done
