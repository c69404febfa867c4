# Round evidence after the fast rung: gpu tests, smoke, every config's bench line
# (default C2 with the CPU baseline), the reference arm, launch lists C2/C4.
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
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_c4.csv python tools/profile_run.py C4 20 > /dev/null 2>&1
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv
