# Round check on one B200: gpu tests, smoke, default bench line.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1200 python -m pytest tests -m gpu -q -x --durations=8 2>&1 | tail -14
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py 2>gpurun_out/bench_err.log | tee gpurun_out/bench_default.json
tail -3 gpurun_out/bench_err.log
