# Round-2 baseline check on one B200: gpu tests, smoke, C2 + C4 bench lines.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1200 python -m pytest tests -m gpu -q -x --durations=8 2>&1 | tail -14
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for c in ${CONFIGS:-C2 C4}; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>gpurun_out/bench_err_$c.log | tee gpurun_out/bench_$c.json
  tail -3 gpurun_out/bench_err_$c.log
done
