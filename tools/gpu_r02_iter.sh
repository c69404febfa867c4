# Round-2 iteration on one B200: gpu tests, C2 bench line, 2-rank spawn (gloo, shared GPU).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
for c in ${CONFIGS:-C2}; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>gpurun_out/bench_err_$c.log | tee gpurun_out/bench_$c.json
  tail -3 gpurun_out/bench_err_$c.log
done
if [ -n "$SPAWN2" ]; then
  EBC_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --config C1 --steps 3 --no-cpu-baseline 2>gpurun_out/bench_err_spawn2.log | tee gpurun_out/bench_spawn2.json
  tail -5 gpurun_out/bench_err_spawn2.log
fi
