set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "every_screen or full_config or random_instances" 2>&1 | tail -5
timeout 300 python tools/quick_time.py 2>&1 | grep -v untimed
timeout 300 python tools/e2e_probe.py C2
timeout 900 python bench.py --config C3 --no-cpu-baseline 2>gpurun_out/bench_err.log | tee gpurun_out/bench_c3.json
