set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python tools/quick_time.py 2>&1 | grep -v untimed
timeout 300 python tools/e2e_probe.py C2
timeout 900 python bench.py 2>gpurun_out/bench_err.log | tee gpurun_out/bench_default.json
