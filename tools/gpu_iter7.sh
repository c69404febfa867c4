set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python tools/quick_time.py 2>&1 | grep -v untimed
EBC200_TC_PRUNE=0 timeout 300 python tools/quick_time.py 2>&1 | grep -v untimed | grep C4
timeout 300 python tools/c5_time.py
timeout 900 python bench.py --config C4 --no-cpu-baseline 2>gpurun_out/bench_err_c4.log | tee gpurun_out/bench_c4.json
