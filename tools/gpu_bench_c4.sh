set -x
timeout 900 python bench.py --config C4 --no-cpu-baseline 2>gpurun_out/bench_err_c4.log | tee gpurun_out/bench_c4.json
timeout 900 python bench.py 2>gpurun_out/bench_err.log | tee gpurun_out/bench_c2.json
tail -3 gpurun_out/bench_err_c4.log
