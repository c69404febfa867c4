# One development iteration on the GPU box: parity tests, quick timings, bench
# line, and an ncu full capture of one k_screen launch (C2).
set -x
mkdir -p gpurun_out
TAG=${1:-iter}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python tools/quick_time.py 2>&1 | tail -12
python bench.py --no-cpu-baseline 2>gpurun_out/bench_${TAG}.err | tee gpurun_out/bench_${TAG}.json
if [ "${NCU:-1}" = "1" ]; then
ncu --set full --clock-control none --import-source on -k regex:k_screen -s 2 -c 1 -o gpurun_out/screen_${TAG} python tools/profile_run.py C2 4 > gpurun_out/ncu_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_${TAG}.log
fi
