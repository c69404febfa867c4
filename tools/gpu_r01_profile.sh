set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python bench.py 2>gpurun_out/bench_c2.err | tee gpurun_out/bench_c2.json
python bench.py --config C4 --steps 2 --no-cpu-baseline 2>gpurun_out/bench_c4.err | tee gpurun_out/bench_c4.json
python bench.py --impl reference --steps 2 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/profile_run.py C2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_screen -s 2 -c 1 -o gpurun_out/screen_c2 python tools/profile_run.py C2 4 > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_screen -s 2 -c 1 -o gpurun_out/screen_c4 python tools/profile_run.py C4 3 >> gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out
