set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 1 --warmup 3 --config C1 2>gpurun_out/torchrun2.err | tee gpurun_out/torchrun2.json
tail -5 gpurun_out/torchrun2.err
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_memcheck.log 2>&1; echo memcheck rc=$?
timeout 600 compute-sanitizer --tool racecheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_racecheck.log 2>&1; echo racecheck rc=$?
timeout 600 compute-sanitizer --tool synccheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_synccheck.log 2>&1; echo synccheck rc=$?
tail -3 gpurun_out/sanitizer_*.log
python bench.py 2>gpurun_out/bench_b.err | tee gpurun_out/bench_b.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_b.csv python tools/profile_run.py C2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_screen -s 2 -c 1 -o gpurun_out/screen_c2_b python tools/profile_run.py C2 4 > gpurun_out/ncu_b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_screen -s 2 -c 1 -o gpurun_out/screen_c4_b python tools/profile_run.py C4 3 >> gpurun_out/ncu_b.log 2>&1
tail -2 gpurun_out/ncu_b.log
