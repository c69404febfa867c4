# Fast-rung check: parity tests touching the ladder, then C2 with the fast rung on/off.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "variant or clustered or fast_rung or full_config or pruning" 2>&1 | tail -5
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>gpurun_out/fast_err.log > gpurun_out/bench_C2_fast.json
cat gpurun_out/bench_C2_fast.json | python -c "import json,sys; d=json.load(sys.stdin); print(d['ms_per_step'], d['window'], d['roofline']['screen_rung'], d['roofline']['frac'], d['clocks'])"
EBC200_TC_FAST=0 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>>gpurun_out/fast_err.log > gpurun_out/bench_C2_nofast.json
cat gpurun_out/bench_C2_nofast.json | python -c "import json,sys; d=json.load(sys.stdin); print(d['ms_per_step'], d['window'], d['roofline']['screen_rung'], d['roofline']['frac'], d['clocks'])"
tail -5 gpurun_out/fast_err.log
