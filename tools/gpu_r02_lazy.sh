# Lazy Greedy check on one B200: gpu tests, bench lines with lazy on and off.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
for c in ${CONFIGS:-C2 C4}; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>gpurun_out/bench_err_$c.log | tee gpurun_out/bench_$c.json
  tail -3 gpurun_out/bench_err_$c.log
  if [ -n "$OFF" ]; then
    EBC200_LAZY=0 timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null > gpurun_out/bench_${c}_nolazy.json
  fi
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/bench_C*.json")):
    try:
        j = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, j["ms_per_step"], j["selected_head"], j.get("summary_value"), j["roofline"]["frac"], j.get("window"))
    except Exception as e:
        print(f, "ERR", e)
PY
