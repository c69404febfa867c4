# Bench line summary per config (no CPU baseline): CONFIGS="C2 C3 C4" bash tools/gpu_cfgs.sh
mkdir -p gpurun_out
for C in ${CONFIGS:-C2 C3 C4}; do
  timeout 900 python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline 2>gpurun_out/cfg_err_$C.log > gpurun_out/cfg_$C.json
  python - "$C" <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/cfg_{c}.json"))
except Exception as e:
    print(c, "FAILED", e); sys.exit()
r = d.get("roofline", {})
print(c, "ms/step %.2f" % d["ms_per_step"], "e2e %.2f" % d["e2e"]["ms_per_step"], "win", d.get("window"), "rung", r.get("screen_rung"),
      "frac %.3f" % r.get("frac", 0), "screen %.2f" % r.get("screen_ms_per_step", 0), "clk", d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"),
      "sel", d["selected_head"])
PY
  tail -2 gpurun_out/cfg_err_$C.log
done
