# A/B of the fused update's slice rows (EBC200_UB_ROWS) with the phase trace
for r in 128 64; do for c in C2 C4; do
  echo "rows=$r $c"; EBC200_UB_ROWS=$r EBC200_LIB_PATH=paper_2105_12026_b200/libebc200_trace.so python tools/ub_trace.py $c 2>&1 | grep -v "^[0-9] "
  EBC200_UB_ROWS=$r timeout 600 python bench.py --config $c --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c rows $r', round(d['ms_per_step'],3), 'upd_us', round(d['update_roofline']['us_per_step'],2))"
done; done
