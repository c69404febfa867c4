set -x
EBC200_LIB_PATH=$PWD/paper_2105_12026_b200/libebc200_fadd2.so timeout 900 python -m pytest tests -m gpu -q -x -k "every_screen or clustered or full_config or pruning" 2>&1 | tail -2
for L in libebc200.so libebc200_fadd2.so; do
  echo "== $L"
  for C in C4 C3 C2; do
  EBC200_LIB_PATH=$PWD/paper_2105_12026_b200/$L timeout 600 python bench.py --config $C --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$C', d['ms_per_step'], d['roofline']['tmem_read']['frac'], d['clocks']['sm_mhz'])"
  done
done
