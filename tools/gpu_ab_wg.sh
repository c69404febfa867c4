set -x
timeout 600 python -m pytest tests -m gpu -q -x -k "every_screen or clustered or full_config" 2>&1 | tail -2
EBC200_LIB_PATH=$PWD/paper_2105_12026_b200/libebc200_wg4.so timeout 600 python -m pytest tests -m gpu -q -x -k "every_screen or clustered or full_config" 2>&1 | tail -2
for L in libebc200.so libebc200_wg4.so; do
  echo "== $L"
  EBC200_LIB_PATH=$PWD/paper_2105_12026_b200/$L timeout 300 python tools/quick_time.py 2>&1 | grep -v untimed
  EBC200_LIB_PATH=$PWD/paper_2105_12026_b200/$L timeout 600 python bench.py --config C4 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('C4 bench', d['ms_per_step'], d['roofline']['tmem_read']['frac'])"
done
