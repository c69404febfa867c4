set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --durations=8 2>&1 | tail -14
timeout 600 compute-sanitizer --tool racecheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_racecheck.log 2>&1; echo racecheck rc=$?
grep -c Hazard gpurun_out/sanitizer_racecheck.log; tail -3 gpurun_out/sanitizer_racecheck.log
python tools/quick_time.py 2>&1 | grep -v untimed
