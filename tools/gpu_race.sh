timeout 600 compute-sanitizer --tool racecheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_racecheck.log 2>&1; echo racecheck rc=$?
tail -3 gpurun_out/sanitizer_racecheck.log
python tools/quick_time.py 2>&1 | grep -v untimed
