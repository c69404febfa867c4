set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_screen_tc -s 2 -c 1 -o gpurun_out/screen_tc_c2 python tools/profile_run.py C2 4 > gpurun_out/ncu_tc.log 2>&1
tail -2 gpurun_out/ncu_tc.log
timeout 600 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/tc_check.py > gpurun_out/sanitizer_racecheck_tc.log 2>&1; echo racecheck rc=$?
tail -2 gpurun_out/sanitizer_racecheck_tc.log
