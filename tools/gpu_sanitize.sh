mkdir -p gpurun_out
for T in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $T --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/sanitizer_$T.log 2>&1; echo "$T rc=$?"; tail -2 gpurun_out/sanitizer_$T.log
done
timeout 600 ncu --set full --clock-control none -k regex:k_update -s 5 -c 1 -o gpurun_out/update_C4 python tools/profile_run.py C4 8 > /dev/null 2>&1; ls gpurun_out/update_C4*
