mkdir -p gpurun_out
for C in C3 C2; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_screen_tc -s 2 -c 1 -o gpurun_out/screen_tc_$C python tools/profile_run.py $C 4 > gpurun_out/ncu_$C.log 2>&1
tail -1 gpurun_out/ncu_$C.log
done
