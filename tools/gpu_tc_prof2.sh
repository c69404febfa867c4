mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_screen_tc -s 2 -c 1 -o gpurun_out/screen_tc2_c2 python tools/profile_run.py C2 4 > gpurun_out/ncu_tc2.log 2>&1
tail -1 gpurun_out/ncu_tc2.log
