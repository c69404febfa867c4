mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c4.csv python tools/profile_run.py C4 20 > /dev/null 2>&1; wc -l gpurun_out/launches_c4.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_screen_tc -s 8 -c 1 -o gpurun_out/screen_tc_C4 python tools/profile_run.py C4 10 > gpurun_out/ncu_C4.log 2>&1; tail -1 gpurun_out/ncu_C4.log
