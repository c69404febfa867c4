mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c5.csv python tools/c5_profile.py > /dev/null 2>&1; wc -l gpurun_out/launches_c5.csv
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python tools/profile_run.py C2 5 > /dev/null 2>&1; wc -l gpurun_out/launches_c2.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_screen_tc -s 2 -c 1 -o gpurun_out/screen_tc_C2 python tools/profile_run.py C2 4 > gpurun_out/ncu_C2.log 2>&1; tail -1 gpurun_out/ncu_C2.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_screen_tc -s 8 -c 1 -o gpurun_out/screen_tc_C4 python tools/profile_run.py C4 10 > gpurun_out/ncu_C4.log 2>&1; tail -1 gpurun_out/ncu_C4.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_screen_tc -s 1 -c 1 -o gpurun_out/screen_tc_C5 python tools/c5_profile.py > gpurun_out/ncu_C5.log 2>&1; tail -1 gpurun_out/ncu_C5.log
