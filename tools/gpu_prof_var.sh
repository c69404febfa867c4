# ncu --set full of one k_screen_tc launch of C2 for a compile-time variant: LIB=... TAG=... bash tools/gpu_prof_var.sh
mkdir -p gpurun_out
EBC200_LIB_PATH=$PWD/$LIB timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_screen_tc -s 2 -c 1 -o gpurun_out/screen_$TAG python tools/profile_run.py ${CFG:-C2} 4 > gpurun_out/ncu_$TAG.log 2>&1
tail -1 gpurun_out/ncu_$TAG.log
