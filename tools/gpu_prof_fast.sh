# ncu --set full of the fast-rung (FP16-rounded) tensor screen on C2 (one launch, step 2)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_screen_tc -s 2 -c 1 -o gpurun_out/screen_fast_C2 python tools/profile_run.py C2 4 > gpurun_out/ncu_fast_C2.log 2>&1
tail -2 gpurun_out/ncu_fast_C2.log
