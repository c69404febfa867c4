set -x
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_screen -s 2 -c 1 -o gpurun_out/screen_gram_c2 python tools/profile_run.py C2 4 > gpurun_out/ncu_gram.log 2>&1
tail -2 gpurun_out/ncu_gram.log
