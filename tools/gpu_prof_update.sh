# ncu of the cached-min update (K4): launch list over a short run + one --set full capture per config
mkdir -p gpurun_out
for c in ${CONFIGS:-C2 C4}; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:k_update --csv python tools/profile_run.py $c 6 > gpurun_out/upd_list_$c.csv 2>gpurun_out/upd_list_$c.err
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_update_fused -s ${SKIP:-3} -c 1 \
    -o gpurun_out/upd_full_$c -f python tools/profile_run.py $c ${KSTEPS:-6} > gpurun_out/upd_full_$c.log 2>&1
  tail -1 gpurun_out/upd_full_$c.log
done
