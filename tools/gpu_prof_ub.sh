# ncu of the fused cached-min update + first lazy batch (k_update_batch) on C2:
# launch list of the per-step kernels over one run, then one --set full capture
# of a mid-run launch (source-correlated: build with -lineinfo).
mkdir -p gpurun_out
c=${CONFIG:-C2}
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_active.avg,sm__cycles_elapsed.avg \
  --clock-control none -k regex:'k_update_batch|k_lazy_topk|k_batch_pack' --csv \
  python tools/profile_run.py $c > gpurun_out/ub_list_$c.csv 2>gpurun_out/ub_list_$c.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_update_batch -s ${SKIP:-20} -c 1 \
  -o gpurun_out/ub_full_$c -f python tools/profile_run.py $c > gpurun_out/ub_full_$c.log 2>&1
tail -1 gpurun_out/ub_full_$c.log
