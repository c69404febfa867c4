# Two ranks on the one GPU of a gpurun box (gloo exchange, host-driven sharded path):
# C1 and C4 bench lines; selections must equal the single-GPU runs.
mkdir -p gpurun_out
for C in C1 C4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
    bench.py --gpus 2 --config $C --steps 3 --warmup 3 > gpurun_out/torchrun2_$C.json 2> gpurun_out/torchrun2_err_$C.log
  echo "$C rc=$?"; tail -c 600 gpurun_out/torchrun2_$C.json; echo; tail -3 gpurun_out/torchrun2_err_$C.log
done
