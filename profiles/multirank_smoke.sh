# Functional check of bench.py under torchrun with 2 ranks on ONE GPU (gloo for the host
# collectives; both ranks on cuda:0).  Not a measurement: two ranks share one device.
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
export SSM_BENCH_BACKEND=gloo
timeout 600 $T --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --variants 0 --cpu-baseline 0 --particles $((1<<22)) > gpurun_out/mr_sharded.log 2>&1
echo "sharded rc=$?"; grep '^{' gpurun_out/mr_sharded.log | cut -c1-300
timeout 900 $T --master-port 29513 bench.py --gpus 2 --steps 3 --warmup 3 --workload smc2 --smc-theta 256 > gpurun_out/mr_smc2.log 2>&1
echo "smc2 rc=$?"; grep '^{' gpurun_out/mr_smc2.log | cut -c1-300; grep -n "Error\|error\|Traceback" gpurun_out/mr_smc2.log | head -20
