T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
export SSM_BENCH_BACKEND=gloo
timeout 900 $T --master-port 29993 bench.py --gpus 2 --steps 3 --warmup 3 --workload smc2 --smc-theta 256 > gpurun_out/mr_smc2.log 2>&1
echo "bench smc2 rc=$?"; grep '^{' gpurun_out/mr_smc2.log | cut -c1-250; grep -m3 "Error" gpurun_out/mr_smc2.log | cut -c1-200
timeout 900 $T --master-port 29994 bench.py --gpus 2 --steps 3 --warmup 3 --workload smc2 > gpurun_out/mr_smc2_1024.log 2>&1
echo "bench smc2 1024 rc=$?"; grep '^{' gpurun_out/mr_smc2_1024.log | cut -c1-250; grep -m3 "Error" gpurun_out/mr_smc2_1024.log | cut -c1-200
