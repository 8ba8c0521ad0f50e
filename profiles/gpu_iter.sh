set -x
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python bench.py --steps 5 --warmup 3 --cpu-baseline 0 --e2e-steps 0 --variants 0 --exact > gpurun_out/b_exact.json 2>&1
python bench.py --steps 5 --warmup 3 --cpu-baseline 0 --e2e-steps 0 --variants 0 > gpurun_out/b_fast.json 2>&1
python bench.py --steps 5 --warmup 3 --dtype float32 --cpu-baseline 0 --e2e-steps 0 --variants 0 > gpurun_out/b_f32.json 2>&1
SKIP=${SKIP:-483} COUNT=${COUNT:-161} bash profiles/run_ncu_launches.sh
