mkdir -p gpurun_out
python -m pytest tests/test_gpu_generic_theta.py tests/test_gpu_theta_mh.py tests/test_gpu_generic.py -q -p no:cacheprovider -x > gpurun_out/gt.log 2>&1; tail -3 gpurun_out/gt.log
(cd _r1tree && python bench_outer.py --configs 3,5 > ../gpurun_out/ab_r1.jsonl 2> ../gpurun_out/ab_r1.err)
SSM_COOP_MAX=0 python bench_outer.py --configs 3,5 > gpurun_out/ab_nocoop.jsonl 2> gpurun_out/ab_nocoop.err
python bench_outer.py --configs 3,5 > gpurun_out/ab_head.jsonl 2> gpurun_out/ab_head.err
for f in ab_r1 ab_nocoop ab_head; do echo == $f; cut -c1-330 gpurun_out/$f.jsonl; tail -2 gpurun_out/$f.err; done
