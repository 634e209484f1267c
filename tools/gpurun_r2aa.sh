# round 2, GPU run AA: randomized rounding -- fp32 compare at one sample; 12 rounding warps (setmaxnreg 80/120)
set -x
O=gpurun_out/r2aa
mkdir -p $O
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
timeout 200 $B --samples 1 > $O/bench_rand1.json 2> $O/bench_rand1.err
timeout 200 $B --samples 4 > $O/bench_rand4.json 2> $O/bench_rand4.err
CM_LIB=tune/r12.so timeout 200 $B --samples 1 > $O/bench_rand1_r12.json 2> $O/bench_rand1_r12.err
CM_LIB=tune/r12.so timeout 200 $B > $O/bench_det_r12.json 2> $O/bench_det_r12.err
timeout 900 python -m pytest tests/test_gpu_randomized.py -q -x --timeout 600 > $O/tests_rand.log 2>&1; echo "rc=$?" >> $O/tests_rand.log
CM_LIB=tune/r12.so timeout 900 python -m pytest tests/test_gpu_randomized.py -q -x --timeout 600 > $O/tests_rand_r12.log 2>&1; echo "rc=$?" >> $O/tests_rand_r12.log
