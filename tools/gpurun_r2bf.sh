# round 2, GPU run BF: the per-S* Philox table compiled into the fused blocked randomized instances only
set -x
O=gpurun_out/r2bf
mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_randomized.py tests/test_gpu_overlap.py tests/test_gpu_scale.py -q -x --timeout 1200 -k "andomized or overlap" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
for k in 1 2 4; do timeout 300 $B --samples $k > $O/r${k}.json 2> $O/r${k}.err; done
timeout 300 $B > $O/bench.json 2> $O/bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 3 -c 1 -o $O/rand1 python bench.py --steps 1 --warmup 3 --samples 1 --batch 40000 --no-e2e --no-cpu-baseline --overlap off > $O/ncu_rand1.log 2>&1
