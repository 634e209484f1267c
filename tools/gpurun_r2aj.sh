# round 2, GPU run AJ: Philox blocks in flight per rounding warp (CM_RAND_ILP 2 / 4 (default) / 8)
set -x
O=gpurun_out/r2aj
mkdir -p $O
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
for v in base ilp2 ilp8; do
  L=""; [ $v != base ] && L="CM_LIB=tune/$v.so"
  for k in 1 2 4; do env $L timeout 200 $B --samples $k > $O/r${k}_$v.json 2> $O/r${k}_$v.err; done
done
timeout 900 python -m pytest tests/test_gpu_randomized.py tests/test_gpu_overlap.py -q -x --timeout 600 > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
