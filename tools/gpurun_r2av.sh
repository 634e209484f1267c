# round 2, GPU run AV: randomized compare as an integer borrow (CM_RAND_CMP=1) vs the fp32 sign
set -x
O=gpurun_out/r2av
mkdir -p $O
CM_LIB=tune/cmp1.so timeout 1200 python -m pytest tests/test_gpu_randomized.py tests/test_gpu_overlap.py -q -x --timeout 600 > $O/tests_cmp1.log 2>&1; echo "rc=$?" >> $O/tests_cmp1.log
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
for v in base cmp1; do
  L=""; [ $v != base ] && L="CM_LIB=tune/$v.so"
  for k in 1 2 4; do env $L timeout 200 $B --samples $k > $O/r${k}_$v.json 2> $O/r${k}_$v.err; done
done
