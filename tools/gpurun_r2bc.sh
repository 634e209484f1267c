# round 2, GPU run BC: randomized rounding with 2-4 samples on 12 scan warps (K1 at 88 / 80 registers)
set -x
O=gpurun_out/r2bc
mkdir -p $O
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
for v in base r12 r12k80; do
  L=""; [ $v != base ] && L="CM_LIB=tune/$v.so"
  for k in 2 4; do env $L timeout 200 $B --samples $k > $O/r${k}_$v.json 2> $O/r${k}_$v.err; done
done
CM_LIB=tune/r12.so timeout 900 python -m pytest tests/test_gpu_randomized.py tests/test_gpu_overlap.py -q -x --timeout 600 > $O/tests_r12.log 2>&1; echo "rc=$?" >> $O/tests_r12.log
