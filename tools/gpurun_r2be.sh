# round 2, GPU run BE: per-S* Philox tables (rounds 0-2 per (node block, q4, sample), lane-parallel) -- parity + A/B
set -x
O=gpurun_out/r2be
mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_randomized.py tests/test_gpu_overlap.py tests/test_gpu_scale.py -q -x --timeout 1200 -k "andomized or overlap" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
for t in 1 0; do
  for k in 1 2 4; do CM_RAND_TAB=$t timeout 300 $B --samples $k > $O/r${k}_tab$t.json 2> $O/r${k}_tab$t.err; done
done
