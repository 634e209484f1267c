# round 2, GPU run K: lean K1 + leaner event rounds / walk bookkeeping; register rebalance (CTA pool balanced)
set -x
O=gpurun_out/r2k
mkdir -p $O
B="python bench.py --layout blk --steps 10 --no-cpu-baseline --no-e2e"
for c in resnet50 unet vgg16 mobilenet fcn8; do timeout 300 $B --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
for f in g2 mix; do timeout 300 $B --family $f > $O/bench_resnet50_$f.json 2> $O/bench_resnet50_$f.err; done
for v in rb12 rb12r80; do for c in resnet50 unet; do CM_LIB=tune/$v.so timeout 120 $B --config $c > $O/bench_${c}_$v.json 2> $O/bench_${c}_$v.err; done; done
CM_LIB=tune/rb12.so timeout 120 $B --family g2 > $O/bench_resnet50_g2_rb12.json 2> $O/bench_resnet50_g2_rb12.err
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_randomized.py tests/test_gpu_overlap.py -q -x --timeout 600 > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
