# round 2, GPU run J: lean K1 with one block body; K1-alone rate; register rebalance (12 rounding warps)
set -x
O=gpurun_out/r2j
mkdir -p $O
B="python bench.py --layout blk --steps 10 --no-cpu-baseline --no-e2e"
for c in resnet50 unet vgg16; do timeout 300 $B --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
CM_LIB=tune/noscan2.so timeout 300 $B > $O/bench_resnet50_noscan2.json 2> $O/bench_resnet50_noscan2.err
for v in rb12 rb12r72; do for c in resnet50 unet vgg16 mobilenet; do CM_LIB=tune/$v.so timeout 300 $B --config $c > $O/bench_${c}_$v.json 2> $O/bench_${c}_$v.err; done; done
CM_LIB=tune/rb12.so timeout 300 $B --family g2 > $O/bench_resnet50_g2_rb12.json 2> $O/bench_resnet50_g2_rb12.err
CM_LIB=tune/rb12.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "blk" > $O/tests_rb12.log 2>&1; echo "rc=$?" >> $O/tests_rb12.log
