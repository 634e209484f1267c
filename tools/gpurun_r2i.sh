# round 2, GPU run I: lean blocked-layout K1 body -- GPU suite, bench per config (blk)
set -x
O=gpurun_out/r2i
mkdir -p $O
B="python bench.py --layout blk --steps 10 --no-cpu-baseline --no-e2e"
timeout 300 $B > $O/bench_resnet50.json 2> $O/bench_resnet50.err
CM_LIB=tune/noscan.so timeout 300 $B > $O/bench_resnet50_noscan_old.json 2> $O/bench_resnet50_noscan_old.err
for c in vgg16 unet mobilenet fcn8; do timeout 300 $B --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 300 $B --samples 1 > $O/bench_rand1.json 2> $O/bench_rand1.err
timeout 300 $B --samples 4 > $O/bench_rand4.json 2> $O/bench_rand4.err
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
