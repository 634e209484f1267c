# round 2, GPU run T: Sn ring (int32 state) -- every config, families, N_theta = 4, randomized, full GPU suite
set -x
O=gpurun_out/r2t
mkdir -p $O
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
for c in resnet50 vgg16 unet mobilenet fcn8; do CM_DEBUG=1 timeout 300 $B --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 300 $B --layout dense > $O/bench_resnet50_dense.json 2> $O/bench_resnet50_dense.err
timeout 300 $B --layout tri4 > $O/bench_resnet50_tri4.json 2> $O/bench_resnet50_tri4.err
for f in g2 mix; do timeout 300 $B --family $f > $O/bench_resnet50_$f.json 2> $O/bench_resnet50_$f.err; done
timeout 300 $B --thetas 0.2,0.4,0.5,0.7 > $O/bench_nt4.json 2> $O/bench_nt4.err
timeout 300 $B --samples 1 > $O/bench_rand1.json 2> $O/bench_rand1.err
timeout 300 $B --samples 4 > $O/bench_rand4.json 2> $O/bench_rand4.err
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
