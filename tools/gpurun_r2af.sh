# round 2, GPU run AF: verification of the current build -- full GPU suite, default bench line, per-config lines
set -x
O=gpurun_out/r2af
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
for c in vgg16 unet mobilenet fcn8; do timeout 300 $B --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
for f in g2 mix; do timeout 300 $B --family $f > $O/bench_resnet50_$f.json 2> $O/bench_resnet50_$f.err; done
timeout 300 $B --thetas 0.2,0.4,0.5,0.7 > $O/bench_nt4.json 2> $O/bench_nt4.err
timeout 300 $B --samples 1 > $O/bench_rand1.json 2> $O/bench_rand1.err
timeout 300 $B --samples 4 > $O/bench_rand4.json 2> $O/bench_rand4.err
timeout 300 $B --layout dense > $O/bench_resnet50_dense.json 2> $O/bench_resnet50_dense.err
timeout 300 $B --max-batch > $O/bench_resnet50_maxbatch.json 2> $O/bench_resnet50_maxbatch.err
