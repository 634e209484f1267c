# round 2, GPU run Q: leaner randomized compare; all configs; N_theta = 4; VGG16 diagnostics; parity subset
set -x
O=gpurun_out/r2q
mkdir -p $O
B="python bench.py --layout blk --steps 10 --no-cpu-baseline --no-e2e"
for c in resnet50 vgg16 unet mobilenet fcn8; do timeout 300 $B --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 300 $B --samples 1 > $O/bench_rand1.json 2> $O/bench_rand1.err
timeout 300 $B --samples 4 > $O/bench_rand4.json 2> $O/bench_rand4.err
timeout 300 $B --thetas 0.2,0.4,0.5,0.7 > $O/bench_nt4.json 2> $O/bench_nt4.err
CM_LIB=tune/noscan.so timeout 300 $B --config vgg16 > $O/bench_vgg16_noscan.json 2> $O/bench_vgg16_noscan.err
CM_LIB=tune/noscan.so timeout 300 $B --config resnet50 > $O/bench_resnet50_noscan.json 2> $O/bench_resnet50_noscan.err
timeout 300 python tools/cta_timeline.py --config vgg16 --layout blk > $O/timeline_vgg16.txt 2>&1
timeout 300 python tools/cta_timeline.py --config resnet50 --layout blk > $O/timeline_resnet50.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_randomized.py tests/test_gpu_overlap.py -q -x --timeout 600 > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
