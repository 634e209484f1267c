# round 2, GPU run S: Sn ring in shared memory (cp.async, 7 quads ahead), masses read at the task end
set -x
O=gpurun_out/r2s
mkdir -p $O
B="python bench.py --layout blk --steps 10 --no-cpu-baseline --no-e2e"
for c in resnet50 vgg16 unet mobilenet fcn8; do CM_DEBUG=1 timeout 300 $B --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 300 $B --family g2 > $O/bench_resnet50_g2.json 2> $O/bench_resnet50_g2.err
timeout 300 $B --thetas 0.2,0.4,0.5,0.7 > $O/bench_nt4.json 2> $O/bench_nt4.err
for v in snr0 snr4 snr16; do
  CM_LIB=tune/$v.so timeout 120 $B > $O/bench_resnet50_$v.json 2> $O/bench_resnet50_$v.err
  CM_LIB=tune/$v.so timeout 120 $B --thetas 0.2,0.4,0.5,0.7 > $O/bench_nt4_$v.json 2> $O/bench_nt4_$v.err
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_randomized.py tests/test_gpu_overlap.py -q -x --timeout 600 > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
