# round 2, GPU run M: two CTAs per SM (4 + 4 warps, 256 TMEM columns each) for finer call overlap
set -x
O=gpurun_out/r2m
mkdir -p $O
B="python bench.py --layout blk --steps 10 --no-cpu-baseline --no-e2e"
timeout 300 $B > $O/bench_resnet50_base.json 2> $O/bench_resnet50_base.err
for v in c2 c2m nsm; do
  CM_LIB=tune/$v.so timeout 120 $B > $O/bench_resnet50_$v.json 2> $O/bench_resnet50_$v.err
  CM_LIB=tune/$v.so timeout 120 $B --family g2 > $O/bench_resnet50_g2_$v.json 2> $O/bench_resnet50_g2_$v.err
  CM_LIB=tune/$v.so timeout 120 $B --config unet > $O/bench_unet_$v.json 2> $O/bench_unet_$v.err
done
CM_LIB=tune/c2.so timeout 300 python tools/cta_timeline.py --layout blk > $O/timeline_c2.txt 2>&1
CM_LIB=tune/c2.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_overlap.py -q -x --timeout 600 -k "blk or overlap" > $O/tests_c2.log 2>&1; echo "rc=$?" >> $O/tests_c2.log
