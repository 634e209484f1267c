# round 2, GPU run N: two CTAs per SM with 128-register launch bounds; randomized rounding rates
set -x
O=gpurun_out/r2n
mkdir -p $O
B="python bench.py --layout blk --steps 10 --no-cpu-baseline --no-e2e"
for v in c2 c2m; do
  CM_LIB=tune/$v.so timeout 120 $B > $O/bench_resnet50_$v.json 2> $O/bench_resnet50_$v.err
  CM_LIB=tune/$v.so timeout 120 $B --family g2 > $O/bench_resnet50_g2_$v.json 2> $O/bench_resnet50_g2_$v.err
  CM_LIB=tune/$v.so timeout 120 $B --config unet > $O/bench_unet_$v.json 2> $O/bench_unet_$v.err
done
CM_LIB=tune/c2.so timeout 300 python tools/cta_timeline.py --layout blk > $O/timeline_c2.txt 2>&1
timeout 300 $B --samples 1 > $O/bench_rand1.json 2> $O/bench_rand1.err
timeout 300 $B --samples 4 > $O/bench_rand4.json 2> $O/bench_rand4.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 3 -c 1 -o $O/fused_rand1 python bench.py --layout blk --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --overlap off --samples 1 > $O/ncu_rand1.log 2>&1
