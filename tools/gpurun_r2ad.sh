# round 2, GPU run AD: 12 scan warps (K1 at 2 stages to fit) vs 2 stages alone, with the current build
set -x
O=gpurun_out/r2ad
mkdir -p $O
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
for v in s12 st2; do
  CM_DEBUG=1 CM_LIB=tune/$v.so timeout 200 $B > $O/bench_$v.json 2> $O/bench_$v.err
  CM_LIB=tune/$v.so timeout 200 $B --config unet > $O/bench_unet_$v.json 2> $O/bench_unet_$v.err
  CM_LIB=tune/$v.so timeout 200 $B --family g2 > $O/bench_g2_$v.json 2> $O/bench_g2_$v.err
  CM_LIB=tune/$v.so timeout 300 python tools/cta_timeline.py > $O/timeline_$v.txt 2>&1
done
