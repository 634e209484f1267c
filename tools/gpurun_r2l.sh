# round 2, GPU run L: warp-role splits without the staged masses (12 rounding warps x 3 stages; 12 scan warps)
set -x
O=gpurun_out/r2l
mkdir -p $O
B="python bench.py --layout blk --steps 10 --no-cpu-baseline --no-e2e"
timeout 300 $B > $O/bench_resnet50_base.json 2> $O/bench_resnet50_base.err
for v in nsm k12s3 s12; do
  CM_LIB=tune/$v.so timeout 120 $B > $O/bench_resnet50_$v.json 2> $O/bench_resnet50_$v.err
  CM_LIB=tune/$v.so timeout 120 $B --family g2 > $O/bench_resnet50_g2_$v.json 2> $O/bench_resnet50_g2_$v.err
  CM_LIB=tune/$v.so timeout 120 $B --config unet > $O/bench_unet_$v.json 2> $O/bench_unet_$v.err
  CM_LIB=tune/$v.so timeout 120 $B --config mobilenet > $O/bench_mobilenet_$v.json 2> $O/bench_mobilenet_$v.err
done
