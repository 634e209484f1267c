# round 2, GPU run AK: rounding vs scan time for randomized rounding (two-kernel pipeline, one chunk);
# VGG16 with 12 rounding warps; ncu of the VGG16 fused kernel
set -x
O=gpurun_out/r2ak
mkdir -p $O
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
for k in 1 4; do
  CM_FUSED=0 CM_WS_MB=16384 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/split_rand$k.csv $B --samples $k --overlap off > $O/split_rand$k.log 2>&1
done
CM_FUSED=0 CM_WS_MB=16384 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/split_det.csv $B --overlap off > $O/split_det.log 2>&1
CM_FUSED=0 CM_WS_MB=16384 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/split_vgg.csv $B --config vgg16 --overlap off > $O/split_vgg.log 2>&1
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
for v in base k1w12; do
  L=""; [ $v != base ] && L="CM_LIB=tune/$v.so"
  env $L timeout 200 $B --config vgg16 > $O/vgg_$v.json 2> $O/vgg_$v.err
  env $L timeout 200 $B --config unet > $O/unet_$v.json 2> $O/unet_$v.err
  env $L timeout 200 $B > $O/res_$v.json 2> $O/res_$v.err
  env $L timeout 200 $B --samples 1 > $O/r1_$v.json 2> $O/r1_$v.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 3 -c 1 -o $O/vgg python bench.py --steps 1 --warmup 3 --config vgg16 --no-e2e --no-cpu-baseline --overlap off > $O/ncu_vgg.log 2>&1
