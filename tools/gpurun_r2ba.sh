# round 2, GPU run BA: 12 scan warps (K1 2 stages, setmaxnreg 72 / 112) on the scan-heavy deterministic workloads
set -x
O=gpurun_out/r2ba
mkdir -p $O
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
for v in base s12 s12r4; do
  L=""; [ $v != base ] && L="CM_LIB=tune/$v.so"
  env $L timeout 200 $B --config vgg16 > $O/vgg_$v.json 2> $O/vgg_$v.err
  env $L timeout 200 $B --family g2 > $O/g2_$v.json 2> $O/g2_$v.err
  env $L timeout 200 $B --family mix > $O/mix_$v.json 2> $O/mix_$v.err
  env $L timeout 200 $B --thetas 0.2,0.4,0.5,0.7 > $O/nt4_$v.json 2> $O/nt4_$v.err
  env $L timeout 200 $B > $O/res_$v.json 2> $O/res_$v.err
done
