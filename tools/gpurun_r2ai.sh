# round 2, GPU run AI: warp split for randomized rounding (rounding warps + scan warps per CTA)
set -x
O=gpurun_out/r2ai
mkdir -p $O
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
for v in base k12s4 k8s4 k10s6; do
  L=""; [ $v != base ] && L="CM_LIB=tune/$v.so"
  env $L timeout 200 $B --samples 1 > $O/r1_$v.json 2> $O/r1_$v.err
  env $L timeout 200 $B --samples 4 > $O/r4_$v.json 2> $O/r4_$v.err
  env $L timeout 200 $B > $O/det_$v.json 2> $O/det_$v.err
done
