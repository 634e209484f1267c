# round 2, GPU run Y: two CTAs per SM -- why occupancy 1? (ncu launch statistics of the variant), rates
set -x
O=gpurun_out/r2y
mkdir -p $O
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
for v in c2 c2s2; do
  CM_DEBUG=1 CM_LIB=tune/$v.so timeout 200 $B > $O/bench_$v.json 2> $O/bench_$v.err
  CM_LIB=tune/$v.so timeout 600 ncu --section LaunchStats --section Occupancy -k regex:fused -s 3 -c 1 --csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --overlap off > $O/ncu_occ_$v.csv 2>&1
done
