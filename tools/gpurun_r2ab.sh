# round 2, GPU run AB: S* bulk copies with an L2 evict-first policy (keep the ring in L2?)
set -x
O=gpurun_out/r2ab
mkdir -p $O
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
timeout 200 $B > $O/bench_base.json 2> $O/bench_base.err
CM_LIB=tune/ef.so timeout 200 $B > $O/bench_ef.json 2> $O/bench_ef.err
CM_LIB=tune/ef.so timeout 200 $B --config unet > $O/bench_unet_ef.json 2> $O/bench_unet_ef.err
CM_LIB=tune/ef.so timeout 200 $B --family g2 > $O/bench_g2_ef.json 2> $O/bench_g2_ef.err
for v in base ef; do
  L=""; [ $v != base ] && L="CM_LIB=tune/$v.so"
  env $L timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fused -s 3 -c 1 --csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --overlap off > $O/ncu_dram_$v.csv 2>&1
done
