# round 2, GPU run AC: ring in L2 -- evict-first S* (now default) + ring stores evict-last / discard after reduce
set -x
O=gpurun_out/r2ac
mkdir -p $O
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
for v in base el disc eldisc; do
  L=""; [ $v != base ] && L="CM_LIB=tune/$v.so"
  env $L timeout 200 $B > $O/bench_$v.json 2> $O/bench_$v.err
  env $L timeout 200 $B --config unet > $O/bench_unet_$v.json 2> $O/bench_unet_$v.err
  env $L timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fused -s 3 -c 1 --csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --overlap off > $O/ncu_dram_$v.csv 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k blk > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
