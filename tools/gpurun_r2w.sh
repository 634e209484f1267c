# round 2, GPU run W: producer slot-wait back-off (8 us cap vs 1 us); synccheck of the pipeline without TMEM
set -x
O=gpurun_out/r2w
mkdir -p $O
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
for v in main sw1k; do
  L=""; [ $v != main ] && L="CM_LIB=tune/$v.so"
  env $L timeout 200 $B > $O/bench_resnet50_$v.json 2> $O/bench_resnet50_$v.err
  env $L timeout 200 $B --thetas 0.2,0.4,0.5,0.7 > $O/bench_nt4_$v.json 2> $O/bench_nt4_$v.err
  env $L timeout 200 $B --family g2 > $O/bench_g2_$v.json 2> $O/bench_g2_$v.err
  env $L timeout 200 $B --samples 1 > $O/bench_rand1_$v.json 2> $O/bench_rand1_$v.err
  env $L timeout 200 $B --samples 4 > $O/bench_rand4_$v.json 2> $O/bench_rand4_$v.err
done
export CM_UNDER_SANITIZER=1
CM_TMEM=0 timeout 900 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_overlap.py -q -k init_keys_all_paths > $O/san_synccheck_notmem.log 2>&1; echo "rc=$?" >> $O/san_synccheck_notmem.log
timeout 900 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_overlap.py -q -k "init_keys_all_paths and v1" > $O/san_synccheck_v1.log 2>&1; echo "rc=$?" >> $O/san_synccheck_v1.log
