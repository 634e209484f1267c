# round 2, GPU run H: scan-alone rate (pipeline without K1), K1 priority, HBM read ceiling, ncu of K1 alone
set -x
O=gpurun_out/r2h
mkdir -p $O
B="python bench.py --layout blk --steps 10 --no-cpu-baseline --no-e2e"
timeout 300 python tools/bw_probe.py --json $O/bw_probe.json > $O/bw_probe.log 2>&1
CM_FUSED=0 timeout 300 $B > $O/bench_pipeline.json 2> $O/bench_pipeline.err
CM_LIB=tune/nok1.so CM_FUSED=0 timeout 300 $B > $O/bench_pipeline_nok1.json 2> $O/bench_pipeline_nok1.err
CM_LIB=tune/k1high.so timeout 300 $B > $O/bench_k1high.json 2> $O/bench_k1high.err
timeout 300 $B --family g2 > $O/bench_g2.json 2> $O/bench_g2.err
timeout 300 $B --family mix > $O/bench_mix.json 2> $O/bench_mix.err
CM_LIB=tune/noscan.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 3 -c 1 -o $O/fused_noscan python bench.py --layout blk --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --overlap off > $O/ncu_noscan.log 2>&1
