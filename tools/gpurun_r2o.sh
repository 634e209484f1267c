# round 2, GPU run O: occupancy of the two-CTA variant; scan-alone and rounding-alone times (one-chunk pipeline)
set -x
O=gpurun_out/r2o
mkdir -p $O
B="python bench.py --layout blk --steps 5 --no-cpu-baseline --no-e2e"
CM_DEBUG=1 CM_LIB=tune/c2.so timeout 120 $B --steps 2 > $O/bench_c2.json 2> $O/bench_c2.err
CM_DEBUG=1 timeout 120 $B --steps 2 > $O/bench_base.json 2> $O/bench_base.err
for f in g1 g2 mix; do CM_FUSED=0 CM_WS_MB=6144 timeout 300 $B --family $f --overlap off > $O/bench_pipe1_$f.json 2> $O/bench_pipe1_$f.err; done
