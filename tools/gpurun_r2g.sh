# round 2, GPU run G: which role limits the fused kernel on the blocked layout
set -x
O=gpurun_out/r2g
mkdir -p $O
B="python bench.py --layout blk --steps 10 --no-cpu-baseline --no-e2e"
timeout 300 $B > $O/bench_base.json 2> $O/bench_base.err
for v in noscan nomass l2input st4 st2; do CM_LIB=tune/$v.so timeout 300 $B > $O/bench_$v.json 2> $O/bench_$v.err; done
CM_FUSED=0 timeout 300 $B > $O/bench_pipeline.json 2> $O/bench_pipeline.err
CM_RING=1536 timeout 300 $B > $O/bench_ring1536.json 2> $O/bench_ring1536.err
CM_RING=384 timeout 300 $B > $O/bench_ring384.json 2> $O/bench_ring384.err
timeout 300 python tools/cta_timeline.py --layout blk > $O/timeline_blk.txt 2>&1
CM_LIB=tune/noscan.so timeout 300 python tools/cta_timeline.py --layout blk > $O/timeline_blk_noscan.txt 2>&1
