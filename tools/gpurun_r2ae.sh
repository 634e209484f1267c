# round 2, GPU run AE: 12 scan warps (setmaxnreg: K1 72 / K2 112 registers), K1 2 stages, Sn ring of 4 quads
set -x
O=gpurun_out/r2ae
mkdir -p $O
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
CM_DEBUG=1 CM_LIB=tune/s12r4.so timeout 200 $B > $O/bench_s12r4.json 2> $O/bench_s12r4.err
CM_DEBUG=1 CM_LIB=tune/s12r4.so timeout 200 $B --config unet > $O/bench_unet_s12r4.json 2> $O/bench_unet_s12r4.err
CM_DEBUG=1 CM_LIB=tune/s12r4.so timeout 200 $B --family g2 > $O/bench_g2_s12r4.json 2> $O/bench_g2_s12r4.err
CM_DEBUG=1 CM_LIB=tune/s12r4.so timeout 200 $B --thetas 0.2,0.4,0.5,0.7 > $O/bench_nt4_s12r4.json 2> $O/bench_nt4_s12r4.err
CM_LIB=tune/s12r4.so timeout 300 python tools/cta_timeline.py > $O/timeline_s12r4.txt 2>&1
