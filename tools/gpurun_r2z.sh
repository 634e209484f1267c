# round 2, GPU run Z: two CTAs per SM forced (ncu: register and shared limits allow 2); 4 K1 stages
set -x
O=gpurun_out/r2z
mkdir -p $O
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
CM_DEBUG=1 CM_FUSED_PER_SM=2 CM_LIB=tune/c2.so timeout 200 $B > $O/bench_c2x2.json 2> $O/bench_c2x2.err
CM_FUSED_PER_SM=2 CM_LIB=tune/c2.so timeout 200 $B --config unet > $O/bench_unet_c2x2.json 2> $O/bench_unet_c2x2.err
CM_FUSED_PER_SM=2 CM_LIB=tune/c2.so timeout 200 $B --family g2 > $O/bench_g2_c2x2.json 2> $O/bench_g2_c2x2.err
CM_FUSED_PER_SM=2 CM_LIB=tune/c2.so timeout 300 python tools/cta_timeline.py > $O/timeline_c2x2.txt 2>&1
CM_DEBUG=1 CM_LIB=tune/st4.so timeout 200 $B > $O/bench_st4.json 2> $O/bench_st4.err
CM_LIB=tune/st4.so timeout 200 $B --config unet > $O/bench_unet_st4.json 2> $O/bench_unet_st4.err
CM_LIB=tune/st4.so timeout 200 $B --config mobilenet > $O/bench_mobilenet_st4.json 2> $O/bench_mobilenet_st4.err
timeout 200 $B > $O/bench_base.json 2> $O/bench_base.err
CM_FUSED_PER_SM=2 CM_LIB=tune/c2.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_overlap.py -q -x --timeout 600 -k "blk or overlap" > $O/tests_c2x2.log 2>&1; echo "rc=$?" >> $O/tests_c2x2.log
