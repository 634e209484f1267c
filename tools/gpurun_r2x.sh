# round 2, GPU run X: timeline and ncu full of the current build (sources unchanged during the call); synccheck diagnostic
set -x
O=gpurun_out/r2x
mkdir -p $O
timeout 300 python tools/cta_timeline.py --layout blk > $O/timeline_resnet50.txt 2>&1
CM_LIB=tune/noscan.so timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-e2e > $O/bench_noscan.json 2> $O/bench_noscan.err
CM_LIB=tune/noscan.so timeout 300 python tools/cta_timeline.py --layout blk > $O/timeline_resnet50_noscan.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 3 -c 1 -o $O/fused_blk python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --overlap off > $O/ncu_blk.log 2>&1
export CM_UNDER_SANITIZER=1
CM_LIB=tune/scanpad.so timeout 900 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_overlap.py -q -k "init_keys_all_paths and pipeline" > $O/san_synccheck_scanpad.log 2>&1; echo "rc=$?" >> $O/san_synccheck_scanpad.log
