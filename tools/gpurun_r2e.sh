# round 2, GPU run E: chunk-major blk blocks, single-LOP3 transpose, relaxed polling
set -x
O=gpurun_out/r2e
mkdir -p $O
for lay in blk dense; do timeout 300 python bench.py --layout $lay --steps 10 --no-cpu-baseline --no-e2e > $O/bench_resnet50_$lay.json 2> $O/bench_resnet50_$lay.err; done
for c in vgg16 unet mobilenet fcn8; do for lay in blk dense; do timeout 300 python bench.py --config $c --layout $lay --steps 10 --no-cpu-baseline --no-e2e > $O/bench_${c}_$lay.json 2> $O/bench_${c}_$lay.err; done; done
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_randomized.py tests/test_gpu_overlap.py -q -x --timeout 600 > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 3 -c 1 -o $O/fused_blk python bench.py --layout blk --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --overlap off > $O/ncu_full.log 2>&1
