# round 2, GPU run F (re-entry): state of HEAD -- full GPU suite, bench per config and layout, ncu of blk and dense
set -x
O=gpurun_out/r2f
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
for lay in blk dense tri4; do timeout 300 python bench.py --layout $lay --steps 10 --no-cpu-baseline --no-e2e > $O/bench_resnet50_$lay.json 2> $O/bench_resnet50_$lay.err; done
for c in vgg16 unet mobilenet fcn8; do for lay in blk dense; do timeout 300 python bench.py --config $c --layout $lay --steps 10 --no-cpu-baseline --no-e2e > $O/bench_${c}_$lay.json 2> $O/bench_${c}_$lay.err; done; done
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for lay in blk dense; do timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 3 -c 1 -o $O/fused_$lay python bench.py --layout $lay --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --overlap off > $O/ncu_$lay.log 2>&1; done
