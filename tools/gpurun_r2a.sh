# round 2, GPU run A: new diagonal loads, int peak, bench lines, N=2 on one GPU, tests, ncu
set -x
O=gpurun_out/r2a
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $O/nvsmi.txt
timeout 300 python tools/int_peak.py --json $O/int_peak.json > $O/int_peak.log 2>&1
timeout 600 python bench.py > $O/bench_resnet50.json 2> $O/bench_resnet50.err
for c in vgg16 unet mobilenet fcn8; do timeout 300 python bench.py --config $c --steps 5 --no-cpu-baseline --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 300 python bench.py --layout tri4 --steps 5 --no-cpu-baseline --no-e2e > $O/bench_tri4.json 2> $O/bench_tri4.err
CM_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --batch 62500 --steps 5 --no-e2e --no-cpu-baseline > $O/bench_n2_one_gpu.json 2> $O/bench_n2_one_gpu.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 3 -c 1 -o $O/fused python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --overlap off > $O/ncu_full.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 2400 python -m pytest tests/test_gpu_scale.py tests/test_gpu_overlap.py -q -x --timeout 1800 > $O/tests_new.log 2>&1; echo "rc=$?" >> $O/tests_new.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 --deselect tests/test_gpu_scale.py --deselect tests/test_gpu_overlap.py > $O/tests_rest.log 2>&1; echo "rc=$?" >> $O/tests_rest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
