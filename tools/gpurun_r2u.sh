# round 2, GPU run U: the profile set of the current build -- default bench line (cpu_baseline, e2e),
# reference arm, launch list, ncu full of the fused kernel, N = 2 ranks on one GPU (gloo), sanitizers
set -x
O=gpurun_out/r2u
mkdir -p $O
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 3 -c 1 -o $O/fused_blk python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --overlap off > $O/ncu_blk.log 2>&1
CM_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --batch 62500 --steps 5 --no-e2e --no-cpu-baseline > $O/bench_n2_one_gpu.json 2> $O/bench_n2_one_gpu.err
timeout 300 python bench.py --batch 125000 --steps 5 --no-e2e --no-cpu-baseline > $O/bench_n1_same_total.json 2> $O/bench_n1_same_total.err
timeout 1500 compute-sanitizer --tool memcheck python -m pytest tests -m gpu -q -x --timeout 1200 -k "not full_launch" > $O/san_memcheck.log 2>&1; echo "rc=$?" >> $O/san_memcheck.log
timeout 900 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_overlap.py -q -k init_keys_all_paths > $O/san_racecheck.log 2>&1; echo "rc=$?" >> $O/san_racecheck.log
timeout 900 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_overlap.py -q -k init_keys_all_paths > $O/san_synccheck.log 2>&1; echo "rc=$?" >> $O/san_synccheck.log
timeout 900 compute-sanitizer --tool initcheck python -m pytest tests/test_gpu_overlap.py tests/test_gpu_parity.py -q -k "init_keys_all_paths or paper_shaped" > $O/san_initcheck.log 2>&1; echo "rc=$?" >> $O/san_initcheck.log
