# round 2, GPU run AZ: per-config ncu --set full captures (DRAM traffic per S* of every bench config),
# N = 2 ranks on one GPU (gloo) vs one rank over the same S*, NVLS test (skip path)
set -x
O=gpurun_out/r2az
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_nvls.py -q -rs --timeout 300 > $O/nvls_tests.log 2>&1; echo "rc=$?" >> $O/nvls_tests.log
for c in vgg16 unet mobilenet fcn8; do
  timeout 900 ncu --set full --clock-control none -k regex:fused -s 3 -c 1 -o $O/fused_$c python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --overlap off > $O/ncu_$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none -k regex:fused -s 3 -c 1 -o $O/fused_resnet50_dense python bench.py --layout dense --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --overlap off > $O/ncu_dense.log 2>&1
CM_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --batch 62500 --steps 5 --no-e2e --no-cpu-baseline > $O/bench_n2_one_gpu.json 2> $O/bench_n2_one_gpu.err
timeout 300 python bench.py --batch 125000 --steps 5 --no-e2e --no-cpu-baseline > $O/bench_n1_same_total.json 2> $O/bench_n1_same_total.err
