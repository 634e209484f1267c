set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python tools/hbm_probe.py > gpurun_out/r2_hbm_probe.json 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 400 > gpurun_out/r2_base_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2_base_tests.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r2_base_bench.json 2> gpurun_out/r2_base_bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 3 -c 1 -o gpurun_out/r2_base python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --overlap off > gpurun_out/r2_base_ncu.log 2>&1
