# round 2, GPU run AR: multimem epilogue wiring test; VGG16 timeline + ncu at the deeper ring
set -x
O=gpurun_out/r2ar
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_nvls.py -q -rs --timeout 300 > $O/nvls_tests.log 2>&1; echo "rc=$?" >> $O/nvls_tests.log
timeout 300 python tools/cta_timeline.py --config vgg16 > $O/timeline_vgg16.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 3 -c 1 -o $O/vgg python bench.py --steps 1 --warmup 3 --config vgg16 --no-e2e --no-cpu-baseline --overlap off > $O/ncu_vgg.log 2>&1
