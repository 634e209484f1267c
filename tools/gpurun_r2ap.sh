# round 2, GPU run AP: NVLS multicast keys with the FABRIC handle type (team of one)
set -x
O=gpurun_out/r2ap
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_nvls.py -q -x --timeout 300 > $O/nvls_tests.log 2>&1; echo "rc=$?" >> $O/nvls_tests.log
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
timeout 200 $B --keys nvls > $O/res_nvls.json 2> $O/res_nvls.err
timeout 200 $B --keys nvls --max-batch > $O/res_nvls_mb.json 2> $O/res_nvls_mb.err
