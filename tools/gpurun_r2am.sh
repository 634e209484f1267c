# round 2, GPU run AM: NVLS multicast keys (a8 in the reduce step) at one device; GPU suite
set -x
O=gpurun_out/r2am
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_nvls.py -q -x --timeout 300 > $O/nvls_tests.log 2>&1; echo "rc=$?" >> $O/nvls_tests.log
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
