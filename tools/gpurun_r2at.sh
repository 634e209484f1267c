# round 2, GPU run AT: new scale tests (randomized rounding at the bench launch, forced 256-slot ring)
set -x
O=gpurun_out/r2at
mkdir -p $O
timeout 2400 python -m pytest tests/test_gpu_scale.py -q -k "randomized or 256" --timeout 1800 -rs > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
