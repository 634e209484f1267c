# round 2, GPU run V: sanitizers after the barrier / workspace fixes
set -x
O=gpurun_out/r2v
mkdir -p $O
export CM_UNDER_SANITIZER=1
timeout 900 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_overlap.py -q -k init_keys_all_paths > $O/san_synccheck.log 2>&1; echo "rc=$?" >> $O/san_synccheck.log
timeout 900 compute-sanitizer --tool initcheck python -m pytest tests/test_gpu_overlap.py tests/test_gpu_parity.py -q -k "init_keys_all_paths or paper_shaped" > $O/san_initcheck.log 2>&1; echo "rc=$?" >> $O/san_initcheck.log
timeout 900 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_overlap.py -q -k init_keys_all_paths > $O/san_racecheck.log 2>&1; echo "rc=$?" >> $O/san_racecheck.log
timeout 1800 compute-sanitizer --tool memcheck python -m pytest tests -m gpu -q -x --timeout 1500 -k "not full_launch" > $O/san_memcheck.log 2>&1; echo "rc=$?" >> $O/san_memcheck.log
