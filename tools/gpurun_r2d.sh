# round 2, GPU run D: timing experiments (variants), timeline, fixed corner test
set -x
O=gpurun_out/r2d
mkdir -p $O
for v in noscan l2input st4 st2; do CM_LIB=tune/$v.so timeout 300 python bench.py --layout blk --steps 10 --no-cpu-baseline --no-e2e > $O/bench_$v.json 2> $O/bench_$v.err; done
CM_LIB=tune/l2input.so timeout 300 python bench.py --layout dense --steps 10 --no-cpu-baseline --no-e2e > $O/bench_l2input_dense.json 2> $O/bench_l2input_dense.err
timeout 300 python tools/cta_timeline.py --layout blk > $O/timeline_blk.txt 2>&1
timeout 300 python tools/cta_timeline.py --layout dense > $O/timeline_dense.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "ieee or edge" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
