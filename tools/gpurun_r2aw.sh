# round 2, GPU run AW: borrow polarity of sub.cc / addc in the integer randomized compare
set -x
O=gpurun_out/r2aw
mkdir -p $O
for v in cmp1 cmp1inv; do
CM_LIB=tune/$v.so timeout 900 python -m pytest tests/test_gpu_randomized.py -q -x --timeout 600 > $O/tests_$v.log 2>&1; echo "rc=$?" >> $O/tests_$v.log
done
