# round 2, GPU run AU: K1 software pipelining (block w's transpose / masses after block w+1's pack)
set -x
O=gpurun_out/r2au
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_randomized.py -q -x --timeout 600 > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
for v in base nopipe; do
  L=""; [ $v != base ] && L="CM_LIB=tune/$v.so"
  env $L timeout 200 $B > $O/res_$v.json 2> $O/res_$v.err
  env $L timeout 200 $B --config vgg16 > $O/vgg_$v.json 2> $O/vgg_$v.err
  env $L timeout 200 $B --config unet > $O/unet_$v.json 2> $O/unet_$v.err
  env $L timeout 200 $B --samples 1 > $O/r1_$v.json 2> $O/r1_$v.err
  env $L timeout 200 $B --family g2 > $O/g2_$v.json 2> $O/g2_$v.err
done
env timeout 200 $B > $O/res_base2.json 2> $O/res_base2.err
