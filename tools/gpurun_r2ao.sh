# round 2, GPU run AO: ring depth by bytes (default ~300 MB of slots, 768..4096), per-config sweep; NVLS retry
set -x
O=gpurun_out/r2ao
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_nvls.py -q -x --timeout 300 > $O/nvls_tests.log 2>&1; echo "rc=$?" >> $O/nvls_tests.log
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
timeout 200 $B --keys nvls > $O/res_nvls.json 2> $O/res_nvls.err
for c in vgg16 unet mobilenet resnet50 fcn8; do
  CM_DEBUG=1 timeout 200 $B --config $c > $O/${c}_auto.json 2> $O/${c}_auto.err
done
for r in 1024 2048 4096; do CM_RING=$r timeout 200 $B --config unet > $O/unet_r$r.json 2> $O/unet_r$r.err; done
for r in 1024 1536; do CM_RING=$r timeout 200 $B --config mobilenet > $O/mobilenet_r$r.json 2> $O/mobilenet_r$r.err; done
CM_RING=1024 timeout 200 $B --config vgg16 > $O/vgg16_r1024.json 2> $O/vgg16_r1024.err
