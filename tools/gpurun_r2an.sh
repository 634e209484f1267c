# round 2, GPU run AN: NVLS multicast keys retry (POSIX-fd multicast object); VGG16 ring / stages experiments
set -x
O=gpurun_out/r2an
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_nvls.py -q -x --timeout 300 > $O/nvls_tests.log 2>&1; echo "rc=$?" >> $O/nvls_tests.log
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
timeout 200 $B --keys nvls > $O/res_nvls.json 2> $O/res_nvls.err
timeout 200 $B --config vgg16 > $O/vgg_base.json 2> $O/vgg_base.err
CM_RING=4096 timeout 200 $B --config vgg16 > $O/vgg_ring4k.json 2> $O/vgg_ring4k.err
CM_LIB=tune/st4.so timeout 200 $B --config vgg16 > $O/vgg_st4.json 2> $O/vgg_st4.err
CM_LIB=tune/st4.so timeout 200 $B --config unet > $O/unet_st4.json 2> $O/unet_st4.err
