# round 2, GPU run BH: VGG16 / U-Net tuning knobs at run time (S* per producer ticket, scan tasks per ticket)
set -x
O=gpurun_out/r2bh
mkdir -p $O
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
timeout 200 $B --config vgg16 > $O/vgg_base.json 2> $O/vgg_base.err
for c in 4 16 32; do CM_CLAIM=$c timeout 200 $B --config vgg16 > $O/vgg_claim$c.json 2> $O/vgg_claim$c.err; done
for t in 2 3; do CM_TASK_CLAIM=$t timeout 200 $B --config vgg16 > $O/vgg_task$t.json 2> $O/vgg_task$t.err; done
timeout 200 $B --config unet > $O/unet_base.json 2> $O/unet_base.err
for c in 2 4 8; do CM_CLAIM=$c timeout 200 $B --config unet > $O/unet_claim$c.json 2> $O/unet_claim$c.err; done
