# round 2, GPU run R: ncu of the current build -- ResNet-50 blk (theta 0.5) and N_theta = 4 (scan-bound)
set -x
O=gpurun_out/r2r
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 3 -c 1 -o $O/fused_blk python bench.py --layout blk --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --overlap off > $O/ncu_blk.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 3 -c 1 -o $O/fused_nt4 python bench.py --layout blk --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --overlap off --thetas 0.2,0.4,0.5,0.7 > $O/ncu_nt4.log 2>&1
