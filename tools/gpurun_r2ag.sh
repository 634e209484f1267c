# round 2, GPU run AG: pipe probes (int_peak --pipes) and ncu full of the randomized-rounding fused kernel (1 and 4 samples)
set -x
O=gpurun_out/r2ag
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python tools/int_peak.py --pipes --json $O/int_peak_pipes.json > $O/int_peak.log 2>&1
B="python bench.py --steps 5 --no-cpu-baseline --no-e2e"
timeout 300 $B --samples 1 > $O/bench_rand1.json 2> $O/bench_rand1.err
timeout 300 $B --samples 4 > $O/bench_rand4.json 2> $O/bench_rand4.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 3 -c 1 -o $O/rand1 python bench.py --steps 1 --warmup 3 --samples 1 --batch 40000 --no-e2e --no-cpu-baseline --overlap off > $O/ncu_rand1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 3 -c 1 -o $O/rand4 python bench.py --steps 1 --warmup 3 --samples 4 --batch 10000 --no-e2e --no-cpu-baseline --overlap off > $O/ncu_rand4.log 2>&1
