# round 2, GPU run AH: randomized rounding with the 32-bit uniform (R1 re-read): GPU suite, rand bench lines, pipe probes
set -x
O=gpurun_out/r2ah
mkdir -p $O
timeout 300 python tools/int_peak.py --pipes --json $O/int_peak_pipes.json > $O/int_peak.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
for k in 1 2 4; do timeout 300 $B --samples $k > $O/bench_rand$k.json 2> $O/bench_rand$k.err; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 3 -c 1 -o $O/rand1 python bench.py --steps 1 --warmup 3 --samples 1 --batch 40000 --no-e2e --no-cpu-baseline --overlap off > $O/ncu_rand1.log 2>&1
