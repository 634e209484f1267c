# round 2, GPU run BB: 12 scan warps for the 2-4 threshold fused instances -- GPU suite, nt2/nt3/nt4 bench lines
set -x
O=gpurun_out/r2bb
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 1800 > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
timeout 300 $B --thetas 0.2,0.4,0.5,0.7 > $O/bench_nt4.json 2> $O/bench_nt4.err
timeout 300 $B --thetas 0.4,0.5,0.7 > $O/bench_nt3.json 2> $O/bench_nt3.err
timeout 300 $B --thetas 0.5,0.7 > $O/bench_nt2.json 2> $O/bench_nt2.err
timeout 300 $B --thetas 0.2,0.4,0.5,0.7 --family g2 > $O/bench_nt4_g2.json 2> $O/bench_nt4_g2.err
timeout 300 $B > $O/bench.json 2> $O/bench.err
