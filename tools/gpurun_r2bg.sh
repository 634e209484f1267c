# round 2, GPU run BG: final profile set of the round-2 build (after the per-S* Philox tables) -- GPU suite, smoke, default bench line
# (cpu_baseline, e2e), reference arm, per-config / family / rounding lines, launch list, ncu full of
# the headline fused kernel, memcheck + racecheck of the changed paths (randomized, multimem wiring)
set -x
O=gpurun_out/r2bg
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
for c in vgg16 unet mobilenet fcn8; do timeout 300 $B --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
for f in g2 mix; do timeout 300 $B --family $f > $O/bench_resnet50_$f.json 2> $O/bench_resnet50_$f.err; done
timeout 300 $B --thetas 0.2,0.4,0.5,0.7 > $O/bench_nt4.json 2> $O/bench_nt4.err
timeout 300 $B --thetas 0.5,0.7 > $O/bench_nt2.json 2> $O/bench_nt2.err
for k in 1 2 4; do timeout 300 $B --samples $k > $O/bench_rand$k.json 2> $O/bench_rand$k.err; done
timeout 300 $B --layout dense > $O/bench_resnet50_dense.json 2> $O/bench_resnet50_dense.err
timeout 300 $B --max-batch > $O/bench_resnet50_maxbatch.json 2> $O/bench_resnet50_maxbatch.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 3 -c 1 -o $O/fused_blk python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --overlap off > $O/ncu_blk.log 2>&1
