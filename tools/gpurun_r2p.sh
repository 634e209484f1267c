set -x
O=gpurun_out/r2p
mkdir -p $O
CM_DEBUG=1 CM_LIB=tune/c2.so timeout 120 python bench.py --layout blk --steps 2 --no-cpu-baseline --no-e2e > $O/bench_c2.json 2> $O/bench_c2.err
nvidia-smi -q | grep -i -A3 "shared\|L1" > $O/smi.txt 2>&1
python -c "import torch; p=torch.cuda.get_device_properties(0); print(p)" > $O/props.txt 2>&1
