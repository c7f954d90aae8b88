#!/bin/bash
# ncu --set full (with source) of one attention launch of the bench step -> gpurun_out/$1.ncu-rep
n=${1:-ncu_attn}
k=${2:-sparse_attn}
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1 || { echo "bench failed"; exit 1; }
ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 8 -c 1 -f -o gpurun_out/$n \
  python bench.py --steps 5 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/$n.log 2>&1
echo "ncu exit $?"
