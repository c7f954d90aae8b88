#!/bin/bash
# ncu --set full (with source) of the attention kernel for each source variant dir
C=paper_2510_12747_b200/csrc
mkdir -p /tmp/ab_orig && cp $C/*.cu $C/*.cuh /tmp/ab_orig/
for v in "$@"; do
  cp /tmp/ab_orig/* $C/ && cp $v/* $C/
  python -c "import paper_2510_12747_b200.build as b; b.build(force=True)" > /dev/null 2>&1 || { echo "$v build failed"; continue; }
  python bench.py --steps 5 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1 || { echo "$v bench failed"; continue; }
  n=$(basename $v)
  ncu --set full --import-source on --clock-control none -k regex:sparse_attn --launch-skip 5 -c 1 -f -o gpurun_out/ncu_$n python bench.py --steps 5 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_$n.log 2>&1
  echo "$v done"
done
cp /tmp/ab_orig/* $C/
