#!/bin/bash
# A/B of source variants: each arg is a directory holding replacement csrc files
# (e.g. variants/base); the bench runs twice per variant, interleaved order A B A B.
C=paper_2510_12747_b200/csrc
mkdir -p /tmp/ab_orig && cp $C/*.cu $C/*.cuh /tmp/ab_orig/
for r in 1 2; do
  for v in "$@"; do
    cp /tmp/ab_orig/* $C/ && cp $v/* $C/
    python -c "import paper_2510_12747_b200.build as b; b.build(force=True)" > /dev/null 2>&1 || { echo "$v build failed"; continue; }
    t=$(python bench.py --steps 300 --warmup 20 --e2e-steps 5 --no-cpu 2>/dev/null | grep -o '"avg_launch_us": [0-9.]*' | cut -d' ' -f2)
    echo "$v run$r attn_us=$t"
  done
done
cp /tmp/ab_orig/* $C/
