#!/bin/bash
# A/B of compile-time variants: each arg is "VAR=val,VAR=val"; bench twice per variant
for v in "$@"; do
  env $(echo $v | tr ',' ' ') python -c "import paper_2510_12747_b200.build as b; b.build(force=True)" > /dev/null 2>&1
  for r in ${RUNS:-1 2}; do
    t=$(python bench.py --steps 300 --warmup 20 --e2e-steps 5 --no-cpu 2>/dev/null | grep -o '"avg_launch_us": [0-9.]*' | cut -d' ' -f2)
    echo "$v run$r attn_us=$t"
  done
done
