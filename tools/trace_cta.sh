#!/bin/bash
# per-CTA end-time distribution of the attention kernel (instrumented build), per variant env
for v in "$@"; do
  env $(echo $v | tr ',' ' ') FVSR_CTA_TIMELINE=1 python -c "import paper_2510_12747_b200.build as b; b.build(force=True)" > /dev/null 2>&1
  env $(echo $v | tr ',' ' ') FVSR_ATTN_TRACE=1 python bench.py --steps 30 --warmup 10 --no-cpu --e2e-steps 1 > /dev/null 2> gpurun_out/trace_cta.txt
  echo "== $v"; grep -A2 "cta timeline" gpurun_out/trace_cta.txt
done
