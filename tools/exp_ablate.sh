#!/bin/bash
# bottleneck ablations of the attention kernel: rebuild with -DFVSR_ATTN_EXP=m, time the bench
for m in ${@:-0 1 2 4 7}; do
  FVSR_ATTN_EXP=$m python -c "import paper_2510_12747_b200.build as b; b.build(force=True)" > /dev/null 2>&1
  python bench.py --steps 200 --warmup 10 --no-cpu --e2e-steps 1 > gpurun_out/abl_$m.json 2> gpurun_out/abl_$m.err
  python -c "
import json
try:
  d=json.load(open('gpurun_out/abl_$m.json')); print('exp=$m attn_us=%.1f' % d['roofline']['avg_launch_us'])
except Exception as e: print('exp=$m failed'); print(open('gpurun_out/abl_$m.err').read()[-600:])
"
done
