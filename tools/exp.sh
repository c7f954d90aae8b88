#!/bin/bash
# attention-kernel experiments: FVSR_ATTN_DEBUG=0 normal, 1 no softmax math, 2 no K/V loads, 3 both
for m in 0 1 2 3; do
  FVSR_ATTN_DEBUG=$m python bench.py --steps 200 --warmup 10 --no-cpu --e2e-steps 1 > gpurun_out/exp_$m.json 2> gpurun_out/exp_$m.err
  python -c "
import json,sys
try:
  d=json.load(open('gpurun_out/exp_$m.json')); print('debug=$m attn_us=%.1f mb_us=%.1f step_ms=%.3f' % (d['roofline']['avg_launch_us'], d['mask_builder']['avg_us'], d['ms_per_step']))
except Exception as e: print('debug=$m failed'); print(open('gpurun_out/exp_$m.err').read()[-1500:])
"
done
