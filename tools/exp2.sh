#!/bin/bash
for sw in 8 16; do
  FVSR_SOFT_WARPS=$sw python bench.py --steps 200 --warmup 10 --no-cpu --e2e-steps 1 > gpurun_out/sw_$sw.json 2> gpurun_out/sw_$sw.err
  python -c "
import json
d=json.load(open('gpurun_out/sw_$sw.json')); print('softwarps=$sw attn_us=%.1f tflops=%.1f step_ms=%.3f' % (d['roofline']['avg_launch_us'], d['roofline']['achieved'], d['ms_per_step']))"
done
FVSR_SOFT_WARPS=16 FVSR_ATTN_TRACE=1 python bench.py --steps 30 --warmup 10 --no-cpu --e2e-steps 1 > /dev/null 2> gpurun_out/trace16.txt; sed -n 38,44p gpurun_out/trace16.txt
