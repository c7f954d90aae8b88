#!/bin/bash
# round-end measurement set: bench line, launch list, attention ncu capture, configs sweep
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
tail -c 400 gpurun_out/bench_final.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:sparse_attn --launch-skip 5 -c 1 -f \
  -o gpurun_out/attn_final python bench.py --steps 10 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
python tools/configs.py --out gpurun_out/configs_final.json > gpurun_out/configs_final.log 2>&1
echo done
