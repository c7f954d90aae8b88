#!/bin/bash
# round-end measurement set (session 3): GPU tests, smoke, bench line, launch list, configs sweep, f-row timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final_tests.log 2>&1; echo TESTS_EXIT $? >> gpurun_out/final_tests.log
tail -2 gpurun_out/final_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo SMOKE_EXIT $? >> gpurun_out/final_smoke.log
tail -2 gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
head -c 400 gpurun_out/bench_final.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
timeout 600 python tools/configs.py --out gpurun_out/configs_final.json > gpurun_out/configs_final.log 2>&1
timeout 300 python tools/f_rows.py --out gpurun_out/f_rows_final.json > gpurun_out/f_rows_final.log 2>&1
echo done
