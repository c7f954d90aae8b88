# Round-end measurement on one B200: GPU tests, bench line (with CPU baseline), BASELINE configs,
# toy-DiT stack, launch list and ncu captures of the three hot kernels.  Outputs in gpurun_out/.
set -u
python -m pytest tests -m gpu -x -q > gpurun_out/final_tests.log 2>&1; tail -1 gpurun_out/final_tests.log
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
python tools/configs.py --out gpurun_out/final_configs.json > gpurun_out/final_configs.log 2>&1
python tools/dit_stream.py > gpurun_out/final_dit.json 2> gpurun_out/final_dit.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
bash tools/ncu_attn.sh final_ncu_attn sparse_attn > /dev/null
bash tools/ncu_attn.sh final_ncu_pack ring_pack > /dev/null
bash tools/ncu_attn.sh final_ncu_select mask_select > /dev/null
ls gpurun_out/final_*
