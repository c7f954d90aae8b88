# mask_select kernel time for experiment variants (ncu launch list); args: variant names ('' = product)
for v in "$@"; do
  if [ "$v" = prod ]; then lib=""; else lib=variants/libfvsr_b200_$v.so; fi
  FVSR_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none -k regex:mask_select -c 40 --csv --log-file gpurun_out/lx_$v.csv python bench.py --steps 10 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
done
