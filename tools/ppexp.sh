# ring_pack kernel time for experiment variants (ncu launch list); args: variant names (prod = product)
for v in "$@"; do
  if [ "$v" = prod ]; then lib=""; else lib=variants/libfvsr_b200_$v.so; fi
  FVSR_LIB=$lib ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:ring_pack -c 40 --csv --log-file gpurun_out/lp_$v.csv python bench.py --steps 10 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
done
