# mask_select kernel time per FVSR_FRONT_QB variant (ncu launch list)
for q in "$@"; do
  if [ "$q" = 6 ]; then lib=""; else lib=variants/libfvsr_b200_qb$q.so; fi
  FVSR_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none -k regex:mask_select -c 40 --csv --log-file gpurun_out/lq$q.csv python bench.py --steps 10 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
done
