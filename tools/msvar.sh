# mask_select time, product vs variants, at the headline config and 1440p locality
for v in prod "$@"; do
  if [ "$v" = prod ]; then lib=""; else lib=variants/libfvsr_b200_$v.so; fi
  FVSR_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none -k regex:mask_select -c 12 --csv --log-file gpurun_out/mv_${v}_1440.csv python tools/point.py 90 160 41 loc 72 72 trunc > /dev/null 2>&1
  FVSR_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none -k regex:mask_select -c 12 --csv --log-file gpurun_out/mv_${v}_768.csv python tools/point.py 48 88 27 > /dev/null 2>&1
done
for v in prod "$@"; do for c in 768 1440; do echo "$v $c $(python tools/launches.py gpurun_out/mv_${v}_$c.csv --skip 4 | head -1)"; done; done
