for r in 1 2; do
for v in 0 1; do
  if [ $v = 1 ]; then export FVSR_NO_TAIL_SPLIT=1; else unset FVSR_NO_TAIL_SPLIT; fi
  t=$(python bench.py --steps 300 --warmup 20 --e2e-steps 5 --no-cpu 2>/dev/null | grep -o '"avg_launch_us": [0-9.]*' | cut -d' ' -f2)
  echo "nosplit=$v run$r attn_us=$t"
done; done
