# A/B/C of the bench step time: product vs variants $1 $2, alternating, $3 rounds
n=${3:-3}
for i in $(seq 1 $n); do
  python bench.py --no-cpu --e2e-steps 1 --steps 400 > gpurun_out/ab_prod_$i.json 2>/dev/null
  for v in $1 $2; do FVSR_LIB=variants/libfvsr_b200_$v.so python bench.py --no-cpu --e2e-steps 1 --steps 400 > gpurun_out/ab_${v}_$i.json 2>/dev/null; done
done
python - $n prod $1 $2 <<'PY'
import json, sys
n = int(sys.argv[1])
for name in sys.argv[2:]:
    xs = [json.load(open(f"gpurun_out/ab_{name}_{i}.json")) for i in range(1, n + 1)]
    print(name, "step", " ".join("%.2f" % (x["ms_per_step"] * 1e3) for x in xs), "attn", " ".join("%.2f" % x["roofline"]["avg_launch_us"] for x in xs))
PY
