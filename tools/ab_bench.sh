# A/B of the bench step time: product library vs variants/libfvsr_b200_$1.so, alternating, $2 rounds
for i in $(seq 1 ${2:-2}); do
  python bench.py --no-cpu --e2e-steps 1 --steps 400 > gpurun_out/ab_prod_$i.json 2>/dev/null
  FVSR_LIB=variants/libfvsr_b200_$1.so python bench.py --no-cpu --e2e-steps 1 --steps 400 > gpurun_out/ab_$1_$i.json 2>/dev/null
done
python - "$1" "${2:-2}" <<'PY'
import json, sys
v, n = sys.argv[1], int(sys.argv[2])
for name in ("prod", v):
    xs = [json.load(open(f"gpurun_out/ab_{name}_{i}.json"))["ms_per_step"] * 1e3 for i in range(1, n + 1)]
    print(name, " ".join("%.2f" % x for x in xs))
PY
