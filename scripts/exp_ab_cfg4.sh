# A/B on the config-4 per-GPU shard: current build vs libnswrank_b200_$1.so
run() {
  timeout 600 python bench.py --config cfg4 --slice 0:12500 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(round(d['value'],3), round(d['ms_per_step'],2), d['config']['tile'], round(r.get('frac'),4))"
}
for rep in 1 2; do
  echo "default $(run)"
  echo "$1 $(NSW_LIB_PATH=paper_2406_10262_b200/libnswrank_b200_$1.so run)"
done
