# config-4 shard: u~ history (default) vs replay (NSW_UHIST=0), same build
run() {
  timeout 600 python bench.py --config cfg4 --slice 0:12500 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(round(d['value'],3), round(d['ms_per_step'],2), d['config']['tile'], round(r.get('frac'),4))"
}
for rep in 1 2; do
  echo "uhist  $(run)"
  echo "replay $(NSW_UHIST=0 run)"
done
