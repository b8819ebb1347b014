run() {
  timeout 600 python bench.py --config cfg4 --slice 0:12500 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(round(d['value'],3), round(d['ms_per_step'],2), d['config']['tile'], round(r.get('frac'),4))"
}
echo "default $(run)"
echo "52,7,256,9 $(NSW_CL_TILE=52,7,256,9 run)"
echo "52,8,224,9 $(NSW_CL_TILE=52,8,224,9 run)"
