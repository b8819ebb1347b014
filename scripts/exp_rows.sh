# 16-warp row tiles vs the default 8-warp tiles on configs 2 / 3 (NSW_MAIN_TILE=R,NT)
run() {
  timeout 900 python bench.py --no-cpu-baseline --no-e2e $1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(round(d['value'],3), round(d['ms_per_step'],3), round(r.get('frac'),4), d['config']['tile'])"
}
echo "cfg2 default $(run '--config cfg2 --steps 10 --warmup 3')"
echo "cfg2 2,512 $(NSW_MAIN_TILE=2,512 run '--config cfg2 --steps 10 --warmup 3')"
echo "cfg3 default $(run '--config cfg3 --steps 5 --warmup 3')"
echo "cfg3 4,512 $(NSW_MAIN_TILE=4,512 run '--config cfg3 --steps 5 --warmup 3')"
