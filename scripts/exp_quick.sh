# quick config-1/2 numbers of the current build (+ optional NSW_MAIN_TILE variants as args)
run() {
  timeout 900 python bench.py --no-cpu-baseline --no-e2e $1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(round(d['value'],3), round(d['ms_per_step'],4), round(r.get('frac'),4), d['config']['workload'][:5], d['config'].get('tile'))"
}
echo "cfg1 $(run '--config cfg1 --steps 300')"
for t in "$@"; do echo "cfg1 tile=$t $(NSW_MAIN_TILE=$t run '--config cfg1 --steps 300')"; done
echo "cfg2 $(run '--config cfg2 --steps 10 --warmup 3')"
