# Main-tile experiment on config 1: default vs 7-per-SM tiles (NSW_MAIN_TILE=R,NT[,MINB]).
for t in "" "8,64,7" "16,32,7" "8,64,6"; do
  echo "== NSW_MAIN_TILE=$t"
  NSW_MAIN_TILE=$t timeout 120 python bench.py --steps 200 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(d['value'], d['ms_per_step'], r.get('fused_ms_per_launch'), d['config']['tile'], r.get('frac'))"
done
