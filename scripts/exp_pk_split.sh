# config 1: packed FMAs per part (D: dots that must agree bitwise, B: backward, F: forward accumulation)
run() {
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 300 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(round(d['value'],2), round(d['ms_per_step']*1e3,2), 'us; fused', round(r['fused_ms_per_launch']*1e3,2))"
}
for rep in 1 2; do
  echo "all   $(run)"
  for t in nob nof nod; do echo "$t   $(NSW_LIB_PATH=paper_2406_10262_b200/libnswrank_b200_$t.so run)"; done
done
