for v in 0 1 2 3; do
  echo "== variant $v"; timeout 300 python bench.py --steps 30 --no-cpu-baseline --no-e2e --variant $v "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(round(d['value'],2), round(r.get('fused_ms_per_launch'),4), d['config']['tile'], round(r.get('frac'),4))"
done
