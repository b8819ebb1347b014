for args in "--inner 100" "--users 148 --inner 2" "--users 148 --inner 100" "--users 148 --inner 200" "--users 888 --inner 100" "--users 888 --inner 2"; do
  echo "== $args"; timeout 120 python bench.py --steps 30 --no-cpu-baseline --no-e2e $args 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(round(d['value'],1), round(r.get('fused_ms_per_launch'),4), d['config']['tile'], round(r.get('frac'),4))"
done
