for args in "--config cfg1" "--config cfg1 --users 888 --inner 2" "--config cfg2 --steps 20" "--config cfg3 --steps 10 --users 5000"; do
  echo "== $args"; timeout 300 python bench.py --steps 30 --no-cpu-baseline --no-e2e $args 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(round(d['value'],2), round(r.get('fused_ms_per_launch'),4), d['config']['tile'], round(r.get('frac'),4), d['config']['workload'])"
done
