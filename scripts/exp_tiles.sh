for args in "--inner 100" "--inner 10" "--inner 2" "--users 888" "--users 148" "--users 296" "--variant 1" "--variant 2"; do
  echo "== $args"; timeout 120 python bench.py --steps 50 --no-cpu-baseline --no-e2e $args 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(d['value'], d['ms_per_step'], r.get('fused_ms_per_launch'), d['config']['tile'], r.get('frac'))"
done
