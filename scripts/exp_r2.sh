python scripts/phase_timing.py
timeout 120 python bench.py --steps 100 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(round(d['value'],1), round(r.get('fused_ms_per_launch'),4), d['config']['tile'], round(r.get('frac'),4))"
python -m pytest tests -q -m gpu -x 2>&1 | tail -3
