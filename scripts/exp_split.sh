# config 1: split step (backward / forward launches; NSW_SPLIT=1) vs fused
run() {
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 300 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(round(d['value'],2), round(d['ms_per_step']*1e3,2), 'us; fused', round(r['fused_ms_per_launch']*1e3,2), 'launches', d['gpu_launches'])"
}
for rep in 1 2; do echo "fused  $(run)"; echo "split7 $(NSW_SPLIT=1 run)"; echo "split6 $(NSW_SPLIT=2 run)"; done
