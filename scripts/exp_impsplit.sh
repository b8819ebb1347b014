# config 1: main wave's impact terms reduced during the tail (default) vs after it (NSW_IMP_SPLIT=0)
run() {
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 400 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(round(d['value'],2), round(d['ms_per_step']*1e3,2), 'us/step; fused', round(r['fused_ms_per_launch']*1e3,2), 'launches', d['gpu_launches'])"
}
for rep in 1 2 3; do echo "split    $(run)"; echo "nosplit  $(NSW_IMP_SPLIT=0 run)"; done
