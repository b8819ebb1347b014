# impact-reduction user chunks (NSW_IMP_CHUNKS) on config 1: step time
run() {
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 400 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(round(d['value'],2), round(d['ms_per_step']*1e3,2), 'us/step; fused', round(r['fused_ms_per_launch']*1e3,2))"
}
echo "default(5) $(run)"
for c in 1 2 3 8 16 32; do echo "chunks $c $(NSW_IMP_CHUNKS=$c run)"; done
