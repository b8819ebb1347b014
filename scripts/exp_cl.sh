# Cluster-tile variants on the config-4 per-GPU shard (NSW_CL_TILE=M,R,NT,CL)
for t in "" "52,8,128,16" "56,8,256,16" "52,4,256,16" "52,8,256,16"; do
  echo "== NSW_CL_TILE=$t"
  NSW_CL_TILE=$t timeout 600 python bench.py --config cfg4 --slice 0:12500 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(round(d['value'],3), round(d['ms_per_step'],2), d['config']['tile'], round(r.get('frac'),4))"
done
