# full-size configs 2 and 3 on one GPU, config-4 per-GPU shard (8-GPU layout)
for args in "--config cfg2 --steps 10 --warmup 3" "--config cfg3 --steps 5 --warmup 3" "--config cfg4 --steps 3 --warmup 3 --slice 0:12500"; do
  echo "== $args"; timeout 900 python bench.py --no-cpu-baseline --no-e2e $args 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(round(d['value'],3), d['ms_per_step'], d['config']['tile'], round(r.get('frac'),4), d['config']['workload'], d['clocks'])"
done
