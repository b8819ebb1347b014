# config-1 per-GPU shards (strong scaling over users, 1 GPU measured)
run() {
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 300 $1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step']*1e3,1), 'us', d['config']['tile'])"
}
for s in 0:1000 0:500 0:250 0:125; do echo "cfg1 $s $(run "--slice $s")"; done
