# Per-GPU shard throughput for the strong-scaling configs (one GPU runs the user block a
# rank of an N-GPU job owns): cfg2 / cfg3 at 2/4/8 GPUs, cfg4 at 4/8 GPUs.
run() {
  timeout 900 python bench.py --no-cpu-baseline --no-e2e $1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(round(d['value'],3), round(d['ms_per_step'],3), round(r.get('frac'),4), d['config']['workload'][:60], d['config'].get('tile'))"
}
for s in 0:1250 0:2500 0:5000; do echo "cfg2 $s $(run "--config cfg2 --slice $s --steps 10 --warmup 3")"; done
for s in 0:6250 0:12500 0:25000; do echo "cfg3 $s $(run "--config cfg3 --slice $s --steps 5 --warmup 3")"; done
echo "cfg4 0:25000 $(run '--config cfg4 --slice 0:25000 --steps 3 --warmup 3')"
