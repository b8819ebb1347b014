# config-1 tail tile register budgets: (2,256) at MINB 1 (138 regs) / 2 / 3
run() {
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 300 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(round(d['value'],2), round(d['ms_per_step']*1e3,2), 'us', d['config']['tile'])"
}
for rep in 1 2; do for t in 2,256,1 2,256,2 2,256,3; do echo "tail $t $(NSW_TAIL_TILE=$t run)"; done; done
