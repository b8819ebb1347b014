# config-1 tail tile: wide (default 2,256) vs smaller tiles that fit beside running main CTAs
run() {
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 300 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(round(d['value'],3), round(d['ms_per_step'],4), d['config']['tile'])"
}
echo "default $(run)"
for t in 4,128 2,128 8,64 1,256; do echo "tail $t $(NSW_TAIL_TILE=$t run)"; done
