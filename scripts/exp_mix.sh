# config 1: main two-warp tile and one-warp tile launched concurrently (NSW_MIX=U1,R,NT,MINB,NS)
run() {
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 300 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(round(d['value'],3), round(d['ms_per_step'],4), d['config']['tile'])"
}
echo "default $(run)"
for x in 444,16,32,7,1 592,16,32,7,1 296,16,32,7,1 148,16,32,7,1; do echo "mix $x $(NSW_MIX=$x run)"; done
