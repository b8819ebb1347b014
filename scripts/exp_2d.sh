# 2-D lane-mapping tiles (cluster kernel, CL=1) vs the row tiles on configs 2 / 3 (NSW_CL_TILE=M,R,NT,CL)
run() {
  timeout 900 python bench.py --no-cpu-baseline --no-e2e $1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(round(d['value'],3), round(d['ms_per_step'],3), round(r.get('frac'),4), d['config']['tile'])"
}
echo "cfg2 default $(run '--config cfg2 --steps 10 --warmup 3')"
for t in 24,4,1024,1 22,4,512,1; do echo "cfg2 $t $(NSW_CL_TILE=$t run '--config cfg2 --steps 10 --warmup 3')"; done
echo "cfg3 default $(run '--config cfg3 --steps 5 --warmup 3')"
for t in 12,8,1024,1 12,8,512,1; do echo "cfg3 $t $(NSW_CL_TILE=$t run '--config cfg3 --steps 5 --warmup 3')"; done
