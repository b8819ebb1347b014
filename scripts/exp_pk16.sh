run() {
  timeout 900 python bench.py --no-cpu-baseline --no-e2e $1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(round(d['value'],3), round(d['ms_per_step'],3), round(r.get('frac'),4), d['config']['tile'])"
}
L=paper_2406_10262_b200/libnswrank_b200_pkall.so
echo "cfg1 default $(run '--steps 300')"
echo "cfg1 16,32 $(NSW_MAIN_TILE=16,32 run '--steps 300')"
echo "cfg1 16,32 pkall $(NSW_LIB_PATH=$L NSW_MAIN_TILE=16,32 run '--steps 300')"
echo "cfg1 8,64,7 pkall $(NSW_LIB_PATH=$L NSW_MAIN_TILE=8,64,7 run '--steps 300')"
echo "cfg3 pkall $(NSW_LIB_PATH=$L run '--config cfg3 --steps 5 --warmup 3')"
