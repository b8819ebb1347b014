# A/B on configs 2 and 3 only: current build vs libnswrank_b200_$1.so
run() {
  timeout 900 python bench.py --no-cpu-baseline --no-e2e $1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(round(d['value'],3), round(d['ms_per_step'],4), round(r.get('frac'),4), d['config']['workload'][:5])"
}
for a in "--config cfg2 --steps 10 --warmup 3" "--config cfg3 --steps 5 --warmup 3"; do
  for rep in 1 2; do
    echo "default  $(run "$a")"
    echo "$1 $(NSW_LIB_PATH=paper_2406_10262_b200/libnswrank_b200_$1.so run "$a")"
  done
done
