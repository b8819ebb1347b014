# A/B of two library builds (default vs libnswrank_b200_$1.so) on configs 1-3 (+ cfg4 shard if $2 == cfg4).
TAG=$1
run() {
  timeout 900 python bench.py --no-cpu-baseline --no-e2e $1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(round(d['value'],3), round(d['ms_per_step'],4), round(r.get('frac'),4), d['config']['workload'][:5])"
}
CFGS=("--config cfg1 --steps 300" "--config cfg2 --steps 10 --warmup 3" "--config cfg3 --steps 5 --warmup 3")
[ "$2" == "cfg4" ] && CFGS+=("--config cfg4 --steps 3 --warmup 3 --slice 0:12500")
for a in "${CFGS[@]}"; do
  for rep in 1 2; do
    echo "default  $(run "$a")"
    echo "$TAG $(NSW_LIB_PATH=paper_2406_10262_b200/libnswrank_b200_$TAG.so run "$a")"
  done
done
