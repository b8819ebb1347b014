# Same-box A/B of library builds on configs 2 / 1 / 3: ab3.sh "LIB..." [rounds]
LIBS=$1; R=${2:-2}
run() { NSW_LIB_PATH=$1 python bench.py --config $2 $3 --no-e2e --no-cpu-baseline | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],2), round(d["roofline"]["frac"],4))'; }
for r in $(seq $R); do
  for lib in $LIBS; do
    echo "$(basename $lib) cfg2: $(run $lib cfg2 '--steps 10 --warmup 3')"
    echo "$(basename $lib) cfg1: $(run $lib cfg1 '--steps 200 --warmup 5')"
    echo "$(basename $lib) cfg3: $(run $lib cfg3 '--users 2960 --steps 5 --warmup 3')"
  done
done
