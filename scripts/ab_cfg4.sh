# Same-box A/B of library builds on the config-4 cluster tile: ab_cfg4.sh "LIB..." [rounds] [users]
LIBS=$1; R=${2:-2}; NU=${3:-1500}
for r in $(seq $R); do
  for lib in $LIBS; do
    echo "$(basename $lib) cfg4[0:$NU]: $(NSW_LIB_PATH=$lib python bench.py --config cfg4 --slice 0:$NU --steps 3 --warmup 3 --no-e2e --no-cpu-baseline | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],3), round(d["roofline"]["frac"],4))')"
  done
done
