# Same-box A/B on config 1 only: ab_cfg1.sh LIB_A LIB_B [rounds]
A=$1; B=$2; R=${3:-3}
for r in $(seq $R); do for lib in $A $B; do
  echo "$(basename $lib) cfg1: $(NSW_LIB_PATH=$lib python bench.py --config cfg1 --steps 300 --warmup 5 --no-e2e --no-cpu-baseline | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],2), round(d["roofline"]["frac"],4))')"
done; done
