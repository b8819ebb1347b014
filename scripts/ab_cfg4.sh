# Same-box A/B on the config-4 shard (12.5k users): ab_cfg4.sh LIB_A LIB_B [rounds]
A=$1; B=$2; R=${3:-2}
for r in $(seq $R); do for lib in $A $B; do
  echo "$(basename $lib) cfg4: $(NSW_LIB_PATH=$lib python bench.py --config cfg4 --slice 0:12500 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],3), round(d["roofline"]["frac"],4))')"
done; done
