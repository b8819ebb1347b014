# A/B of row-tile shapes on configs 2 and 3 (experiment build libnswrank_b200_exp.so)
L=paper_2406_10262_b200/libnswrank_b200_exp.so
for t in "4,256,1" "3,384,1" "4,288,1" "5,224,1"; do
  echo "cfg2 tile $t: $(NSW_LIB_PATH=$L NSW_MAIN_TILE=$t python bench.py --config cfg2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],2), d["config"]["tile"], d["roofline"]["frac"])')"
done
for t in "8,256,1" "6,352,1" "7,288,1" "5,416,1"; do
  echo "cfg3 tile $t: $(NSW_LIB_PATH=$L NSW_MAIN_TILE=$t python bench.py --config cfg3 --users 2960 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],2), d["config"]["tile"], d["roofline"]["frac"])')"
done
