run() { echo "$1 $2: $(NSW_LIB_PATH=paper_2406_10262_b200/$1 $2 python bench.py --config cfg1 --steps 200 --warmup 5 --no-e2e --no-cpu-baseline | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["roofline"]["frac"],4), d["config"]["tile"])')"; }
for r in 1 2; do
run libnswrank_b200.so ""
run libnswrank_b200.so "env NSW_MAIN_TILE=4,128,3"
run libnswrank_b200_kany.so "env NSW_MAIN_TILE=4,128,3"
run libnswrank_b200_kany.so ""
done
