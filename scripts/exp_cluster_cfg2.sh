# A/B: config 2 on 2-CTA cluster tiles (two users per SM) vs the 1-CTA tile
L=paper_2406_10262_b200/libnswrank_b200_exp.so
run() { python bench.py --config cfg2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],2), d["config"]["tile"], round(d["roofline"]["frac"],4))'; }
echo "1-CTA tile: $(NSW_LIB_PATH=$L run)"
for t in "21,2,256,2" "22,4,256,2" "21,4,128,2"; do
  echo "cluster $t: $(NSW_LIB_PATH=$L NSW_CL_TILE=$t run)"
done
