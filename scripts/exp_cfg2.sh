for t in "4,256" "2,512" "4,128"; do
  NSW_MAIN_TILE=$t timeout 600 python bench.py --config cfg2 --users 2000 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tile $t', round(d['value'],2), d['config']['tile'], round(d['roofline']['frac'],3))"
done
