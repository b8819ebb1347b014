for U in 444 500 592 700; do
  timeout 300 python bench.py --users $U --steps 100 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('U=$U', round(d['value'],1), d['config']['tile'])"
  NSW_MAIN_TILE=8,64 timeout 300 python bench.py --users $U --steps 100 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('U=$U 8,64', round(d['value'],1), d['config']['tile'])"
done
