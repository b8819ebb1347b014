for tc in 1 0; do NSW_TAIL_CONCURRENT=$tc timeout 300 python bench.py --steps 200 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('concurrent', $tc, d['value'], d['e2e']['value'], d['roofline']['frac'])"; done
NSW_TAIL_CONCURRENT=1 python scripts/phase_timing.py | grep "launch\|total"
python -m pytest tests -q -m gpu -x 2>&1 | tail -2
