# Same-box A/B of the tensor-core adjoint (NSW_TC=1) against the FFMA sweep
# on the config-2 tile: parity tests first, then bench lines and phase timing
# (timing-only diagnostics builds libnswrank_b200_tcx{1,2,3}.so: no staging
# stores / no MMAs / neither).
TAG=${1:-tc}
timeout 600 python -m pytest tests/test_gpu_tiles.py -q -k "tensor_core" -s > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "float32 and -2" -s >> gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest -2 rc=$?"
grep -E "tc-|ragged-tc" gpurun_out/${TAG}_pytest.log
run() { timeout 300 python bench.py --config cfg2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],2), round(d["roofline"]["frac"],4))'; }
for r in 1 2; do
  echo "ffma cfg2: $(NSW_TC=0 run)"
  echo "tc   cfg2: $(NSW_TC=1 run)"
done
pt() { timeout 300 python scripts/phase_timing.py --config cfg2 --users 1184 2>&1 | grep -E "backward levels|forward iter|total per CTA|Adam"; }
echo "-- ffma"; NSW_TC=0 pt
echo "-- tc"; NSW_TC=1 pt
for x in 4 8 16 12; do echo "-- tcx$x"; NSW_TC=1 NSW_LIB_PATH=$PWD/paper_2406_10262_b200/libnswrank_b200_tcx$x.so pt; done
