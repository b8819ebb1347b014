set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
python -m pytest tests -m gpu -q -x -rs --durations=15 > gpurun_out/r02a_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/r02a_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a_smoke.log 2>&1; echo "smoke rc=$?"; cat gpurun_out/r02a_smoke.log | tail -5
python bench.py > gpurun_out/r02a_bench.jsonl 2> gpurun_out/r02a_bench.err; echo "bench rc=$?"; cat gpurun_out/r02a_bench.jsonl; tail -3 gpurun_out/r02a_bench.err
python bench.py --impl reference > gpurun_out/r02a_bench_ref.jsonl 2>&1; echo "ref rc=$?"; cat gpurun_out/r02a_bench_ref.jsonl | tail -2
