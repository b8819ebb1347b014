# Session re-entry check on the GPU box: GPU suite + smoke, default bench line,
# and one source-level ncu capture of the config-2 main tile (one wave of users).
TAG=${1:-r02c}
bash scripts/gpu_tests.sh $TAG
python bench.py > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"; cat gpurun_out/${TAG}_bench.jsonl
ncu --set full --import-source on --clock-control none -k regex:step_kernel -s 2 -c 1 -o gpurun_out/${TAG}_src \
    python bench.py --slice 0:148 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_src.log 2>&1; echo "ncu rc=$?"
