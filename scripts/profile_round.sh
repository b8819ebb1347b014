# Round profile refresh (run on the GPU box): bench lines, launch list, full
# ncu capture of the fused step kernels.  Outputs under gpurun_out/$TAG_*.
TAG=${1:-r01b}
set -x
python bench.py > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_reference.jsonl 2> gpurun_out/${TAG}_ref.err
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:step_kernel -s 4 -c 2 -o gpurun_out/${TAG}_full \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_full.log 2>&1
