# Round profile refresh (run on the GPU box): bench lines (default config 2,
# the other configs, the reference arm), per-GPU shard lines, the launch list
# and one ncu --set full capture of the fused step kernels.  Outputs under
# gpurun_out/$TAG_*.
TAG=${1:-r02}
set -x
python bench.py > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err
python bench.py --impl reference > gpurun_out/${TAG}_bench_reference.jsonl 2> gpurun_out/${TAG}_ref.err
python bench.py --gpus 2 --steps 10 --no-cpu-baseline > gpurun_out/${TAG}_bench_gpus2.jsonl 2>> gpurun_out/${TAG}_bench.err
for c in cfg1 cfg3; do
  python bench.py --config $c --steps 20 --no-cpu-baseline --no-e2e >> gpurun_out/${TAG}_bench_configs.jsonl 2>> gpurun_out/${TAG}_bench.err
done
python bench.py --config cfg4 --slice 0:12500 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/${TAG}_bench_configs.jsonl 2>> gpurun_out/${TAG}_bench.err
for s in 0:1250 0:2500 0:5000; do   # the user block rank 0 of an 8 / 4 / 2-GPU config-2 job owns
  python bench.py --slice $s --steps 20 --no-cpu-baseline --no-e2e >> gpurun_out/${TAG}_bench_shards_cfg2.jsonl 2>> gpurun_out/${TAG}_bench.err
done
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:step_kernel -s 4 -c 2 -o gpurun_out/${TAG}_full \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_full.log 2>&1
