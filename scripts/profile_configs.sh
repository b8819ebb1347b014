# Per-config ncu evidence: one --set full capture of the fused step
# kernel of configs 2, 3 (user slices: same tile, fewer waves) and the config-4
# cluster tile, plus raw pipe / DRAM / shared-memory metrics.  Run on the GPU box.
TAG=${1:-r01e}
M="gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__warps_active.avg.per_cycle_active,smsp__issue_active.avg.pct_of_peak_sustained_active"
for spec in "cfg2 --config cfg2 --slice 0:1184 --steps 2" "cfg3 --config cfg3 --slice 0:1184 --steps 2" "cfg4 --config cfg4 --slice 0:540 --steps 2" "cfg1 --config cfg1 --steps 2"; do
  set -- $spec
  name=$1; shift
  python bench.py "$@" --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1 || { echo "$name bench failed"; continue; }
  ncu --set full --import-source on --clock-control none -k regex:step_kernel -s 4 -c 1 -o gpurun_out/${TAG}_${name}_full \
      python bench.py "$@" --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_${name}_ncu.log 2>&1
  ncu -i gpurun_out/${TAG}_${name}_full.ncu-rep --page details > gpurun_out/${TAG}_ncu_${name}_details.txt 2>&1
  ncu -i gpurun_out/${TAG}_${name}_full.ncu-rep --page raw --csv --metrics $M > gpurun_out/${TAG}_ncu_${name}_raw.csv 2>&1
done
