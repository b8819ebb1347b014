# Source-level ncu capture of one fused-step tile (by mangled-name regex) for a library build:
# ncu_src_tile.sh TAG LIB REGEX [bench args...]
TAG=$1; LIB=$2; RX=$3; shift 3
NSW_LIB_PATH=$LIB ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:$RX -s 3 -c 1 \
  -o gpurun_out/${TAG} python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/${TAG}.log 2>&1
echo "$TAG rc=$?"
