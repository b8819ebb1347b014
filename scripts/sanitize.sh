# compute-sanitizer memcheck / racecheck / synccheck over the GPU parity,
# cluster, operator and tolerance tests (small shapes; every kernel family:
# single-CTA step tiles incl. cp.async.bulk + mbarrier, cluster tiles with
# st.async DSMEM pushes, the operator seam, impact/finalize/tolerance kernels)
tag=${1:-r02}
SEL="tests/test_gpu_parity.py::test_fp64_small_shapes_vs_oracle tests/test_gpu_parity.py::test_fp32_small_shapes_close_to_oracle tests/test_gpu_cluster.py::test_cluster_fp64_vs_oracle tests/test_gpu_ops.py tests/test_gpu_tolerance.py tests/test_gpu_tiles.py::test_production_tile_one_step tests/test_gpu_tiles.py::test_cfg4_cluster_tile_one_step tests/test_gpu_two_shards.py"
for tool in memcheck racecheck synccheck; do
  t0=$(date +%s)
  timeout ${SAN_TIMEOUT:-900} compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 30 \
    --log-file gpurun_out/${tag}_sanitizer_${tool}.log python -m pytest -q -m gpu $SEL > gpurun_out/${tag}_sanitizer_${tool}.pytest.log 2>&1
  rc=$?
  echo "$tool rc=$rc seconds=$(( $(date +%s) - t0 ))" | tee -a gpurun_out/${tag}_sanitizer_summary.txt
  tail -3 gpurun_out/${tag}_sanitizer_${tool}.log | tee -a gpurun_out/${tag}_sanitizer_summary.txt
  tail -2 gpurun_out/${tag}_sanitizer_${tool}.pytest.log | tee -a gpurun_out/${tag}_sanitizer_summary.txt
done
