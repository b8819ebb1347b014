# The GPU suite against the checked build (NSW_CHECKS=1: shared-memory bounds
# checks on every vector access, NaN-poisoned shared memory, mbarrier wait
# timeouts, canary guard bands around every solver buffer).  Stands in for
# compute-sanitizer, which is closed on the GPU pool.
#   build first (CPU):  python -m paper_2406_10262_b200.build --tag checked -D NSW_CHECKS=1
tag=${1:-r02}
NSW_LIB_PATH=paper_2406_10262_b200/libnswrank_b200_checked.so timeout ${CHECK_TIMEOUT:-1500} \
  python -m pytest tests -m gpu -q -rs > gpurun_out/${tag}_checked_pytest.log 2>&1
echo "checked-build GPU suite rc=$?"
tail -5 gpurun_out/${tag}_checked_pytest.log
grep -c "NSW_CHECKS" gpurun_out/${tag}_checked_pytest.log
# positive control: an out-of-bounds write 8 bytes past a solver buffer must be
# caught by the guard band when the buffer is freed
NSW_LIB_PATH=paper_2406_10262_b200/libnswrank_b200_checked.so python - > gpurun_out/${tag}_checked_control.log 2>&1 <<'PY'
import numpy as np, torch
from paper_2406_10262_b200 import DeviceSolver, DeviceOptions, SolverConfig
rel = np.full((3, 20), 0.5); expo = 1.0 / np.log2(np.arange(2, 6))
s = DeviceSolver(rel, expo, 20, 5, SolverConfig(sinkhorn_max_iters=5, outer_max_iters=3), DeviceOptions(dtype="float64"))
local, _ = s.exchange_buffers()
from cuda.bindings import runtime as rt
print("memset past the end:", rt.cudaMemset(local + 21 * 8, 0, 8))
torch.cuda.synchronize()
s.close()
print("NOT DETECTED")
PY
echo "positive control rc=$? (expect 134: abort on the overwritten guard band)"
cat gpurun_out/${tag}_checked_control.log | tail -3
