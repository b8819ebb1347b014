# GPU test session: the -m gpu suite and the smoke, logs under gpurun_out/
tag=${1:-r02}
python -m pytest tests -m gpu -q -rs --durations=20 > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/${tag}_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"; tail -5 gpurun_out/${tag}_smoke.log
