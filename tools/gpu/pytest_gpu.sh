# GPU parity suite on the box; log under gpurun_out/
timeout 1700 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -25 gpurun_out/pytest_gpu.log
