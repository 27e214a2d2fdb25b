mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
python tools/profile_step.py > gpurun_out/prof_plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_micro32 -s 1 -c 1 -o gpurun_out/prof_cur python tools/profile_step.py > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/pytest_gpu.log
