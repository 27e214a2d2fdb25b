set -x
(nproc; lscpu | grep -E "Model name|Socket|Core|Thread|NUMA node\(s\)"; free -g; df -h /dev/shm; nvidia-smi -L) > gpurun_out/sys.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c5.log 2> gpurun_out/bench_c5.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
tail -3 gpurun_out/pytest_gpu.log
