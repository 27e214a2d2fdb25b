# Full verification + evidence pass on the GPU box for the current tree:
# GPU parity tests, smoke, default bench (with CPU baseline), reference arm,
# launch list, one ncu --set full capture of k_micro32.  Outputs in gpurun_out/.
#   gpurun --timeout 2400 -- 'bash tools/refresh.sh TAG'
TAG=${1:-cur}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu --timeout 300 -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu_$TAG.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launches rc=$?"
python tools/profile_step.py > gpurun_out/prof_plain_$TAG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_micro32 -s 1 -c 1 \
  -o gpurun_out/prof_$TAG python tools/profile_step.py > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/bench_$TAG.json
for c in c3 c4 c4s c5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err; echo "bench $c rc=$?"
done
