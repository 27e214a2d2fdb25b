# A/B of two library builds on the GPU box: parity tests on the new build,
# then bench launch/step times for both (alternating, 2 runs each).
#   bash tools/ab.sh [old.so] [new.so]
OLD=${1:-libmm2d_old.so}; NEW=${2:-libmm2d.so}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 -x > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ab_pytest.log
for r in 1 2; do
  for L in $OLD $NEW; do
    MM2D_LIBRARY=paper_2509_21832_b200/$L timeout 120 python bench.py --steps 300 --warmup 5 --no-cpu-baseline | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['roofline']['launch_ms'],4), round(d['ms_per_step'],4))"
  done
done
