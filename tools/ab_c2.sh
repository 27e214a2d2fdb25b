# A/B of library builds at C2 only: GPU tests on the default build, then
# bench kernel/step times per library, alternating, 3 rounds.
#   bash tools/ab_c2.sh TAG "libA.so libB.so ..."
TAG=$1; LIBS=$2
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 300 -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu_$TAG.log)"
for r in 1 2 3; do
  for L in $LIBS; do
    MM2D_LIBRARY=paper_2509_21832_b200/$L timeout 300 python bench.py --steps 500 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${TAG}_${L}_c2_$r.json 2>/dev/null
    python tools/cmp_bench.py gpurun_out/ab_${TAG}_${L}_c2_$r.json
  done
done
