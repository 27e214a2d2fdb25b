# A/B of the prep kernel variants: GPU tests on the default build, then
# per-kernel times (bench kernel_ms) at C2 and C5 for each library, alternating.
#   bash tools/ab_prep.sh TAG "libmm2d.so libmm2d_untiled.so"
TAG=$1; LIBS=${2:-"libmm2d.so libmm2d_untiled.so"}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 300 -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu_$TAG.log)"
for r in 1 2; do
  for L in $LIBS; do
    for c in c2 c5; do
      st=300; [ $c = c5 ] && st=20
      MM2D_LIBRARY=paper_2509_21832_b200/$L timeout 300 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/ab_${TAG}_${L}_${c}_$r.json 2>/dev/null
      python tools/cmp_bench.py gpurun_out/ab_${TAG}_${L}_${c}_$r.json
    done
  done
done
