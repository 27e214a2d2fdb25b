# A/B of library builds on the GPU box: 2D parity tests on each new build,
# then bench launch/step times (alternating, 2 rounds).
#   bash tools/ab.sh "libA.so libB.so[:LY] ..."      (LY sets MM2D_LY)
LIBS=${1:-"libmm2d_old.so libmm2d.so"}
mkdir -p gpurun_out
for spec in $LIBS; do
  L=${spec%%:*}
  [ "$L" = libmm2d_old.so ] && continue
  MM2D_LIBRARY=paper_2509_21832_b200/$L timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 -x > gpurun_out/ab_pytest_$L.log 2>&1; echo "$L pytest rc=$? $(tail -1 gpurun_out/ab_pytest_$L.log)"
done
for r in 1 2; do
  for spec in $LIBS; do
    L=${spec%%:*}; LY=""; [ "$spec" != "$L" ] && LY=${spec#*:}
    env MM2D_LIBRARY=paper_2509_21832_b200/$L ${LY:+MM2D_LY=$LY} timeout 120 python bench.py --steps 300 --warmup 5 --no-cpu-baseline | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$spec', round(d['roofline']['launch_ms'],4), round(d['ms_per_step'],4))"
  done
done
