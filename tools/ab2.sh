# A/B of library builds on the GPU box (round 2): optional parity tests on
# each candidate, then alternating device timings on C5 and C2.
#   bash tools/ab2.sh "libmm2d_base.so libmm2d.so" [pytest-args|-]
LIBS=${1:-"libmm2d_base.so libmm2d.so"}
PT=${2:-"tests/test_gpu_parity.py tests/test_specular.py"}
mkdir -p gpurun_out
if [ "$PT" != "-" ]; then
for L in $LIBS; do
  [ "$L" = libmm2d_base.so ] && continue
  MM2D_LIBRARY=paper_2509_21832_b200/$L timeout 900 python -m pytest $PT -q -m gpu -x > gpurun_out/ab_pytest_$L.log 2>&1; echo "$L pytest rc=$? $(tail -1 gpurun_out/ab_pytest_$L.log)"
done
fi
for r in 1 2; do
  for cfg in c5 c2; do
    for L in $LIBS; do
      n=30; [ $cfg = c2 ] && n=300
      MM2D_LIBRARY=paper_2509_21832_b200/$L timeout 300 python bench.py --config $cfg --steps $n --warmup 5 --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg $L', 'micro', round(r['launch_ms'],4), 'step', round(d['ms_per_step'],4), 'frac', round(r['frac'],4), 'sm', d['clocks']['sm_mhz'])"
    done
  done
done
