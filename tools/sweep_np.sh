# micro-kernel variants: node pairs per thread x rows per band (C2, 200 steps)
for NP in ${NPS:-4 8}; do for LY in ${LYS:-32 48 64}; do
  r=$(MM2D_NP=$NP MM2D_LY=$LY timeout 90 python bench.py --steps 200 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4f %.4f' % (d['roofline']['launch_ms'], d['ms_per_step']))")
  echo "np=$NP ly=$LY micro_ms/step_ms $r"
done; done
for NP in ${NPS:-4 8}; do MM2D_NP=$NP timeout 240 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 2>&1 | tail -1; done
